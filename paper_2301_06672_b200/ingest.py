"""GPU ingest: PQ code assignment and coarse assignment.

Mirrors the reference's encode-side functions with the same names, argument
meaning and errors; the arithmetic runs in csrc/ingest.cuh through the C ABI
(`ivfpq_pq_encode*`, `ivfpq_assign*`):

* `pq_encode`            pq.py:92-110        -- bit-exact for sub_d <= 4
* `assign_to_centroids`  kmeans.py:49-69     -- decision-level parity
* `populate_lists`       index.py:93-96 grouping + pq.py:54-63 residuals,
                         all on the device (used to build 10M/100M indexes)
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .index import IvfPqIndex, PQCodebook
from .validation import check_matrix


def pq_encode(residuals, cb: PQCodebook) -> np.ndarray:
    """Nearest sub-centroid per subspace, ties to the lower code (pq.py:92-110).
    One residual (d,) -> (s,); a batch (n, d) -> (n, s) uint8."""
    arr = np.ascontiguousarray(residuals, dtype=np.float32)
    single = arr.ndim == 1
    if single:
        arr = arr[None, :]
    if arr.ndim != 2 or arr.shape[1] != cb.d:
        raise ValueError(f"residuals must have {cb.d} dimensions")
    centers = np.ascontiguousarray(cb.centers, dtype=np.float32)
    codes = np.empty((arr.shape[0], cb.s), dtype=np.uint8)
    _lib.require_gpu()
    _lib.check(_lib.lib.ivfpq_pq_encode(_lib.ptr(arr), arr.shape[0], arr.shape[1], _lib.ptr(centers), cb.s, cb.p,
                                        _lib.ptr(codes)))
    return codes[0] if single else codes


def assign_to_centroids(X, centroids) -> tuple[np.ndarray, np.ndarray]:
    """Nearest centroid per row under squared L2, ties to the lower id
    (kmeans.py:49-69): (assignments int64, squared distances float32)."""
    X = check_matrix(X, "X")
    centroids = check_matrix(centroids, "centroids")
    if X.shape[1] != centroids.shape[1]:
        raise ValueError("X and centroids must have the same dimension")
    assign = np.empty(X.shape[0], dtype=np.int64)
    d2 = np.empty(X.shape[0], dtype=np.float32)
    _lib.require_gpu()
    _lib.check(_lib.lib.ivfpq_assign(_lib.ptr(X), X.shape[0], X.shape[1], _lib.ptr(centroids), centroids.shape[0],
                                     _lib.ptr(assign), _lib.ptr(d2)))
    return assign, d2


def assign_device(x, centroids, stream=None):
    """Device tensors: x f32[n,d], centroids f32[nc,d] -> (assign i64[n], d2 f32[n])."""
    import torch
    n = x.shape[0]
    a = torch.empty(n, dtype=torch.int64, device=x.device)
    d2 = torch.empty(n, dtype=torch.float32, device=x.device)
    st = stream if stream is not None else torch.cuda.current_stream(x.device).cuda_stream
    _lib.check(_lib.lib.ivfpq_assign_device(x.data_ptr(), n, x.shape[1], centroids.data_ptr(), centroids.shape[0],
                                            a.data_ptr(), d2.data_ptr(), ctypes.c_void_p(st)))
    return a, d2


def pq_encode_device(x, centers, p: int, coarse=None, assign=None, stream=None):
    """Device tensors -> codes u8[n, s].  With `coarse` and `assign` the rows
    are encoded as residuals fl(x - coarse[assign]) (compute_residuals,
    pq.py:54-63) formed inside the kernel."""
    import torch
    n, d = x.shape
    s = centers.shape[0]
    codes = torch.empty((n, s), dtype=torch.uint8, device=x.device)
    st = stream if stream is not None else torch.cuda.current_stream(x.device).cuda_stream
    _lib.check(_lib.lib.ivfpq_pq_encode_device(
        x.data_ptr(), n, d, coarse.data_ptr() if coarse is not None else None,
        assign.data_ptr() if assign is not None else None, centers.data_ptr(), s, p, codes.data_ptr(),
        ctypes.c_void_p(st)))
    return codes


def populate_lists(data, coarse: np.ndarray, cb: PQCodebook, chunk: int = 1 << 22) -> IvfPqIndex:
    """Assign every row to its nearest coarse centroid, encode its residual
    and group rows into inverted lists in ascending id order (index.py:93-96:
    `np.nonzero(assign == c)` per list) -- on the GPU, `chunk` rows at a time.
    `data` may be a numpy array or a CUDA tensor."""
    import torch
    _lib.require_gpu()
    coarse_t = torch.from_numpy(np.ascontiguousarray(coarse, dtype=np.float32)).cuda()
    centers_t = torch.from_numpy(np.ascontiguousarray(cb.centers, dtype=np.float32)).cuda()
    n = data.shape[0]
    assign = torch.empty(n, dtype=torch.int64, device="cuda")
    codes = torch.empty((n, cb.s), dtype=torch.uint8, device="cuda")
    for lo in range(0, n, chunk):
        xb = data[lo:lo + chunk]
        xb = xb if isinstance(xb, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(xb, dtype=np.float32))
        xb = xb.cuda()
        a, _ = assign_device(xb, coarse_t)
        assign[lo:lo + xb.shape[0]] = a
        codes[lo:lo + xb.shape[0]] = pq_encode_device(xb, centers_t, cb.p, coarse_t, a)
    order = torch.sort(assign, stable=True).indices   # ascending ids within each list
    off = torch.zeros(coarse.shape[0] + 1, dtype=torch.int64, device="cuda")
    off[1:] = torch.cumsum(torch.bincount(assign, minlength=coarse.shape[0]), 0)
    return IvfPqIndex.from_csr(np.asarray(coarse, dtype=np.float32), cb, off.cpu().numpy(), order.cpu().numpy(),
                               codes[order].cpu().numpy())
