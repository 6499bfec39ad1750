"""IVFPQ search -- the reference `ivfpq8.search` API (search.py:23-221) backed
by the sm_100a kernels through the C ABI.

Drop-in: same names, signatures, return types and ValueError wording.  The
heavy entry point `search_batch` is one C-ABI call (`ivfpq_search`): coarse
selection (K1), per-(query, list) LUT build + encode (K2), code scan (K3) and
top-k merge (K4) all run on the GPU.  The sub-ops `select_clusters`,
`build_lut`, `scan_list` and `top_k` are routed to the same device routines
through the conformance hooks of the ABI.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

from . import _lib, minifloat
from .datasets import NeighborLists
from .index import IvfPqIndex, PQCodebook, device_index
from .validation import check_matrix, check_vector

__all__ = [
    "LUT_PRECISIONS",
    "Lut",
    "SearchParams",
    "TopKResult",
    "select_clusters",
    "build_lut",
    "scan_list",
    "top_k",
    "search",
    "search_batch",
    "search_device",
    "recall",
]

# precision name -> stored bytes per table entry (search.py:38)
LUT_PRECISIONS = {"f32": 4, "f16": 2, "e5m3": 1, "e4m4": 1}
_SPECS = {"e5m3": minifloat.E5M3, "e4m4": minifloat.E4M4}
_ENTRY_DTYPE = {"f32": np.float32, "f16": np.uint16, "e5m3": np.uint8, "e4m4": np.uint8}


def _check_precision(precision: str) -> str:
    if precision not in LUT_PRECISIONS:
        raise ValueError(f"unknown LUT precision {precision!r}; expected one of {sorted(LUT_PRECISIONS)}")
    return precision


@dataclass(frozen=True)
class SearchParams:
    """search.py:51-62."""

    k: int = 10
    nprobe: int = 1
    precision: str = "f32"

    def __post_init__(self):
        if self.k < 1:
            raise ValueError("k must be at least 1")
        if self.nprobe < 1:
            raise ValueError("nprobe must be at least 1")
        _check_precision(self.precision)


@dataclass
class Lut:
    """search.py:65-82: entries (s, 2^p) as f32 / uint16 bits / uint8 codes."""

    entries: np.ndarray
    precision: str

    def decoded(self) -> np.ndarray:
        if self.precision == "f32":
            return self.entries
        if self.precision == "f16":
            return minifloat.decode_f16_array(self.entries)
        return minifloat.decode_array(self.entries, _SPECS[self.precision])


class TopKResult(NamedTuple):
    ids: np.ndarray
    distances: np.ndarray
    short: bool


def _nprobe_in_range(idx: IvfPqIndex, nprobe: int) -> None:
    if not 1 <= nprobe <= idx.nlist:
        raise ValueError(f"nprobe={nprobe} out of range 1..{idx.nlist}")


def select_clusters(idx: IvfPqIndex, q: np.ndarray, nprobe: int) -> np.ndarray:
    """search.py:91-97 on the device (K1): ascending distance, ties by id."""
    _nprobe_in_range(idx, nprobe)
    q = check_vector(q, idx.d)
    out = np.empty(nprobe, dtype=np.int64)
    h = device_index(idx)
    _lib.check(_lib.lib.ivfpq_select_clusters(h.handle, q.ctypes.data, 1, nprobe, out.ctypes.data))
    return out


def build_lut(cb: PQCodebook, residual_query: np.ndarray, precision: str = "f32") -> Lut:
    """search.py:114-127 on the device (the K2 routine of the search kernel)."""
    _check_precision(precision)
    rq = check_vector(residual_query, cb.d, "residual_query")
    _lib.require_gpu()
    out = np.empty((cb.s, cb.n_codes), dtype=_ENTRY_DTYPE[precision])
    centers = np.ascontiguousarray(cb.centers, dtype=np.float32)
    _lib.check(_lib.lib.ivfpq_build_lut(centers.ctypes.data, cb.s, cb.p, cb.sub_d, rq.ctypes.data,
                                        _lib.LUT_CODES[precision], out.ctypes.data))
    return Lut(entries=out, precision=precision)


def scan_list(ids: np.ndarray, codes: np.ndarray, lut: Lut) -> tuple[np.ndarray, np.ndarray]:
    """search.py:130-142 on the device (the K3 arithmetic of the search kernel)."""
    entries = np.ascontiguousarray(lut.entries, dtype=_ENTRY_DTYPE[_check_precision(lut.precision)])
    s, n_codes = entries.shape
    if codes.shape != (ids.shape[0], s):
        raise ValueError("codes shape must be (len(ids), s)")
    # range check on the caller's array, before any narrowing (search.py:137-138)
    if codes.size and codes.max() >= n_codes:
        raise ValueError("code byte out of range for the table")
    if codes.size and not np.issubdtype(codes.dtype, np.integer):
        raise IndexError("arrays used as indices must be of integer (or boolean) type")
    if codes.size and codes.min() < 0:
        # the reference indexes table[j, codes[:, j]]: numpy wraps negative
        # indices in [-n_codes, -1] and raises IndexError below that
        if codes.min() < -n_codes:
            raise IndexError(f"index {int(codes.min())} is out of bounds for axis 1 with size {n_codes}")
        codes = np.where(codes < 0, codes + n_codes, codes)
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    p = int(n_codes).bit_length() - 1
    if 1 << p != n_codes:
        raise ValueError("table width must be a power of two")
    _lib.require_gpu()
    out = np.empty(ids.shape[0], dtype=np.float32)
    _lib.check(_lib.lib.ivfpq_scan_list(codes.ctypes.data, ids.shape[0], s, p, entries.ctypes.data,
                                        _lib.LUT_CODES[lut.precision], out.ctypes.data))
    return ids, out


def top_k(ids: np.ndarray, distances: np.ndarray, k: int) -> TopKResult:
    """search.py:145-155 on the device (the K4 block top-k)."""
    if ids.shape[0] == 0:
        raise ValueError("top_k requires at least one candidate")
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    dists = np.ascontiguousarray(distances, dtype=np.float32)
    _lib.require_gpu()
    m = min(ids.shape[0], k)
    oi = np.empty(m, dtype=np.int64)
    od = np.empty(m, dtype=np.float32)
    _lib.check(_lib.lib.ivfpq_top_k(ids.ctypes.data, dists.ctypes.data, ids.shape[0], k, oi.ctypes.data,
                                    od.ctypes.data))
    return TopKResult(ids=oi, distances=od, short=ids.shape[0] < k)


def search(idx: IvfPqIndex, q: np.ndarray, params: SearchParams) -> TopKResult:
    """search.py:158-184: one query; only the reached candidates are returned."""
    q = check_vector(q, idx.d)
    lists, n_short = search_batch(idx, q[None, :], params)
    keep = lists.ids[0] >= 0
    return TopKResult(ids=lists.ids[0][keep], distances=lists.distances[0][keep], short=bool(n_short))


def search_batch(idx: IvfPqIndex, queries, params: SearchParams) -> tuple[NeighborLists, int]:
    """search.py:187-203: one device call; short rows padded with -1 / +inf."""
    queries = check_matrix(queries, "queries")
    if queries.shape[1] != idx.d:
        raise ValueError(f"queries have d={queries.shape[1]}, index has d={idx.d}")
    _nprobe_in_range(idx, params.nprobe)
    h = device_index(idx)
    nq = queries.shape[0]
    ids = np.empty((nq, params.k), dtype=np.int64)
    dists = np.empty((nq, params.k), dtype=np.float32)
    n_short = _lib.ctypes.c_int64(0)
    _lib.check(_lib.lib.ivfpq_search(h.handle, queries.ctypes.data, nq, params.k, params.nprobe,
                                     _lib.LUT_CODES[params.precision], ids.ctypes.data, dists.ctypes.data,
                                     _lib.ctypes.byref(n_short)))
    return NeighborLists(ids=ids, distances=dists), int(n_short.value)


def search_device(dev, queries, params: SearchParams, out_ids, out_dists, out_short, stream=None) -> None:
    """Device-resident batch search on torch CUDA tensors (no host copies):
    queries f32 [nq, d], out_ids int64 [nq, k], out_dists f32 [nq, k],
    out_short int32 [nq].  `dev` is a DeviceIndex; `stream` a cudaStream_t
    handle (int) or None for the current torch stream."""
    if stream is None:
        import torch
        stream = torch.cuda.current_stream(dev.device).cuda_stream
    _lib.check(_lib.lib.ivfpq_search_device(dev.handle, queries.data_ptr(), queries.shape[0], params.k,
                                            params.nprobe, _lib.LUT_CODES[params.precision], out_ids.data_ptr(),
                                            out_dists.data_ptr(), out_short.data_ptr(), stream))


def recall(results: NeighborLists, gt: NeighborLists) -> tuple[np.ndarray, float]:
    """search.py:206-221: per-query |ids ∩ gt| / gt.k; padding ids never match."""
    if results.n_queries != gt.n_queries:
        raise ValueError(f"result rows ({results.n_queries}) != ground-truth rows ({gt.n_queries})")
    if gt.k == 0:
        raise ValueError("ground truth has no neighbors per query")
    res = results.ids
    hits = (res[:, :, None] == gt.ids[:, None, :]) & (res[:, :, None] >= 0)
    per_query = hits.any(axis=2).sum(axis=1) / gt.k
    return per_query, float(per_query.mean())
