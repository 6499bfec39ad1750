"""Index construction on the GPU: `build_index(data, nlist, s, p, seed)` with
the reference's signature and validation (index.py:73-97).

Training is outside the search path: the k-means
here are Lloyd iterations seeded from a random sample, NOT the reference's
k-means++ (kmeans.py:79-89), so centroids and codebooks differ from a
reference-built index.  Every assignment step runs on the product kernels --
coarse `assign_to_centroids` (csrc/ingest.cuh assign_kernel) and the
bit-exact `pq_encode` -- and the final lists are grouped exactly as the
reference does (ascending ids per list).  Torch is used only for device
buffers and the per-cluster means.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .index import IvfPqIndex, PQCodebook
from .ingest import assign_device, populate_lists, pq_encode_device
from .validation import check_matrix


def _means(x, a, k, old):
    """Per-cluster means of rows x (n, m) under labels a; empty clusters keep
    their previous centroid.  Float64 sums, deterministic: rows sorted by label,
    then one sequential sum per (segment, column) (torch.segment_reduce; a
    dim-0 cumsum of a tall, narrow matrix runs one thread per column)."""
    import torch
    order = torch.sort(a, stable=True).indices
    cnt = torch.bincount(a, minlength=k)
    sums = torch.segment_reduce(x[order].double(), "sum", lengths=cnt, axis=0)
    return torch.where(cnt[:, None] > 0, (sums / cnt.clamp(min=1)[:, None]).float(), old)


def train_coarse_gpu(x, nlist: int, seed: int, iters: int = 12):
    """Lloyd k-means on device rows x (n, d) -> centroids (nlist, d)."""
    import torch
    g = torch.Generator(device=x.device).manual_seed(seed)
    c = x[torch.randperm(x.shape[0], generator=g, device=x.device)[:nlist]].contiguous()
    for _ in range(iters):
        a, _ = assign_device(x, c)
        c = _means(x, a, nlist, c).contiguous()
    return c


def train_pq_gpu(res, s: int, p: int, seed: int, iters: int = 12):
    """Per-subspace Lloyd k-means (k = 2^p) on device residuals (n, d) ->
    centers (s, 2^p, d/s); assignments by the bit-exact pq_encode kernel."""
    import torch
    n, d = res.shape
    sub = d // s
    K = 1 << p
    g = torch.Generator(device=res.device).manual_seed(seed)
    pick = torch.randperm(n, generator=g, device=res.device)[:K]
    centers = res[pick].reshape(K, s, sub).transpose(0, 1).contiguous()   # (s, K, sub)
    x3 = res.reshape(n, s, sub)
    sub_id = torch.arange(s, device=res.device)[None, :] * K
    for _ in range(iters):
        codes = pq_encode_device(res, centers, p).long()                   # (n, s)
        # all subspaces at once: segment means over the (subspace, code) key
        key = (codes + sub_id).reshape(-1)
        centers = _means(x3.reshape(n * s, sub), key, s * K, centers.reshape(s * K, sub)).reshape(s, K, sub)
        centers = centers.contiguous()
    return centers


def build_index(data, nlist: int, s: int, p: int, seed: int = 0, train_n: int = 262_144,
                iters: int = 12) -> IvfPqIndex:
    """Coarse k-means, residuals, one global PQ codebook, encode every row
    (index.py:73-97), all on the GPU.  Deterministic under `seed`."""
    import torch
    X = check_matrix(data, "data")
    n, d = X.shape
    if n < max(nlist, 1 << p):
        raise ValueError(f"need at least max(nlist, 2^p) = {max(nlist, 1 << p)} rows, got {n}")
    if d % s != 0:
        raise ValueError(f"d={d} not divisible by s={s}")
    if not 1 <= p <= 8:
        raise ValueError("p must be in 1..8 (one byte per sub-code)")
    _lib.require_gpu()
    coarse_seed, pq_seed = (int(v) for v in np.random.SeedSequence(seed).generate_state(2))
    x = torch.from_numpy(X).cuda()
    g = torch.Generator(device="cuda").manual_seed(coarse_seed)
    tr = x[torch.randperm(n, generator=g, device="cuda")[:min(n, max(train_n, 8 * nlist))]].contiguous()
    import sys
    import time
    t0 = time.time()
    coarse = train_coarse_gpu(tr, nlist, coarse_seed, iters)
    a, _ = assign_device(tr, coarse)
    res = (tr - coarse[a]).contiguous()
    torch.cuda.synchronize()
    t1 = time.time()
    centers = train_pq_gpu(res, s, p, pq_seed, iters)
    cb = PQCodebook(centers=centers.cpu().numpy(), p=p)
    del tr, res
    t2 = time.time()
    out = populate_lists(x, coarse.cpu().numpy(), cb)
    print(f"[build_index] coarse {t1 - t0:.1f}s pq {t2 - t1:.1f}s populate {time.time() - t2:.1f}s", file=sys.stderr,
          flush=True)
    return out
