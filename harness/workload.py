"""Benchmark workload: synthetic data, an (untimed) GPU index builder and exact
ground truth.  Harness code, not the product: it uses torch ops as plumbing to
produce the inputs of the search path quickly at BASELINE.json sizes.

Index training is OUT OF SCOPE for the hot path:
coarse k-means and per-subspace PQ k-means here are plain Lloyd iterations on
a subsample; assignment/encoding take the nearest centroid.  The search
kernels consume the resulting arrays exactly like a reference-built index.
"""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# BASELINE.json configs (SURVEY.md 8d generator proposals)
CONFIGS = {
    "cfg1": dict(n=100_000, d=128, nlist=1024, s=64, p=8, nq=1_000, nprobe=32, k=10, comps=16, spread=0.3, seed=1),
    "cfg2": dict(n=1_000_000, d=128, nlist=4096, s=64, p=8, nq=10_000, nprobe=32, k=10, comps=64, spread=0.3,
                 seed=2),
    "cfg3p8": dict(n=1_000_000, d=960, nlist=4096, s=240, p=8, nq=10_000, nprobe=32, k=10, comps=64, spread=0.3,
                   seed=3),
    "cfg3p5": dict(n=1_000_000, d=960, nlist=4096, s=240, p=5, nq=10_000, nprobe=32, k=10, comps=64, spread=0.3,
                   seed=3),
    "cfg4": dict(n=10_000_000, d=96, nlist=16384, s=48, p=8, nq=10_000, nprobe=32, k=100, comps=256, spread=0.3,
                 seed=4),
    "cfg5": dict(n=100_000_000, d=96, nlist=65536, s=32, p=8, nq=10_000, nprobe=64, k=10, comps=1024, spread=0.3,
                 seed=5),
}


def make_data(cfg):
    from paper_2301_06672_b200.datasets import synth_gaussian_mixture_chunked
    X = synth_gaussian_mixture_chunked(cfg["n"] + cfg["nq"], cfg["d"], cfg["comps"], cfg["spread"], cfg["seed"])
    return X[:cfg["n"]], X[cfg["n"]:]


def _nearest(x, c, chunk=65536):
    """argmin_j ||x_i - c_j||^2 (expanded form, fp32 tensor cores off)."""
    import torch
    cn = (c * c).sum(1)
    out = torch.empty(x.shape[0], dtype=torch.int64, device=x.device)
    for lo in range(0, x.shape[0], chunk):
        xb = x[lo:lo + chunk]
        d = cn[None, :] - 2.0 * (xb @ c.T)
        out[lo:lo + chunk] = d.argmin(1)
    return out


def _segment_means(x, a, k, old):
    """Deterministic per-cluster means (sort + float64 prefix sums; no atomics)."""
    import torch
    order = torch.sort(a, stable=True).indices
    cs = torch.zeros((x.shape[0] + 1, x.shape[1]), dtype=torch.float64, device=x.device)
    cs[1:] = torch.cumsum(x[order].double(), 0)
    cnt = torch.bincount(a, minlength=k)
    hi = torch.cumsum(cnt, 0)
    lo = hi - cnt
    sums = cs[hi] - cs[lo]
    return torch.where(cnt[:, None] > 0, (sums / cnt.clamp(min=1)[:, None]).float(), old)


def _kmeans(x, k, iters, seed):
    import torch
    g = torch.Generator(device=x.device).manual_seed(seed)
    c = x[torch.randperm(x.shape[0], generator=g, device=x.device)[:k]].clone()
    for _ in range(iters):
        c = _segment_means(x, _nearest(x, c), k, c)
    return c


def _pq_train_encode(res, s, p, train_n, iters, seed):
    """Batched per-subspace k-means (k = 2^p) and encode.  res: (n, d) cuda."""
    import torch
    n, d = res.shape
    sub = d // s
    K = 1 << p
    g = torch.Generator(device=res.device).manual_seed(seed)
    tr = res[torch.randperm(n, generator=g, device=res.device)[:train_n]].reshape(-1, s, sub).transpose(0, 1)
    c = tr[:, torch.randperm(tr.shape[1], generator=g, device=res.device)[:K]].clone()   # (s, K, sub)
    tr = tr.contiguous()

    def assign(xs):  # xs (s, m, sub) -> (s, m)
        cn = (c * c).sum(2)
        return (cn[:, None, :] - 2.0 * torch.bmm(xs, c.transpose(1, 2))).argmin(2)

    for _ in range(iters):
        a = torch.cat([assign(tr[:, lo:lo + 16384]) for lo in range(0, tr.shape[1], 16384)], 1)
        c = torch.stack([_segment_means(tr[j], a[j], K, c[j]) for j in range(s)])
    codes = torch.empty((n, s), dtype=torch.uint8, device=res.device)
    for lo in range(0, n, 16384):
        xs = res[lo:lo + 16384].reshape(-1, s, sub).transpose(0, 1).contiguous()
        codes[lo:lo + 16384] = assign(xs).T.to(torch.uint8)
    return c, codes


def build_index_gpu(base: np.ndarray, nlist: int, s: int, p: int, seed: int = 0, train_n: int = 262_144,
                    iters: int = 12):
    """Returns an IvfPqIndex (CSR-backed) built on cuda:0."""
    import torch
    from paper_2301_06672_b200.index import IvfPqIndex, PQCodebook
    x = torch.from_numpy(base).cuda()
    g = torch.Generator(device="cuda").manual_seed(seed)
    tr = x[torch.randperm(x.shape[0], generator=g, device="cuda")[:max(train_n, nlist * 8)]]
    coarse = _kmeans(tr, nlist, iters, seed)
    assign = _nearest(x, coarse)
    res = x - coarse[assign]
    centers, codes = _pq_train_encode(res, s, p, min(train_n, x.shape[0]), iters, seed + 1)
    order = torch.sort(assign, stable=True).indices
    off = torch.zeros(nlist + 1, dtype=torch.int64, device="cuda")
    off[1:] = torch.cumsum(torch.bincount(assign, minlength=nlist), 0)
    idx = IvfPqIndex.from_csr(coarse.cpu().numpy(), PQCodebook(centers=centers.cpu().numpy(), p=p),
                              off.cpu().numpy(), order.cpu().numpy(), codes[order].cpu().numpy())
    del x, res, tr
    torch.cuda.empty_cache()
    return idx


def ground_truth_gpu(base: np.ndarray, queries: np.ndarray, k: int) -> np.ndarray:
    """Exact k-NN ids (ties -> lower id) with the product's K7 kernel
    (`brute_force_knn`, bit-identical to the reference's datasets.py:179-201)."""
    from paper_2301_06672_b200.datasets import brute_force_knn
    return brute_force_knn(base, queries, k).ids


def recall_at(ids: np.ndarray, gt: np.ndarray) -> float:
    hits = (ids[:, :, None] == gt[:, None, :]) & (ids[:, :, None] >= 0)
    return float((hits.any(2).sum(1) / gt.shape[1]).mean())
