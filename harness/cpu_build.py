"""Deterministic CPU workload builder for bench.py (numpy + host BLAS only).

Both bench arms (`--impl ours` and `--impl reference`) build their inputs
here, so they search IDENTICAL arrays -- and the reference arm never loads
the product library (`paper_2301_06672_b200/libivfpq_b200.so`) nor anything
else of the GPU path.  This module imports neither the product package nor
`oracle/`; it only produces synthetic inputs of the BASELINE.json shapes:

* data: the chunked Gaussian-mixture recipe of SURVEY.md 8(d) (means from
  default_rng(seed), chunk i from default_rng([seed, i])), the same draw as
  `paper_2301_06672_b200.datasets.synth_gaussian_mixture_chunked`;
* index: Lloyd k-means on a subsample (coarse quantizer, then one global PQ
  codebook on the residuals -- the structure of reference index.py:73-97;
  training itself is out of scope), every row
  assigned and encoded by nearest-centroid argmin in the expanded BLAS form,
  lists = ascending ids per cluster (index.py:93-96).  Which codes the
  encoder picks at near-ties does not matter here: the arrays are the search
  path's INPUT, handed unchanged to both arms;
* ground truth: exact k-NN (ties -> lower id) by a BLAS shortlist re-ranked
  with the reference's sequential float32 distance (datasets.py:166-201).

Work is split over host threads (numpy's BLAS and reductions release the
GIL).
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_NT = max(1, len(os.sched_getaffinity(0)))


def _pool():
    return ThreadPoolExecutor(_NT)


def synth_chunked(n: int, d: int, n_components: int, spread: float, seed: int, chunk: int = 1 << 20) -> np.ndarray:
    """SURVEY.md 8(d) chunked mixture: means U[0,1)^d from default_rng(seed);
    chunk i draws labels then N(0, spread^2) noise from default_rng([seed, i])."""
    means = np.random.default_rng(seed).random((n_components, d)).astype(np.float32)
    X = np.empty((n, d), dtype=np.float32)

    def one(i):
        lo = i * chunk
        hi = min(n, lo + chunk)
        rng = np.random.default_rng([seed, i])
        labels = rng.integers(0, n_components, size=hi - lo)
        X[lo:hi] = means[labels] + np.float32(spread) * rng.standard_normal((hi - lo, d), dtype=np.float32)

    with _pool() as ex:
        list(ex.map(one, range((n + chunk - 1) // chunk)))
    return X


def _nearest(x: np.ndarray, c: np.ndarray, rows: int = 8192) -> np.ndarray:
    """argmin_j |x_i - c_j|^2 in the expanded form |c|^2 - 2 x.c (first index
    on ties), threaded over row blocks."""
    cn = np.einsum("ij,ij->i", c, c)
    out = np.empty(x.shape[0], dtype=np.int64)

    def one(lo):
        hi = min(x.shape[0], lo + rows)
        d = cn[None, :] - 2.0 * (x[lo:hi] @ c.T)
        out[lo:hi] = np.argmin(d, axis=1)

    with _pool() as ex:
        list(ex.map(one, range(0, x.shape[0], rows)))
    return out


def _lloyd(x: np.ndarray, k: int, iters: int, rng: np.random.Generator) -> np.ndarray:
    c = x[np.sort(rng.choice(x.shape[0], k, replace=False))].copy()
    for _ in range(iters):
        a = _nearest(x, c)
        cnt = np.bincount(a, minlength=k)
        sums = np.zeros((k, x.shape[1]), dtype=np.float64)
        np.add.at(sums, a, x)
        nz = cnt > 0
        c[nz] = (sums[nz] / cnt[nz, None]).astype(np.float32)
    return c


def _pq_nearest(res: np.ndarray, centers: np.ndarray, rows: int = 16384) -> np.ndarray:
    """codes[i, j] = argmin_m |res_i[j-th subvector] - centers[j, m]|^2."""
    s, K, sub = centers.shape
    codes = np.empty((res.shape[0], s), dtype=np.uint8)
    cn = np.einsum("jmt,jmt->jm", centers, centers)

    def one(lo):
        hi = min(res.shape[0], lo + rows)
        r = res[lo:hi].reshape(hi - lo, s, sub).transpose(1, 0, 2)          # (s, b, sub)
        d = cn[:, None, :] - 2.0 * np.matmul(r, centers.transpose(0, 2, 1))  # (s, b, K)
        codes[lo:hi] = np.argmin(d, axis=2).T

    with _pool() as ex:
        list(ex.map(one, range(0, res.shape[0], rows)))
    return codes


def build_index_cpu(base: np.ndarray, nlist: int, s: int, p: int, seed: int = 0, train_n: int = 131_072,
                    iters: int = 10):
    """-> (coarse f32 [nlist, d], centers f32 [s, 2^p, d/s], list_off i64
    [nlist+1], ids i64 [n], codes u8 [n, s]) in CSR list order."""
    n, d = base.shape
    rng = np.random.default_rng(seed)
    tr = base[np.sort(rng.choice(n, min(n, max(train_n, 8 * nlist)), replace=False))]
    coarse = _lloyd(tr, nlist, iters, rng)
    a_tr = _nearest(tr, coarse)
    res_tr = tr - coarse[a_tr]
    K, sub = 1 << p, d // s
    pq_tr = res_tr[np.sort(rng.choice(res_tr.shape[0], min(res_tr.shape[0], 64 * K), replace=False))]
    centers = pq_tr[np.sort(rng.choice(pq_tr.shape[0], K, replace=False))].reshape(K, s, sub).transpose(1, 0, 2).copy()
    for _ in range(iters):
        codes = _pq_nearest(pq_tr, centers)
        for j in range(s):
            x = pq_tr[:, j * sub:(j + 1) * sub]
            cnt = np.bincount(codes[:, j], minlength=K)
            sums = np.zeros((K, sub), dtype=np.float64)
            np.add.at(sums, codes[:, j], x)
            nz = cnt > 0
            centers[j][nz] = (sums[nz] / cnt[nz, None]).astype(np.float32)
    assign = _nearest(base, coarse)
    order = np.argsort(assign, kind="stable")          # ascending ids within each list
    counts = np.bincount(assign, minlength=nlist)
    off = np.zeros(nlist + 1, dtype=np.int64)
    np.cumsum(counts, out=off[1:])
    res = base[order] - coarse[assign[order]]
    codes = _pq_nearest(res, centers)
    return coarse, np.ascontiguousarray(centers), off, order.astype(np.int64), codes


def ground_truth_cpu(base: np.ndarray, queries: np.ndarray, k: int, margin: int = 32, rows: int = 256) -> np.ndarray:
    """Exact top-k ids by squared L2, ties -> lower id (datasets.py:179-201):
    BLAS shortlist of k + margin, re-ranked with the sequential float32
    distance of datasets.py:166-176."""
    bn = np.einsum("ij,ij->i", base, base)
    out = np.empty((queries.shape[0], k), dtype=np.int64)
    m = min(base.shape[0], k + margin)

    def one(lo):
        hi = min(queries.shape[0], lo + rows)
        q = queries[lo:hi]
        approx = bn[None, :] - 2.0 * (q @ base.T)
        cand = np.argpartition(approx, m - 1, axis=1)[:, :m]
        cand.sort(axis=1)
        acc = np.zeros(cand.shape, dtype=np.float32)
        for t in range(base.shape[1]):                      # sequential over t, one rounding per op
            diff = base[cand, t] - q[:, t:t + 1]
            acc = acc + diff * diff
        for r in range(hi - lo):
            o = np.lexsort((cand[r], acc[r]))[:k]
            out[lo + r] = cand[r][o]

    with _pool() as ex:
        list(ex.map(one, range(0, queries.shape[0], rows)))
    return out
