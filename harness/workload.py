"""Benchmark workload: synthetic data, an (untimed) GPU index builder and exact
ground truth.  Harness code, not the product: it uses torch ops as plumbing to
produce the inputs of the search path quickly at BASELINE.json sizes.

Index training is OUT OF SCOPE for the hot path:
the index comes from the package's GPU builder (Lloyd iterations on a
subsample; assignment and bit-exact PQ encoding by the product kernels).  The
search kernels consume the resulting arrays exactly like a reference-built
index.
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


def build_index_gpu(base: np.ndarray, nlist: int, s: int, p: int, seed: int = 0, train_n: int = 262_144,
                    iters: int = 12):
    """The product's GPU index builder (paper_2301_06672_b200.train.build_index):
    Lloyd training on a subsample, coarse assignment + bit-exact pq_encode of
    every row by the product kernels."""
    from paper_2301_06672_b200.train import build_index
    return build_index(base, nlist, s, p, seed=seed, train_n=train_n, iters=iters)


def ground_truth_gpu(base: np.ndarray, queries: np.ndarray, k: int) -> np.ndarray:
    """Exact k-NN ids (ties -> lower id) with the product's K7 kernel
    (`brute_force_knn`, bit-identical to the reference's datasets.py:179-201)."""
    from paper_2301_06672_b200.datasets import brute_force_knn
    return brute_force_knn(base, queries, k).ids


def recall_at(ids: np.ndarray, gt: np.ndarray) -> float:
    hits = (ids[:, :, None] == gt[:, None, :]) & (ids[:, :, None] >= 0)
    return float((hits.any(2).sum(1) / gt.shape[1]).mean())
