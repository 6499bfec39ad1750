"""Benchmark workload: BASELINE.json configs, synthetic data, index builders
and exact ground truth.  Harness code, not the product.

Index training is OUT OF SCOPE for the hot path;
the search kernels consume the resulting arrays exactly like a
reference-built index.  Two builders:

* "cpu" (harness/cpu_build.py, numpy + host BLAS only): deterministic, used by
  BOTH bench arms at cfg1/cfg2 so they search identical arrays, and the only
  one the reference arm may use (it must not load the product library);
* "gpu" (the package's `train.build_index`: Lloyd on a subsample, assignment
  and bit-exact pq_encode by the product kernels): for cfg3..cfg5, whose CPU
  build would take hours.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from harness import cpu_build  # noqa: E402  (numpy only)

# BASELINE.json configs; generator (comps, spread) per SURVEY.md 8(d); cfg3 and
# cfg5 re-calibrated with harness/calibrate.py (profiles/r02_calibration_*.jsonl):
# the SURVEY proposals (64 / 1024 components, spread 0.3) put recall@10 at
# 0.46 (cfg3 p8), 0.20 (cfg3 p5), 0.60 (cfg5) -- PQ-limited, not IVF-limited.
# ~12-15 points per component (cfg3: 81920 comps, spread 0.15; cfg5: 6.55M
# comps, spread 0.1) keeps the IVF ceiling responsive to nprobe (cfg3: 0.94 at
# P 32) and lifts recall@10 at the headline nprobe above 0.8 (calibration
# sample: 0.82 cfg3 p5, 0.84 cfg5; p5's 32 codewords cap it near 0.78 at
# 65536 comps).
CONFIGS = {
    "cfg1": dict(n=100_000, d=128, nlist=1024, s=64, p=8, nq=1_000, nprobe=32, k=10, comps=16, spread=0.3, seed=1),
    "cfg2": dict(n=1_000_000, d=128, nlist=4096, s=64, p=8, nq=10_000, nprobe=32, k=10, comps=64, spread=0.3,
                 seed=2),
    "cfg3p8": dict(n=1_000_000, d=960, nlist=4096, s=240, p=8, nq=10_000, nprobe=32, k=10, comps=81920,
                   spread=0.15, seed=3),
    "cfg3p5": dict(n=1_000_000, d=960, nlist=4096, s=240, p=5, nq=10_000, nprobe=32, k=10, comps=81920,
                   spread=0.15, seed=3),
    "cfg4": dict(n=10_000_000, d=96, nlist=16384, s=48, p=8, nq=10_000, nprobe=32, k=100, comps=256, spread=0.3,
                 seed=4),
    "cfg5": dict(n=100_000_000, d=96, nlist=65536, s=32, p=8, nq=10_000, nprobe=64, k=10, comps=6_553_600,
                 spread=0.1, seed=5),
}
DEFAULT_BUILDER = {"cfg1": "cpu", "cfg2": "cpu"}


def make_data(cfg):
    """(base, queries): one chunked mixture draw of n + nq rows, split."""
    X = cpu_build.synth_chunked(cfg["n"] + cfg["nq"], cfg["d"], cfg["comps"], cfg["spread"], cfg["seed"])
    return X[:cfg["n"]], X[cfg["n"]:]


def build_arrays(cfg, base, builder: str):
    """-> dict(coarse, centers, off, ids, codes) in CSR list order."""
    if builder == "cpu":
        coarse, centers, off, ids, codes = cpu_build.build_index_cpu(base, cfg["nlist"], cfg["s"], cfg["p"],
                                                                     seed=cfg["seed"])
        return dict(coarse=coarse, centers=centers, off=off, ids=ids, codes=codes)
    idx = build_index_gpu(base, cfg["nlist"], cfg["s"], cfg["p"], seed=cfg["seed"])
    off, ids, codes = idx.csr()
    return dict(coarse=idx.coarse, centers=idx.cb.centers, off=off, ids=ids, codes=codes)


def arrays_digest(arr: dict, queries: np.ndarray) -> str:
    """Short hash of the search inputs (both bench arms print it: same inputs)."""
    h = hashlib.sha1()
    for k in ("coarse", "centers", "off", "ids", "codes"):
        h.update(np.ascontiguousarray(arr[k]).data)
    h.update(np.ascontiguousarray(queries).data)
    return h.hexdigest()[:16]


def to_index(arr: dict, p: int):
    """Product index object over the arrays (loads the product library)."""
    from paper_2301_06672_b200.index import IvfPqIndex, PQCodebook
    return IvfPqIndex.from_csr(arr["coarse"], PQCodebook(centers=arr["centers"], p=p), arr["off"], arr["ids"],
                               arr["codes"])


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
