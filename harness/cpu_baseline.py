"""CPU baseline for bench.py: the oracle's numpy restatement of the reference
search loop (oracle/ivfpq_np.py = search.py:158-203 step for step), run over a
bounded query sample in a spawn-started process pool (one single-threaded
worker per host core; SPEC.md:437 allows query-parallel search over a shared
immutable index).  This is test/bench infrastructure: it never runs on the
product path.
"""

from __future__ import annotations

import os
import tempfile
import time

import numpy as np

_STATE = {}


def _init(path):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    z = {k: np.load(os.path.join(path, k + ".npy"), mmap_mode="r") for k in ("coarse", "centers", "off", "ids", "codes")}
    off = np.asarray(z["off"])
    s = z["centers"].shape[0]
    _STATE["coarse"] = np.ascontiguousarray(z["coarse"])
    _STATE["centers"] = np.ascontiguousarray(z["centers"])
    _STATE["ids"] = [np.asarray(z["ids"][off[c]:off[c + 1]]) for c in range(off.size - 1)]
    _STATE["codes"] = [np.asarray(z["codes"][off[c]:off[c + 1]]).reshape(-1, s) for c in range(off.size - 1)]


def _work(args):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if root not in sys.path:
        sys.path.insert(0, root)
    from oracle import ivfpq_np as onp
    q, k, nprobe, prec = args
    t0 = time.perf_counter()
    ids, d, ns = onp.search_batch(_STATE["coarse"], _STATE["centers"], _STATE["ids"], _STATE["codes"], q, k, nprobe,
                                  prec)
    return ids, time.perf_counter() - t0


class CpuBaseline:
    """Holds a worker pool with the index loaded; `run` times one sample."""

    def __init__(self, arrays: dict, workers: int | None = None):
        """arrays: coarse, centers, off, ids, codes (CSR list order, codes (n, s))."""
        import multiprocessing as mp
        self.workers = workers or len(os.sched_getaffinity(0))
        self.tmp = tempfile.TemporaryDirectory(prefix="ivfpq_cpu_")
        for name in ("coarse", "centers", "off", "ids", "codes"):
            np.save(os.path.join(self.tmp.name, name + ".npy"), arrays[name])
        self.pool = mp.get_context("spawn").Pool(self.workers, initializer=_init, initargs=(self.tmp.name,))
        # warm every worker (imports + index load) outside any timed sample
        d = arrays["coarse"].shape[1]
        self.pool.map(_work, [(np.zeros((1, d), np.float32), 1, 1, "f32")] * self.workers)

    def run(self, queries: np.ndarray, k: int, nprobe: int, prec: str):
        """Returns (qps, ids, wall_s) for the sample, split evenly over workers."""
        shards = [s for s in np.array_split(queries, self.workers) if s.shape[0]]
        t0 = time.perf_counter()
        res = self.pool.map(_work, [(s, k, nprobe, prec) for s in shards])
        wall = time.perf_counter() - t0
        ids = np.concatenate([r[0] for r in res])
        return queries.shape[0] / wall, ids, wall

    def size_for(self, queries: np.ndarray, k: int, nprobe: int, prec: str, seconds: float) -> int:
        """Query count that takes about `seconds` of wall time, from a short
        pilot run (4 queries per worker); clamped to [workers, len(queries)]."""
        pilot = queries[:4 * self.workers]
        qps, _, _ = self.run(pilot, k, nprobe, prec)
        return int(min(queries.shape[0], max(self.workers, qps * seconds)))

    def close(self):
        self.pool.terminate()
        self.tmp.cleanup()
