"""Generator calibration probe (SURVEY.md 8d "the component count decides
whether recall responds to nprobe -- calibrate it"), run on the GPU box:

for a BASELINE config shape and candidate (components, spread) pairs, build
the index (product GPU builder), exact ground truth (K7) for a query sample,
and report per nprobe the IVF ceiling (fraction of the true top-10 whose list
is probed) and recall@10 for the f32 and e5m3 LUTs.

  python -m harness.calibrate --config cfg5 --cand 1024:0.3 262144:0.1 --nprobe 16 64 256
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--cand", nargs="+", required=True, help="comps:spread pairs")
    ap.add_argument("--nprobe", nargs="+", type=int, default=[8, 16, 32, 64, 128])
    ap.add_argument("--nq", type=int, default=1000)
    ap.add_argument("--out", default="gpurun_out/calibration.jsonl")
    a = ap.parse_args()
    import paper_2301_06672_b200 as pkg
    from harness import workload as W
    for cand in a.cand:
        comps, spread = cand.split(":")
        cfg = dict(W.CONFIGS[a.config], comps=int(comps), spread=float(spread))
        t0 = time.time()
        cfg_n = dict(cfg, nq=a.nq)
        base, queries = W.make_data(cfg_n)
        td = time.time()
        arr = W.build_arrays(cfg, base, "gpu")
        t1 = time.time()
        gt = W.ground_truth_gpu(base, queries, 10)
        print(f"[cal] data {td - t0:.1f}s build {t1 - td:.1f}s gt {time.time() - t1:.1f}s", file=sys.stderr, flush=True)
        del base
        idx = W.to_index(arr, cfg["p"])
        list_of = np.empty(cfg["n"], dtype=np.int64)
        list_of[arr["ids"]] = np.repeat(np.arange(cfg["nlist"]), np.diff(arr["off"]))
        sizes = np.diff(arr["off"])
        row = {"config": a.config, "comps": int(comps), "spread": float(spread), "build_s": round(t1 - t0, 1),
               "list_len": [int(sizes.min()), int(np.median(sizes)), int(sizes.max())], "P": {}}
        for P in a.nprobe:
            probes = np.empty((queries.shape[0], P), dtype=np.int64)
            h = pkg.device_index(idx)
            pkg._lib.check(pkg._lib.lib.ivfpq_select_clusters(h.handle, queries.ctypes.data, queries.shape[0], P,
                                                              probes.ctypes.data))
            ceil = float(np.mean([np.isin(list_of[gt[i]], probes[i]).mean() for i in range(gt.shape[0])]))
            r = {"ivf_ceiling": round(ceil, 4)}
            for prec in ("f32", "e5m3"):
                lists, _ = pkg.search_batch(idx, queries, pkg.SearchParams(k=10, nprobe=P, precision=prec))
                r[prec] = round(W.recall_at(lists.ids, gt), 4)
            row["P"][P] = r
        print(json.dumps(row), flush=True)
        os.makedirs(os.path.dirname(a.out), exist_ok=True)
        with open(a.out, "a") as f:
            f.write(json.dumps(row) + "\n")


if __name__ == "__main__":
    main()
