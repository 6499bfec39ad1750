"""Small driver for ncu captures: builds a BASELINE config index (untimed),
then runs `--reps` batch searches per requested LUT dtype through the same
device entry point bench.py times.  Usage (on the GPU box):

  python -m harness.profile_run --config cfg2 --dtypes e5m3 f16 f32 --reps 2
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--dtypes", nargs="+", default=["e5m3"])
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--nprobe", type=int, default=None)
    ap.add_argument("--nq", type=int, default=0)
    ap.add_argument("--builder", choices=["cpu", "gpu"], default=None)
    a = ap.parse_args()
    import torch
    from harness import workload as W
    from paper_2301_06672_b200.index import DeviceIndex
    from paper_2301_06672_b200.search import SearchParams, search_device
    cfg = W.CONFIGS[a.config]
    base, queries = W.make_data(cfg)
    if a.nq:
        queries = queries[:a.nq]
    # the same index bench.py measures (its default builder for the config)
    idx = W.to_index(W.build_arrays(cfg, base, a.builder or W.DEFAULT_BUILDER.get(a.config, "gpu")), cfg["p"])
    del base
    dev = DeviceIndex(idx, 0)
    q = torch.from_numpy(queries).cuda()
    k, P = cfg["k"], a.nprobe or cfg["nprobe"]
    oi = torch.empty((q.shape[0], k), dtype=torch.int64, device="cuda")
    od = torch.empty((q.shape[0], k), dtype=torch.float32, device="cuda")
    osh = torch.empty(q.shape[0], dtype=torch.int32, device="cuda")
    for prec in a.dtypes:
        for _ in range(a.reps):
            search_device(dev, q, SearchParams(k=k, nprobe=P, precision=prec), oi, od, osh)
    torch.cuda.synchronize()
    print("profile_run done", a.config, a.dtypes, q.shape[0], "queries")


if __name__ == "__main__":
    main()
