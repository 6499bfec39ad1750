"""Times the scan kernel alone (CUDA events, L2 flushed) for the given LUT
dtypes on a BASELINE config; used for kernel experiments."""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--dtypes", nargs="+", default=["e5m3"])
    ap.add_argument("--nprobe", type=int, default=None)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--scan-mode", type=int, default=0, help="ivfpq_set_scan_kernel mode (2: prefer row chunks)")
    a = ap.parse_args()
    import numpy as np
    import torch
    from harness import workload as W
    from paper_2301_06672_b200 import _lib
    from paper_2301_06672_b200.index import DeviceIndex
    cfg = W.CONFIGS[a.config]
    cache = f"/tmp/ivfpq_ts_{a.config}.npz"   # same-call reuse across library variants
    if os.path.exists(cache):
        from paper_2301_06672_b200.index import IvfPqIndex, PQCodebook
        z = np.load(cache)
        idx = IvfPqIndex.from_csr(z["coarse"], PQCodebook(centers=z["centers"], p=cfg["p"]), z["off"], z["ids"],
                                  z["codes"])
        queries = z["queries"]
        del z
    else:
        base, queries = W.make_data(cfg)
        arr = W.build_arrays(cfg, base, W.DEFAULT_BUILDER.get(a.config, "gpu"))   # the bench's index
        del base
        idx = W.to_index(arr, cfg["p"])
        np.save(cache.replace(".npz", "_q.npy"), queries)
        np.savez(cache, queries=queries, **arr)
    _lib.check(_lib.lib.ivfpq_set_scan_kernel(a.scan_mode))
    dev = DeviceIndex(idx, 0)
    q = torch.from_numpy(queries).cuda()
    k, P = cfg["k"], a.nprobe or cfg["nprobe"]
    nq = q.shape[0]
    st = torch.cuda.current_stream().cuda_stream
    keys = torch.empty((nq, P), dtype=torch.int64, device="cuda")
    okeys = torch.empty((nq, k), dtype=torch.int64, device="cuda")
    ncand = torch.empty(nq, dtype=torch.int64, device="cuda")
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib.ivfpq_select_device(dev.handle, q.data_ptr(), nq, P, keys.data_ptr(), st))
    for prec in a.dtypes:
        ts = []
        for r in range(a.reps + 1):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _lib.check(_lib.lib.ivfpq_scan_device(dev.handle, q.data_ptr(), nq, keys.data_ptr(), P, k,
                                                  _lib.LUT_CODES[prec], okeys.data_ptr(), ncand.data_ptr(), st))
            e1.record()
            e1.synchronize()
            if r:
                ts.append(e0.elapsed_time(e1))
        print(f"{a.config} {prec} nprobe {P} mode {a.scan_mode}: scan {np.mean(ts):.3f} ms (min {np.min(ts):.3f})",
              flush=True)


if __name__ == "__main__":
    main()
