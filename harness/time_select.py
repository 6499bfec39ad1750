"""Times K1 (coarse select) alone on a BASELINE config (CUDA events)."""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--nprobe", type=int, default=None)
    ap.add_argument("--mode", type=int, default=0, help="0 auto (tensor core), 1 SIMT, 2 TC + all re-done")
    a = ap.parse_args()
    import numpy as np
    import torch
    from harness import workload as W
    from paper_2301_06672_b200 import _lib
    from paper_2301_06672_b200.index import DeviceIndex, IvfPqIndex, PQCodebook
    cfg = W.CONFIGS[a.config]
    rng = np.random.default_rng(0)
    # K1 only needs the centroids: random unit-cube coarse + queries of the config's shape
    coarse = rng.random((cfg["nlist"], cfg["d"]), dtype=np.float32)
    queries = rng.random((cfg["nq"], cfg["d"]), dtype=np.float32)
    s, p = cfg["s"], cfg["p"]
    idx = IvfPqIndex.from_csr(coarse, PQCodebook(np.zeros((s, 1 << p, cfg["d"] // s), np.float32), p),
                              np.zeros(cfg["nlist"] + 1, np.int64), np.zeros(0, np.int64), np.zeros((0, s), np.uint8))
    dev = DeviceIndex(idx, 0)
    _lib.check(_lib.lib.ivfpq_set_select_kernel(a.mode))
    q = torch.from_numpy(queries).cuda()
    P = a.nprobe or cfg["nprobe"]
    keys = torch.empty((q.shape[0], P), dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    ts = []
    for r in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(_lib.lib.ivfpq_select_device(dev.handle, q.data_ptr(), q.shape[0], P, keys.data_ptr(), st))
        e1.record()
        e1.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    n = _lib.ctypes.c_int64()
    _lib.check(_lib.lib.ivfpq_debug_select_flagged(dev.handle, _lib.ctypes.byref(n)))
    print(f"{a.config} select nprobe {P} mode {a.mode}: {np.mean(ts):.3f} ms  flagged={n.value}")


if __name__ == "__main__":
    main()
