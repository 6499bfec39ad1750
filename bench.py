#!/usr/bin/env python
"""IVFPQ search benchmark: QPS at recall@10 per LUT dtype on B200 vs the CPU
reference algorithm (BASELINE.json metric, configs[1] = cfg2 by default).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one search of the whole query batch (10K queries at cfg2) through
coarse select (K1), per-(query, list) LUT build + fp8 encode (K2), code scan
(K3) and top-k merge (K4).  Inputs are resident in HBM for `value`; `e2e`
times the C-ABI host entry point (`ivfpq_search`) with pinned host buffers,
H2D of queries and D2H of results inside the timed region.  L2 is flushed
(256 MiB write) between timed steps.  N>1 (torchrun): lists are sharded over
the ranks, every rank searches the whole batch, top-k keys are merged with an
NCCL all-gather (strong scaling: total work fixed).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "QPS at recall@10 per LUT dtype (fp32/fp16/custom fp8), 1–8 B200 vs CPU"
PRECS = ["f32", "f16", "e5m3", "e4m4"]
THROTTLE_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
                 0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
                 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--nprobe", type=int, default=None)
    ap.add_argument("--dtype", default="e5m3", choices=PRECS)
    ap.add_argument("--cpu-sample", type=int, default=0, help="queries in the CPU baseline sample (0 = auto)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--sweep", action="store_true", help="also sweep nprobe 8..256 for every dtype")
    ap.add_argument("--quick", action="store_true", help="skip per-dtype table and roofline")
    ap.add_argument("--builder", choices=["cpu", "gpu"], default=None,
                    help="index builder (default: cpu at cfg1/cfg2, gpu above; the reference arm always uses cpu)")
    return ap.parse_args()


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------ clocks ----
class Clocks:
    """SM clock + clock-event reasons sampled DURING the timed region by an
    NVML thread (~1 kHz; the timed region is tens of ms, far below
    nvidia-smi's 200 ms polling period).  Idle samples are dropped."""

    def __init__(self):
        import threading
        self.rows = []
        self.stop_ev = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            idx = int(os.environ.get("LOCAL_RANK", "0"))
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            if vis and vis.split(",")[idx].strip().isdigit():
                idx = int(vis.split(",")[idx])
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # noqa: BLE001 -- no NVML: report null clocks
            log(f"[bench] NVML unavailable: {e}")
            self.nv = None
            return
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        nv, h = self.nv, self.h
        while not self.stop_ev.is_set():
            try:
                self.rows.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                                  nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.001)

    def stop(self):
        if self.nv is None:
            return None
        self.stop_ev.set()
        self.t.join()
        rows = self.rows
        if not rows:
            return None
        busy = [r for r in rows if not (r[1] & 0x1)] or rows
        reasons = set()
        for r in busy:
            for bit, name in THROTTLE_BITS.items():
                if r[1] & bit and bit != 0x1:
                    reasons.add(name)
        return {"sm_mhz": float(np.median([r[0] for r in busy])), "sm_max_mhz": int(self.max_mhz),
                "reasons": sorted(reasons), "samples": len(rows), "busy_samples": len(busy), "source": "nvml"}


# ---------------------------------------------------------------- workload ----
def load_workload(args, rank, world):
    """Rank 0 generates the data and builds the index arrays (untimed; the
    deterministic CPU builder at cfg1/cfg2, identical in both arms); other
    ranks load them from a shared temp dir.  Returns (cfg, arrays, base,
    queries)."""
    from harness import workload as W
    cfg = dict(W.CONFIGS[args.config])
    cfg["name"] = args.config
    cfg["builder"] = args.builder or W.DEFAULT_BUILDER.get(args.config, "gpu")
    shared = os.path.join(tempfile.gettempdir(), f"ivfpq_bench_{args.config}_{os.environ.get('MASTER_PORT', '0')}")
    base = None
    if rank == 0:
        t0 = time.time()
        base, queries = W.make_data(cfg)
        t1 = time.time()
        arr = W.build_arrays(cfg, base, cfg["builder"])
        log(f"[bench] data {t1 - t0:.1f}s, index build ({cfg['builder']}) {time.time() - t1:.1f}s")
        if world > 1:
            os.makedirs(shared, exist_ok=True)
            np.savez(os.path.join(shared, "w.npz"), queries=queries, **arr)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        if rank != 0:
            z = np.load(os.path.join(shared, "w.npz"))
            arr = {k: z[k] for k in ("coarse", "centers", "off", "ids", "codes")}
            queries = z["queries"]
        dist.barrier()
    cfg["digest"] = W.arrays_digest(arr, queries)
    return cfg, arr, base, queries


def workload_desc(cfg, nprobe, dtype):
    return (f"{cfg['name']}: {cfg['n'] // 1000}K x {cfg['d']} synthetic Gaussian mixture ({cfg['comps']} comps, "
            f"spread {cfg['spread']}), nlist {cfg['nlist']}, pq_dim {cfg['s']}, pq_bits {cfg['p']}, "
            f"nprobe {nprobe}, k {cfg['k']}, {cfg['nq']} queries, LUT {dtype}")


def config_dict(cfg, P, dtype, world):
    """The `config` object, identical in both arms (same_config)."""
    return {"workload": workload_desc(cfg, P, dtype), "n": cfg["n"], "d": cfg["d"], "nlist": cfg["nlist"],
            "pq_dim": cfg["s"], "pq_bits": cfg["p"], "nprobe": P, "k": cfg["k"], "queries": cfg["nq"], "lut": dtype,
            "parallelism": "single GPU" if world == 1 else f"lists sharded over {world} GPUs",
            "index": f"{cfg['builder']} builder (harness/workload.py), inputs sha1 {cfg['digest']}",
            "l2": "flushed between timed steps (256 MiB write)"}


# -------------------------------------------------------------- our arm -----
class Searcher:
    """1 GPU: ivfpq_search_device; N GPUs: list-sharded protocol over NCCL."""

    def __init__(self, idx, rank, world):
        import torch
        from paper_2301_06672_b200 import parallel
        from paper_2301_06672_b200.index import DeviceIndex
        self.torch = torch
        self.world = world
        self.idx = idx
        if world == 1:
            self.dev = DeviceIndex(idx, 0)
        else:
            off, _, _ = idx.csr()
            shards = parallel.shard_lists(np.diff(off), idx.cb.s, world)
            self.dev = DeviceIndex(idx, torch.cuda.current_device(), owned=shards[rank])
            self.ops = parallel.CudaShardOps(self.dev)
            self.gather = parallel.torch_all_gather()

    def search(self, q, k, nprobe, prec, out=None):
        from paper_2301_06672_b200 import parallel
        from paper_2301_06672_b200.search import SearchParams, search_device
        torch = self.torch
        if self.world == 1:
            if out is None:
                out = (torch.empty((q.shape[0], k), dtype=torch.int64, device=q.device),
                       torch.empty((q.shape[0], k), dtype=torch.float32, device=q.device),
                       torch.empty(q.shape[0], dtype=torch.int32, device=q.device))
            search_device(self.dev, q, SearchParams(k=k, nprobe=nprobe, precision=prec), *out)
            return out
        return parallel.sharded_search(self.ops, q, k, nprobe, prec, self.gather)


def timed_steps(fn, steps, flush, torch, world):
    """Per-step CUDA-event times (ms) with an L2 flush between steps; max over ranks."""
    import torch.distributed as dist
    times = []
    for _ in range(steps):
        flush()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    t = torch.tensor(times, dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.cpu().numpy()


def run_ours(args, rank, world):
    import torch
    import torch.distributed as dist
    from harness.workload import recall_at
    from paper_2301_06672_b200 import _lib

    from harness import workload as W
    cfg, arr, base, queries = load_workload(args, rank, world)
    gt = None
    if rank == 0:
        t0 = time.time()
        gt = W.ground_truth_gpu(base, queries, 10)   # K7, exact (datasets.py:179-201)
        log(f"[bench] ground truth {time.time() - t0:.1f}s")
    del base
    idx = W.to_index(arr, cfg["p"])
    P = args.nprobe or cfg["nprobe"]
    k = cfg["k"]
    nq = queries.shape[0]
    srch = Searcher(idx, rank, world)
    q_dev = torch.from_numpy(queries).cuda()
    flush_buf = torch.empty(64 << 20, dtype=torch.float32, device="cuda")   # 256 MiB > 126 MB L2

    def flush():
        flush_buf.zero_()

    out = None if world > 1 else srch.search(q_dev, k, P, args.dtype)
    step = lambda: srch.search(q_dev, k, P, args.dtype, out)
    for _ in range(args.warmup):
        res = step()
    torch.cuda.synchronize()
    n0 = _lib.launch_count()
    clocks = Clocks()
    times = timed_steps(step, args.steps, flush, torch, world)
    clk = clocks.stop()
    launches = _lib.launch_count() - n0
    res = step()
    ids = res[0].cpu().numpy()
    rec = recall_at(ids[:, :10], gt) if rank == 0 else 0.0
    ms = float(times.mean())
    value = nq / (ms / 1e3)

    # ---- e2e through the reference-facing host API (pinned host buffers)
    e2e = measure_e2e(srch, queries, k, P, args.dtype, args.steps, flush, torch, world)

    line = {"metric": METRIC, "value": round(value, 1), "unit": "queries/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": f"f32 accumulate, {args.dtype} LUT", "data": "synthetic",
            "impl": "ours", "config": config_dict(cfg, P, args.dtype, world),
            f"recall@10": round(rec, 4), "e2e": e2e, "gpu_launches": int(launches), "clocks": clk}

    if not args.quick:
        line["per_dtype"] = per_dtype(srch, q_dev, gt, k, P, flush, torch, world, nq)
        if world == 1:
            line["roofline"] = roofline(srch, idx, q_dev, k, P, args.dtype, flush, torch, args.config)
    if args.sweep:
        line["sweep"] = sweep(srch, q_dev, gt, k, flush, torch, world, nq, cfg["nlist"])
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(arr, queries, gt, k, P, args.dtype, args.cpu_sample)
    if rank == 0:
        print(json.dumps(line), flush=True)


def measure_e2e(srch, queries, k, P, prec, steps, flush, torch, world):
    from paper_2301_06672_b200 import _lib
    import torch.distributed as dist
    nq, d = queries.shape
    qh = torch.from_numpy(queries).pin_memory()
    oi = torch.empty((nq, k), dtype=torch.int64).pin_memory()
    od = torch.empty((nq, k), dtype=torch.float32).pin_memory()
    times = []
    for i in range(steps + 1):
        flush()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        if world == 1:
            ns = _lib.ctypes.c_int64()
            _lib.check(_lib.lib.ivfpq_search(srch.dev.handle, qh.data_ptr(), nq, k, P, _lib.LUT_CODES[prec],
                                             oi.data_ptr(), od.data_ptr(), _lib.ctypes.byref(ns)))
        else:
            qd = qh.cuda(non_blocking=True)
            ids, dists, short = srch.search(qd, k, P, prec)
            oi.copy_(ids, non_blocking=True)
            od.copy_(dists, non_blocking=True)
            torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if i > 0:   # first call absorbs scratch allocation
            times.append(dt)
    t = torch.tensor(times, dtype=torch.float64)
    if world > 1:
        t = t.cuda()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t = t.cpu()
    mean = float(t.mean())
    return {"value": round(nq / mean, 1), "unit": "queries/s", "h2d_bytes_per_step": int(nq * d * 4),
            "d2h_bytes_per_step": int(nq * k * 12 + (nq * 4 if world == 1 else 0)),
            "ms_per_step": round(mean * 1e3, 4), "api": "ivfpq_search (C ABI, host buffers)" if world == 1
            else "sharded_search (torch.distributed NCCL) + host copies"}


def per_dtype(srch, q_dev, gt, k, P, flush, torch, world, nq, steps=3):
    """QPS and recall@10 per LUT dtype at the same nprobe (recall on rank 0)."""
    from harness.workload import recall_at
    out = {}
    for prec in PRECS:
        try:
            o = None if world > 1 else srch.search(q_dev, k, P, prec)
        except ValueError as e:   # e.g. an f32 LUT that does not fit shared memory (cfg3 p8: 240 KiB)
            out[prec] = {"unsupported": str(e)[:160]}
            continue
        fn = lambda: srch.search(q_dev, k, P, prec, o)
        res = fn()
        torch.cuda.synchronize()
        t = timed_steps(fn, steps, flush, torch, world)
        res = fn()
        out[prec] = {"qps": round(nq / (float(t.mean()) / 1e3), 1), "ms": round(float(t.mean()), 4),
                     "recall@10": round(recall_at(res[0].cpu().numpy()[:, :10], gt), 4) if gt is not None else None}
    return out


def sweep(srch, q_dev, gt, k, flush, torch, world, nq, nlist):
    out = {}
    for P in [8, 16, 32, 64, 128, 256]:
        if P > nlist:
            continue
        out[str(P)] = per_dtype(srch, q_dev, gt, k, P, flush, torch, world, nq, steps=2)
    return out


def roofline(srch, idx, q_dev, k, P, prec, flush, torch, cfg_name):
    """Dominant kernel = the scan kernel (K2+K3+K4).  Algorithmic bytes per
    launch = sum over queries of the code bytes of the lists actually probed
    (SURVEY.md 8d): B = sum_q sum_{c in probes(q)} L_c * pq_dim."""
    from paper_2301_06672_b200 import _lib
    nq = q_dev.shape[0]
    st = torch.cuda.current_stream().cuda_stream
    keys = torch.empty((nq, P), dtype=torch.int64, device="cuda")
    okeys = torch.empty((nq, k), dtype=torch.int64, device="cuda")
    ncand = torch.empty(nq, dtype=torch.int64, device="cuda")
    sel = lambda: _lib.check(_lib.lib.ivfpq_select_device(srch.dev.handle, q_dev.data_ptr(), nq, P,
                                                          keys.data_ptr(), st))
    scan = lambda: _lib.check(_lib.lib.ivfpq_scan_device(srch.dev.handle, q_dev.data_ptr(), nq, keys.data_ptr(),
                                                         P, k, _lib.LUT_CODES[prec], okeys.data_ptr(),
                                                         ncand.data_ptr(), st))
    sel()
    scan()
    torch.cuda.synchronize()
    t_sel = timed_steps(sel, 3, flush, torch, 1).mean()
    t_scan = timed_steps(scan, 3, flush, torch, 1).mean()
    off, _, _ = idx.csr()
    lens = torch.from_numpy(np.diff(off)).cuda()
    gid = keys & 0xFFFFFFFF
    B = float(lens[gid].sum().item()) * idx.cb.s
    achieved = B / (t_scan / 1e3) / 1e9
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    # DRAM bytes (read + write) of ONE scan launch, measured by ncu on this
    # config, nprobe and dtype (profiles/scan_traffic.json, with the capture
    # it came from); null when no capture exists for this exact workload
    traffic, traffic_src = None, None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "scan_traffic.json")))
        ent = tr.get(f"{cfg_name}/nprobe{P}/{prec}")
        if ent:
            traffic, traffic_src = ent["bytes"], ent["source"]
    except (OSError, ValueError, KeyError):
        pass
    return {"bound": "hbm", "kernel": f"scan_ws_kernel<{prec}> (K2 LUT build + K3 scan + K4 top-k)",
            "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
            "traffic": traffic, "traffic_source": traffic_src, "algorithmic_bytes_per_launch": int(B),
            "scan_ms": round(float(t_scan), 4),
            "select_ms": round(float(t_sel), 4),
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if "hbm_gbs" in peaks else "fallback 6.65 TB/s"}


def cpu_baseline(arr, queries, gt, k, P, prec, n_sample):
    from harness.cpu_baseline import CpuBaseline
    from harness.workload import recall_at
    cb = CpuBaseline(arr)
    n = n_sample or cb.size_for(queries, k, P, prec, seconds=20.0)  # pilot underestimates QPS ~2x
    qps, ids, wall = cb.run(queries[:n], k, P, prec)
    cb.close()
    return {"value": round(qps, 2), "unit": "queries/s", "cores": cb.workers, "kind": "port",
            "sample": f"first {n} of the {queries.shape[0]} queries, {prec} LUT, nprobe {P}, k {k}; oracle/ivfpq_np "
                      f"(numpy restatement of search.py:158-203) in {cb.workers} single-thread worker processes",
            "wall_s": round(wall, 2), "recall@10": round(recall_at(ids[:, :10], gt[:n]), 4)}


# --------------------------------------------------------- reference arm ----
def run_reference(args, rank, world):
    """The reference's CPU algorithm (oracle port of search.py) on the box's
    host cores, same workload / metric / config; rank 0 only.  Its inputs come
    from the CPU builder (numpy + host BLAS): this process never loads the
    product library."""
    if rank != 0:
        return
    from harness import cpu_build
    from harness.cpu_baseline import CpuBaseline
    from harness.workload import recall_at
    args.builder = "cpu"
    cfg, arr, base, queries = load_workload(args, 0, 1)
    P = args.nprobe or cfg["nprobe"]
    k = cfg["k"]
    cb = CpuBaseline(arr)
    # each step is a bounded sample sized so the whole run is ~90 s of host time
    n = args.cpu_sample or cb.size_for(queries, k, P, args.dtype, seconds=90.0 / (args.warmup + args.steps))
    nq = queries.shape[0]
    total_q, total_t, hits = 0, 0.0, []
    for i in range(args.warmup + args.steps):
        rows = (i * n + np.arange(n)) % nq
        qps, ids, wall = cb.run(queries[rows], k, P, args.dtype)
        if i >= args.warmup:
            total_q += rows.size
            total_t += wall
            hits.append((rows, ids[:, :10]))
    cb.close()
    # recall on the timed rows: exact ground truth on the CPU (datasets.py:179-201)
    rows = np.concatenate([h[0] for h in hits])
    uniq, inv = np.unique(rows, return_inverse=True)
    gt = cpu_build.ground_truth_cpu(base, queries[uniq], 10)[inv]
    rec = recall_at(np.concatenate([h[1] for h in hits]), gt)
    value = total_q / total_t
    line = {"metric": METRIC, "value": round(value, 2), "unit": "queries/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(1e3 * total_t / args.steps, 2), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": f"f32 accumulate, {args.dtype} LUT",
            "data": "synthetic", "impl": "reference", "config": config_dict(cfg, P, args.dtype, world),
            "recall@10": round(float(rec), 4),
            "cpu_baseline": {"value": round(value, 2), "unit": "queries/s", "cores": cb.workers, "kind": "port",
                             "sample": f"{n} queries per step, oracle/ivfpq_np (numpy restatement of the reference "
                                       f"search_batch, search.py:187-203) in {cb.workers} single-thread processes"},
            "e2e": {"value": round(value, 2), "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def spawn_ranks(n):
    """`bench.py --gpus N` outside torchrun: re-launch this command as N ranks
    (one per GPU) under torch.distributed.run on 127.0.0.1."""
    import socket
    import subprocess
    import torch
    have = torch.cuda.device_count()
    if have < n:
        log(f"[bench] --gpus {n} needs {n} CUDA devices, found {have}")
        sys.exit(1)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.run(cmd).returncode)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        spawn_ranks(args.gpus)
    if args.impl == "reference":
        run_reference(args, rank, world)   # rank 0 only; no process group needed
        return
    import torch
    if world > 1:
        import torch.distributed as dist
        lr = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(lr)
        dist.init_process_group("nccl", device_id=torch.device("cuda", lr))
    run_ours(args, rank, world)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
