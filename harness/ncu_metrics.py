"""Parse the ncu metric CSVs of harness/ncu_triple.sh (HERE, no GPU) into

* profiles/scan_traffic.json: per-launch DRAM bytes (read + write) of
  scan_ws_kernel keyed "<cfg>/nprobe<P>/<dtype>" (bench.py's roofline.traffic);
* a summary table: time, issue activity, shared-memory wavefronts per LD
  instruction and bank conflicts per LUT dtype, DRAM and L2 bytes, compared
  with the reference bank model's expected wavefronts for random 256-entry
  gathers (bankmodel.py:96-118 via SURVEY.md 8d: f32 3.15, f16 2.78, fp8 2.00).

  python harness/ncu_metrics.py gpurun_out/triple_cfg2.csv --config cfg2 --nprobe 32 [--update]
"""

from __future__ import annotations

import argparse
import csv
import json
import os
import re
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DT_OF = {"0": "f32", "1": "f16", "2": "e5m3", "3": "e4m4"}   # scan_ws_kernel<DT, ...>
BANK_MODEL = {"f32": 3.15, "f16": 2.78, "e5m3": 2.00, "e4m4": 2.00}


def load(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    per = defaultdict(dict)
    for r in rows:
        m = re.search(r"scan_ws_kernel<(?:WsCfg<[^>]*>, )?(\d+),", r["Kernel Name"])
        if not m:
            continue
        key = (r["ID"], DT_OF[m.group(1)])
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(unit, 1)
        per[key][r["Metric Name"]] = v * scale
    return per


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--config", required=True)
    ap.add_argument("--nprobe", type=int, required=True)
    ap.add_argument("--update", action="store_true", help="write profiles/scan_traffic.json")
    a = ap.parse_args()
    per = load(a.csv)
    out = {}
    print(f"# {a.config} nprobe {a.nprobe}: scan_ws_kernel, one launch per LUT dtype ({os.path.basename(a.csv)})")
    print(f"{'dtype':6s} {'ms':>8s} {'issue%':>7s} {'Ginst':>7s} {'wf/LD':>6s} {'model':>6s} {'conflicts':>11s} "
          f"{'DRAM GB':>8s} {'L2 GB':>8s}")
    for (kid, dt), m in sorted(per.items(), key=lambda kv: int(kv[0][0])):
        wf = m["l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum"] / m["smsp__sass_inst_executed_op_shared_ld.sum"]
        dram = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
        print(f"{dt:6s} {m['gpu__time_duration.sum']:8.3f} "
              f"{m['smsp__issue_active.avg.pct_of_peak_sustained_active']:7.1f} {m['smsp__inst_executed.sum'] / 1e9:7.3f} "
              f"{wf:6.2f} {BANK_MODEL[dt]:6.2f} {m['l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum'] / 1e6:10.1f}M "
              f"{dram / 1e9:8.3f} {m['lts__t_bytes.sum'] / 1e9:8.1f}")
        out[dt] = int(dram)
    if a.update:
        p = os.path.join(ROOT, "profiles", "scan_traffic.json")
        try:
            tr = json.load(open(p))
        except (OSError, ValueError):
            tr = {}
        tr = {k: v for k, v in tr.items() if "/" in k or k.startswith("_")}
        for dt, b in out.items():
            tr[f"{a.config}/nprobe{a.nprobe}/{dt}"] = {"bytes": b, "source": f"profiles/{os.path.basename(a.csv)}"}
        tr["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum of one scan_ws_kernel launch (bytes), measured by "
                       "ncu (harness/ncu_triple.sh) on the bench's index for the config / nprobe / LUT dtype")
        json.dump(tr, open(p, "w"), indent=1, sort_keys=True)
        print("updated", p)


if __name__ == "__main__":
    main()
