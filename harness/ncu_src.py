"""Summarise an ncu report of the scan kernel (run HERE on the CPU box):
headline metrics, per-region executed-instruction histogram of the SASS
(with stall samples) and the opcode mix of the hottest regions.

  python harness/ncu_src.py gpurun_out/prof.ncu-rep [--kernel scan_ws] [--bucket 0x400]
  python harness/ncu_src.py gpurun_out/<tag>          (CSVs from harness/ncu_capture.sh)
"""

from __future__ import annotations

import argparse
import csv
import io
import re
import subprocess
from collections import Counter, defaultdict

METRICS = [
    "gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smsp__sass_inst_executed_op_shared_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_bytes.sum", "launch__registers_per_thread",
]


def ncu(*args) -> str:
    return subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout


def _page(rep: str, page: str) -> str:
    """A report's page as CSV text: from the .ncu-rep, or from the CSVs that
    harness/ncu_capture.sh exported next to it (<tag>_raw.csv / <tag>_src.csv)."""
    if rep.endswith(".ncu-rep"):
        args = ["-i", rep, "--page", page, "--csv"] + (["--print-source", "sass"] if page == "source" else [])
        return ncu(*args)
    return open(f"{rep}_{'raw' if page == 'raw' else 'src'}.csv").read()


def raw_metrics(rep: str, kernel: str) -> list[dict]:
    rows = list(csv.reader(io.StringIO(_page(rep, "raw"))))
    hdr = rows[0]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        if kernel in d.get("Kernel Name", ""):
            out.append(d)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--kernel", default="scan_ws")
    ap.add_argument("--bucket", type=lambda x: int(x, 0), default=0x400)
    ap.add_argument("--top", type=int, default=40)
    a = ap.parse_args()
    for d in raw_metrics(a.rep, a.kernel):
        print("==", d["Kernel Name"][:90])
        for m in METRICS:
            if m in d:
                print(f"   {m:62s} {d[m]}")
        st = {k: float(v.replace(",", "")) for k, v in d.items()
              if k.startswith("smsp__average_warp_latency_issue_stalled_") or
              k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
        tot = sum(st.values()) or 1.0
        top = sorted(st.items(), key=lambda kv: -kv[1])[:10]
        print("   stalls: " + ", ".join(f"{k.split('stalled_')[-1]} {v / tot * 100:.1f}%" for k, v in top))
    src = list(csv.reader(io.StringIO(_page(a.rep, "source"))))
    hdr = src[1]
    iI = hdr.index("Instructions Executed")
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in src[2:]:
        try:
            data.append((int(r[0], 16), r[1].strip(), float(r[iS] or 0), float(r[iI] or 0)))
        except (ValueError, IndexError):
            pass
    base = data[0][0]
    tot = sum(x[3] for x in data)
    tots = sum(x[2] for x in data) or 1.0
    print(f"== SASS: {len(data)} instructions, {tot / 1e6:.1f} M warp-instructions executed")
    b = defaultdict(lambda: [0.0, 0.0, Counter()])
    for addr, s, ss, ie in data:
        k = (addr - base) // a.bucket
        b[k][0] += ie
        b[k][1] += ss
        op = re.sub(r"^@!?U?P\w+\s+", "", s).split()[0] if s else "?"
        b[k][2][op] += ie
    for k in sorted(b):
        ie, ss, ops = b[k]
        if ie / tot > 0.004 or ss / tots > 0.004:
            mix = " ".join(f"{o}:{v / ie * 100:.0f}" for o, v in ops.most_common(5)) if ie else ""
            print(f"  {k * a.bucket:6x} {ie / tot * 100:6.2f}% inst {ss / tots * 100:6.2f}% samples  {mix}")


if __name__ == "__main__":
    main()
