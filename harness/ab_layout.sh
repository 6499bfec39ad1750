#!/bin/bash
# Warp layout A (scan-mode 3) vs B (scan-mode 4) on one config, scan kernel
# alone (harness/time_scan.py).  On the box: CFG=cfg3p8 bash harness/ab_layout.sh [dtypes...]
D=${@:-e5m3 f16}
C=${CFG:-cfg3p8}
for m in 3 4; do
  echo "== scan-mode $m"
  timeout 600 python harness/time_scan.py --config $C --reps 3 --scan-mode $m --dtypes $D 2>&1 | grep -v "^\[build"
done
