#!/bin/bash
# Warp layout A vs B and the scanners' L2 prefetch on one config (scan kernel
# alone, harness/time_scan.py).  On the box: CFG=cfg3p8 bash harness/ab_cfg3.sh [dtypes...]
D=${@:-e5m3 f16}
C=${CFG:-cfg3p8}
for m in 3 4; do for spf in 0 1; do
  echo "== scan-mode $m spf $spf"
  IVFPQ_WS_SPF=$spf timeout 600 python harness/time_scan.py --config $C --reps 3 --scan-mode $m --dtypes $D 2>&1 | grep -v "^\[build"
done; done
