#!/bin/bash
# Sweep of the scan kernel's LUT pipeline shape (LUT budget -> G lists per job,
# NBUF slots) on a config (default cfg2).  Usage: DTYPES="e5m3 f16" bash harness/sweep_scan.sh [cfg]
CFG=${1:-cfg2}
D=${DTYPES:-e5m3}
for cfg in "64 0" "48 0" "32 0" "64 2" "48 3"; do
  set -- $cfg
  echo -n "[budget=$1 nbuf=$2] "
  IVFPQ_LUT_BUDGET_KB=$1 IVFPQ_WS_NBUF=$2 timeout 120 python harness/time_scan.py --config $CFG --reps 3 --dtypes $D 2>&1 \
    | grep -E "scan" | tr '\n' ' '; echo
done
