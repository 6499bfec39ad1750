#!/bin/bash
# Sweep of the scan kernel's LUT pipeline shape (LUT budget -> G lists per job, NBUF slots) on cfg2.
export IVFPQ_WS_PLAN_PRINT=1
D=${DTYPES:-e5m3}
for cfg in "64 0" "48 4" "48 3" "32 6" "32 4" "32 3" "16 6" "80 2" "64 2"; do
  set -- $cfg
  IVFPQ_LUT_BUDGET_KB=$1 IVFPQ_WS_NBUF=$2 timeout 100 python harness/time_scan.py --reps 3 --dtypes $D 2>&1 \
    | grep -E "plan|scan" | tr '\n' ' '; echo " [budget=$1 nbuf=$2]"
done
