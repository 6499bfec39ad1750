#!/bin/bash
# Sweep of the scan kernel's pipeline depths (LUT budget -> G, LUT slots, code stages) on cfg2.
export IVFPQ_WS_PLAN_PRINT=1
for cfg in "64 0 0" "48 3 2" "48 0 0" "32 4 2" "32 5 3" "32 0 0" "64 2 2" "80 0 0"; do
  set -- $cfg
  IVFPQ_LUT_BUDGET_KB=$1 IVFPQ_WS_NBUF=$2 IVFPQ_WS_SD=$3 timeout 100 python harness/time_scan.py --reps 3 2>&1 \
    | grep -E "plan|scan" | tr '\n' ' '; echo " [budget=$1 nbuf=$2 sd=$3]"
done
