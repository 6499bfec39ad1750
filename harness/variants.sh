#!/bin/bash
# Times the scan kernel for each library variant in harness/variants/ (plus
# the in-tree build) on cfg2.  Usage (on the box): bash harness/variants.sh [dtypes...]
D=${@:-e5m3 f16 f32}
echo "== base"; timeout 90 python harness/time_scan.py --reps 5 --dtypes $D 2>&1 | grep scan
for f in harness/variants/*.so; do
  echo "== $f"; IVFPQ_LIB=$PWD/$f timeout 90 python harness/time_scan.py --reps 5 --dtypes $D 2>&1 | grep scan
done
