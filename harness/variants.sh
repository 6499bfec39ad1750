#!/bin/bash
# Times the scan kernel for each library variant in harness/variants/ (plus
# the in-tree build) on a config.  Usage (on the box):
#   CFG=cfg5 bash harness/variants.sh [dtypes...]
D=${@:-e5m3 f16 f32}
C=${CFG:-cfg2}
echo "== base"; timeout 600 python harness/time_scan.py --config $C --reps 5 --dtypes $D 2>&1 | grep scan
for f in harness/variants/*.so; do
  echo "== $f"; IVFPQ_LIB=$PWD/$f timeout 300 python harness/time_scan.py --config $C --reps 5 --dtypes $D 2>&1 | grep scan
done
