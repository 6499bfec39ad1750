#!/bin/bash
# Builds scan-kernel variants into harness/variants/ (make variant, in parallel).
# Usage: bash harness/variants_build.sh name1 "-DFLAG..." [name2 "-DFLAG..." ...]
cd "$(dirname "$0")/../paper_2301_06672_b200/csrc"
rm -f ../../harness/variants/*.so
while [ $# -ge 2 ]; do
  ( make -s -j5 variant VAR=$1 EXTRA="$2" > /tmp/var_$1.log 2>&1 || { echo "variant $1 failed"; tail -5 /tmp/var_$1.log; } ) &
  shift 2
done
wait
rm -rf build_*/
ls -la ../../harness/variants/
