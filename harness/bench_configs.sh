#!/bin/bash
# bench.py lines for several BASELINE configs (one process each); on the box:
#   bash harness/bench_configs.sh <tag> cfg4 cfg5 ...  -> gpurun_out/<tag>_bench_<cfg>.json
TAG=$1; shift
O=gpurun_out; mkdir -p $O
for C in "$@"; do
  timeout 1500 python bench.py --config $C > $O/${TAG}_bench_$C.json 2> $O/${TAG}_bench_$C.err
  echo "$C rc=$?"; tail -c 600 $O/${TAG}_bench_$C.json; echo
done
