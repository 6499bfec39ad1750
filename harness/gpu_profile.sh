#!/bin/bash
# One GPU call: bench line, launch list of the bench command, ncu --set full
# of the scan kernel (e5m3, f16, f32) and the tensor-core coarse kernel.
# Usage (on the box): bash harness/gpu_profile.sh <tag>
set -x
TAG=${1:-r01}
O=gpurun_out
mkdir -p $O
timeout 600 python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'ivfpq|scan_ws|coarse|ws_plan|merge_keys|finalize' -c 400 --csv \
  --log-file $O/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --quick --no-cpu > $O/ncu_launch_$TAG.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'scan_ws_kernel|coarse_tc_kernel' -c 4 \
  -o $O/full_$TAG -f python -m harness.profile_run --config cfg2 --dtypes e5m3 f16 f32 --reps 1 > $O/ncu_full_$TAG.log 2>&1
ls -la $O
