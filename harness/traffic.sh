#!/bin/bash
# DRAM traffic (read + write bytes) of one scan_ws_kernel launch per LUT dtype,
# on the index bench.py builds for the config.  Run on the box:
#   bash harness/traffic.sh cfg2 [nprobe] -> gpurun_out/traffic_<cfg>.csv
CFG=${1:-cfg2}; NP=${2:-}
O=gpurun_out; mkdir -p $O
ARGS="--config $CFG --dtypes f32 f16 e5m3 e4m4 --reps 1 ${NP:+--nprobe $NP}"
timeout 900 python -m harness.profile_run $ARGS > $O/traffic_${CFG}_plain.log 2>&1 && \
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:scan_ws_kernel --csv --log-file $O/traffic_${CFG}${NP:+_p$NP}.csv python -m harness.profile_run $ARGS \
  > $O/traffic_${CFG}_ncu.log 2>&1
tail -2 $O/traffic_${CFG}_ncu.log
