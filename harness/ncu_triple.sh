#!/bin/bash
# The ncu evidence north_star asks for, on the scan kernel of the bench's index:
#   shared-memory bank conflicts and wavefronts per LD for the f32 / f16 / e5m3
#   (+ e4m4) LUTs, DRAM bytes, issue activity and instruction counts.
# One ncu pass per config (metrics only, not --set full).  On the box:
#   bash harness/ncu_triple.sh cfg2 [nprobe]   -> gpurun_out/triple_<cfg>.csv
CFG=${1:-cfg2}; NP=${2:-}
O=gpurun_out; mkdir -p $O
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
M=$M,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum
M=$M,smsp__sass_inst_executed_op_shared_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum
M=$M,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum
ARGS="--config $CFG --dtypes f32 f16 e5m3 e4m4 --reps 1 ${NP:+--nprobe $NP}"
timeout 1200 python -m harness.profile_run $ARGS > $O/triple_${CFG}_plain.log 2>&1 && \
timeout 1500 ncu --metrics $M --clock-control none -k regex:scan_ws_kernel --csv \
  --log-file $O/triple_${CFG}${NP:+_p$NP}.csv python -m harness.profile_run $ARGS > $O/triple_${CFG}_ncu.log 2>&1
tail -2 $O/triple_${CFG}_ncu.log
