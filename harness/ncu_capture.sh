#!/bin/bash
# One ncu --set full capture of the scan kernel on the box, exported to small
# CSVs (raw metrics + SASS source page) so gpurun_out stays under its 64 MiB
# copy-back limit.  Usage: bash harness/ncu_capture.sh <tag> <profile_run args...>
TAG=$1; shift
O=gpurun_out; mkdir -p $O
timeout 900 python -m harness.profile_run "$@" > $O/${TAG}_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:scan_ws_kernel -c 1 -o /tmp/${TAG} -f \
  python -m harness.profile_run "$@" > $O/${TAG}_ncu.log 2>&1
ncu -i /tmp/${TAG}.ncu-rep --page raw --csv > $O/${TAG}_raw.csv 2>/dev/null
ncu -i /tmp/${TAG}.ncu-rep --page source --csv --print-source sass > $O/${TAG}_src.csv 2>/dev/null
ls -la $O/${TAG}_*
