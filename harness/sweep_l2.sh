#!/bin/bash
# Code-stream knobs of the scan kernel for code stores larger than L2: the
# scanners' L2 policy for code loads (IVFPQ_WS_POL 0 evict_last [default],
# 1 evict_normal, 2 evict_first) and the bulk-prefetch distance in rounds of
# pairs (IVFPQ_WS_PFD, default 2).  On the box: CFG=cfg5 bash harness/sweep_l2.sh [dtypes...]
D=${@:-e5m3}
C=${CFG:-cfg5}
run() { timeout 900 python harness/time_scan.py --config $C --reps 3 --dtypes $D 2>&1 | grep "scan "; }
for pol in 0 1 2; do echo "== pol $pol"; IVFPQ_WS_POL=$pol run; done
for pfd in 1 3 4; do echo "== pfd $pfd"; IVFPQ_WS_PFD=$pfd run; done
