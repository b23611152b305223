#!/bin/bash
# ncu --set full of the deterministic dual insert (k_dual_rounds) at lambda $1 (tools/prof_dual.py, workers 1)
set -u
O=gpurun_out/dualcap
mkdir -p "$O" /tmp/cap
L=${1:-1.0}
timeout 900 ncu --nvtx --nvtx-include "prof/" --set full --clock-control none --import-source on \
  -o /tmp/cap/dr_$L -f python tools/prof_dual.py $L 1 > "$O/log_$L.txt" 2>&1
ncu -i /tmp/cap/dr_$L.ncu-rep --page raw --csv > "$O/ncu_dual_rounds_${L}_raw.csv" 2>/dev/null
ncu -i /tmp/cap/dr_$L.ncu-rep --page source --csv --kernel-name "regex:k_dual_rounds" > /tmp/cap/src_dr.csv 2>/dev/null &&
  python tools/ncu_src_top.py /tmp/cap/src_dr.csv 25 > "$O/src_top_k_dual_rounds_$L.txt" 2>&1
echo done
