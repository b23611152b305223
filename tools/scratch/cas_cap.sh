#!/bin/bash
# ncu --set full of the CAS engine's dual insert at lambda 1.0 (tools/prof_dual.py)
set -u
O=gpurun_out/cas
mkdir -p "$O" /tmp/cap
L=${1:-1.0}
timeout 900 ncu --nvtx --nvtx-include "prof/" --set full --clock-control none --import-source on \
  -o /tmp/cap/dual_$L -f python tools/prof_dual.py $L 8 > "$O/log_$L.txt" 2>&1
ncu -i /tmp/cap/dual_$L.ncu-rep --page raw --csv > "$O/ncu_dual_cas_${L}_raw.csv" 2>/dev/null
ncu -i /tmp/cap/dual_$L.ncu-rep --page source --csv --kernel-name "regex:k_cas" > /tmp/cap/src_cas.csv 2>/dev/null &&
  python tools/ncu_src_top.py /tmp/cap/src_cas.csv 25 > "$O/src_top_k_cas_$L.txt" 2>&1
echo done
ncu -i /tmp/cap/dual_$L.ncu-rep --page source --print-source cuda,sass --csv --kernel-name "regex:k_cas" > /tmp/cap/srcl_cas.csv 2>/dev/null &&
  python tools/ncu_cuda_lines.py /tmp/cap/srcl_cas.csv 40 > "$O/cuda_lines_k_cas_$L.txt" 2>&1
