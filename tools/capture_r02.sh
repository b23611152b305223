#!/bin/bash
# Round-2 capture on the B200 (run through gpurun from the repo root):
#   gpurun --timeout 2400 -- 'bash tools/capture_r02.sh'
# writes gpurun_out/r02/: the bench's timed-region launch list (cold,
# serialised: shares, not absolutes), one ncu --set full capture of the C2
# find + insert pair at lambda 0.5 and 1.0 (raw metrics + per-kernel source
# hot spots), and traffic.json (DRAM bytes per launch for bench.py's roofline).
set -u
O=gpurun_out/r02
mkdir -p "$O" /tmp/cap
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file "$O/launches.csv" python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
for L in 0.5 1.0; do
  timeout 900 ncu --nvtx --nvtx-include "prof/" --set full --clock-control none --import-source on \
    -o /tmp/cap/c2_$L -f python tools/prof_c2.py $L > /dev/null 2>&1
  ncu -i /tmp/cap/c2_$L.ncu-rep --page raw --csv > "$O/ncu_c2_${L}_raw.csv" 2>/dev/null
  for K in k_find_fused k_meta_tps k_values_write k_scatter k_segfin; do
    ncu -i /tmp/cap/c2_$L.ncu-rep --page source --csv --kernel-name "regex:$K" > /tmp/cap/src_$K.csv 2>/dev/null &&
      python tools/ncu_src_top.py /tmp/cap/src_$K.csv 12 > "$O/src_top_${K}_$L.txt" 2>&1
  done
done
python tools/traffic_from_ncu.py "$O/ncu_c2_0.5_raw.csv" "$O/ncu_c2_1.0_raw.csv" > "$O/traffic.json"
echo done > "$O/DONE"
