#!/bin/bash
# Round-2 closing capture on the B200 (from the repo root):
#   gpurun --timeout 3000 -- 'bash tools/capture_r02b.sh'
# writes gpurun_out/final2/ (copied to profiles/r02/final2/ afterwards)
set -u
O=gpurun_out/final2
mkdir -p "$O" /tmp/cap
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -3 > "$O/gpu_tests.txt"
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > "$O/smoke.txt" 2>&1
python bench.py > "$O/bench.json" 2> "$O/bench.err"
python bench.py --impl reference --steps 2 --warmup 3 > "$O/bench_ref.json" 2>> "$O/bench.err"
timeout 300 python tools/dual_time.py dual,single > "$O/dual_time.json" 2>> "$O/bench.err"
# launch list of the bench's timed region (cold, serialised: shares, not absolutes)
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file "$O/launches.csv" python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-extras > /dev/null 2>&1
for L in 0.5 1.0; do
  timeout 900 ncu --nvtx --nvtx-include "prof/" --set full --clock-control none --import-source on \
    -o /tmp/cap/c2_$L -f python tools/prof_c2.py $L > /dev/null 2>&1
  ncu -i /tmp/cap/c2_$L.ncu-rep --page raw --csv > "$O/ncu_c2_${L}_raw.csv" 2>/dev/null
  for K in k_find_fused k_meta_tps k_values_write; do
    ncu -i /tmp/cap/c2_$L.ncu-rep --page source --csv --kernel-name "regex:$K" > /tmp/cap/src_$K.csv 2>/dev/null &&
      python tools/ncu_src_top.py /tmp/cap/src_$K.csv 12 > "$O/src_top_${K}_$L.txt" 2>&1
  done
done
python tools/traffic_from_ncu.py "$O/ncu_c2_0.5_raw.csv" "$O/ncu_c2_1.0_raw.csv" > "$O/traffic.json"
echo done > "$O/DONE"
