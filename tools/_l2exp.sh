for v in unset 32 64 128; do
  if [ $v = unset ]; then unset HKV_L2_FETCH; else export HKV_L2_FETCH=$v; fi
  echo "== $v"
  python tools/stage_times.py 27 0.5 2>&1 | grep -v Warn
  ncu --nvtx --nvtx-include "prof/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/prof_c2.py 0.5 > gpurun_out/l2_$v.csv 2>/dev/null
done
