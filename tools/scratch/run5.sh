timeout 900 python -m pytest tests/test_gpu_boundary.py -x -q 2>&1 | tail -1
for v in old new old new; do
  if [ $v = old ]; then export HKV_LIB=tools/scratch/lib_old.so; else unset HKV_LIB; fi
  python bench.py --no-e2e --no-cpu-baseline --no-extras 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['value'], [(k, round(v['find_ms'],4), round(v['insert_ms'],4)) for k,v in d['breakdown'].items()])"
done
