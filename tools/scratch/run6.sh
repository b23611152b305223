timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "dual" 2>&1 | tail -1
HKV_DUAL_ROUNDS=2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -k "dual" 2>&1 | tail -1
for r in 0 1; do echo "== rounds $r"; HKV_DUAL_ROUNDS=$r MODE=dual timeout 300 python tools/scratch/qt.py 0.5,1.0 insert_or_assign,find 2>&1 | grep lambda; done
