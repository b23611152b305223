HKV_COLLECT=2 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q 2>&1 | tail -1
timeout 300 python tools/scratch/qt.py 0.5,0.75,1.0 insert_or_assign 2>&1 | grep lambda
