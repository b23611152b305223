timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_collector.py -x -q 2>&1 | tail -1
timeout 300 python tools/scratch/qt.py 0.5,1.0 insert_or_assign,insert_and_evict 2>&1 | grep lambda
