timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -k "dual" 2>&1 | tail -1
MODE=dual timeout 300 python tools/scratch/qt.py 0.5,1.0 insert_or_assign 2>&1 | grep lambda
