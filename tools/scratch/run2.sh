timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -k "dual" 2>&1 | tail -2
timeout 900 python tools/stage_times.py 27 0.5,1.0 dual insert_or_assign,find 2>&1 | grep lambda
