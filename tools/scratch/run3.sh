timeout 1500 python -m pytest tests -m gpu -x -q -k "not sanitizer" 2>&1 | tail -2
timeout 300 python tools/scratch/qt.py 0.5,1.0 insert_or_assign,insert_and_evict 2>&1 | grep lambda
