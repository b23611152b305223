timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/scratch/qt.py 0.5,0.75,1.0 insert_or_assign,insert_and_evict,find 2>&1 | grep lambda
