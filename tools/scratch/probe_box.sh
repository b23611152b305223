free -g; nproc; lscpu | grep -i "model name\|socket\|numa node(s)"; cat /sys/kernel/mm/transparent_hugepage/enabled; cat /proc/sys/vm/nr_hugepages; python - <<'PY'
import sys, time
sys.path.insert(0, 'baseline/_ref')
import numpy as np
t=time.time()
import cachekv
from cachekv import CacheTable, TableConfig
t0=time.time()
tb = CacheTable(TableConfig(capacity=2**27, value_dim=64))
print("ref 2^27 construct s", time.time()-t0, flush=True)
k = cachekv.workloads.uniform_distinct_keys(2**20, 0, stream_offset=2**44)
v = np.random.default_rng(0).standard_normal((2**20, 64), dtype=np.float32)
t0=time.time(); tb.insert_or_assign(k, v); print("ins 1M into empty s", time.time()-t0, flush=True)
t0=time.time(); f,_=tb.find(k); print("find 1M s", time.time()-t0, f.mean(), flush=True)
PY
