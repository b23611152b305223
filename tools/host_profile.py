"""Host-side cost of one public-API call (the GPU work is tiny here, so the
wall time per call is the Python + C-ABI + launch overhead)."""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2603_17168_b200 as hkv  # noqa: E402

t = hkv.CacheTable(hkv.TableConfig(capacity=2**20, value_dim=64))
t.validate_keys = False
k = torch.arange(1, 1025, device="cuda", dtype=torch.int64)
v = torch.randn(1024, 64, device="cuda")
for _ in range(20):
    t.insert_or_assign(k, v)
    t.find(k)
torch.cuda.synchronize()
for name, fn in (("insert_or_assign", lambda: t.insert_or_assign(k, v)), ("find", lambda: t.find(k)),
                 ("restore", lambda: t.restore() if t_snap else None)):
    if name == "restore":
        t.snapshot()
        t_snap = True
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    for _ in range(200):
        fn()
    h1 = time.perf_counter()
    torch.cuda.synchronize()
    h2 = time.perf_counter()
    print(f"{name}: host issue {1e6 * (h1 - h0) / 200:.1f} us/call, incl. drain {1e6 * (h2 - h0) / 200:.1f} us/call")
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    t.insert_or_assign(k, v)
    t.find(k)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
