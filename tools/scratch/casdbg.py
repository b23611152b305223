import os, sys, torch
sys.path.insert(0, ".")
import bench
import paper_2603_17168_b200 as hkv
from paper_2603_17168_b200 import workloads as W
cap, dim, B = 2**27, 64, 2**20
mode = os.environ.get("MODE", "dual")
t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, mode=mode, workers=8))
t.validate_keys = False
bench.fill_table(t, 1.0, cap, dim, B, torch, W)
t.snapshot()
vals = torch.randn((B, dim), device="cuda")
for r in range(3):
    k = W.uniform_distinct_keys_torch(B, 0, stream_offset=2**45 + r * B)
    t.counters.reset()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(); t.insert_or_assign(k, vals); e1.record(); torch.cuda.synchronize()
    print(r, round(e0.elapsed_time(e1), 3), t.counters.as_dict(), flush=True)
    t.restore()
