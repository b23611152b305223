"""pipeline latency floor: insert_or_assign of small batches on the C2 table"""
import sys, torch
sys.path.insert(0, ".")
import bench
import paper_2603_17168_b200 as hkv
from paper_2603_17168_b200 import workloads as W
cap, dim = 2**27, 64
t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim))
t.validate_keys = False
bench.fill_table(t, 0.5, cap, dim, 2**20, torch, W)
t.snapshot()
st = torch.cuda.current_stream()
for n in [1024, 16384, 262144, 1048576]:
    vals = torch.randn((n, dim), device="cuda")
    ms = []
    for i in range(6):
        k = W.uniform_distinct_keys_torch(n, 0, stream_offset=2**44 + i * n)
        torch.cuda.synchronize(); torch.cuda._sleep(400_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st); t.insert_or_assign(k, vals); e1.record(st)
        torch.cuda.synchronize(); t.restore()
        if i: ms.append(e0.elapsed_time(e1))
    ms.sort()
    print(f"n {n}: {1000*ms[len(ms)//2]:.1f} us", flush=True)
