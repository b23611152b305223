import sys, os, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2603_17168_b200 as hkv
from paper_2603_17168_b200 import workloads as W
lg = int(sys.argv[1]) if len(sys.argv) > 1 else 24
mode = sys.argv[2] if len(sys.argv) > 2 else "single"
cap, dim, B = 2**lg, 64, 2**20
t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, workers=8, mode=mode))
t.validate_keys = False
vals = torch.randn((B, dim), device="cuda")
off = 0
while t.size() < cap // 2:
    n = min(B, cap // 2 - t.size())
    t.insert_or_assign(W.uniform_distinct_keys_torch(n, 0, stream_offset=off), vals[:n]); off += n
t.snapshot()
k = W.uniform_distinct_keys_torch(B, 0, stream_offset=2**44)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("x")
for r in range(2):
    t.insert_or_assign(k, vals); t.restore()
q = W.uniform_distinct_keys_torch(B, 0, stream_offset=0)
t.insert_or_assign(q, vals)
torch.cuda.synchronize()
print("ok")
