"""Dual-mode insert for ncu: 2^27 slots, dim 64, lambda argv[1], engine
workers argv[2] (1: serial dataflow, > 1: CAS engine; the fill always uses
the serial engine); one insert_or_assign of 1M fresh keys inside NVTX range
"prof"."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2603_17168_b200 as hkv  # noqa: E402
from paper_2603_17168_b200 import workloads as W  # noqa: E402

lam = float(sys.argv[1]) if len(sys.argv) > 1 else 0.5
workers = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cap, dim, B = 2**27, 64, 2**20
t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, mode="dual"))
t.validate_keys = False
vals = torch.randn((B, dim), device="cuda")
off = 0
while t.size() < int(lam * cap) and off < 40 * cap:
    n = B if lam >= 1.0 else min(B, int(lam * cap) - t.size())
    t.insert_or_assign(W.uniform_distinct_keys_torch(n, 0, stream_offset=off), vals[:n])
    off += n
t.snapshot()
t.set_workers(workers)
for i in range(3):
    if i == 2:
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_push("prof")
    t.insert_or_assign(W.uniform_distinct_keys_torch(B, 0, stream_offset=2**44 + i * B), vals)
    if i == 2:
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
    t.restore()
torch.cuda.synchronize()
print("ok")
