"""Short C2 workload for ncu: one 2^27-slot dim-64 table at lambda (argv[1],
default 1.0), two warm-up rounds of find + insert_or_assign (+ restore), then
one round inside an NVTX range "prof" so ncu can filter with
--nvtx --nvtx-include "prof/".

    ncu --nvtx --nvtx-include "prof/" --set full ... python tools/prof_c2.py 1.0
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2603_17168_b200 as hkv  # noqa: E402
from paper_2603_17168_b200 import workloads as W  # noqa: E402

lam = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
lg = int(sys.argv[2]) if len(sys.argv) > 2 else 27
cap, dim, B = 2**lg, 64, 2**20
t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim))
t.validate_keys = False
vals = torch.randn((B, dim), device="cuda", generator=torch.Generator(device="cuda").manual_seed(0))
off = 0
target = int(lam * cap)
while t.size() < target and off < 40 * cap:
    n = B if lam >= 1.0 else min(B, target - t.size())
    t.insert_or_assign(W.uniform_distinct_keys_torch(n, 0, stream_offset=off), vals[:n])
    off += n
t.snapshot()
# resident queries: the first keys of the fill stream that are still present
cand = W.uniform_distinct_keys_torch(4 * B, 0, stream_offset=max(0, off - 4 * B))
f = t.contains(cand)
q = cand[f.bool()][:B]
if q.numel() < B:
    q = torch.cat([q, q[: B - q.numel()]])
q = q[torch.randperm(B, device="cuda")].contiguous()
for i in range(3):
    if i == 2:
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_push("prof")
    t.find(q)
    t.insert_or_assign(W.uniform_distinct_keys_torch(B, 0, stream_offset=2**44 + i * B), vals)
    t.restore()
    if i == 2:
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("prof_c2 done", lam, t.load_factor())
