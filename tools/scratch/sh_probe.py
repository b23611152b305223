import os, sys, time, torch, json
import torch.distributed as dist
sys.path.insert(0, os.getcwd())
import paper_2603_17168_b200 as hkv
from paper_2603_17168_b200 import workloads as W
from paper_2603_17168_b200.sharded import ShardedCacheTable
dist.init_process_group("nccl")
torch.cuda.set_device(0)
cap, dim, B = 2**27, 64, 2**20
t = ShardedCacheTable(hkv.TableConfig(capacity=cap, value_dim=dim))
t.local.validate_keys = False
vals = torch.randn((B, dim), device="cuda")
off = 0
while off < cap // 2:
    t.insert_or_assign(W.uniform_distinct_keys_torch(B, 0, stream_offset=off), vals); off += B
t.local.snapshot()
k = W.uniform_distinct_keys_torch(B, 0, stream_offset=2**44)
st = torch.cuda.current_stream()
def ev():
    e = torch.cuda.Event(enable_timing=True); e.record(st); return e
import paper_2603_17168_b200.sharded as S
orig_plan, orig_pack, orig_local = t._plan, t._a2a_packed, t.local.insert_or_assign
marks = []
def plan(keys):
    marks.append(("plan0", ev(), time.perf_counter())); r = orig_plan(keys); marks.append(("plan1", ev(), time.perf_counter())); return r
def pack(cols, send, recv):
    marks.append(("pack0", ev(), time.perf_counter())); r = orig_pack(cols, send, recv); marks.append(("pack1", ev(), time.perf_counter())); return r
def local(*a, **kw):
    marks.append(("loc0", ev(), time.perf_counter())); r = orig_local(*a, **kw); marks.append(("loc1", ev(), time.perf_counter())); return r
t._plan, t._a2a_packed, t.local.insert_or_assign = plan, pack, local
for rep in range(4):
    marks.clear()
    torch.cuda.synchronize()
    e0 = ev(); h0 = time.perf_counter()
    t.insert_or_assign(k, vals)
    e1 = ev(); h1 = time.perf_counter()
    torch.cuda.synchronize()
    t.local.restore(); torch.cuda.synchronize()
    out = {"total_ms": round(e0.elapsed_time(e1), 3), "host_ms": round(1e3*(h1-h0), 3)}
    prev = e0; ph = h0
    for name, e, h in marks:
        out[name] = (round(prev.elapsed_time(e), 3), round(1e3*(h-ph), 3)); prev = e; ph = h
    out["tail"] = (round(prev.elapsed_time(e1), 3), round(1e3*(h1-ph), 3))
    print(json.dumps(out), flush=True)
dist.destroy_process_group()
