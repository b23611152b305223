"""quick C2 insert timing: python tools/scratch/qt.py lambdas [ops] (env HKV_LIB selects a build)"""
import os, sys, time
import torch
sys.path.insert(0, ".")
import bench
import paper_2603_17168_b200 as hkv
from paper_2603_17168_b200 import workloads as W
import os
if os.environ.get("FETCH"):
    torch.cuda.init(); torch.zeros(1, device="cuda")
    from cuda.bindings import runtime as rt
    print("set fetch", rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitMaxL2FetchGranularity, int(os.environ["FETCH"])),
          rt.cudaDeviceGetLimit(rt.cudaLimit.cudaLimitMaxL2FetchGranularity))
lams = [float(x) for x in sys.argv[1].split(",")]
ops = sys.argv[2].split(",") if len(sys.argv) > 2 else ["insert_or_assign", "find"]
cap, dim, B = 2**27, 64, 2**20
mode = os.environ.get("MODE", "single")
workers = int(os.environ.get("WORKERS", "1"))
t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, mode=mode, workers=workers))
t.validate_keys = False
vals = torch.randn((B, dim), device="cuda")
ins = [W.uniform_distinct_keys_torch(B, 0, stream_offset=2**44 + i * B) for i in range(6)]
st = torch.cuda.current_stream()
junk = torch.empty(2**28, dtype=torch.uint8, device="cuda")
for lam in lams:
    t0 = time.time()
    bench.fill_table(t, lam, cap, dim, B, torch, W)
    t.snapshot()
    q = W.uniform_distinct_keys_torch(B, 0, stream_offset=0)
    res = {}
    for op in ops:
        ms = []
        for i in range(6):
            torch.cuda.synchronize(); junk.fill_(1); torch.cuda._sleep(400_000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            if op == "insert_or_assign": t.insert_or_assign(ins[i], vals)
            elif op == "insert_and_evict": t.insert_and_evict(ins[i], vals)
            elif op == "find": t.find(q)
            e1.record(st)
            torch.cuda.synchronize()
            if op.startswith("insert"): t.restore()
            if i: ms.append(e0.elapsed_time(e1))
        ms.sort()
        res[op] = round(1000 * ms[len(ms) // 2], 1)
    print(f"lambda {lam} size {t.size()/cap:.3f} fill {time.time()-t0:.1f}s us {res}", flush=True)
