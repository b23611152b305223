import sys, os, ctypes as C, torch, json
sys.path.insert(0, os.getcwd())
import paper_2603_17168_b200 as hkv
from paper_2603_17168_b200 import _lib, workloads as W
lib = _lib.load()
lg = int(sys.argv[1]) if len(sys.argv) > 1 else 27
lams = [float(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0.5", "1.0"])]
cap, dim, B = 2**lg, 64, 2**20
st = torch.cuda.current_stream()
STAGES = ["prep", "sort", "segments", "apply", "finalize", "values_write"]
for lam in lams:
    t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim))
    t.validate_keys = False
    vals = torch.randn((B, dim), device="cuda")
    off = 0
    tgt = int(cap * lam)
    while t.size() < tgt and off < 4 * cap:
        n = B if lam >= 1 else min(B, tgt - t.size())
        t.insert_or_assign(W.uniform_distinct_keys_torch(n, 0, stream_offset=off), vals[:n]); off += n
    t.snapshot()
    ins = [W.uniform_distinct_keys_torch(B, 0, stream_offset=2**44 + i * B) for i in range(12)]
    res = {"lambda": lam}
    for level in (0, 1, 2):
        lib.hkv_set_kernel_timing(level)
        ms = []
        for i in range(12):
            torch.cuda.synchronize(); torch.cuda._sleep(400_000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st); t.insert_or_assign(ins[i], vals); e1.record(st)
            torch.cuda.synchronize(); t.restore(); torch.cuda.synchronize()
            if i >= 2: ms.append(e0.elapsed_time(e1))
        res[f"level{level}_ms"] = round(sorted(ms)[len(ms)//2], 4)
        if level == 2:
            for name in STAGES:
                m, n = C.c_double(), C.c_int64()
                lib.hkv_kernel_times(name.encode(), C.byref(m), C.byref(n))
                if n.value: res[name] = round(1e3 * m.value / n.value, 1)
        else:
            for name in STAGES:
                m, n = C.c_double(), C.c_int64()
                lib.hkv_kernel_times(name.encode(), C.byref(m), C.byref(n))
    lib.hkv_set_kernel_timing(0)
    print(json.dumps(res), flush=True)
    del t; torch.cuda.empty_cache()
