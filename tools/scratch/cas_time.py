import sys, os, torch, json
sys.path.insert(0, os.getcwd())
import paper_2603_17168_b200 as hkv
from paper_2603_17168_b200 import workloads as W
lg = 27; cap, dim, B = 2**lg, 64, 2**20
for mode in ("single", "dual"):
    t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, workers=8, mode=mode))
    t.validate_keys = False
    vals = torch.randn((B, dim), device="cuda")
    off = 0
    while t.size() < cap // 2:
        n = min(B, cap // 2 - t.size())
        t.insert_or_assign(W.uniform_distinct_keys_torch(n, 0, stream_offset=off), vals[:n]); off += n
    t.snapshot()
    res = {}
    for name, k in (("fresh", W.uniform_distinct_keys_torch(B, 0, stream_offset=2**44)),
                    ("hits", W.uniform_distinct_keys_torch(B, 0, stream_offset=12345))):
        ms = []
        for r in range(4):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); a.record(); t.insert_or_assign(k, vals); b.record(); torch.cuda.synchronize()
            ms.append(a.elapsed_time(b)); t.restore()
        res[name] = round(sorted(ms)[1], 3)
    print(json.dumps({"lib": os.environ.get("HKV_LIB", "default"), "mode": mode, **res}), flush=True)
    del t; torch.cuda.empty_cache()
