import sys, time, torch, numpy as np
sys.path.insert(0, ".")
import paper_2603_17168_b200 as hkv
from paper_2603_17168_b200 import workloads as W
cap, dim, B = 2**24, 8, 2**20
t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, mode="dual"))
t.validate_keys = False
vals = torch.randn((B, dim), device="cuda")
zk = torch.from_numpy(W.zipf_keys(B, 4 * cap, 0.99, seed=1).view(np.int64)).cuda()
for name, keys in [("zipf", zk), ("one_key", torch.full((B,), 12345, dtype=torch.int64, device="cuda"))]:
    for r in range(2):
        torch.cuda.synchronize(); t0 = time.time()
        o = t.insert_or_assign(keys, vals)
        torch.cuda.synchronize()
        print(name, r, f"{(time.time()-t0)*1e3:.2f} ms", torch.bincount(o.to(torch.int64), minlength=4).tolist())
assert t.check_consistency()
print("ok")
