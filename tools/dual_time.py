"""Dual-mode (and single-mode CAS) insert_or_assign timings at the C2 shape:
2^27 slots, dim 64, 1M fresh keys per batch, lambda 0.5 / 1.0; each engine
from the same snapshot (serial-engine fill).  Prints one JSON line."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2603_17168_b200 as hkv  # noqa: E402
from paper_2603_17168_b200 import workloads as W  # noqa: E402

cap, dim, B, reps = 2**27, 64, 2**20, 3
modes = sys.argv[1].split(",") if len(sys.argv) > 1 else ["dual", "single"]
gen = torch.Generator(device="cuda").manual_seed(9)
vals = torch.randn((B, dim), device="cuda", generator=gen)
fresh = [W.uniform_distinct_keys_torch(B, 0, stream_offset=2**45 + r * B) for r in range(reps + 1)]
out = {}
for mode in modes:
    for lam in (0.5, 1.0):
        t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, mode=mode, workers=1))
        t.validate_keys = False
        bench._fill(t, lam, cap, dim, B, torch, W)
        t.snapshot()
        k = f"{mode}_{lam:.2f}"
        if mode == "dual":
            ms, o = bench._timed(torch, lambda r: t.insert_or_assign(fresh[r], vals), reps, after=t.restore)
            out[f"{k}_serial"] = bench._rec(ms, B, {"outcomes": bench._mix(torch, o)})
        t.set_workers(8)
        ms, o = bench._timed(torch, lambda r: t.insert_or_assign(fresh[r], vals), reps, after=t.restore)
        out[f"{k}_cas"] = bench._rec(ms, B, {"outcomes": bench._mix(torch, o)})
        t.set_workers(1)
        res = torch.from_numpy(t.occupied_keys().view(np.int64)).cuda()
        hits = res[torch.randint(0, res.numel(), (B,), device="cuda", generator=gen)]
        del res
        ms, _ = bench._timed(torch, lambda r: t.find(hits), reps)
        out[f"{k}_find"] = bench._rec(ms, B)
        t.set_workers(8)
        t.counters.reset()
        t.insert_or_assign(fresh[0], vals)
        out[f"{k}_cas"]["counters"] = t.counters.as_dict()
        assert t.check_consistency()
        del t
        torch.cuda.empty_cache()
print(json.dumps(out))
