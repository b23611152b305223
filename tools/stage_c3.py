"""Warm per-stage device times of C3 (zipf insert_and_evict at lambda 1).

    python tools/stage_c3.py [log2_capacity] [policy]
"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2603_17168_b200 as hkv  # noqa: E402
from paper_2603_17168_b200 import _lib  # noqa: E402
from paper_2603_17168_b200 import workloads as W  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 27
pol = sys.argv[2] if len(sys.argv) > 2 else "kLfu"
cap, dim, B = 2**lg, 64, 2**20
lib = _lib.load()
t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, score_policy=pol))
t.validate_keys = False
vals = torch.randn((B, dim), device="cuda")
off = base = 0
while t.size() < cap and off < 40 * cap:
    sc = torch.arange(base, base + B, device="cuda", dtype=torch.int64) if pol == "kCustomized" else None
    t.insert_or_assign(W.uniform_distinct_keys_torch(B, 1, stream_offset=off), vals, sc)
    off += B
    base += B
zk = [torch.from_numpy(W.zipf_keys(B, 4 * cap, 0.99, seed=s).view(np.int64)).cuda() for s in range(12)]
STAGES = ["prep", "sort", "segments", "apply", "finalize", "values_write"]
for s in range(12):
    if s == 8:
        lib.hkv_set_kernel_timing(2)
    sc = torch.arange(base, base + B, device="cuda", dtype=torch.int64) if pol == "kCustomized" else None
    base += B
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    t.insert_and_evict(zk[s], vals, sc)
    b.record()
    torch.cuda.synchronize()
    if s >= 8:
        print(f"batch {s}: {1e3 * a.elapsed_time(b):.1f} us")
lib.hkv_set_kernel_timing(0)
parts = []
for name in STAGES:
    ms, n = C.c_double(), C.c_int64()
    lib.hkv_kernel_times(name.encode(), C.byref(ms), C.byref(n))
    if n.value:
        parts.append(f"{name} {1e3 * ms.value / n.value:.1f}")
print(pol, " | ".join(parts))
