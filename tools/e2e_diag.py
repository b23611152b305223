"""Where the end-to-end (host buffer) time of bench.py's e2e step goes.

    python tools/e2e_diag.py [log2_capacity]

Times raw pinned copies of the step's sizes (H2D 264 MB, D2H 257 MB), then
find / insert_or_assign through the public API with pinned host tensors,
split into host-side phases with perf_counter.
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2603_17168_b200 as hkv  # noqa: E402
from paper_2603_17168_b200 import workloads as W  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 27
cap, dim, B = 2**lg, 64, 2**20
dev = torch.device("cuda")


def wall(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(ts))


hv = torch.randn((B, dim)).pin_memory()
dv = torch.empty((B, dim), device=dev)
hout = torch.empty((B, dim)).pin_memory()
ms = wall(lambda: dv.copy_(hv, non_blocking=True))
print(f"raw H2D 256 MB pinned: {ms:.2f} ms = {hv.numel() * 4 / ms / 1e6:.1f} GB/s")
ms = wall(lambda: hout.copy_(dv, non_blocking=True))
print(f"raw D2H 256 MB pinned: {ms:.2f} ms = {hv.numel() * 4 / ms / 1e6:.1f} GB/s")
s2 = torch.cuda.Stream()


def duplex():
    with torch.cuda.stream(s2):
        hout.copy_(dv, non_blocking=True)
    dv2.copy_(hv, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)


dv2 = torch.empty_like(dv)
ms = wall(duplex)
print(f"raw H2D || D2H 256 MB each: {ms:.2f} ms = {2 * hv.numel() * 4 / ms / 1e6:.1f} GB/s total")

t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim))
vals = torch.randn((B, dim), device=dev)
off = 0
while t.size() < cap // 2:
    n = min(B, cap // 2 - t.size())
    t.insert_or_assign(W.uniform_distinct_keys_torch(n, 0, stream_offset=off), vals[:n])
    off += n
t.snapshot()
hq = W.uniform_distinct_keys_torch(B, 0, stream_offset=0).cpu().pin_memory()
hk = W.uniform_distinct_keys_torch(B, 0, stream_offset=2**44).cpu().pin_memory()
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f, v = t.find(hq)
    t1 = time.perf_counter()
    o = t.insert_or_assign(hk, hv)
    t2 = time.perf_counter()
    t.restore()
    torch.cuda.synchronize()
    print(f"rep {rep}: find(host) {1e3 * (t1 - t0):.2f} ms  insert_or_assign(host) {1e3 * (t2 - t1):.2f} ms")
import cProfile  # noqa: E402
import pstats  # noqa: E402

pr = cProfile.Profile()
pr.enable()
for rep in range(3):
    f, v = t.find(hq)
    o = t.insert_or_assign(hk, hv)
    t.restore()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
