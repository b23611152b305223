"""Host-side issue cost vs device time per op on a C2-sized table.

    python tools/diag_host.py [log2_capacity]

Prints, per iteration, the host time spent inside find / insert_or_assign /
restore and the device time (CUDA events) of find and insert_or_assign, then
a cProfile of the loop (top entries by cumulative time).
"""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2603_17168_b200 as hkv  # noqa: E402
from paper_2603_17168_b200 import workloads as W  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 27
cap, dim, B = 2**lg, 64, 2**20
t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim))
t.validate_keys = False
vals = torch.randn((B, dim), device="cuda")
off = 0
while t.size() < cap // 2:
    n = min(B, cap // 2 - t.size())
    t.insert_or_assign(W.uniform_distinct_keys_torch(n, 0, stream_offset=off), vals[:n])
    off += n
t.snapshot()
q = W.uniform_distinct_keys_torch(B, 0, stream_offset=0)
ins = [W.uniform_distinct_keys_torch(B, 0, stream_offset=2**44 + i * B) for i in range(20)]
torch.cuda.synchronize()
st = torch.cuda.current_stream()
if "--ktimer" in sys.argv:
    hkv._lib.load().hkv_set_kernel_timing(1)
if "--smi" in sys.argv:
    import bench

    _clk = bench.Clocks(0)
    _clk.start()
    _clk.wait_first_sample()


def it(i, log):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    h0 = time.perf_counter()
    e[0].record(st)
    t.find(q)
    e[1].record(st)
    h1 = time.perf_counter()
    e[2].record(st)
    t.insert_or_assign(ins[i], vals)
    e[3].record(st)
    h2 = time.perf_counter()
    t.restore()
    h3 = time.perf_counter()
    if log:
        torch.cuda.synchronize()
        print(f"it {i}: host find {1e3*(h1-h0):.3f} ms ins {1e3*(h2-h1):.3f} ms restore {1e3*(h3-h2):.3f} ms | "
              f"dev find {e[0].elapsed_time(e[1]):.3f} ins {e[2].elapsed_time(e[3]):.3f}", flush=True)


for i in range(5):
    it(i, True)
for i in range(20):
    it(i, True)
pr = cProfile.Profile()
pr.enable()
for i in range(5, 15):
    it(i, False)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
for i in range(15, 20):
    it(i, True)
