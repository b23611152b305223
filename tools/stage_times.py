"""Warm per-stage device times of the single-mode mutation pipeline on C2.

    python tools/stage_times.py [log2_capacity] [lambdas, e.g. 0.5,1.0] [single|dual] [ops, e.g. insert_or_assign,find]

Fills a dim-64 table to lambda 0.5 and 1.0, then runs insert_or_assign of
1M fresh keys (snapshot restored after each), assign of 1M resident keys and
find, with the library's event timers on each stage (prep, sort, segments,
apply, finalize, values_write, ...).  Prints the mean per stage and the
whole-op time from events around the call.
"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2603_17168_b200 as hkv  # noqa: E402
from paper_2603_17168_b200 import _lib  # noqa: E402
from paper_2603_17168_b200 import workloads as W  # noqa: E402

STAGES = ["prep", "sort", "segments", "count", "alloc", "scatter", "segfin", "big", "apply", "finalize", "evict_select", "values_read", "values_write", "assign_apply", "find", "find_gather",
          "dual_ranks", "dual_flow"]
lg = int(sys.argv[1]) if len(sys.argv) > 1 else 27
cap, dim, B = 2**lg, 64, 2**20
lib = _lib.load()
st = torch.cuda.current_stream()


def stage_report(label, reps, total_ms):
    parts = []
    for name in STAGES:
        ms, n = C.c_double(), C.c_int64()
        lib.hkv_kernel_times(name.encode(), C.byref(ms), C.byref(n))
        if n.value:
            parts.append(f"{name} {1e3 * ms.value / reps:.1f}")
    print(f"{label}: total {1e3 * total_ms / reps:.1f} us | " + " | ".join(parts), flush=True)


mode = sys.argv[3] if len(sys.argv) > 3 else "single"
t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, mode=mode))
t.validate_keys = False
vals = torch.randn((B, dim), device="cuda")
off = 0
reps = 10
ins = [W.uniform_distinct_keys_torch(B, 0, stream_offset=2**44 + i * B) for i in range(reps)]
for lam in [float(x) for x in (sys.argv[2].split(',') if len(sys.argv) > 2 else ['0.5', '1.0'])]:
    bench.fill_table(t, lam, cap, dim, B, torch, W)
    t.snapshot()
    q = W.uniform_distinct_keys_torch(B, 0, stream_offset=0)
    torch.cuda.synchronize()
    ops = sys.argv[4].split(",") if len(sys.argv) > 4 else ["insert_or_assign", "assign", "find"]
    for op in ops:
        for warm in (True, False):
            lib.hkv_set_kernel_timing(0 if warm else 2)
            tot = 0.0
            for i in range(2 if warm else reps):
                torch.cuda._sleep(400_000)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                if op == "insert_or_assign":
                    t.insert_or_assign(ins[i], vals)
                elif op == "insert_and_evict":
                    t.insert_and_evict(ins[i], vals)
                elif op == "assign":
                    t.assign(q, vals)
                else:
                    t.find(q)
                e1.record(st)
                if op.startswith("insert"):
                    t.restore()
                torch.cuda.synchronize()
                tot += e0.elapsed_time(e1)
            lib.hkv_set_kernel_timing(0)
            if not warm:
                stage_report(f"lambda {lam} {op}", reps, tot)
