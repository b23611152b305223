"""Per-config measurements for every BASELINE.json config that fits one GPU
(SURVEY.md 8(d) C1, C2 extras, C3, C4, dual mode).  bench.py keeps the
headline (C2); this prints one JSON object per measurement so the other
8(d) rows carry B200 numbers too.

    python tools/bench_configs.py [--only c1,c2x,c3,c4,dual] [--reps 5]

Every number: median over `reps` device-timed repeats (CUDA events around
the public-API call on its stream, inputs resident in HBM), the table's
metadata restored from an HBM snapshot between mutation repeats (outside
the timed region).  Outcome mixes are reported so the byte model can be
applied.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_17168_b200 as hkv  # noqa: E402
from paper_2603_17168_b200 import workloads as W  # noqa: E402

B = 2**20


def ev():
    return torch.cuda.Event(enable_timing=True)


def timed(fn, reps, after=None):
    """median device ms of fn() over reps (after() runs untimed between reps)."""
    st = torch.cuda.current_stream()
    out = None
    ms = []
    for r in range(reps + 1):
        a, b = ev(), ev()
        a.record(st)
        out = fn(r)
        b.record(st)
        torch.cuda.synchronize()
        if r > 0:
            ms.append(a.elapsed_time(b))
        if after is not None:
            after()
    torch.cuda.synchronize()
    return statistics.median(ms), out


def outcome_mix(o):
    c = torch.bincount(o.to(torch.int64), minlength=7).cpu().tolist()
    names = ["inserted", "updated", "rejected", "evicted", "found", "not_found", "erased"]
    return {n: v for n, v in zip(names, c) if v}


def emit(rec):
    print(json.dumps(rec), flush=True)


def fill(t, lam, cap, dim, seed=0, batch=B):
    vals = torch.randn((batch, dim), device="cuda", generator=torch.Generator(device="cuda").manual_seed(seed))
    target = int(round(lam * cap))
    off = 0
    while t.size() < target and off < 40 * cap:
        n = batch if lam >= 1.0 else min(batch, target - t.size())
        t.insert_or_assign(W.uniform_distinct_keys_torch(n, seed, stream_offset=off), vals[:n])
        off += n
    return off


def resident_sample(t, n, gen):
    res = torch.from_numpy(t.occupied_keys().view(np.int64)).cuda()
    idx = torch.randint(0, res.numel(), (n,), device="cuda", generator=gen)
    return res[idx].contiguous()


def c1(reps):
    """configs[0]: 2^20 slots, dim 8, kLru; prefill 0.5; insert_or_assign 1M fresh; find 1M mixed."""
    cap, dim = 2**20, 8
    t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, score_policy="kLru"))
    t.validate_keys = False
    pk = torch.from_numpy(W.uniform_distinct_keys(524288, 0).view(np.int64)).cuda()
    pv = torch.from_numpy(np.random.default_rng(0).standard_normal((524288, dim)).astype(np.float32)).cuda()
    t.insert_or_assign(pk, pv)
    t.snapshot()
    ik = torch.from_numpy(W.uniform_distinct_keys(B, 0, stream_offset=2**41).view(np.int64)).cuda()
    iv = torch.randn((B, dim), device="cuda")
    ms_i, o = timed(lambda r: t.insert_or_assign(ik, iv), reps, after=t.restore)
    emit({"config": "C1", "op": "insert_or_assign", "capacity": cap, "dim": dim, "lambda": 0.5, "ms": ms_i,
          "bkvs": B / ms_i / 1e6, "outcomes": outcome_mix(o)})
    t.insert_or_assign(ik, iv)
    q = torch.cat([ik[: B // 2], W.uniform_distinct_keys_torch(B // 2, 0, stream_offset=2**40)])
    ms_f, (f, _) = timed(lambda r: t.find(q), reps)
    emit({"config": "C1", "op": "find", "capacity": cap, "dim": dim, "lambda": round(t.load_factor(), 4),
          "ms": ms_f, "bkvs": B / ms_f / 1e6, "hit_rate": float(f.float().mean())})
    # assign of the same mixed batch (half resident; 128 ops per bucket: the dense-duplicate path)
    ms_a, o = timed(lambda r: t.assign(q, iv), reps)
    emit({"config": "C1", "op": "assign", "capacity": cap, "dim": dim, "lambda": round(t.load_factor(), 4),
          "ms": ms_a, "bkvs": B / ms_a / 1e6, "outcomes": outcome_mix(o)})


def c2_extras(reps, lg=27):
    """C2 table (2^27 slots, dim 64): miss-find, contains, find_ptr, assign, insert_and_evict, erase."""
    cap, dim = 2**lg, 64
    gen = torch.Generator(device="cuda").manual_seed(7)
    for lam in (0.5, 1.0):
        t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, score_policy="kLru"))
        t.validate_keys = False
        fill(t, lam, cap, dim)
        t.snapshot()
        q = resident_sample(t, B, gen)
        miss = W.uniform_distinct_keys_torch(B, 0, stream_offset=2**40)
        vals = torch.randn((B, dim), device="cuda", generator=gen)
        base = {"config": "C2", "capacity": cap, "dim": dim, "lambda": round(t.load_factor(), 4)}
        for name, fn in (("find_hit", lambda r: t.find(q)), ("find_miss", lambda r: t.find(miss)),
                         ("contains_hit", lambda r: t.contains(q)), ("find_ptr_hit", lambda r: t.find_ptr(q))):
            ms, _ = timed(fn, reps)
            emit({**base, "op": name, "ms": ms, "bkvs": B / ms / 1e6})
        ms, o = timed(lambda r: t.assign(q, vals), reps)
        emit({**base, "op": "assign_hit", "ms": ms, "bkvs": B / ms / 1e6, "outcomes": outcome_mix(o)})
        fresh = [W.uniform_distinct_keys_torch(B, 0, stream_offset=2**44 + r * B) for r in range(reps + 1)]
        ms, out = timed(lambda r: t.insert_and_evict(fresh[r], vals), reps, after=t.restore)
        emit({**base, "op": "insert_and_evict_fresh", "ms": ms, "bkvs": B / ms / 1e6,
              "outcomes": outcome_mix(out[0])})
        ms, o = timed(lambda r: t.insert_or_assign(q, vals), reps, after=t.restore)
        emit({**base, "op": "insert_or_assign_update", "ms": ms, "bkvs": B / ms / 1e6,
              "outcomes": outcome_mix(o)})
        ms, o = timed(lambda r: t.erase(q), reps, after=t.restore)
        emit({**base, "op": "erase_hit", "ms": ms, "bkvs": B / ms / 1e6, "outcomes": outcome_mix(o)})
        # export_batch_if through the C-ABI into device buffers: 1M entries with
        # score >= 1 (the service's native predicate) from cursor 0
        import ctypes as C

        ok = torch.empty(B, dtype=torch.int64, device="cuda")
        ov = torch.empty((B, dim), dtype=torch.float32, device="cuda")
        osc = torch.empty(B, dtype=torch.int64, device="cuda")
        cnt, nxt = C.c_int64(), C.c_int64()

        def exp(r):
            hkv._lib.check(t._lib.hkv_export(t._h, 0, B, 1, 1, None, 0, C.c_void_p(ok.data_ptr()),
                                             C.c_void_p(ov.data_ptr()), C.c_void_p(osc.data_ptr()), C.byref(cnt),
                                             C.byref(nxt), t._sp()))

        ms, _ = timed(exp, reps)
        scanned = nxt.value if nxt.value > 0 else cap
        emit({**base, "op": "export_batch_if_1M", "ms": ms, "rows_scanned": scanned, "exported": cnt.value,
              "scan_gbs": round(scanned * 16 / ms / 1e6, 1),
              "bkvs": cnt.value / ms / 1e6})
        del t
        torch.cuda.empty_cache()


def c3(reps, lg=27, batches=24):
    """configs[2]: C2 table at lambda 1, zipf alpha 0.99 over 4x capacity, insert_and_evict, kLfu and kCustomized."""
    cap, dim = 2**lg, 64
    for pol in ("kLfu", "kCustomized"):
        t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, score_policy=pol))
        t.validate_keys = False
        vals = torch.randn((B, dim), device="cuda")
        off = 0
        op_base = 0
        while t.size() < cap and off < 40 * cap:  # uniform pre-fill to lambda = 1
            k = W.uniform_distinct_keys_torch(B, 1, stream_offset=off)
            sc = torch.arange(op_base, op_base + B, device="cuda", dtype=torch.int64) if pol == "kCustomized" else None
            t.insert_or_assign(k, vals, sc)
            off += B
            op_base += B
        zk = [torch.from_numpy(W.zipf_keys(B, 4 * cap, 0.99, seed=s).view(np.int64)).cuda() for s in range(batches)]
        ms_all, mixes = [], []
        for s in range(batches):
            sc = torch.arange(op_base, op_base + B, device="cuda", dtype=torch.int64) if pol == "kCustomized" else None
            op_base += B
            a, b = ev(), ev()
            a.record()
            o, ek, evv, es = t.insert_and_evict(zk[s], vals, sc)
            b.record()
            torch.cuda.synchronize()
            ms_all.append(a.elapsed_time(b))
            mixes.append(outcome_mix(o))
        tail = ms_all[batches // 2:]
        ms = statistics.median(tail)
        emit({"config": "C3", "op": "insert_and_evict_zipf", "policy": pol, "capacity": cap, "dim": dim,
              "lambda": round(t.load_factor(), 4), "alpha": 0.99, "universe": 4 * cap, "batches": batches,
              "ms": ms, "bkvs": B / ms / 1e6, "outcomes_last": mixes[-1],
              "note": f"median of the last {len(tail)} of {batches} consecutive 1M zipf batches after a uniform "
                      "fill to lambda 1 (no restore: continuous ingestion)"})
        del t
        torch.cuda.empty_cache()


def host_mem_gb():
    try:
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemAvailable"):
                return int(ln.split()[1]) / 2**20
    except Exception:
        pass
    return 0.0


def c4(reps, lg=None):
    """configs[3]: dim 128 values in mapped pinned host memory (fast_tier_budget 0, and 50/50); find + assign."""
    dim = 128
    if lg is None:
        lg = 27 if host_mem_gb() > 160 else 26
    cap = 2**lg
    gen = torch.Generator(device="cuda").manual_seed(3)
    for split in (0.0, 0.5, 1.0):
        budget = int(split * (cap // 128))
        t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, score_policy="kLru", fast_tier_budget=budget))
        t.validate_keys = False
        fill(t, 0.5, cap, dim)
        q = resident_sample(t, B, gen)
        vals = torch.randn((B, dim), device="cuda", generator=gen)
        base = {"config": "C4", "capacity": cap, "dim": dim, "lambda": round(t.load_factor(), 4),
                "hbm_fraction_of_buckets": split}
        ms, _ = timed(lambda r: t.find(q), reps)
        emit({**base, "op": "find_hit", "ms": ms, "bkvs": B / ms / 1e6})
        ms, _ = timed(lambda r: t.find_ptr(q), reps)
        emit({**base, "op": "find_ptr_hit", "ms": ms, "bkvs": B / ms / 1e6})
        ms, _ = timed(lambda r: t.assign(q, vals), reps)
        emit({**base, "op": "assign_hit", "ms": ms, "bkvs": B / ms / 1e6})
        del t
        torch.cuda.empty_cache()


def dual(reps, lg=27):
    """Dual-bucket mode (D1/D2, table.py:1088-1119) on the C2 shape: find + insert_or_assign at lambda 0.5 / 1."""
    cap, dim = 2**lg, 64
    gen = torch.Generator(device="cuda").manual_seed(5)
    for lam in (0.5, 1.0):
        t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, score_policy="kLru", mode="dual"))
        t.validate_keys = False
        fill(t, lam, cap, dim)
        t.snapshot()
        q = resident_sample(t, B, gen)
        vals = torch.randn((B, dim), device="cuda", generator=gen)
        base = {"config": "dual", "capacity": cap, "dim": dim, "lambda": round(t.load_factor(), 4)}
        ms, _ = timed(lambda r: t.find(q), reps)
        emit({**base, "op": "find_hit", "ms": ms, "bkvs": B / ms / 1e6})
        fresh = [W.uniform_distinct_keys_torch(B, 0, stream_offset=2**44 + r * B) for r in range(reps + 1)]
        ms, o = timed(lambda r: t.insert_or_assign(fresh[r], vals), reps, after=t.restore)
        emit({**base, "op": "insert_or_assign_fresh", "ms": ms, "bkvs": B / ms / 1e6, "outcomes": outcome_mix(o)})
        del t
        torch.cuda.empty_cache()


def cas(reps, lg=27):
    """The concurrent slot-CAS engine (workers > 1, hkv_cas.cu) on the C2
    shape: insert_or_assign / insert_and_evict of 1M fresh keys, single mode
    at lambda 0.5 / 0.75 / 1 and dual mode at 0.5 / 1."""
    cap, dim = 2**lg, 64
    gen = torch.Generator(device="cuda").manual_seed(6)
    for mode, lams in (("single", (0.5, 0.75, 1.0)), ("dual", (0.5, 1.0))):
        for lam in lams:
            t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, score_policy="kLru", mode=mode,
                                               workers=8))
            t.validate_keys = False
            fill(t, lam, cap, dim)
            t.snapshot()
            vals = torch.randn((B, dim), device="cuda", generator=gen)
            base = {"config": f"cas-{mode}", "capacity": cap, "dim": dim, "lambda": round(t.load_factor(), 4)}
            fresh = [W.uniform_distinct_keys_torch(B, 0, stream_offset=2**44 + r * B) for r in range(reps + 1)]
            ms, o = timed(lambda r: t.insert_or_assign(fresh[r], vals), reps, after=t.restore)
            emit({**base, "op": "insert_or_assign_fresh", "ms": ms, "bkvs": B / ms / 1e6, "outcomes": outcome_mix(o)})
            ms, o = timed(lambda r: t.insert_and_evict(fresh[r], vals)[0], reps, after=t.restore)
            emit({**base, "op": "insert_and_evict_fresh", "ms": ms, "bkvs": B / ms / 1e6, "outcomes": outcome_mix(o)})
            q = resident_sample(t, B, gen)
            ms, o = timed(lambda r: t.insert_or_assign(q, vals), reps, after=t.restore)
            emit({**base, "op": "insert_or_assign_hits", "ms": ms, "bkvs": B / ms / 1e6, "outcomes": outcome_mix(o)})
            del t
            torch.cuda.empty_cache()


def peer(reps, lg=27, world=2):
    """Sharded find over peer memory, `world` virtual shards of 2^lg / world
    slots on this one GPU (hkv_find_peer with same-process peers: the kernel
    path of NVLink peer reads, minus NVLink), vs the local find of one table
    of the same total size."""
    cap, dim = 2**lg, 64
    cl = cap // world
    bl = cl // 128
    gen = torch.Generator(device="cuda").manual_seed(11)
    shards = [hkv.CacheTable(hkv.TableConfig(capacity=cl, value_dim=dim, score_policy="kLru")) for _ in range(world)]
    for s in shards:
        s.validate_keys = False
    vals = torch.randn((B, dim), device="cuda", generator=gen)
    off = 0
    while sum(s.size() for s in shards) < cap // 2:
        k = W.uniform_distinct_keys_torch(B, 0, stream_offset=off)
        off += B
        owner = torch.div(W.fmix64_torch(k) & (bl * world - 1), bl, rounding_mode="floor")
        for r in range(world):
            sel = owner == r
            shards[r].insert_or_assign(k[sel].contiguous(), vals[: int(sel.sum())])
    for s in shards:
        s._set_peers_local(shards)
    q = W.uniform_distinct_keys_torch(B, 0, stream_offset=int(torch.randint(0, off - B, (1,)).item()))
    out = torch.empty((B, dim), device="cuda")
    ms, (f, _) = timed(lambda r: shards[0]._find_peer(q, out), reps)
    emit({"config": "C5-virtual", "op": "find_peer", "shards": world, "capacity": cap, "dim": dim,
          "lambda": round(sum(s.size() for s in shards) / cap, 4), "hit_rate": float(f.float().mean().item()),
          "ms": ms, "bkvs": B / ms / 1e6,
          "note": "all shards on one GPU: measures the peer-find kernel, not NVLink"})
    del shards
    torch.cuda.empty_cache()


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--only", default="c1,c2x,c3,c4,dual,cas,peer")
    p.add_argument("--reps", type=int, default=5)
    p.add_argument("--lg", type=int, default=27)
    a = p.parse_args()
    torch.cuda.set_device(0)
    which = set(a.only.split(","))
    t0 = time.time()
    if "peer" in which:
        peer(a.reps, a.lg)
    if "cas" in which:
        cas(a.reps, a.lg)
    if "c1" in which:
        c1(a.reps)
    if "c2x" in which:
        c2_extras(a.reps, a.lg)
    if "c3" in which:
        c3(a.reps, a.lg)
    if "c4" in which:
        c4(a.reps)
    if "dual" in which:
        dual(a.reps, a.lg)
    emit({"done_s": round(time.time() - t0, 1), "device": torch.cuda.get_device_name(0)})


if __name__ == "__main__":
    main()
