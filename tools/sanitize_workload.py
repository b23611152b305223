"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): every kernel family of the library on tiny tables.

    compute-sanitizer --tool memcheck python tools/sanitize_workload.py [parts]

parts (comma list, default all): single, dual, cas, host, single_key, peer, export
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_17168_b200 as hkv  # noqa: E402

parts = set((sys.argv[1] if len(sys.argv) > 1 else "single,dual,cas,host,single_key,peer,export").split(","))
rng = np.random.default_rng(0)
cap, dim = 128 * 64, 8


def batch(n, universe):
    k = rng.integers(1, universe, size=n, dtype=np.uint64)
    return k, rng.standard_normal((n, dim)).astype(np.float32)


def mutate(t, policy="kLru"):
    for j in range(4):
        k, v = batch(3000, 3 * cap)
        s = rng.integers(0, 100, size=len(k), dtype=np.uint64) if policy == "kCustomized" else None
        t.insert_or_assign(k, v, s)
        t.insert_and_evict(k[::2], v[::2], None if s is None else s[::2])
        vi = v[:500].copy()
        t.find_or_insert(k[:500], vi, None if s is None else s[:500])
        t.find(k)
        t.contains(k)
        t.find_ptr(k)
        t.assign(k[:700], v[:700])
        t.assign_scores(k[:300], None if s is None else s[:300])
        t.erase(k[:200])
    assert t.check_consistency()


if "single" in parts:
    for pol in ("kLru", "kLfu", "kCustomized"):
        mutate(hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, score_policy=pol)), pol)
    # long segments (>= 16 ops per bucket): the long-segment engine and the assign aggregation path
    t = hkv.CacheTable(hkv.TableConfig(capacity=128 * 16, value_dim=dim))
    k, v = batch(40000, 6000)
    t.insert_or_assign(k, v)
    t.assign(k, v)
    t.insert_and_evict(k, v)
if "dual" in parts:
    mutate(hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, mode="dual")))
if "cas" in parts:
    mutate(hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, workers=4)))
    mutate(hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, mode="dual", workers=4)))
if "host" in parts:
    t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, fast_tier_budget=16))
    k, v = batch(5000, 3 * cap)
    kt, vt = torch.from_numpy(k.view(np.int64)).pin_memory(), torch.from_numpy(v).pin_memory()
    t.insert_or_assign(kt, vt)
    t.find(kt)
    t.find_or_insert(kt, vt.clone())
if "single_key" in parts:
    for mode in ("single", "dual"):
        t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, mode=mode))
        for key in rng.integers(1, 3 * cap, size=400, dtype=np.uint64):
            t.upsert_single(int(key), np.ones(dim, np.float32))
            if mode == "dual":
                t.upsert_dual(int(key) + 1, np.ones(dim, np.float32))
            r = t.lookup(int(key))
            t.find_in_bucket(0, int(key))
            if r.found:
                t.read_value(r.value_handle)
if "peer" in parts:
    shards = [hkv.CacheTable(hkv.TableConfig(capacity=cap // 2, value_dim=dim)) for _ in range(2)]
    for s in shards:
        s._set_peers_local(shards)
    k, v = batch(3000, 3 * cap)
    shards[0].insert_or_assign(k, v)
    shards[0]._find_peer(torch.from_numpy(k.view(np.int64)).cuda())
if "export" in parts:
    t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim))
    k, v = batch(5000, 3 * cap)
    t.insert_or_assign(k, v)
    t.export_batch_if(None, 0, 1000)
    t.export_batch_if(5, 100, 3000)
    t.export_batch_if(lambda kk, ss: ss % 2 == 0, 0, 4000)
torch.cuda.synchronize()
print("sanitize workload ok:", ",".join(sorted(parts)))
