"""Subprocess body of tests/test_gpu_collector.py::test_grouping_forced: run
with HKV_COLLECT=2 (collector on every batch) or 0 (sorted grouping on every
batch).  Dense batches (configs[0] shape: 128 ops per bucket), zipf batches
with long same-key runs under every policy, and contended random scripts,
each against the oracle, bit-exact; prints "collector forced ok"."""

import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import paper_2603_17168_b200 as hkv  # noqa: E402
from oracle.oracle import OracleTable  # noqa: E402
from paper_2603_17168_b200.workloads import uniform_distinct_keys, zipf_keys  # noqa: E402
from refdiff import make_script, outputs_equal, run_impl  # noqa: E402


def check_state(t, o, what):
    st = t.export_state()
    for name, ref in (("keys", o.keys), ("digests", o.digests), ("scores", o.scores), ("values", o.values)):
        assert st[name].tobytes() == ref.tobytes(), f"{what}: {name}"
    assert st["size"] == o.size() and st["clock"] == o.clock, what
    assert t.counters.as_dict() == o.counters, what


def main():
    assert torch.cuda.is_available()
    # configs[0]: 2^20 slots, dim 8, prefill 0.5, a 1M insert_and_evict batch
    cap, dim = 2**20, 8
    t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim))
    o = OracleTable(cap, dim)
    k0 = uniform_distinct_keys(cap // 2, 0)
    v0 = np.random.default_rng(0).standard_normal((len(k0), dim)).astype(np.float32)
    assert np.array_equal(t.insert_or_assign(k0, v0), o.insert_or_assign(k0, v0))
    k1 = uniform_distinct_keys(cap, 0, stream_offset=2**41)
    v1 = np.random.default_rng(1).standard_normal((len(k1), dim)).astype(np.float32)
    a, b = t.insert_and_evict(k1, v1), o.insert_and_evict(k1, v1)
    assert all(x.tobytes() == y.tobytes() for x, y in zip(a, b)), "c1 insert_and_evict"
    check_state(t, o, "c1")
    # zipf hot buckets and same-key runs, every policy
    for policy in ("kLru", "kLfu", "kEpochLru", "kEpochLfu", "kCustomized"):
        cap, dim = 128 * 64, 4
        t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, score_policy=policy))
        o = OracleTable(cap, dim, "single", policy)
        rng = np.random.default_rng(7)
        for j in range(8):
            keys = zipf_keys(30_000, 6 * cap, 0.99, seed=j)
            vals = rng.standard_normal((len(keys), dim)).astype(np.float32)
            sc = rng.integers(0, 60, size=len(keys), dtype=np.uint64) if policy == "kCustomized" else None
            op = ["insert_or_assign", "insert_and_evict", "find_or_insert", "erase"][j % 4]
            args = {"keys": keys[: len(keys) // 2]} if op == "erase" else {"keys": keys, "values": vals, "scores": sc}
            assert outputs_equal(run_impl(o, op, args), run_impl(t, op, args)), f"zipf {policy} {j} {op}"
        check_state(t, o, f"zipf {policy}")
    # contended random scripts
    for policy in ("kLru", "kLfu", "kCustomized"):
        cap, dim = 128 * 64, 8
        t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, score_policy=policy))
        o = OracleTable(cap, dim, "single", policy)
        for j, (op, a) in enumerate(make_script(900 + len(policy), cap, dim, policy, n_batches=30, batch=3000,
                                                universe_scale=3.0, dup_frac=0.3)):
            assert outputs_equal(run_impl(o, op, a), run_impl(t, op, a)), f"script {policy} {j} {op}"
        check_state(t, o, f"script {policy}")
    print("collector forced ok", os.environ.get("HKV_COLLECT"))


if __name__ == "__main__":
    main()
