"""Differential test: C oracle vs the reference package run live (needs
/root/reference; skipped on the GPU box, where the golden fixtures stand in)."""

import numpy as np
import pytest

from refdiff import make_script, outputs_equal, ref_state, run_impl, run_reference
from oracle.oracle import OracleTable

MODES = ["single", "dual"]
POLICIES = ["kLru", "kLfu", "kEpochLru", "kEpochLfu", "kCustomized"]


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("policy", POLICIES)
@pytest.mark.parametrize("seed", [0, 1])
def test_oracle_matches_reference(reference_pkg, mode, policy, seed):
    cap, dim = 128 * 16, 3
    budget = None if seed == 0 else 5
    ref = reference_pkg.CacheTable(reference_pkg.TableConfig(capacity=cap, value_dim=dim, mode=mode,
                                                             score_policy=policy, fast_tier_budget=budget))
    ora = OracleTable(cap, dim, mode, policy, budget)
    outcomes_seen = set()
    for j, (op, a) in enumerate(make_script(seed, cap, dim, policy, n_batches=30, batch=400, universe_scale=3.0)):
        r = run_reference(ref, op, a)
        o = run_impl(ora, op, a)
        assert outputs_equal(r, o), f"op {j} {op}"
        if op in ("insert_or_assign", "insert_and_evict", "find_or_insert"):
            outcomes_seen |= set(np.unique(np.asarray(o[0])).tolist())
    st = ref_state(ref)
    assert st["keys"].tobytes() == ora.keys.tobytes()
    assert st["scores"].tobytes() == ora.scores.tobytes()
    assert st["digests"].tobytes() == ora.digests.tobytes()
    assert st["values"].tobytes() == ora.values.tobytes()
    assert int(st["size"]) == ora.size() and int(st["clock"]) == ora.clock
    assert ref.counters.as_dict() == ora.counters
    assert ref.first_eviction_lambda == ora.first_eviction_lambda
    assert 0 in outcomes_seen and 1 in outcomes_seen  # inserted and updated exercised


def test_oracle_workload_sizes(reference_pkg):
    """C1-shaped run (2^16 slots here to stay fast): prefill to 0.5, fresh batch, mixed find."""
    from cachekv.workloads import uniform_distinct_keys

    cap, dim = 2**16, 8
    ref = reference_pkg.CacheTable(reference_pkg.TableConfig(capacity=cap, value_dim=dim))
    ora = OracleTable(cap, dim)
    k0 = uniform_distinct_keys(cap // 2, seed=0)
    v0 = np.random.default_rng(0).standard_normal((len(k0), dim)).astype(np.float32)
    assert np.array_equal(ref.insert_or_assign(k0, v0), ora.insert_or_assign(k0, v0))
    k1 = uniform_distinct_keys(cap, 0, stream_offset=2**41)
    v1 = np.random.default_rng(1).standard_normal((len(k1), dim)).astype(np.float32)
    a, b = ref.insert_and_evict(k1, v1), ora.insert_and_evict(k1, v1)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    q = np.concatenate([k0[::3], k1[::2]])
    fr, vr = ref.find(q)
    fo, vo = ora.find(q, threads=4)
    assert np.array_equal(fr, fo) and vr.tobytes() == vo.tobytes()


def _norm_lookup(r):
    if not r.found:
        return (False, -1, -1, None, None)
    return (True, r.bucket_index, r.slot_index, int(r.value_handle.tier), r.value_handle.offset)


def _norm_upsert(r):
    return (int(r.kind), r.evicted_key, r.evicted_score)


def single_key_script(seed, cap, dim, mode, policy, n=4000):
    """Mixed single-key ops (lookup / find_in_bucket / upsert_single /
    upsert_dual) on a small key universe so buckets fill, hits repeat and
    full-bucket decisions happen; explicit scores where the policy allows
    (and sometimes where it does not: a usage error only on the miss path)."""
    rng = np.random.default_rng(seed)
    universe = rng.integers(1, 2**63, size=3 * cap, dtype=np.uint64)
    ops = []
    for i in range(n):
        key = int(universe[rng.integers(0, len(universe))])
        val = rng.standard_normal(dim).astype(np.float32)
        r = rng.random()
        score = None
        if policy == "kCustomized":
            score = int(rng.integers(0, 50)) if rng.random() < 0.95 else None
        elif rng.random() < 0.03:
            score = 7
        if r < 0.25:
            ops.append(("lookup", key))
        elif r < 0.35:
            ops.append(("find_in_bucket", int(rng.integers(0, cap // 128)), key))
        elif r < 0.7 or mode == "single":
            ops.append(("upsert_single", key, val, score))
        else:
            ops.append(("upsert_dual", key, val, score))
    return ops


def apply_single(t, op, ref):
    try:
        if op[0] == "lookup":
            r = t.lookup(op[1])
            return _norm_lookup(r) if ref else r
        if op[0] == "find_in_bucket":
            r = t.find_in_bucket(op[1], op[2])
            return _norm_lookup(r) if ref else r
        r = getattr(t, op[0])(op[1], op[2], op[3])
        return _norm_upsert(r) if ref else r
    except ValueError as e:
        return ("ValueError", str(e))


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("policy", POLICIES)
def test_oracle_single_key_api_matches_reference(reference_pkg, mode, policy):
    cap, dim = 128 * 8, 2
    ref = reference_pkg.CacheTable(reference_pkg.TableConfig(capacity=cap, value_dim=dim, mode=mode,
                                                             score_policy=policy, fast_tier_budget=5))
    ora = OracleTable(cap, dim, mode, policy, 5)
    kinds = set()
    for j, op in enumerate(single_key_script(3, cap, dim, mode, policy)):
        a = apply_single(ref, op, True)
        b = apply_single(ora, op, False)
        assert a == b, (j, op[0], a, b)
        if op[0].startswith("upsert") and a[0] != "ValueError":
            kinds.add(a[0])
    st = ref_state(ref)
    assert st["keys"].tobytes() == ora.keys.tobytes()
    assert st["scores"].tobytes() == ora.scores.tobytes()
    assert st["values"].tobytes() == ora.values.tobytes()
    assert int(st["size"]) == ora.size() and int(st["clock"]) == ora.clock
    assert ref.counters.as_dict() == ora.counters
    assert ref.first_eviction_lambda == ora.first_eviction_lambda
    assert {0, 1}.issubset(kinds) and (3 in kinds or 2 in kinds)
