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
