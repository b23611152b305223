"""Host-side logic of the B200 package that runs without a GPU: config
validation, the role gate (mirrors the reference's gate tests), workload
generators pinned to the reference."""

import threading
import time

import numpy as np
import pytest

import paper_2603_17168_b200 as hkv
from paper_2603_17168_b200 import workloads
from paper_2603_17168_b200.gate import Role, RoleGate


def test_table_config_validation_messages():
    with pytest.raises(ValueError, match="multiple of 128"):
        hkv.TableConfig(capacity=100, value_dim=1)
    with pytest.raises(ValueError, match="power of two"):
        hkv.TableConfig(capacity=128 * 3, value_dim=1)
    with pytest.raises(ValueError, match="value_dim"):
        hkv.TableConfig(capacity=128, value_dim=0)
    with pytest.raises(ValueError, match="fast_tier_budget"):
        hkv.TableConfig(capacity=256, value_dim=1, fast_tier_budget=3)
    with pytest.raises(ValueError, match="bucket_slots"):
        hkv.TableConfig(capacity=256, value_dim=1, bucket_slots=64)
    c = hkv.TableConfig(capacity=1024, value_dim=2, mode="dual", score_policy="kLfu")
    assert c.mode is hkv.Mode.dual and c.score_policy is hkv.PolicyId.kLfu and c.fast_tier_budget == 8


def test_outcome_codes_match_reference():
    assert [int(o) for o in hkv.Outcome] == [0, 1, 2, 3, 4, 5, 6]
    assert [o.name for o in hkv.Outcome] == ["Inserted", "Updated", "Rejected", "Evicted", "Found", "NotFound",
                                             "Erased"]


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        hkv.CacheTable(hkv.TableConfig(capacity=1024, value_dim=4))


def test_workloads_match_reference(reference_pkg):
    from cachekv import workloads as W

    for s in (0, 3):
        assert np.array_equal(W.uniform_distinct_keys(4096, s, 2**41), workloads.uniform_distinct_keys(4096, s, 2**41))
        assert np.array_equal(W.zipf_keys(4096, 10**6, 0.99, s), workloads.zipf_keys(4096, 10**6, 0.99, s))


# ---- role gate: compatibility matrix and fairness (reference pkg/tests/test_gate.py ideas) ----

def test_gate_compatibility_matrix():
    g = RoleGate()
    a = g.acquire(Role.Reader)
    b = g.try_acquire(Role.Reader)
    assert b is not None
    assert g.try_acquire(Role.Updater) is None
    assert g.try_acquire(Role.Inserter) is None
    a.release()
    b.release()
    i = g.acquire(Role.Inserter)
    assert g.try_acquire(Role.Inserter) is None
    assert g.try_acquire(Role.Reader) is None
    i.release()
    u = g.acquire(Role.Updater)
    u2 = g.try_acquire(Role.Updater)
    assert u2 is not None
    u.release()
    u2.release()


def test_gate_double_release():
    g = RoleGate()
    h = g.acquire(Role.Reader)
    h.release()
    with pytest.raises(RuntimeError):
        h.release()


def test_gate_phase_fair_inserter_not_starved():
    g = RoleGate()
    r1 = g.acquire(Role.Reader)
    got = []

    def inserter():
        with g.acquire(Role.Inserter):
            got.append("I")

    th = threading.Thread(target=inserter)
    th.start()
    time.sleep(0.05)
    # a later reader must queue behind the waiting inserter
    assert g.try_acquire(Role.Reader) is None
    r1.release()
    th.join(2)
    assert got == ["I"]


def test_gate_stress_audit():
    events = []
    g = RoleGate(event_hook=events.append)
    roles = [Role.Reader, Role.Updater, Role.Inserter]

    def worker(seed):
        rng = np.random.default_rng(seed)
        for _ in range(300):
            with g.acquire(roles[int(rng.integers(0, 3))]):
                pass

    ths = [threading.Thread(target=worker, args=(s,)) for s in range(6)]
    [t.start() for t in ths]
    [t.join() for t in ths]
    active = {}
    for _, ev, role, _cnt in events:
        if ev == "acquire":
            others = {r for r, c in active.items() if c > 0}
            assert not others or others == {role}
            if role is Role.Inserter:
                assert not others
            active[role] = active.get(role, 0) + 1
        else:
            active[role] -= 1
    assert all(c == 0 for c in active.values())
