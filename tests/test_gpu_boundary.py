"""Drop-in boundary on the B200: the native role gate seen straight through
the C-ABI (two host threads, two streams), live TxnCounters, empty-batch
bookkeeping, and the reference's OWN experiment runners (bench.py
run_lf_sweep / run_digest_ablation / stress_gate with check=True, from the
installed reference in baseline/_ref) driving the B200 CacheTable.

Run on a B200: python -m pytest tests -m gpu
"""

import ctypes as C
import os
import sys
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle.oracle import OracleTable  # noqa: E402

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def hkv():
    if not torch.cuda.is_available():
        pytest.fail("gpu test ran without a CUDA device")
    import paper_2603_17168_b200 as p

    return p


def _vp(t):
    return C.c_void_p(t.data_ptr())


def test_gate_fences_an_inserter_and_a_reader_on_two_streams(hkv):
    """Thread A: insert_or_assign on stream sA, held back on the device by a
    spin kernel.  Thread B (starts after A's call returned): find on stream
    sB.  Without the gate's device fence B's find would run first and miss
    every key; with it the result equals serial execution (all found, the
    inserted rows).  Then the mirror case: a delayed reader, then an erase."""
    lib = hkv._lib.load()
    cap, dim, n = 128 * 4096, 16, 200_000
    t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim))
    keys = torch.from_numpy(np.random.default_rng(3).integers(1, 2**62, n, dtype=np.int64)).cuda()
    vals = torch.randn(n, dim, device="cuda")
    out = torch.zeros(n, dim, device="cuda")
    found = torch.zeros(n, dtype=torch.uint8, device="cuda")
    outc = torch.empty(n, dtype=torch.uint8, device="cuda")
    sA, sB = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    issued = threading.Event()

    def inserter():
        with torch.cuda.stream(sA):
            torch.cuda._sleep(200_000_000)  # ~0.1 s of device time ahead of the insert
        hkv._lib.check(lib.hkv_upsert(t._h, 0, _vp(keys), _vp(vals), None, n, _vp(outc), None, None, None, None,
                                      None, 0, C.c_void_p(sA.cuda_stream)))
        issued.set()

    def reader():
        issued.wait()
        hkv._lib.check(lib.hkv_find(t._h, _vp(keys), n, _vp(out), _vp(found), 0, C.c_void_p(sB.cuda_stream)))

    ta, tb = threading.Thread(target=inserter), threading.Thread(target=reader)
    ta.start(), tb.start()
    ta.join(), tb.join()
    torch.cuda.synchronize()
    assert bool((found == 1).all()), "reader overlapped the inserter on the device"
    assert torch.equal(out, vals)

    # a delayed reader, then an inserter (erase) on another stream: the find
    # must still see every key
    found.zero_()
    out.zero_()
    issued.clear()

    def reader2():
        with torch.cuda.stream(sB):
            torch.cuda._sleep(200_000_000)
        hkv._lib.check(lib.hkv_find(t._h, _vp(keys), n, _vp(out), _vp(found), 0, C.c_void_p(sB.cuda_stream)))
        issued.set()

    def eraser():
        issued.wait()
        hkv._lib.check(lib.hkv_erase(t._h, _vp(keys), n, _vp(outc), C.c_void_p(sA.cuda_stream)))

    ta, tb = threading.Thread(target=reader2), threading.Thread(target=eraser)
    ta.start(), tb.start()
    ta.join(), tb.join()
    torch.cuda.synchronize()
    assert bool((found == 1).all()), "inserter overlapped the reader on the device"
    assert torch.equal(out, vals)
    assert bool((outc == 6).all()) and t.size() == 0


def test_gate_device_mirror_and_nested_roles(hkv):
    """An explicit reader hold: the same thread's finds pass through, a
    nested mutation is refused (it would deadlock), the device mirror word
    never lets a mutation run under a reader group."""
    t = hkv.CacheTable(hkv.TableConfig(capacity=128 * 64, value_dim=4))
    k = np.arange(1, 101, dtype=np.uint64)
    t.insert_or_assign(k, np.ones((100, 4), np.float32))
    g = t.gate
    with g.acquire(hkv.Role.Reader, torch.cuda.current_stream()):
        f, _ = t.find(k)
        assert f.all()
        assert g.active_state() == (hkv.Role.Reader, 1)
        with pytest.raises(ValueError, match="incompatible role"):
            t.erase(k)
    assert g.active_state() == (None, 0)
    with g.acquire(hkv.Role.Inserter):
        assert (t.erase(k[:10]) == 6).all()  # inserter covers every role
        assert t.contains(k[:10]).sum() == 0
    assert t.size() == 90
    groups = g.groups_admitted()
    t.find(k)
    t.find(k)  # a reader after a reader: same group continues? no -- each call drained the gate
    assert g.groups_admitted() >= groups


def test_counters_are_live(hkv):
    """table.counters.reset() resets the device counters (reference callers:
    bench.py:198-205, service.py:288-289)."""
    cap = 128 * 256
    t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=2))
    o = OracleTable(cap, 2)
    k = np.arange(1, 5001, dtype=np.uint64)
    v = np.ones((5000, 2), np.float32)
    t.insert_or_assign(k, v)
    o.insert_or_assign(k, v)
    assert t.counters.as_dict() == o.counters
    t.counters.reset()
    assert t.counters.digest_line_loads == 0 and t.counters.as_dict() == dict.fromkeys(o.counters, 0)
    t.find(k[:1000])
    snap = t.counters.snapshot()
    assert snap.digest_line_loads == 1000 and snap.value_copies_fast == 1000
    assert isinstance(snap, hkv.TxnCounters)
    t.counters.merge(snap)
    assert t.counters.digest_line_loads == 2000


def test_empty_host_batch_leaves_first_eviction_unset(hkv):
    """an empty upsert (CPU tensors -> hkv_upsert_host) must not
    latch first_eviction_lambda."""
    t = hkv.CacheTable(hkv.TableConfig(capacity=128 * 8, value_dim=3))
    e = t.insert_or_assign(torch.empty(0, dtype=torch.int64), torch.empty((0, 3)))
    assert len(e) == 0
    assert t.first_eviction_lambda is None
    ek = torch.empty(0, dtype=torch.int64, device="cuda")
    t.insert_or_assign(ek, torch.empty((0, 3), device="cuda"))
    t.insert_and_evict(ek, torch.empty((0, 3), device="cuda"))
    assert t.first_eviction_lambda is None and t.size() == 0
    # and it still latches correctly when evictions happen
    o = OracleTable(128 * 8, 3)
    k = np.arange(1, 3001, dtype=np.uint64)
    v = np.zeros((3000, 3), np.float32)
    t.insert_or_assign(k, v)
    o.insert_or_assign(k, v)
    assert t.first_eviction_lambda == o.first_eviction_lambda is not None


def test_batch_size_bound(hkv):
    lib = hkv._lib.load()
    t = hkv.CacheTable(hkv.TableConfig(capacity=128 * 8, value_dim=1))
    rc = lib.hkv_erase(t._h, C.c_void_p(8), 2**31, C.c_void_p(8), None)
    assert rc == hkv._lib.HKV_EINVAL
    assert b"batch too large" in lib.hkv_last_error()


# ----- the reference's own runners against the B200 class -------------------------------
def _reference_bench(hkv):
    sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
    try:
        import cachekv.bench as rb
        from cachekv.gate import Role as RefRole
    except Exception:
        pytest.skip("baseline/_ref (the installed reference) is absent")
    return rb, RefRole


@pytest.fixture
def ref_bench_on_b200(hkv, monkeypatch):
    rb, RefRole = _reference_bench(hkv)
    ours = {r: RefRole(r.value) for r in hkv.Role}

    class B200Table(hkv.CacheTable):
        # the reference's audit keys its counts on its own Role enum
        def __init__(self, config, gate_event_hook=None):
            hook = None if gate_event_hook is None else (
                lambda ev, _h=gate_event_hook: _h((ev[0], ev[1], ours[ev[2]], ev[3])))
            super().__init__(config, gate_event_hook=hook)

    def cfg(**kw):
        return hkv.TableConfig(**kw)

    monkeypatch.setattr(rb, "CacheTable", B200Table)
    monkeypatch.setattr(rb, "TableConfig", cfg)
    return rb


def test_reference_lf_sweep_runs_on_b200(ref_bench_on_b200):
    rep = ref_bench_on_b200.run_lf_sweep(capacity=2**17, dim=8, batch=2**12, check=True)
    assert rep.metric("find_miss_loads_per_op") == [1.0] * 4
    assert all(v == 1.0 for v in rep.metric("find_hit_loads_per_op"))


def test_reference_lf_sweep_dual_runs_on_b200(ref_bench_on_b200):
    rep = ref_bench_on_b200.run_lf_sweep(capacity=2**15, dim=4, mode="dual", batch=2**11, check=True)
    assert rep.metric("find_miss_loads_per_op") == [2.0] * 4


def test_reference_digest_ablation_runs_on_b200(ref_bench_on_b200):
    rep = ref_bench_on_b200.run_digest_ablation(capacity=2**16, misses=2**14, check=True)
    assert min(rep.metric("compare_ratio_off_over_on")) >= 100


def test_reference_stress_gate_runs_on_b200(ref_bench_on_b200):
    rep = ref_bench_on_b200.stress_gate(threads=6, total_ops=3000, capacity=2**13, dim=4, check=True)
    assert rep.metric("matrix_violations") == [0] and rep.metric("dual_inserters") == [0]
    assert rep.metric("torn_reads") == [0] and rep.metric("gate_events")[0] >= 6000


# ----- single-key API (table.py:562-620) vs the oracle ----------------------------------
MODES = ["single", "dual"]
POLICIES = ["kLru", "kLfu", "kEpochLru", "kEpochLfu", "kCustomized"]


def _norm(r):
    if hasattr(r, "found"):
        if not r.found:
            return (False, -1, -1, None, None)
        return (True, r.bucket_index, r.slot_index, int(r.value_handle.tier), r.value_handle.offset)
    return (int(r.kind), r.evicted_key, r.evicted_score)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("policy", POLICIES)
def test_single_key_api_matches_oracle(hkv, mode, policy):
    """lookup / find_in_bucket / upsert_single / upsert_dual interleaved with
    batch upserts: every result, then the raw state and counters, equal the
    oracle's (pinned to the reference by test_oracle_reference.py)."""
    from test_oracle_reference import single_key_script

    cap, dim = 128 * 8, 2
    t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, mode=mode, score_policy=policy,
                                       fast_tier_budget=5))
    o = OracleTable(cap, dim, mode, policy, 5)
    rng = np.random.default_rng(5)
    for j, op in enumerate(single_key_script(4, cap, dim, mode, policy, n=2500)):
        if j % 500 == 499:  # a batch in between: the summary the single-key ops invalidated is rebuilt
            k = rng.integers(1, 2**63, size=300, dtype=np.uint64)
            v = rng.standard_normal((300, dim)).astype(np.float32)
            s = rng.integers(0, 50, size=300, dtype=np.uint64) if policy == "kCustomized" else None
            assert np.array_equal(t.insert_and_evict(k, v, s)[0], o.insert_and_evict(k, v, s)[0])
        results = []
        for impl in (t, o):
            try:
                if op[0] == "lookup":
                    r = impl.lookup(op[1])
                elif op[0] == "find_in_bucket":
                    r = impl.find_in_bucket(op[1], op[2])
                else:
                    r = getattr(impl, op[0])(op[1], op[2], op[3])
                results.append(_norm(r) if impl is t else r)
            except ValueError as e:
                results.append(("ValueError", str(e)))
        assert results[0] == results[1], (j, op[0], results)
    st = t.export_state()
    assert st["keys"].tobytes() == o.keys.tobytes() and st["scores"].tobytes() == o.scores.tobytes()
    assert st["values"].tobytes() == o.values.tobytes() and st["digests"].tobytes() == o.digests.tobytes()
    assert st["size"] == o.size() and st["clock"] == o.clock and st["fel"] == o.first_eviction_lambda
    assert t.counters.as_dict() == o.counters
    assert t.check_consistency()
    # a value handle reads the row the lookup found
    res = o.occupied_keys()
    r = t.lookup(int(res[0]))
    f, v = o.find(res[:1])
    assert r.found and np.array_equal(t.read_value(r.value_handle), v[0])
