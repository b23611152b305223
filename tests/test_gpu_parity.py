"""Parity of the B200 table (CUDA kernels through the C-ABI) with the oracle
and with the reference's recorded outputs.  Bit-exact everywhere: keys,
digests, scores, values, outcomes, evicted tuples, counters.

Run on a B200: python -m pytest tests -m gpu
"""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from golden_replay import CASE_FILES, load_case, replay  # noqa: E402
from oracle.oracle import OracleTable  # noqa: E402
from refdiff import make_script, outputs_equal, run_impl  # noqa: E402

pytestmark = pytest.mark.gpu

MODES = ["single", "dual"]
POLICIES = ["kLru", "kLfu", "kEpochLru", "kEpochLfu", "kCustomized"]


@pytest.fixture(scope="module")
def hkv():
    if not torch.cuda.is_available():
        pytest.fail("gpu test ran without a CUDA device")
    import paper_2603_17168_b200 as p

    return p


def make_table(hkv, cap, dim, mode="single", policy="kLru", budget=None, unified=False, **kw):
    return hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, mode=mode, score_policy=policy,
                                          fast_tier_budget=budget, admit_ties_unified=unified, **kw))


def assert_same_state(t, o):
    st = t.export_state()
    assert st["keys"].tobytes() == o.keys.tobytes(), "keys"
    assert st["digests"].tobytes() == o.digests.tobytes(), "digests"
    assert st["scores"].tobytes() == o.scores.tobytes(), "scores"
    assert st["values"].tobytes() == o.values.tobytes(), "values"
    assert np.array_equal(st["occupancy"], o.occupancy), "occupancy"
    assert st["size"] == o.size(), "size"
    assert st["clock"] == o.clock, "clock"
    assert st["fel"] == o.first_eviction_lambda, "first_eviction_lambda"


@pytest.mark.parametrize("path", CASE_FILES, ids=[os.path.basename(p)[:-4] for p in CASE_FILES])
def test_replays_reference_fixture(hkv, path):
    """Every op of a script recorded from the reference itself."""
    meta, ops, state, ctr = load_case(path)
    t = make_table(hkv, meta["capacity"], meta["dim"], meta["mode"], meta["policy"], meta["budget"],
                   meta["unified"], overflow_in_hbm=False)
    assert replay(t, ops) is None
    st = t.export_state()
    for name in ("keys", "digests", "scores", "occupancy", "values"):
        assert st[name].tobytes() == state[name].tobytes(), name
    assert st["size"] == int(state["size"])
    assert st["clock"] == int(state["clock"])
    fel = st["fel"]
    assert (-1.0 if fel is None else fel) == float(state["fel"])
    assert t.counters.as_dict() == ctr
    assert t.check_consistency()


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("policy", POLICIES)
def test_oracle_differential_contended(hkv, mode, policy):
    """Random scripts with heavy bucket contention and in-batch duplicates."""
    cap, dim = 128 * 64, 8
    t = make_table(hkv, cap, dim, mode, policy, budget=16, overflow_in_hbm=(policy == "kLfu"))
    o = OracleTable(cap, dim, mode, policy, 16)
    for j, (op, a) in enumerate(make_script(100 + 10 * MODES.index(mode) + POLICIES.index(policy), cap, dim, policy, n_batches=40,
                                            batch=3000, universe_scale=3.0, dup_frac=0.3)):
        r_t = run_impl(t, op, a)
        r_o = run_impl(o, op, a)
        assert outputs_equal(r_o, r_t), f"op {j} {op}"
    assert_same_state(t, o)
    assert t.counters.as_dict() == o.counters
    assert t.check_consistency()


def _c1_inputs(cap, dim):
    from paper_2603_17168_b200.workloads import uniform_distinct_keys

    k0 = uniform_distinct_keys(cap // 2, seed=0)
    v0 = np.random.default_rng(0).standard_normal((len(k0), dim)).astype(np.float32)
    k1 = uniform_distinct_keys(cap, 0, stream_offset=2**41)
    v1 = np.random.default_rng(1).standard_normal((len(k1), dim)).astype(np.float32)
    return k0, v0, k1, v1


@pytest.mark.parametrize("mode", MODES)
def test_c1_config_bit_exact(hkv, mode):
    """BASELINE config 1: 2^20 slots, dim 8, kLru; prefill to 0.5, a 1M fresh
    insert_and_evict batch, then a 1M mixed find — all bit-exact."""
    cap, dim = 2**20, 8
    k0, v0, k1, v1 = _c1_inputs(cap, dim)
    t = make_table(hkv, cap, dim, mode)
    o = OracleTable(cap, dim, mode)
    assert np.array_equal(t.insert_or_assign(k0, v0), o.insert_or_assign(k0, v0))
    a = t.insert_and_evict(k1, v1)
    b = o.insert_and_evict(k1, v1)
    assert all(x.tobytes() == y.tobytes() for x, y in zip(a, b))
    q = np.concatenate([k0[::3], k1[::2], k1[1::7] + np.uint64(1)])
    ft, vt = t.find(q)
    fo, vo = o.find(q)
    assert np.array_equal(ft, fo) and vt.tobytes() == vo.tobytes()
    assert_same_state(t, o)
    assert t.counters.as_dict() == o.counters


def test_torch_io_matches_numpy_io(hkv):
    cap, dim = 2**16, 64
    t = make_table(hkv, cap, dim)
    o = OracleTable(cap, dim)
    rng = np.random.default_rng(3)
    keys = rng.integers(1, 2**63, size=50_000, dtype=np.uint64)
    vals = rng.standard_normal((len(keys), dim)).astype(np.float32)
    kd = torch.from_numpy(keys.view(np.int64)).cuda().view(torch.uint64)
    vd = torch.from_numpy(vals).cuda()
    out_t = t.insert_or_assign(kd, vd)
    out_o = o.insert_or_assign(keys, vals)
    assert np.array_equal(out_t.cpu().numpy(), out_o)
    f, v = t.find(kd)
    fo, vo = o.find(keys)
    assert np.array_equal(f.cpu().numpy(), fo) and v.cpu().numpy().tobytes() == vo.tobytes()
    # int64 view of the same keys is accepted bit-identically
    f2, v2 = t.find(kd.view(torch.int64))
    assert torch.equal(f, f2) and torch.equal(v, v2)


def test_sentinel_keys_raise_without_mutation(hkv):
    t = make_table(hkv, 1024, 4)
    good = np.arange(1, 11, dtype=np.uint64)
    t.insert_or_assign(good, np.ones((10, 4), np.float32))
    before = t.export_state()
    bad = torch.tensor([5, -2, 7], dtype=torch.int64, device="cuda")  # -2 == LOCKED
    with pytest.raises(ValueError):
        t.insert_or_assign(bad, torch.zeros((3, 4), device="cuda"))
    with pytest.raises(ValueError):
        t.erase(bad)
    with pytest.raises(ValueError):
        t.insert_or_assign(np.array([1, 2**64 - 1], dtype=np.uint64), np.zeros((2, 4), np.float32))
    after = t.export_state()
    for k in ("keys", "digests", "scores", "values"):
        assert before[k].tobytes() == after[k].tobytes()
    assert before["clock"] == after["clock"] and before["size"] == after["size"]
    # the table keeps working afterwards
    assert np.array_equal(t.contains(good), np.ones(10, bool))


def test_empty_batches(hkv):
    t = make_table(hkv, 1024, 4)
    e = np.zeros(0, dtype=np.uint64)
    v = np.zeros((0, 4), np.float32)
    assert len(t.insert_or_assign(e, v)) == 0
    o, ek, ev, es = t.insert_and_evict(e, v)
    assert len(o) == len(ek) == len(ev) == len(es) == 0
    f, out = t.find(e)
    assert len(f) == 0 and out.shape == (0, 4)
    assert len(t.erase(e)) == 0 and len(t.assign(e, v)) == 0
    assert t.size() == 0


def test_tiered_values_pinned_host(hkv):
    """Values of buckets >= fast_tier_budget live in mapped pinned host memory."""
    cap, dim = 2**15, 128
    budget = (cap // 128) // 2
    t = make_table(hkv, cap, dim, budget=budget)
    o = OracleTable(cap, dim, fast_tier_budget=budget)
    rng = np.random.default_rng(9)
    keys = rng.integers(1, 2**63, size=cap, dtype=np.uint64)
    vals = rng.standard_normal((cap, dim)).astype(np.float32)
    assert np.array_equal(t.insert_or_assign(keys, vals), o.insert_or_assign(keys, vals))
    assert np.array_equal(t.assign(keys[::2], vals[1::2]), o.assign(keys[::2], vals[1::2]))
    f1, t1, off1 = t.find_ptr(keys)
    f2, t2, off2 = o.find_ptr(keys)
    assert np.array_equal(f1, f2) and np.array_equal(t1, t2) and np.array_equal(off1, off2)
    assert t1.any() and (~t1.astype(bool)[f1]).any()
    ft, vt = t.find(keys)
    fo, vo = o.find(keys)
    assert np.array_equal(ft, fo) and vt.tobytes() == vo.tobytes()
    assert t.counters.as_dict() == o.counters
    assert_same_state(t, o)


def test_export_native_and_callable_predicates(hkv):
    cap, dim = 2**14, 4
    t = make_table(hkv, cap, dim, policy="kCustomized")
    o = OracleTable(cap, dim, score_policy="kCustomized")
    rng = np.random.default_rng(5)
    keys = rng.integers(1, 2**63, size=cap, dtype=np.uint64)
    vals = rng.standard_normal((cap, dim)).astype(np.float32)
    sc = rng.integers(0, 100, size=cap, dtype=np.uint64)
    t.insert_or_assign(keys, vals, sc)
    o.insert_or_assign(keys, vals, sc)
    for cursor, mc, ms in ((0, 10**9, None), (0, 777, 50), (5000, 3, 0), (cap - 1, 5, None), (123, 4096, 99)):
        a = t.export_batch_if(ms, cursor, mc)
        b = o.export_batch_if(ms, cursor, mc)
        assert a[3] == b[3]
        assert all(x.tobytes() == y.tobytes() for x, y in zip(a[:3], b[:3]))
    # callable predicate (reference contract: numpy (keys, scores) chunk -> mask)
    a = t.export_batch_if(lambda k, s: (s % np.uint64(3)) == 0, 0, 10**9)
    full = o.export_batch_if(None, 0, 10**9)
    m = (full[2] % np.uint64(3)) == 0
    assert np.array_equal(a[0], full[0][m]) and np.array_equal(a[2], full[2][m])
    assert a[1].tobytes() == full[1][m].tobytes()


def test_snapshot_restore(hkv):
    cap, dim = 2**14, 16
    t = make_table(hkv, cap, dim)
    rng = np.random.default_rng(1)
    k = rng.integers(1, 2**63, size=cap // 2, dtype=np.uint64)
    t.insert_or_assign(k, np.ones((len(k), dim), np.float32))
    t.snapshot()
    s0 = t.export_state()
    t.insert_or_assign(k + np.uint64(1), np.ones((len(k), dim), np.float32))
    t.restore()
    s1 = t.export_state()
    for name in ("keys", "digests", "scores", "occupancy"):
        assert s0[name].tobytes() == s1[name].tobytes()
    assert s0["size"] == s1["size"] and s0["clock"] == s1["clock"]


def test_full_size_properties_dim64(hkv):
    """C2-shaped (2^24 slots here), dim 64: fill to lambda=1 by 1M batches and
    check size-independent properties: consistency, every resident key found
    with the value it was written with, evicted + resident = offered."""
    cap, dim, batch = 2**24, 64, 2**20
    t = make_table(hkv, cap, dim)
    offered = 0
    total_ev = 0
    seed_base = 2**40
    while offered < cap + 2 * batch:
        keys = torch.arange(seed_base + offered, seed_base + offered + batch, device="cuda", dtype=torch.int64)
        vals = (keys.to(torch.float32) / 1e12).unsqueeze(1).expand(batch, dim).contiguous()
        o, ek, ev, es = t.insert_and_evict(keys, vals)
        oc = torch.bincount(o.long(), minlength=7).cpu()
        total_ev += int(oc[3])
        assert int(oc[2]) == 0  # LRU with fresh ticks never rejects
        assert ek.numel() == int(oc[3])
        offered += batch
    assert t.size() == offered - total_ev  # every insert is Inserted or Evicted; nothing lost
    assert t.check_consistency()
    res = torch.from_numpy(t.occupied_keys().view(np.int64)).cuda()
    f, v = t.find(res)
    assert bool(f.all())
    expect = (res.to(torch.float32) / 1e12).unsqueeze(1).expand(-1, dim)
    assert torch.equal(v, expect)
    assert res.numel() == t.size()


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("policy", POLICIES)
def test_zipf_same_key_runs(hkv, policy, mode):
    """Zipf batches (alpha 0.99, small universe): one key fills thousands of
    consecutive sorted positions of its bucket, so the collapsed same-key
    runs (hits, rejections under Lfu, erase misses, find_or_insert reads) are
    exercised against the one-at-a-time oracle, bit-exact incl. counters."""
    from paper_2603_17168_b200.workloads import zipf_keys

    cap, dim = 128 * 32, 4
    t = make_table(hkv, cap, dim, mode, policy=policy)
    o = OracleTable(cap, dim, mode, policy)
    rng = np.random.default_rng(11)
    custom = policy == "kCustomized"
    for j in range(14):
        keys = zipf_keys(20_000, 6 * cap, 0.99, seed=j)
        vals = rng.standard_normal((len(keys), dim)).astype(np.float32)
        sc = rng.integers(0, 60, size=len(keys), dtype=np.uint64) if custom else None
        op = ["insert_or_assign", "insert_and_evict", "find_or_insert", "insert_and_evict", "erase", "assign",
              "insert_or_assign"][j % 7]
        if op == "erase":
            args = {"keys": keys[: len(keys) // 2]}
        elif op == "assign":
            args = {"keys": keys, "values": vals}
        else:
            args = {"keys": keys, "values": vals, "scores": sc}
        r_t = run_impl(t, op, args)
        r_o = run_impl(o, op, args)
        assert outputs_equal(r_o, r_t), f"batch {j} {op}"
        if policy in ("kEpochLru", "kEpochLfu") and j % 4 == 3:
            t.set_epoch(j)
            o.set_epoch(j)
    assert_same_state(t, o)
    assert t.counters.as_dict() == o.counters
    assert t.check_consistency()


@pytest.mark.parametrize("dim", [1, 3, 4, 8, 12, 64, 132])
@pytest.mark.parametrize("mode", MODES)
def test_find_paths_ragged(hkv, dim, mode):
    """find through every kernel path (fused thread-per-key probe + warp row
    copy for dim % 4 == 0, probe + gather otherwise), ragged batch sizes that
    leave partial warps, caller-provided `out` (misses untouched) and
    out=None (misses zeroed) — bit-exact against the oracle."""
    cap = 128 * 64
    t = make_table(hkv, cap, dim, mode)
    o = OracleTable(cap, dim, mode)
    rng = np.random.default_rng(dim)
    keys = rng.integers(1, 2**63, size=int(cap * 0.9), dtype=np.uint64)
    vals = rng.standard_normal((len(keys), dim)).astype(np.float32)
    t.insert_or_assign(keys, vals)
    o.insert_or_assign(keys, vals)
    for n in (1, 31, 33, 1000, 4097):
        q = np.concatenate([keys[rng.integers(0, len(keys), size=n - n // 3)],
                            rng.integers(1, 2**63, size=n // 3, dtype=np.uint64)])
        ft, vt = t.find(q)
        fo, vo = o.find(q)
        assert np.array_equal(ft, fo) and vt.tobytes() == vo.tobytes(), f"n={n}"
        pre = np.full((n, dim), 7.0, np.float32)
        ot = torch.from_numpy(pre.copy()).cuda()
        ft2, vt2 = t.find(torch.from_numpy(q.view(np.int64)).cuda(), out=ot)
        oo = pre.copy()
        fo2, _ = o.find(q, out=oo)
        assert np.array_equal(ft2.cpu().numpy(), fo2) and vt2.cpu().numpy().tobytes() == oo.tobytes(), f"out= n={n}"
    assert t.counters.as_dict() == o.counters


@pytest.mark.parametrize("mode", MODES)
def test_checkpoint_round_trip(hkv, mode, tmp_path):
    """save_checkpoint / load_checkpoint restore the exact state: the loaded
    table matches the original byte for byte and keeps matching the oracle
    through further mutations (ticks, epoch, first-eviction lambda included)."""
    cap, dim = 128 * 32, 8
    t = make_table(hkv, cap, dim, mode, "kEpochLru", budget=8)
    o = OracleTable(cap, dim, mode, "kEpochLru", 8)
    rng = np.random.default_rng(21)
    for j in range(6):
        if j == 3:
            t.set_epoch(5)
            o.set_epoch(5)
        k = rng.integers(1, 3 * cap, size=1500).astype(np.uint64)
        v = rng.standard_normal((len(k), dim)).astype(np.float32)
        assert np.array_equal(t.insert_or_assign(k, v), o.insert_or_assign(k, v))
        assert np.array_equal(t.erase(k[:100]), o.erase(k[:100]))
    path = tmp_path / "table.npz"
    t.save_checkpoint(path)
    t2 = hkv.CacheTable.load_checkpoint(path)
    a, b = t.export_state(), t2.export_state()
    for name in ("keys", "digests", "scores", "values", "occupancy"):
        assert a[name].tobytes() == b[name].tobytes(), name
    assert (a["size"], a["clock"], a["fel"]) == (b["size"], b["clock"], b["fel"])
    for j in range(3):
        k = rng.integers(1, 3 * cap, size=1500).astype(np.uint64)
        v = rng.standard_normal((len(k), dim)).astype(np.float32)
        r2 = t2.insert_and_evict(k, v)
        ro = o.insert_and_evict(k, v)
        assert all(x.tobytes() == y.tobytes() for x, y in zip(r2, ro))
    assert_same_state(t2, o)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("pinned", [True, False])
def test_host_buffer_entry_points(hkv, mode, pinned):
    """hkv_find_host / hkv_upsert_host (CPU tensors in and out, PCIe copies
    pipelined inside the library) give the oracle's results bit-exactly: a
    batch spanning several ring cycles of find chunks, a caller `out` whose
    miss rows stay untouched, and host scores under kCustomized."""
    cap, dim = 2**18, 64
    rng = np.random.default_rng(11)
    for policy in ("kLru", "kCustomized"):
        t = make_table(hkv, cap, dim, mode, policy)
        o = OracleTable(cap, dim, mode=mode, score_policy=policy)
        pin = (lambda x: x.pin_memory()) if pinned else (lambda x: x)
        for step in range(3):
            n = 300_001 if step == 0 else 123_457  # 300k rows = 5 find chunks of 64k (ring of 3)
            keys = rng.integers(1, 2**40, size=n, dtype=np.uint64)
            keys[: n // 10] = keys[n // 10: 2 * (n // 10)]  # in-batch duplicates
            vals = rng.standard_normal((n, dim)).astype(np.float32)
            sc = rng.integers(0, 2**20, size=n, dtype=np.uint64) if policy == "kCustomized" else None
            kh = pin(torch.from_numpy(keys.view(np.int64)))
            vh = pin(torch.from_numpy(vals))
            sh = None if sc is None else pin(torch.from_numpy(sc.view(np.int64)))
            out_t = t.insert_or_assign(kh, vh, sh)
            assert out_t.device.type == "cpu"
            assert np.array_equal(out_t.numpy(), o.insert_or_assign(keys, vals, sc)), (policy, step)
            q = np.concatenate([keys[: n // 2], rng.integers(2**41, 2**42, size=n // 2, dtype=np.uint64)])
            qh = pin(torch.from_numpy(q.view(np.int64)))
            f, v = t.find(qh)
            fo, vo = o.find(q)
            assert f.device.type == "cpu" and np.array_equal(f.numpy(), fo)
            assert v.numpy().tobytes() == vo.tobytes()
            # caller-provided out: miss rows keep their contents
            base = rng.standard_normal((len(q), dim)).astype(np.float32)
            out = pin(torch.from_numpy(base.copy()))
            f2, v2 = t.find(qh, out=out)
            assert v2 is out and np.array_equal(f2.numpy(), fo)
            exp = np.where(fo[:, None], vo, base)
            assert v2.numpy().tobytes() == exp.tobytes()
            # find_or_insert with a host values_inout: found rows come back in place
            fk = np.concatenate([keys[: n // 4], rng.integers(2**42, 2**43, size=n // 4, dtype=np.uint64)])
            fv = rng.standard_normal((len(fk), dim)).astype(np.float32)
            fsc = rng.integers(0, 2**20, size=len(fk), dtype=np.uint64) if policy == "kCustomized" else None
            fvh = pin(torch.from_numpy(fv.copy()))
            fo_t = t.find_or_insert(pin(torch.from_numpy(fk.view(np.int64))), fvh,
                                    None if fsc is None else pin(torch.from_numpy(fsc.view(np.int64))))
            fv_o = fv.copy()
            fo_o = o.find_or_insert(fk, fv_o, fsc)
            assert np.array_equal(fo_t.numpy(), fo_o) and fvh.numpy().tobytes() == fv_o.tobytes()
        assert_same_state(t, o)
    # sentinel keys through the host path: ValueError, no mutation
    t = make_table(hkv, 1024, 4, mode)
    t.insert_or_assign(np.arange(1, 11, dtype=np.uint64), np.ones((10, 4), np.float32))
    before = t.export_state()
    with pytest.raises(ValueError):
        t.insert_or_assign(torch.tensor([5, -2, 7], dtype=torch.int64), torch.zeros((3, 4)))
    after = t.export_state()
    for k in ("keys", "digests", "scores", "values"):
        assert before[k].tobytes() == after[k].tobytes()
    assert before["clock"] == after["clock"] and before["size"] == after["size"]


def test_host_buffer_concurrent_readers(hkv):
    """Reader groups may overlap (gate.py role matrix): two host threads
    calling find through the host-buffer path on one table and stream get
    their own correct results (the staging ring is held per call)."""
    import threading

    cap, dim = 2**16, 16
    t = make_table(hkv, cap, dim)
    o = OracleTable(cap, dim)
    rng = np.random.default_rng(5)
    keys = rng.integers(1, 2**50, size=30_000, dtype=np.uint64)
    vals = rng.standard_normal((len(keys), dim)).astype(np.float32)
    t.insert_or_assign(keys, vals)
    o.insert_or_assign(keys, vals)
    qs = [np.concatenate([keys[j::7], rng.integers(2**51, 2**52, size=5000, dtype=np.uint64)]) for j in range(2)]
    exp = [o.find(q) for q in qs]
    errs = []

    def worker(j):
        try:
            qh = torch.from_numpy(qs[j].view(np.int64)).pin_memory()
            for _ in range(6):
                f, v = t.find(qh)
                if not (np.array_equal(f.numpy(), exp[j][0]) and v.numpy().tobytes() == exp[j][1].tobytes()):
                    errs.append(j)
        except Exception as e:  # noqa: BLE001
            errs.append(repr(e))

    th = [threading.Thread(target=worker, args=(j,)) for j in range(2)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errs, errs


@pytest.mark.parametrize("world", [2, 4])
def test_peer_find_virtual_shards(hkv, world):
    """hkv_find_peer over `world` shards of one process (same device: the
    code path of NVLink peer memory, without IPC) equals the global oracle
    table bucket for bucket: found flags and rows bit-exact, misses zeroed."""
    from paper_2603_17168_b200.workloads import fmix64_array

    cap_l, dim = 128 * 256, 12
    shards = [make_table(hkv, cap_l, dim) for _ in range(world)]
    o = OracleTable(cap_l * world, dim)
    rng = np.random.default_rng(9)
    bl = cap_l // 128
    gmask = np.uint64(bl * world - 1)
    for step in range(3):
        keys = rng.integers(1, 2**60, size=40_000, dtype=np.uint64)
        vals = rng.standard_normal((len(keys), dim)).astype(np.float32)
        o.insert_or_assign(keys, vals)
        owner = ((fmix64_array(keys) & gmask) // np.uint64(bl)).astype(np.int64)
        for r in range(world):
            sel = owner == r
            if sel.any():
                shards[r].insert_or_assign(keys[sel], vals[sel])
    for s in shards:
        s._set_peers_local(shards)
    q = np.concatenate([keys[::3], rng.integers(2**61, 2**62, size=7000, dtype=np.uint64)])
    fo, vo = o.find(q)
    qd = torch.from_numpy(q.view(np.int64)).cuda()
    for s in shards:  # every rank sees the whole table
        f, v = s._find_peer(qd)
        assert np.array_equal(f.cpu().numpy(), fo)
        assert v.cpu().numpy().tobytes() == vo.tobytes()


def test_peer_find_preconditions(hkv):
    """Peer find needs every shard's value rows in HBM, single mode and the
    digest filter: anything else is a usage error before any launch."""
    t = make_table(hkv, 128 * 64, 8)
    tiered = make_table(hkv, 128 * 64, 8, budget=8)
    dual = make_table(hkv, 128 * 64, 8, mode="dual")
    for bad in (tiered, dual):
        with pytest.raises(ValueError):
            bad._set_peers_local([bad])
    with pytest.raises(ValueError):
        t._set_peers_local([t, tiered])
    with pytest.raises(ValueError):  # no peers set yet
        t._find_peer(torch.ones(4, dtype=torch.int64, device="cuda"))


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("policy", ["kLru", "kLfu", "kCustomized"])
def test_oracle_differential_sparse_duplicates(hkv, mode, policy):
    """The sparse regime (a few ops per bucket: sorted-walk assign, no
    long-segment engine) with in-batch duplicates, against the oracle."""
    cap, dim = 128 * 1024, 4
    t = make_table(hkv, cap, dim, mode, policy)
    o = OracleTable(cap, dim, mode, policy)
    for j, (op, a) in enumerate(make_script(700 + 10 * MODES.index(mode) + POLICIES.index(policy), cap, dim, policy,
                                            n_batches=30, batch=4000, universe_scale=0.3, dup_frac=0.3)):
        r_t = run_impl(t, op, a)
        r_o = run_impl(o, op, a)
        assert outputs_equal(r_o, r_t), f"op {j} {op}"
    assert_same_state(t, o)
    assert t.counters.as_dict() == o.counters
    assert t.check_consistency()
