"""The concurrent upsert engine (TableConfig.workers > 1: LOCKED-sentinel
slot CAS + bucket locks, hkv_cas.cu) — the reference's threaded engine
(table.py:1185-1241), which is serializable but not serial-in-batch-order
under contention.  Checked the way SURVEY.md 8(c)(3) prescribes:

  * contention-free batches (every op owns its candidate buckets): results
    and raw state bit-exact against the oracle;
  * contended batches (in-batch duplicates, many ops per bucket, hot keys):
    the policy invariants -- consistency (occupancy, size, digests), no
    duplicate keys, size identity, residents after <= residents before +
    batch keys, every evicted key was resident or in the batch and its score
    does not exceed the evicting op's insert score, every resident key's row
    holds a value written for it, find_or_insert returns stored rows.

Run on a B200: python -m pytest tests -m gpu
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle.oracle import OracleTable, fmix64_array  # noqa: E402

pytestmark = pytest.mark.gpu
MODES = ["single", "dual"]


@pytest.fixture(scope="module")
def hkv():
    if not torch.cuda.is_available():
        pytest.fail("gpu test ran without a CUDA device")
    import paper_2603_17168_b200 as p

    return p


def buckets_of(keys, nb, dual):
    h = fmix64_array(keys)
    b1 = (h & np.uint64(nb - 1)).astype(np.int64)
    if not dual:
        return b1, b1
    h2 = fmix64_array(h ^ np.uint64(0x9E3779B97F4A7C15))
    return b1, (h2 & np.uint64(nb - 1)).astype(np.int64)


def contention_free(rng, n, nb, dual, taken):
    """n fresh keys whose candidate buckets are pairwise disjoint and avoid
    `taken` (so their ops commute: any order gives the serial result)."""
    out = []
    while len(out) < n:
        k = rng.integers(1, 2**63, size=4 * n, dtype=np.uint64)
        b1, b2 = buckets_of(k, nb, dual)
        for key, x, y in zip(k, b1, b2):
            if x in taken or y in taken:
                continue
            taken.add(int(x))
            taken.add(int(y))
            out.append(key)
            if len(out) == n:
                break
    return np.array(out, dtype=np.uint64)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("policy", ["kLru", "kCustomized"])
def test_cas_contention_free_is_bit_exact(hkv, mode, policy):
    cap, dim = 128 * 128, 8
    nb = cap // 128
    dual = mode == "dual"
    t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, mode=mode, score_policy=policy, workers=8))
    o = OracleTable(cap, dim, mode, policy)
    rng = np.random.default_rng(1)
    custom = policy == "kCustomized"
    iters, per = (600, 40) if not dual else (1500, 20)
    outcomes = set()
    for it in range(iters):
        # fresh keys (free inserts, then evictions / rejections once buckets
        # fill) plus hits of resident keys, all on pairwise disjoint buckets
        used = set()
        fresh = contention_free(rng, per, nb, dual, used)
        res = o.occupied_keys()
        hits = []
        for key in res[rng.permutation(len(res))[:64]]:
            x, y = buckets_of(np.array([key], np.uint64), nb, dual)
            x, y = int(x[0]), int(y[0])
            if x in used or y in used:
                continue
            used |= {x, y}
            hits.append(key)
            if len(hits) == 8:
                break
        keys = np.concatenate([fresh, np.array(hits, dtype=np.uint64)])
        keys = keys[rng.permutation(len(keys))]
        vals = rng.standard_normal((len(keys), dim)).astype(np.float32)
        sc = rng.integers(0, 1000, size=len(keys), dtype=np.uint64) if custom else None
        op = "insert_and_evict" if it % 2 else "insert_or_assign"
        a = getattr(t, op)(keys, vals, sc)
        b = getattr(o, op)(keys, vals, sc)
        if op == "insert_and_evict":
            for x, y in zip(a, b):
                assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8)), it
            a = a[0]
        else:
            assert np.array_equal(a, b), it
        outcomes |= set(np.unique(a).tolist())
    st = t.export_state()
    assert st["keys"].tobytes() == o.keys.tobytes()
    assert st["scores"].tobytes() == o.scores.tobytes()
    assert st["digests"].tobytes() == o.digests.tobytes()
    assert st["values"].tobytes() == o.values.tobytes()
    assert st["size"] == o.size() and st["clock"] == o.clock
    assert t.check_consistency()
    assert {0, 1}.issubset(outcomes) and (3 in outcomes or 2 in outcomes)


def check_invariants(t, before_keys, batch_keys, vals, outcomes, ek, es, s_in, written):
    st = t.export_state()
    keys = st["keys"].reshape(-1)
    resident = keys[keys < np.uint64(0xFFFFFFFFFFFFFFFE)]
    assert t.check_consistency()
    assert len(np.unique(resident)) == len(resident), "duplicate keys"
    assert st["size"] == len(resident)
    assert st["size"] == len(before_keys) + int((outcomes == 0).sum()), "size identity"
    allowed = np.union1d(before_keys, batch_keys)
    assert np.isin(resident, allowed).all(), "a resident key came from nowhere"
    if ek is not None:
        assert np.isin(ek, allowed).all(), "an evicted key was never resident"
        ev_ops = np.flatnonzero(outcomes == 3)
        assert len(ev_ops) == len(ek)
        assert (es <= s_in[ev_ops]).all(), "evicted a score above the admitted one"
    # every resident batch key holds a row written for it in this batch
    rows = np.flatnonzero(np.isin(keys, batch_keys))
    for r in rows[:: max(1, len(rows) // 2000)]:
        k = int(keys[r])
        assert any(np.array_equal(st["values"][r], vals[j]) for j in written[k]), "row not written by its key"
    return resident


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("policy", ["kLru", "kLfu", "kCustomized"])
def test_cas_contended_invariants(hkv, mode, policy):
    from paper_2603_17168_b200.workloads import zipf_keys

    cap, dim = 128 * 64, 4
    t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, mode=mode, score_policy=policy, workers=4))
    rng = np.random.default_rng(2)
    custom = policy == "kCustomized"
    resident = np.zeros(0, dtype=np.uint64)
    clock = 0
    for it in range(12):
        if it % 3 == 2:
            keys = zipf_keys(20_000, 3 * cap, 0.99, seed=it)  # hot keys: thousands of same-key ops
        else:
            keys = rng.integers(1, 4 * cap, size=6000, dtype=np.uint64)  # duplicates + full buckets
        n = len(keys)
        vals = rng.standard_normal((n, dim)).astype(np.float32)
        sc = rng.integers(0, 100, size=n, dtype=np.uint64) if custom else None
        if custom:
            s_in = sc
        elif policy == "kLru":
            s_in = np.arange(clock + 1, clock + n + 1, dtype=np.uint64)
        else:
            s_in = np.ones(n, dtype=np.uint64)
        written = {}
        for j, k in enumerate(keys.tolist()):
            written.setdefault(k, []).append(j)
        o, ek, ev, es = t.insert_and_evict(keys, vals, sc)
        clock += n
        resident = check_invariants(t, resident, keys, vals, o, ek, es, s_in, written)
        assert set(np.unique(o).tolist()) <= {0, 1, 2, 3}
    # find returns exactly the stored rows; find_or_insert reads them back
    f, v = t.find(resident)
    assert f.all()
    vi = np.zeros((len(resident), dim), np.float32)
    oi = t.find_or_insert(resident, vi, np.zeros(len(resident), np.uint64) if custom else None)
    assert (oi == 4).all() and np.array_equal(vi, v)


@pytest.mark.parametrize("mode", MODES)
def test_cas_c2_shape_invariants(hkv, mode):
    """1M-key batches at 2^24 slots, dim 64, filled past lambda = 1 with the
    concurrent engine (single and dual: full-bucket decisions through the
    eviction summary, which check_consistency verifies group by group):
    invariants at scale, every resident key found with its row."""
    cap, dim, B = 2**24, 64, 2**20
    t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, mode=mode, workers=8))
    total_ins = 0
    for j in range(20):
        keys = torch.arange(j * B + 1, (j + 1) * B + 1, device="cuda", dtype=torch.int64)
        vals = (keys.to(torch.float32) / 1e7).unsqueeze(1).expand(B, dim).contiguous()
        o = t.insert_or_assign(keys, vals)
        total_ins += int((o == 0).sum())
        assert int((o == 2).sum()) == 0  # fresh LRU ticks always admit
    assert t.size() == min(total_ins, cap) == total_ins
    assert t.check_consistency()
    res = torch.from_numpy(t.occupied_keys().view(np.int64)).cuda()
    assert torch.unique(res).numel() == res.numel()
    f, v = t.find(res)
    assert bool(f.all())
    assert torch.equal(v, (res.to(torch.float32) / 1e7).unsqueeze(1).expand(-1, dim))
