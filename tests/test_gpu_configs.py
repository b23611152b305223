"""Bit-exact parity at the configurations bench.py and tools/bench_configs.py
report, against the C oracle (the reference engine's serial
restatement, pinned to the reference in tests/test_oracle_reference.py):

  C2      2^24-slot dim-64 kLru table filled by bench.py's protocol to
          lambda 0.50 / 0.75 / 1.00, then the bench's exact step (1M fresh-key
          insert_or_assign + 1M resident-key find) at each lambda;
          and one full 2^27-slot lambda = 1.00 point;
  C3      zipf alpha 0.99 (universe 4 x capacity), 1M-key insert_and_evict
          batches at 2^24 under kLfu and kCustomized (score = global op index,
          reference bench.py:336-338) after a full fill: long same-key runs,
          k_meta_long / the run collapse at bench scale;
  C4      2^22 slots, dim 128, values in mapped pinned host memory
          (fast_tier_budget 0) and split 50/50: find + assign.

Outcomes, found flags, returned values, evicted tuples in batch order and the
raw table state (keys, digests, scores, values, occupancy, size, clock,
first_eviction_lambda) must be byte-identical.

Run on a B200: python -m pytest tests -m gpu
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle.oracle import OracleTable  # noqa: E402
from paper_2603_17168_b200.workloads import uniform_distinct_keys, zipf_keys  # noqa: E402

pytestmark = pytest.mark.gpu
B = 2**20


@pytest.fixture(scope="module")
def hkv():
    if not torch.cuda.is_available():
        pytest.fail("gpu test ran without a CUDA device")
    import paper_2603_17168_b200 as p

    return p


def same_state(t, o, values=True):
    st = t.export_state()
    for name, ref in (("keys", o.keys), ("digests", o.digests), ("scores", o.scores)):
        assert np.array_equal(st[name], ref), name
    if values:
        assert np.array_equal(st["values"].view(np.uint32), o.values.view(np.uint32)), "values"
    assert np.array_equal(st["occupancy"], o.occupancy), "occupancy"
    assert st["size"] == o.size() and st["clock"] == o.clock, "size/clock"
    assert st["fel"] == o.first_eviction_lambda, "first_eviction_lambda"


class Vals:
    """Distinct value rows per batch without generating 256 MB of randoms
    each time: one random block plus the batch number."""

    def __init__(self, dim, n=B):
        self.base = np.random.default_rng(7).standard_normal((n, dim)).astype(np.float32)

    def __call__(self, j, n):
        return self.base[:n] + np.float32(j)


def fill_both(t, o, lam, vals, batch=B, start_off=0):
    """bench.py fill_table (keys of uniform_distinct_keys seed 0 from
    start_off) applied to both tables; outcomes compared batch by batch."""
    cap = t.config.capacity
    target = int(round(lam * cap))
    off = start_off
    j = 0
    while True:
        size = t.size()
        assert size == o.size()
        if size >= target or off > 40 * cap:
            return off
        n = batch if lam >= 1.0 else min(batch, target - size)
        k = uniform_distinct_keys(n, 0, stream_offset=off)
        v = vals(j, n)
        a = t.insert_or_assign(k, v)
        b = o.insert_or_assign(k, v)
        assert np.array_equal(a, b), f"fill batch at offset {off}"
        off += n
        j += 1


def bench_step(t, o, step, vals, rng):
    """bench.py one_op: insert_or_assign of 1M fresh keys, find of 1M
    resident keys (sampled uniformly from the table's keys)."""
    k = uniform_distinct_keys(B, 0, stream_offset=2**44 + step * B)
    v = vals(1000 + step, B)
    a = t.insert_or_assign(k, v)
    b = o.insert_or_assign(k, v)
    assert np.array_equal(a, b), "insert_or_assign outcomes"
    res = o.occupied_keys()
    q = res[rng.integers(0, len(res), size=B)]
    q[::97] = uniform_distinct_keys(len(q[::97]), 0, stream_offset=2**40)  # a few misses
    ft, vt = t.find(q)
    fo, vo = o.find(q, threads=8)
    assert np.array_equal(ft, fo), "found"
    assert np.array_equal(vt.view(np.uint32), vo.view(np.uint32)), "find values"
    return np.bincount(a, minlength=7)


def test_c2_lambda_sweep_2pow24_dim64(hkv):
    cap, dim = 2**24, 64
    t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, score_policy="kLru"))
    o = OracleTable(cap, dim)
    vals = Vals(dim)
    rng = np.random.default_rng(0)
    off = 0
    mixes = {}
    for i, lam in enumerate((0.5, 0.75, 1.0)):
        off = fill_both(t, o, lam, vals, start_off=off)
        same_state(t, o)
        mixes[lam] = bench_step(t, o, i, vals, rng)
        same_state(t, o)
    assert t.counters.as_dict() == o.counters
    assert mixes[1.0][3] > 0 and mixes[0.5][0] > 0  # evictions at lambda 1, inserts at 0.5
    assert t.check_consistency()


def test_c2_full_2pow27_lambda1(hkv):
    """The bench's own table size: 2^27 slots, dim 64, filled to lambda = 1
    by bench.py's protocol, then its step (oracle needs ~34 GB of host RAM)."""
    cap, dim = 2**27, 64
    t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, score_policy="kLru"))
    o = OracleTable(cap, dim)
    vals = Vals(dim)
    fill_both(t, o, 1.0, vals)
    mix = bench_step(t, o, 0, vals, np.random.default_rng(1))
    assert mix[3] == B  # every fresh key evicts at lambda = 1
    same_state(t, o)
    assert t.counters.as_dict() == o.counters


@pytest.mark.parametrize("policy", ["kLfu", "kCustomized"])
def test_c3_zipf_insert_and_evict_2pow24(hkv, policy):
    cap, dim = 2**24, 64
    t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, score_policy=policy))
    o = OracleTable(cap, dim, "single", policy)
    vals = Vals(dim)
    custom = policy == "kCustomized"
    # full fill (kCustomized: score = global op index, reference bench.py:336-338)
    op = 0
    j = 0
    while t.size() < cap:
        k = uniform_distinct_keys(B, 0, stream_offset=j * B)
        v = vals(j, B)
        s = np.arange(op, op + B, dtype=np.uint64) if custom else None
        assert np.array_equal(t.insert_or_assign(k, v, s), o.insert_or_assign(k, v, s))
        op += B
        j += 1
    for b in range(4):
        k = zipf_keys(B, 4 * cap, 0.99, seed=b)
        v = vals(500 + b, B)
        s = np.arange(op, op + B, dtype=np.uint64) if custom else None
        rt = t.insert_and_evict(k, v, s)
        ro = o.insert_and_evict(k, v, s)
        for x, y, name in zip(rt, ro, ("outcomes", "evicted keys", "evicted values", "evicted scores")):
            assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8)), (b, name)
        op += B
    same_state(t, o)
    assert t.counters.as_dict() == o.counters


@pytest.mark.parametrize("budget_frac", [0.0, 0.5])
def test_c4_tiered_dim128(hkv, budget_frac):
    cap, dim = 2**22, 128
    bc = cap // 128
    budget = int(bc * budget_frac)
    t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, fast_tier_budget=budget))
    o = OracleTable(cap, dim, fast_tier_budget=budget)
    vals = Vals(dim)
    fill_both(t, o, 0.5, vals)
    res = o.occupied_keys()
    rng = np.random.default_rng(2)
    q = res[rng.integers(0, len(res), size=B)]
    ft, vt = t.find(q)
    fo, vo = o.find(q, threads=8)
    assert np.array_equal(ft, fo) and np.array_equal(vt.view(np.uint32), vo.view(np.uint32))
    v = vals(77, B)
    assert np.array_equal(t.assign(q, v), o.assign(q, v))
    fp_t = t.find_ptr(q[:4096])
    fp_o = o.find_ptr(q[:4096])
    for x, y in zip(fp_t, fp_o):
        assert np.array_equal(np.asarray(x), np.asarray(y))
    same_state(t, o)
    assert t.counters.as_dict() == o.counters
