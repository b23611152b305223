"""The collector grouping of single-mode batches (hkv_collect.cu: count,
allocate, scatter, per-segment order; singletons recorded straight from the
count pass; segments of more than 16 ops sorted by a block each) against the
one-at-a-time oracle, bit-exact.

The library picks the collector for batches with fewer than 2 ops per bucket
on average, unless the previous batch on the stream was skewed (more than 8
segments of more than 16 ops), and the sorted grouping otherwise.  These tests
drive both choices in-process with batch shapes, and run a subprocess with
HKV_COLLECT=2 (collector on every batch: dense batches, zipf hot buckets,
long same-key runs) and HKV_COLLECT=0 (sorted grouping on every batch).

Run on a B200: python -m pytest tests -m gpu
"""

import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle.oracle import OracleTable  # noqa: E402
from refdiff import make_script, outputs_equal, run_impl  # noqa: E402

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def hkv():
    if not torch.cuda.is_available():
        pytest.fail("gpu test ran without a CUDA device")
    import paper_2603_17168_b200 as p

    return p


def same_state(t, o):
    st = t.export_state()
    for name, ref in (("keys", o.keys), ("digests", o.digests), ("scores", o.scores), ("values", o.values)):
        assert st[name].tobytes() == ref.tobytes(), name
    assert np.array_equal(st["occupancy"], o.occupancy)
    assert st["size"] == o.size() and st["clock"] == o.clock and st["fel"] == o.first_eviction_lambda


@pytest.mark.parametrize("policy", ["kLru", "kLfu", "kCustomized"])
def test_collector_sparse_scripts(hkv, policy):
    """Sparse batches (n < buckets: the collector by default) touching every
    batch API, with in-batch duplicates, hits, evictions and erases."""
    cap, dim = 2**20, 8  # 8192 buckets
    t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, score_policy=policy))
    o = OracleTable(cap, dim, "single", policy)
    for j, (op, a) in enumerate(make_script(500 + len(policy), cap, dim, policy, n_batches=60, batch=6000,
                                            universe_scale=0.02, dup_frac=0.3)):
        assert outputs_equal(run_impl(o, op, a), run_impl(t, op, a)), f"op {j} {op}"
    same_state(t, o)
    assert t.counters.as_dict() == o.counters
    assert t.check_consistency()


def test_collector_fill_to_full_and_evict(hkv):
    """C2 shape at 2^24 slots: 128K-key batches (1 op per bucket) filled to
    lambda 1, then insert_and_evict and find_or_insert batches, each checked."""
    from paper_2603_17168_b200.workloads import uniform_distinct_keys

    cap, dim, B = 2**24, 16, 2**17
    t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim))
    o = OracleTable(cap, dim)
    rng = np.random.default_rng(3)
    off = 0
    for j in range(int(1.3 * cap / B)):
        k = uniform_distinct_keys(B, 7, stream_offset=off)
        off += B
        v = rng.standard_normal((B, dim)).astype(np.float32)
        if j % 5 == 4:
            a, b = t.insert_and_evict(k, v), o.insert_and_evict(k, v)
            assert all(x.tobytes() == y.tobytes() for x, y in zip(a, b)), f"batch {j}"
        else:
            assert np.array_equal(t.insert_or_assign(k, v), o.insert_or_assign(k, v)), f"batch {j}"
    q = np.concatenate([uniform_distinct_keys(B // 2, 7, stream_offset=off - B), k[:100] + np.uint64(5)])
    vq = rng.standard_normal((len(q), dim)).astype(np.float32)
    vt, vo = vq.copy(), vq.copy()
    assert np.array_equal(t.find_or_insert(q, vt), o.find_or_insert(q, vo)) and vt.tobytes() == vo.tobytes()
    same_state(t, o)
    assert t.counters.as_dict() == o.counters


def test_skew_hint_switches_grouping(hkv):
    """uniform -> zipf (collector with big segments; the hint flips) -> zipf
    (sorted grouping) -> uniform (sorted, hint clears) -> uniform (collector):
    every batch bit-exact whichever grouping ran."""
    from paper_2603_17168_b200.workloads import uniform_distinct_keys, zipf_keys

    cap, dim, B = 2**22, 4, 2**14  # 32768 buckets, sparse batches
    t = hkv.CacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, score_policy="kLfu"))
    o = OracleTable(cap, dim, "single", "kLfu")
    rng = np.random.default_rng(5)
    batches = [uniform_distinct_keys(B, 1), zipf_keys(B, 4 * cap, 0.99, seed=1), zipf_keys(B, 4 * cap, 0.99, seed=2),
               uniform_distinct_keys(B, 1, stream_offset=B), uniform_distinct_keys(B, 1, stream_offset=2 * B)]
    for j, k in enumerate(batches):
        v = rng.standard_normal((len(k), dim)).astype(np.float32)
        a, b = t.insert_and_evict(k, v), o.insert_and_evict(k, v)
        assert all(x.tobytes() == y.tobytes() for x, y in zip(a, b)), f"batch {j}"
    same_state(t, o)
    assert t.counters.as_dict() == o.counters


@pytest.mark.parametrize("forced", ["2", "0"])
def test_grouping_forced(forced):
    """HKV_COLLECT=2: the collector on every batch (dense C1-shaped batches,
    zipf hot buckets, long same-key runs); HKV_COLLECT=0: the sorted grouping
    on every batch.  A subprocess, since the choice is read once per process."""
    env = dict(os.environ, HKV_COLLECT=forced)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "collector_forced.py")], env=env,
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "collector forced ok" in r.stdout
