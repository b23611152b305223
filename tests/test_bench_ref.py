"""The reference arm's closed-form fill (bench_ref.ClosedFormFill) equals the
reference package's own fill under bench.py's protocol, bit for bit (needs
/root/reference: CPU only)."""

import numpy as np
import pytest

import bench_ref


def reference_fill(cachekv, capacity, dim, batch, lam):
    """bench.py fill_table, driven through the reference's insert_or_assign."""
    from cachekv.workloads import uniform_distinct_keys

    t = cachekv.CacheTable(cachekv.TableConfig(capacity=capacity, value_dim=dim, score_policy="kLru"))
    target = int(round(lam * capacity))
    off = 0
    vals = np.zeros((batch, dim), dtype=np.float32)
    while True:
        size = t.size()
        if size >= target or off > 40 * capacity:
            break
        n = batch if lam >= 1.0 else min(batch, target - size)
        t.insert_or_assign(uniform_distinct_keys(n, 0, stream_offset=off), vals[:n])
        off += n
    return t


@pytest.mark.parametrize("capacity,batch", [(128 * 64, 1024), (128 * 256, 4096)])
def test_closed_form_fill_matches_reference(reference_pkg, capacity, batch):
    from cachekv.workloads import uniform_distinct_keys

    lams = [0.5, 0.75, 1.0]
    cf = bench_ref.ClosedFormFill(capacity, batch, lams, uniform_distinct_keys)
    for lam in lams:
        ref = reference_fill(reference_pkg, capacity, 2, batch, lam)
        keys, dig, sc, occ, size, clock = cf.state(lam)
        assert np.array_equal(ref._keys, keys), lam
        assert np.array_equal(ref._digests, dig), lam
        assert np.array_equal(ref._scores, sc), lam
        assert np.array_equal(ref._occupancy, occ), lam
        assert ref._size == size and ref._clock == clock, lam


def test_inject_then_reference_ops_match_filled(reference_pkg):
    """A table built by inject() behaves like the filled one (next batch)."""
    from cachekv.workloads import uniform_distinct_keys

    capacity, batch, dim = 128 * 64, 1024, 2
    cf = bench_ref.ClosedFormFill(capacity, batch, [0.75], uniform_distinct_keys)
    a = reference_fill(reference_pkg, capacity, dim, batch, 0.75)
    b = reference_pkg.CacheTable(reference_pkg.TableConfig(capacity=capacity, value_dim=dim))
    bench_ref.inject(b, cf.state(0.75))
    k = uniform_distinct_keys(batch, 0, stream_offset=2**44)
    v = np.ones((batch, dim), np.float32)
    assert np.array_equal(a.insert_or_assign(k, v), b.insert_or_assign(k, v))
    assert np.array_equal(a._keys, b._keys) and np.array_equal(a._scores, b._scores)
