"""Reference arm of bench.py: the UNMODIFIED reference package
(`cachekv.CacheTable(workers=1)`, installed into the git-ignored
baseline/_ref by baseline/install_ref.sh) timed on this host's cores at the
C2 configuration itself (2^27 slots, dim 64, kLru, 1M-key batches,
lambda 0.50 / 0.75 / 1.00).

Filling a 2^27-slot reference table through its own insert_or_assign would
take ~10-20 min per lambda, so the fill is computed in
closed form and written into the reference table's arrays (untimed set-up;
only the reference's find / insert_or_assign are timed):

  bench.py's fill protocol inserts the distinct key stream
  uniform_distinct_keys(seed 0) in 1M batches, LRU, no hits.  Under serial
  semantics key j of the stream takes tick j + 1; a
  bucket's i-th insert goes to slot i while the bucket has room, and once it
  is full the minimum score is always its oldest entry, which sits in slot
  i mod 128 (table.py:1079-1086, 1165-1181).  So the final bucket holds the
  last min(c, 128) keys of its c inserts, key i at slot i mod 128 with score
  = its tick.  The number of stream keys the protocol consumes follows from
  size = sum_b min(c_b, 128) after each batch.
  tests/test_bench_ref.py checks this state bit-exactly against the
  reference's own fill at small capacity.

Nothing here imports the B200 package: the GPU table plays no part in this
arm.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(ROOT, "baseline", "_ref")
SLOTS = 128
EMPTY = np.uint64(0xFFFFFFFFFFFFFFFF)


def import_reference():
    """The installed reference package (baseline/_ref), or None."""
    if REF_DIR not in sys.path and os.path.isdir(os.path.join(REF_DIR, "cachekv")):
        sys.path.insert(0, REF_DIR)
    try:
        import cachekv  # noqa: F401
        from cachekv import workloads as _w  # noqa: F401
    except Exception:
        return None
    import cachekv

    return cachekv


def _fmix64(x):
    k = x.copy()
    with np.errstate(over="ignore"):
        k ^= k >> np.uint64(33)
        k *= np.uint64(0xFF51AFD7ED558CCD)
        k ^= k >> np.uint64(33)
        k *= np.uint64(0xC4CEB9FE1A85EC53)
        k ^= k >> np.uint64(33)
    return k


class ClosedFormFill:
    """Closed-form result of bench.py's fill protocol (fill_table) for one
    capacity: keys of the stream, sorted once by (bucket, stream index)."""

    def __init__(self, capacity: int, batch: int, lambdas, uniform_distinct_keys, seed: int = 0):
        self.capacity = capacity
        self.buckets = capacity // SLOTS
        mask = np.uint64(self.buckets - 1)
        # stream length each lambda's fill consumes: every lambda is filled
        # from an empty table (bench.py fill_table), so each is simulated
        # from zero over the same key stream; size = sum_b min(c_b, 128)
        # is what t.size() returns between batches
        self.consumed = {}
        buf_k = np.zeros(0, np.uint64)
        buf_b = np.zeros(0, np.int64)
        have = 0

        def buckets_of(lo, hi):
            nonlocal have, buf_k, buf_b
            if hi > have:
                grow = max(hi - have, have // 4, batch)
                k = uniform_distinct_keys(grow, seed, stream_offset=have)
                buf_k = np.concatenate([buf_k, k])
                buf_b = np.concatenate([buf_b, (_fmix64(k) & mask).astype(np.int64)])
                have += grow
            return buf_b[lo:hi]

        for lam in sorted(lambdas):
            target = int(round(lam * capacity))
            counts = np.zeros(self.buckets, dtype=np.int64)
            off = size = 0
            while size < target and off <= 40 * capacity:
                n = batch if lam >= 1.0 else min(batch, target - size)
                counts += np.bincount(buckets_of(off, off + n), minlength=self.buckets)
                size = int(np.minimum(counts, SLOTS).sum())
                off += n
            self.consumed[lam] = off
        used = max(self.consumed.values()) if self.consumed else 0
        self.keys = buf_k[:used].copy()
        del buf_k, buf_b
        h = _fmix64(self.keys)
        bkt = (h & mask).astype(np.uint64)
        # one sort of (bucket << 32 | stream index): every lambda's state is a prefix filter of it
        order_key = (bkt << np.uint64(32)) | np.arange(len(self.keys), dtype=np.uint64)
        order_key.sort()
        self.sorted_b = (order_key >> np.uint64(32)).astype(np.int64)
        self.sorted_j = (order_key & np.uint64(0xFFFFFFFF)).astype(np.int64)
        self.digests_by_j = ((h >> np.uint64(32)) & np.uint64(0xFF)).astype(np.uint8)

    def state(self, lam):
        """(keys (B,128) u64, digests u8, scores u64, occupancy i64, size, clock)."""
        used = self.consumed[lam]
        sel = self.sorted_j < used
        b = self.sorted_b[sel]
        j = self.sorted_j[sel]
        cnt = np.bincount(b, minlength=self.buckets)
        start = np.concatenate([[0], np.cumsum(cnt)[:-1]])
        i = np.arange(len(b), dtype=np.int64) - start[b]  # insertion index inside the bucket
        keep = i >= (cnt[b] - SLOTS)  # the last 128 inserts of each bucket stay
        b, j, i = b[keep], j[keep], i[keep]
        slot = i % SLOTS
        keys = np.full((self.buckets, SLOTS), EMPTY, dtype=np.uint64)
        dig = np.zeros((self.buckets, SLOTS), dtype=np.uint8)
        sc = np.zeros((self.buckets, SLOTS), dtype=np.uint64)
        keys[b, slot] = self.keys[j]
        dig[b, slot] = self.digests_by_j[j]
        sc[b, slot] = (j + 1).astype(np.uint64)
        occ = np.minimum(cnt, SLOTS).astype(np.int64)
        return keys, dig, sc, occ, int(occ.sum()), int(used)


def inject(table, st):
    """Write a closed-form state into a reference CacheTable's arrays
    (table.py:143-149); values stay as allocated."""
    keys, dig, sc, occ, size, clock = st
    np.copyto(table._keys, keys)
    np.copyto(table._digests, dig)
    np.copyto(table._scores, sc)
    np.copyto(table._occupancy, occ)
    table._size = size
    table._clock = clock


def time_reference(cachekv, capacity, dim, batch, lambdas, steps, warmup, log=None):
    """Times the reference's find + insert_or_assign per lambda on one
    reference table (state injected per lambda, restored after each insert).
    Returns (value B-KV/s, detail, setup_s)."""
    from cachekv import CacheTable, TableConfig
    from cachekv.workloads import uniform_distinct_keys

    t0 = time.time()
    cf = ClosedFormFill(capacity, batch, lambdas, uniform_distinct_keys)
    table = CacheTable(TableConfig(capacity=capacity, value_dim=dim, score_policy="kLru", workers=1))
    setup = time.time() - t0
    rng = np.random.default_rng(1)
    vals = rng.standard_normal((batch, dim), dtype=np.float32)
    detail = {}
    tot_keys = 0
    tot_s = 0.0
    for lam in lambdas:
        s0 = time.time()
        st = cf.state(lam)
        inject(table, st)
        saved = (st[0], st[1], st[2], st[3], st[4], st[5])
        resident = st[0][st[0] != EMPTY]
        setup += time.time() - s0
        d = {"lambda_actual": round(st[4] / capacity, 4), "find_s": [], "insert_s": []}
        for s in range(warmup + steps):
            q = resident[rng.integers(0, len(resident), size=batch)]
            k = uniform_distinct_keys(batch, 0, stream_offset=2**44 + s * batch)
            a = time.perf_counter()
            found, _ = table.find(q)
            b = time.perf_counter()
            table.insert_or_assign(k, vals)
            c = time.perf_counter()
            r0 = time.time()
            inject(table, saved)  # back to the lambda state (untimed)
            setup += time.time() - r0
            assert found.all()
            if s >= warmup:
                d["find_s"].append(b - a)
                d["insert_s"].append(c - b)
                tot_keys += 2 * batch
                tot_s += (b - a) + (c - b)
            if log:
                log(f"reference lambda {lam} step {s}: find {b - a:.2f} s insert {c - b:.2f} s")
        detail[f"{lam:.2f}"] = {"lambda_actual": d["lambda_actual"],
                                "find_bkvs": len(d["find_s"]) * batch / sum(d["find_s"]) / 1e9,
                                "insert_or_assign_bkvs": len(d["insert_s"]) * batch / sum(d["insert_s"]) / 1e9}
    return tot_keys / tot_s / 1e9, detail, setup
