"""Differential driver: run one random op script on the reference
`cachekv.CacheTable` and on another table implementation (the C oracle, or
the B200 table) and compare every output and the raw state bit-exactly.

Used by tests/test_oracle_reference.py (CPU, needs /root/reference) and by
tests/golden/make_golden.py (which records the reference's outputs as
fixtures so the GPU box, which has no /root/reference, can replay them).
"""

from __future__ import annotations

import numpy as np

SLOTS = 128


def make_script(seed: int, capacity: int, dim: int, policy: str, n_batches: int = 12,
                batch: int = 700, universe_scale: float = 1.5, dup_frac: float = 0.2):
    """A seeded list of (op, args) touching every batch API, with duplicates,
    contention, absent keys and epoch changes."""
    rng = np.random.default_rng(seed)
    universe = max(8, int(capacity * universe_scale))
    # Keys are drawn from a bounded universe so repeats / hits happen often.
    base = rng.integers(1, 2**62, size=universe, dtype=np.uint64)
    base = np.unique(base)
    ops = []
    custom = policy == "kCustomized"
    epoch = 0
    for bi in range(n_batches):
        kind = rng.choice(["upsert", "evict", "foi", "find", "assign", "ascore", "erase", "export", "contains",
                           "ptr"], p=[0.22, 0.16, 0.1, 0.12, 0.08, 0.08, 0.08, 0.06, 0.05, 0.05])
        n = int(rng.integers(0, batch + 1)) if bi % 5 == 4 else batch
        keys = base[rng.integers(0, len(base), size=n)]
        if n and dup_frac > 0:
            nd = int(n * dup_frac)
            src = rng.integers(0, n, size=nd)
            dst = rng.integers(0, n, size=nd)
            keys[dst] = keys[src]
        vals = rng.standard_normal((n, dim)).astype(np.float32)
        scores = rng.integers(0, 50, size=n, dtype=np.uint64) if custom else None
        if rng.random() < 0.15 and policy in ("kEpochLru", "kEpochLfu"):
            epoch += 1
            ops.append(("set_epoch", {"epoch": epoch}))
        if kind == "upsert":
            ops.append(("insert_or_assign", {"keys": keys, "values": vals, "scores": scores}))
        elif kind == "evict":
            ops.append(("insert_and_evict", {"keys": keys, "values": vals, "scores": scores}))
        elif kind == "foi":
            ops.append(("find_or_insert", {"keys": keys, "values": vals, "scores": scores}))
        elif kind == "find":
            ops.append(("find", {"keys": keys}))
        elif kind == "contains":
            ops.append(("contains", {"keys": keys}))
        elif kind == "ptr":
            ops.append(("find_ptr", {"keys": keys}))
        elif kind == "assign":
            ops.append(("assign", {"keys": keys, "values": vals}))
        elif kind == "ascore":
            ops.append(("assign_scores", {"keys": keys, "scores": scores}))
        elif kind == "erase":
            ops.append(("erase", {"keys": keys[: n // 3]}))
        elif kind == "export":
            cursor = int(rng.integers(0, capacity))
            ops.append(("export", {"cursor": cursor, "max_count": int(rng.integers(1, capacity // 2 + 2)),
                                   "min_score": int(rng.integers(0, 20)) if rng.random() < 0.5 else None}))
    return ops


def run_reference(table, op, a):
    """Apply one op to a reference cachekv.CacheTable; normalise outputs."""
    if op == "set_epoch":
        table.set_epoch(a["epoch"])
        return ()
    if op == "insert_or_assign":
        return (table.insert_or_assign(a["keys"], a["values"], a["scores"]),)
    if op == "insert_and_evict":
        o, ek, ev, es = table.insert_and_evict(a["keys"], a["values"], a["scores"])
        return (o, ek, ev, es)
    if op == "find_or_insert":
        v = a["values"].copy()
        o = table.find_or_insert(a["keys"], v, a["scores"])
        return (o, v)
    if op == "find":
        f, v = table.find(a["keys"])
        return (f, v)
    if op == "contains":
        return (table.contains(a["keys"]),)
    if op == "find_ptr":
        return table.find_ptr(a["keys"])
    if op == "assign":
        return (table.assign(a["keys"], a["values"]),)
    if op == "assign_scores":
        return (table.assign_scores(a["keys"], a["scores"]),)
    if op == "erase":
        return (table.erase(a["keys"]),)
    if op == "export":
        ms = a["min_score"]
        pred = None if ms is None else (lambda k, s, ms=ms: s >= np.uint64(ms))
        k, v, s, nxt = table.export_batch_if(pred, a["cursor"], a["max_count"])
        return (k, v, s, -1 if nxt is None else nxt)
    raise ValueError(op)


def run_impl(table, op, a):
    """Apply one op to an OracleTable-like / B200 CacheTable (numpy I/O)."""
    if op == "set_epoch":
        table.set_epoch(a["epoch"])
        return ()
    if op == "export":
        k, v, s, nxt = table.export_batch_if(a["min_score"], a["cursor"], a["max_count"])
        return (k, v, s, -1 if nxt is None else nxt)
    if op == "find_or_insert":
        v = a["values"].copy()
        o = table.find_or_insert(a["keys"], v, a["scores"])
        return (o, v)
    return run_reference(table, op, a)


def ref_state(t):
    return {
        "keys": t._keys.copy(), "digests": t._digests.copy(), "scores": t._scores.copy(),
        "occupancy": t._occupancy.copy(), "values": np.concatenate(
            [t.store._fast.reshape(-1, t.config.value_dim), t.store._overflow.reshape(-1, t.config.value_dim)]),
        "size": np.int64(t._size), "clock": np.uint64(t._clock),
        "fel": np.float64(-1.0 if t.first_eviction_lambda is None else t.first_eviction_lambda),
    }


def outputs_equal(a, b) -> bool:
    if len(a) != len(b):
        return False
    for x, y in zip(a, b):
        x = np.asarray(x)
        y = np.asarray(y)
        if x.dtype == bool or y.dtype == bool:
            x = x.astype(np.uint8)
            y = y.astype(np.uint8)
        if x.shape != y.shape:
            return False
        if x.tobytes() != y.astype(x.dtype).tobytes():
            return False
    return True
