"""ctypes wrapper over liboracle.so — the CPU restatement of the reference engine.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference leg of bench.py.  Never by the product package.

`OracleTable` mirrors the reference `cachekv.CacheTable` batch API
(/root/reference/pkg/src/cachekv/table.py:138-1305) on numpy arrays, with the
same argument meaning, outcome codes and return shapes.  Validation errors
follow the reference's messages (table.py:108-127, 164-188).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

SLOTS = 128
EMPTY_KEY = 0xFFFFFFFFFFFFFFFF
LOCKED_KEY = 0xFFFFFFFFFFFFFFFE
POLICIES = {"kLru": 0, "kLfu": 1, "kEpochLru": 2, "kEpochLfu": 3, "kCustomized": 4}

_u64p = C.POINTER(C.c_uint64)
_u8p = C.POINTER(C.c_uint8)
_f32p = C.POINTER(C.c_float)
_i64p = C.POINTER(C.c_int64)


def build() -> str:
    """Compile liboracle.so with the committed Makefile (gcc only)."""
    src = os.path.join(_HERE, "hkv_oracle.c")
    if (not os.path.exists(_LIB_PATH)) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        L.ot_create.restype = C.c_void_p
        L.ot_create.argtypes = [C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.c_int64, C.c_int32, C.c_int32]
        L.ot_destroy.argtypes = [C.c_void_p]
        L.ot_clone.restype = C.c_void_p
        L.ot_clone.argtypes = [C.c_void_p]
        L.ot_fmix64.restype = C.c_uint64
        L.ot_fmix64.argtypes = [C.c_uint64]
        L.ot_find.argtypes = [C.c_void_p, _u64p, C.c_int64, _f32p, _u8p]
        L.ot_find_mt.argtypes = [C.c_void_p, _u64p, C.c_int64, _f32p, _u8p, C.c_int32]
        L.ot_contains.argtypes = [C.c_void_p, _u64p, C.c_int64, _u8p]
        L.ot_find_ptr.argtypes = [C.c_void_p, _u64p, C.c_int64, _u8p, _u8p, _i64p]
        L.ot_upsert.restype = C.c_int64
        L.ot_upsert.argtypes = [C.c_void_p, C.c_int32, _u64p, _f32p, _u64p, C.c_int64, _u8p,
                                _u64p, _f32p, _u64p, _u64p, C.c_uint64]
        L.ot_assign.argtypes = [C.c_void_p, _u64p, _f32p, _u64p, C.c_int32, C.c_int64, _u8p, _u64p, C.c_uint64]
        L.ot_erase.argtypes = [C.c_void_p, _u64p, C.c_int64, _u8p]
        L.ot_export.restype = C.c_int64
        L.ot_export.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int32, C.c_uint64, _u64p,
                                _f32p, _u64p, _i64p]
        for name, rt in (("ot_keys", _u64p), ("ot_digests", _u8p), ("ot_scores", _u64p),
                         ("ot_occ", _i64p), ("ot_values", _f32p), ("ot_counters", _i64p)):
            getattr(L, name).restype = rt
            getattr(L, name).argtypes = [C.c_void_p]
        L.ot_size.restype = C.c_int64
        L.ot_size.argtypes = [C.c_void_p]
        L.ot_set_size.argtypes = [C.c_void_p, C.c_int64]
        L.ot_clock.restype = C.c_uint64
        L.ot_clock.argtypes = [C.c_void_p]
        L.ot_set_clock.argtypes = [C.c_void_p, C.c_uint64]
        L.ot_epoch.restype = C.c_uint64
        L.ot_epoch.argtypes = [C.c_void_p]
        L.ot_set_epoch.argtypes = [C.c_void_p, C.c_uint64]
        L.ot_fel.restype = C.c_int32
        L.ot_fel.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
        L.ot_set_fel.argtypes = [C.c_void_p, C.c_int32, C.c_double]
        L.ot_lookup_one.argtypes = [C.c_void_p, C.c_int64, C.c_uint64, _i64p]
        L.ot_upsert_one.restype = C.c_int32
        L.ot_upsert_one.argtypes = [C.c_void_p, C.c_int32, C.c_uint64, _f32p, C.c_int32, C.c_uint64, _i64p, _u64p]
        L.ot_snapshot.restype = C.c_void_p
        L.ot_snapshot.argtypes = [C.c_void_p]
        L.ot_restore.argtypes = [C.c_void_p, C.c_void_p]
        L.ot_snap_free.argtypes = [C.c_void_p]
    return _lib


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


def fmix64(x: int) -> int:
    return int(lib().ot_fmix64(C.c_uint64(x)))


def fmix64_array(x: np.ndarray) -> np.ndarray:
    """hashing.py:32-40 restated (numpy uint64 wrap-around)."""
    k = np.asarray(x, dtype=np.uint64).copy()
    with np.errstate(over="ignore"):
        k ^= k >> np.uint64(33)
        k *= np.uint64(0xFF51AFD7ED558CCD)
        k ^= k >> np.uint64(33)
        k *= np.uint64(0xC4CEB9FE1A85EC53)
        k ^= k >> np.uint64(33)
    return k


class OracleTable:
    """Serial CPU restatement of cachekv.CacheTable (table.py:138)."""

    def __init__(self, capacity: int, value_dim: int, mode: str = "single", score_policy: str = "kLru",
                 fast_tier_budget=None, digest_filter: bool = True, admit_ties_unified: bool = False,
                 _handle=None):
        # table.py:108-127
        if capacity <= 0 or capacity % SLOTS:
            raise ValueError("capacity must be a positive multiple of 128")
        bc = capacity // SLOTS
        if bc & (bc - 1):
            raise ValueError("bucket count must be a power of two")
        if value_dim < 1:
            raise ValueError("value_dim must be >= 1")
        if fast_tier_budget is None:
            fast_tier_budget = bc
        if not (0 <= fast_tier_budget <= bc):
            raise ValueError("fast_tier_budget out of range")
        self.capacity, self.dim, self.bucket_count = capacity, value_dim, bc
        self.mode, self.policy = mode, score_policy
        self.fast_tier_budget = fast_tier_budget
        self.digest_filter, self.admit_ties_unified = digest_filter, admit_ties_unified
        L = lib()
        self._h = _handle or L.ot_create(capacity, value_dim, int(mode == "dual"), POLICIES[score_policy],
                                         fast_tier_budget, int(digest_filter), int(admit_ties_unified))
        if not self._h:
            raise MemoryError("oracle allocation failed")

    def __del__(self):
        h = getattr(self, "_h", None)
        sn = getattr(self, "_snap", None)
        if sn:
            lib().ot_snap_free(sn)
            self._snap = None
        if h:
            lib().ot_destroy(h)
            self._h = None

    def clone(self) -> "OracleTable":
        return OracleTable(self.capacity, self.dim, self.mode, self.policy, self.fast_tier_budget,
                           self.digest_filter, self.admit_ties_unified, _handle=lib().ot_clone(self._h))

    def snapshot(self):
        """Metadata snapshot (keys, digests, scores, occupancy, size, clock)."""
        old = getattr(self, "_snap", None)
        if old:
            lib().ot_snap_free(old)
        self._snap = lib().ot_snapshot(self._h)

    def restore(self):
        lib().ot_restore(self._h, self._snap)

    # ----- raw state views (numpy views into the C arrays) ------------------------
    @property
    def keys(self):
        return np.ctypeslib.as_array(lib().ot_keys(self._h), (self.bucket_count, SLOTS))

    @property
    def digests(self):
        return np.ctypeslib.as_array(lib().ot_digests(self._h), (self.bucket_count, SLOTS))

    @property
    def scores(self):
        return np.ctypeslib.as_array(lib().ot_scores(self._h), (self.bucket_count, SLOTS))

    @property
    def occupancy(self):
        return np.ctypeslib.as_array(lib().ot_occ(self._h), (self.bucket_count,))

    @property
    def values(self):
        return np.ctypeslib.as_array(lib().ot_values(self._h), (self.capacity, self.dim))

    @property
    def counters(self) -> dict:
        c = np.ctypeslib.as_array(lib().ot_counters(self._h), (6,))
        names = ("digest_line_loads", "full_key_compares", "score_scans", "slot_lock_retries",
                 "value_copies_fast", "value_copies_overflow")
        return {n: int(v) for n, v in zip(names, c)}

    @property
    def clock(self) -> int:
        return int(lib().ot_clock(self._h))

    @clock.setter
    def clock(self, v: int):
        lib().ot_set_clock(self._h, v)

    @property
    def epoch(self) -> int:
        return int(lib().ot_epoch(self._h))

    def set_epoch(self, e: int):
        if e < self.epoch:
            raise ValueError("epoch may not decrease")
        if e > 0xFFFFFFFF:
            raise ValueError("epoch must fit in 32 bits")
        lib().ot_set_epoch(self._h, e)

    def size(self) -> int:
        return int(lib().ot_size(self._h))

    def set_size(self, s: int):
        lib().ot_set_size(self._h, s)

    def load_factor(self) -> float:
        return self.size() / self.capacity

    @property
    def first_eviction_lambda(self):
        v = C.c_double()
        return float(v.value) if lib().ot_fel(self._h, C.byref(v)) else None

    def set_first_eviction_lambda(self, v):
        lib().ot_set_fel(self._h, int(v is not None), 0.0 if v is None else float(v))

    # ----- coercion (table.py:164-188) ------------------------------------------
    def _keys(self, keys):
        k = np.ascontiguousarray(keys, dtype=np.uint64)
        if k.ndim != 1:
            raise ValueError("keys must be one-dimensional")
        if len(k) and (k >= np.uint64(LOCKED_KEY)).any():
            raise ValueError("keys must not equal a reserved sentinel value")
        return k

    def _values(self, values, n):
        v = np.ascontiguousarray(values, dtype=np.float32)
        if v.shape != (n, self.dim):
            raise ValueError("values must have shape (len(keys), value_dim)")
        return v

    def _scores(self, scores, n):
        if scores is None:
            if self.policy == "kCustomized":
                raise ValueError("kCustomized requires explicit scores")
            return None
        if self.policy != "kCustomized":
            raise ValueError("explicit scores require the kCustomized policy")
        s = np.ascontiguousarray(scores, dtype=np.uint64)
        if s.shape != (n,):
            raise ValueError("scores must have shape (len(keys),)")
        return s

    # ----- API ---------------------------------------------------------------
    def find(self, keys, out=None, threads: int = 1):
        k = self._keys(keys)
        n = len(k)
        if out is None:
            out = np.zeros((n, self.dim), dtype=np.float32)
        found = np.zeros(n, dtype=np.uint8)
        if threads > 1:
            lib().ot_find_mt(self._h, _p(k, _u64p), n, _p(out, _f32p), _p(found, _u8p), threads)
        else:
            lib().ot_find(self._h, _p(k, _u64p), n, _p(out, _f32p), _p(found, _u8p))
        return found.astype(bool), out

    def contains(self, keys):
        k = self._keys(keys)
        found = np.zeros(len(k), dtype=np.uint8)
        lib().ot_contains(self._h, _p(k, _u64p), len(k), _p(found, _u8p))
        return found.astype(bool)

    def find_ptr(self, keys):
        k = self._keys(keys)
        n = len(k)
        found = np.zeros(n, dtype=np.uint8)
        tier = np.zeros(n, dtype=np.uint8)
        off = np.zeros(n, dtype=np.int64)
        lib().ot_find_ptr(self._h, _p(k, _u64p), n, _p(found, _u8p), _p(tier, _u8p), _p(off, _i64p))
        return found.astype(bool), tier, off

    def _upsert(self, op, k, v, s, collect, ticks=None, clock_advance=0):
        n = len(k)
        outcomes = np.zeros(n, dtype=np.uint8)
        if collect:
            ek = np.zeros(n, dtype=np.uint64)
            es = np.zeros(n, dtype=np.uint64)
            ev = np.zeros((n, self.dim), dtype=np.float32)
        else:
            ek = es = ev = None
        t = None if ticks is None else np.ascontiguousarray(ticks, dtype=np.uint64)
        ne = lib().ot_upsert(self._h, op, _p(k, _u64p), _p(v, _f32p), _p(s, _u64p), n, _p(outcomes, _u8p),
                             _p(ek, _u64p), _p(ev, _f32p), _p(es, _u64p), _p(t, _u64p), clock_advance)
        if collect:
            return outcomes, ek[:ne].copy(), ev[:ne].copy(), es[:ne].copy()
        return outcomes

    def insert_or_assign(self, keys, values, scores=None, ticks=None, clock_advance=0):
        k = self._keys(keys)
        v = self._values(values, len(k))
        s = self._scores(scores, len(k))
        return self._upsert(0, k, v, s, False, ticks, clock_advance)

    def insert_and_evict(self, keys, values, scores=None, ticks=None, clock_advance=0):
        k = self._keys(keys)
        v = self._values(values, len(k))
        s = self._scores(scores, len(k))
        return self._upsert(0, k, v, s, True, ticks, clock_advance)

    def find_or_insert(self, keys, values_inout, scores=None, ticks=None, clock_advance=0):
        k = self._keys(keys)
        v = values_inout
        if (not isinstance(v, np.ndarray) or v.dtype != np.float32 or v.shape != (len(k), self.dim)
                or not v.flags.c_contiguous):
            raise ValueError("values_inout must be a C-contiguous float32 array of shape (n, value_dim)")
        s = self._scores(scores, len(k))
        return self._upsert(1, k, v, s, False, ticks, clock_advance)

    def assign(self, keys, values):
        k = self._keys(keys)
        v = self._values(values, len(k))
        out = np.zeros(len(k), dtype=np.uint8)
        lib().ot_assign(self._h, _p(k, _u64p), _p(v, _f32p), None, 0, len(k), _p(out, _u8p), None, 0)
        return out

    def assign_scores(self, keys, scores=None, ticks=None, clock_advance=0):
        k = self._keys(keys)
        s = self._scores(scores, len(k))
        out = np.zeros(len(k), dtype=np.uint8)
        t = None if ticks is None else np.ascontiguousarray(ticks, dtype=np.uint64)
        lib().ot_assign(self._h, _p(k, _u64p), None, _p(s, _u64p), int(scores is None), len(k), _p(out, _u8p),
                        _p(t, _u64p), clock_advance)
        return out

    def erase(self, keys):
        k = self._keys(keys)
        out = np.zeros(len(k), dtype=np.uint8)
        lib().ot_erase(self._h, _p(k, _u64p), len(k), _p(out, _u8p))
        return out

    # ----- single-key API (table.py:562-620) ---------------------------------
    def _lookup_one(self, bucket, key):
        res = np.zeros(3, dtype=np.int64)
        lib().ot_lookup_one(self._h, bucket, int(key), _p(res, _i64p))
        if res[0] != 4:
            return (False, -1, -1, None, None)
        b, s = int(res[1]), int(res[2])
        row = b * SLOTS + s
        fast = b < self.fast_tier_budget
        off = row * self.dim if fast else (row - self.fast_tier_budget * SLOTS) * self.dim
        return (True, b, s, 0 if fast else 1, off)

    def lookup(self, key):
        """-> (found, bucket, slot, tier, offset) (table.py:562-568)."""
        return self._lookup_one(-1, key)

    def find_in_bucket(self, bucket_index, key):
        if not (0 <= bucket_index < self.bucket_count):
            raise IndexError("bucket index out of range")
        return self._lookup_one(int(bucket_index), key)

    def _upsert_one(self, dual, key, value, score):
        key = int(key)
        if key >= LOCKED_KEY:
            raise ValueError("keys must not equal a reserved sentinel value")
        v = np.ascontiguousarray(value, dtype=np.float32).reshape(-1)
        if v.shape != (self.dim,):
            raise ValueError("value must have value_dim elements")
        res = np.zeros(3, dtype=np.int64)
        ev = np.zeros(2, dtype=np.uint64)
        rc = lib().ot_upsert_one(self._h, dual, key, _p(v, _f32p), int(score is not None),
                                 0 if score is None else int(score), _p(res, _i64p), _p(ev, _u64p))
        if rc == 1:
            raise ValueError("kCustomized requires an explicit score")
        if rc == 2:
            raise ValueError("explicit scores require the kCustomized policy")
        kind = int(res[0])
        return (kind, int(ev[0]), int(ev[1])) if kind == 3 else (kind, None, None)

    def upsert_single(self, key, value, score=None):
        """-> (kind, evicted_key, evicted_score) (table.py:584-599)."""
        return self._upsert_one(0, key, value, score)

    def upsert_dual(self, key, value, score=None):
        if self.mode != "dual":
            raise ValueError("upsert_dual requires dual mode")
        return self._upsert_one(1, key, value, score)

    def export_batch_if(self, min_score=None, cursor=None, max_count=1):
        """export_batch_if with the native `score >= min_score` predicate
        (service.py:263-268); None = always-true predicate."""
        if cursor is None:
            cursor = 0
        if not (0 <= cursor < self.capacity):
            raise ValueError("cursor out of range")
        if max_count < 1:
            raise ValueError("max_count must be >= 1")
        m = min(max_count, self.capacity)
        ok = np.zeros(m, dtype=np.uint64)
        os_ = np.zeros(m, dtype=np.uint64)
        ov = np.zeros((m, self.dim), dtype=np.float32)
        nxt = C.c_int64()
        cnt = lib().ot_export(self._h, cursor, m, int(min_score is not None),
                              0 if min_score is None else int(min_score),
                              _p(ok, _u64p), _p(ov, _f32p), _p(os_, _u64p), C.byref(nxt))
        return ok[:cnt].copy(), ov[:cnt].copy(), os_[:cnt].copy(), (None if nxt.value < 0 else int(nxt.value))

    def occupied_keys(self):
        flat = self.keys.reshape(-1)
        return flat[flat < np.uint64(LOCKED_KEY)].copy()

    def check_consistency(self) -> bool:
        keys = self.keys
        user = keys < np.uint64(LOCKED_KEY)
        occ = user.sum(axis=1)
        if not np.array_equal(occ, self.occupancy):
            raise RuntimeError("occupancy counters disagree with bucket contents")
        if int(occ.sum()) != self.size():
            raise RuntimeError("size counter disagrees with occupancy")
        if user.any():
            ub, us = np.nonzero(user)
            h = fmix64_array(keys[ub, us])
            expect = ((h >> np.uint64(32)) & np.uint64(0xFF)).astype(np.uint8)
            if not np.array_equal(expect, self.digests[ub, us]):
                raise RuntimeError("stored digest mismatch")
        return True
