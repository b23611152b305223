"""B200 CacheTable — drop-in mirror of the reference `cachekv.CacheTable`.

Same class, method names, argument meaning, return shapes, outcome codes and
ValueError messages as /root/reference/pkg/src/cachekv/table.py:94-1305; the
work runs in sm_100a kernels behind the C-ABI (include/hkv_b200.h):

  find / contains / find_ptr      hkv_find / hkv_contains / hkv_find_ptr
  insert_or_assign / insert_and_evict / find_or_insert   hkv_upsert
  assign / assign_scores          hkv_assign
  erase                           hkv_erase
  export_batch_if                 hkv_export
  size / load_factor              hkv_size

I/O: torch CUDA tensors (primary; keys torch.uint64 or bit-identical
torch.int64) or numpy arrays (compatibility: copied host<->device, results
returned as numpy, exactly like the reference).  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import enum
import os
import sys
import time
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np
import torch

from . import _lib
from .gate import Role, RoleGate
from .metrics import DeviceTxnCounters, TxnCounters
from .scoring import EpochState, PolicyId

BUCKET_SLOTS = 128
EMPTY_KEY = 0xFFFFFFFFFFFFFFFF
LOCKED_KEY = 0xFFFFFFFFFFFFFFFE
_LOCKED = np.uint64(LOCKED_KEY)
_TRACE = bool(os.environ.get("HKV_TRACE"))


class Mode(enum.Enum):  # table.py:63-65
    single = "single"
    dual = "dual"


class Outcome(enum.IntEnum):  # table.py:68-75
    Inserted = 0
    Updated = 1
    Rejected = 2
    Evicted = 3
    Found = 4
    NotFound = 5
    Erased = 6


class Tier(enum.IntEnum):  # store.py:27-29
    Fast = 0
    Overflow = 1


class ConsistencyError(RuntimeError):
    pass


@dataclass(frozen=True)
class ValueHandle:  # store.py:30-33
    tier: Tier
    offset: int  # element index into the tier arena


@dataclass(frozen=True)
class LookupResult:  # table.py:78-83
    found: bool
    bucket_index: int = -1
    slot_index: int = -1
    value_handle: Optional[ValueHandle] = None


@dataclass(frozen=True)
class UpsertResult:  # table.py:86-91
    kind: Outcome
    evicted_key: Optional[int] = None
    evicted_score: Optional[int] = None
    evicted_value: Optional[np.ndarray] = None


class _OneResult(C.Structure):  # hkv_one_result (include/hkv_b200.h)
    _fields_ = [("kind", C.c_int32), ("slot", C.c_int32), ("bucket", C.c_int64), ("evicted_key", C.c_uint64),
                ("evicted_score", C.c_uint64)]


_POLICY_CODE = {PolicyId.kLru: 0, PolicyId.kLfu: 1, PolicyId.kEpochLru: 2, PolicyId.kEpochLfu: 3,
                PolicyId.kCustomized: 4}


@dataclass
class TableConfig:
    """table.py:94-131; `allocator` is accepted only as None (values live in
    HBM or mapped pinned host memory).  `workers` picks the upsert engine as
    in the reference: 1 = serial batch-order semantics (bit-exact with the
    reference's default engine), > 1 = concurrent slot-CAS upserts (the
    reference's threaded engine, table.py:1185-1241: serializable, order under
    contention unspecified)."""

    capacity: int
    value_dim: int
    mode: Mode = Mode.single
    score_policy: PolicyId = PolicyId.kLru
    fast_tier_budget: Optional[int] = None
    bucket_slots: int = BUCKET_SLOTS
    digest_filter: bool = True
    admit_ties_unified: bool = False
    record_events: bool = False
    workers: int = 1
    allocator: Optional[Callable] = None
    # B200 extensions
    device: Optional[int] = None
    overflow_in_hbm: bool = False

    def __post_init__(self):
        if isinstance(self.mode, str):
            self.mode = Mode(self.mode)
        if isinstance(self.score_policy, str):
            self.score_policy = PolicyId(self.score_policy)
        if self.bucket_slots != BUCKET_SLOTS:
            raise ValueError(f"bucket_slots is fixed at {BUCKET_SLOTS}")
        if self.capacity <= 0 or self.capacity % BUCKET_SLOTS != 0:
            raise ValueError("capacity must be a positive multiple of 128")
        bc = self.capacity // BUCKET_SLOTS
        if bc & (bc - 1) != 0:
            raise ValueError("bucket count must be a power of two")
        if self.value_dim < 1:
            raise ValueError("value_dim must be >= 1")
        if self.fast_tier_budget is None:
            self.fast_tier_budget = bc
        if not (0 <= self.fast_tier_budget <= bc):
            raise ValueError("fast_tier_budget out of range")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        if self.allocator is not None:
            raise ValueError("custom allocators are not supported: values live in HBM / mapped pinned memory")

    @property
    def bucket_count(self) -> int:
        return self.capacity // BUCKET_SLOTS


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


class CacheTable:
    """B200-resident cache-semantic hash table (table.py:138)."""

    def __init__(self, config: TableConfig, gate_event_hook=None):
        self.config = config
        self._lib = _lib.load()
        if not torch.cuda.is_available():
            raise RuntimeError("CacheTable needs a CUDA device (no CPU fallback)")
        dev = torch.cuda.current_device() if config.device is None else int(config.device)
        self.device = torch.device("cuda", dev)
        cfg = _lib.HkvConfig(
            capacity=config.capacity, value_dim=config.value_dim, mode=0 if config.mode is Mode.single else 1,
            score_policy=_POLICY_CODE[config.score_policy], fast_tier_budget=config.fast_tier_budget,
            digest_filter=int(config.digest_filter), admit_ties_unified=int(config.admit_ties_unified),
            overflow_in_hbm=int(config.overflow_in_hbm), device=dev, workers=int(config.workers))
        h = C.c_void_p()
        _lib.check(self._lib.hkv_create(C.byref(cfg), C.byref(h)))
        self._h = h
        self._bucket_mask = config.bucket_count - 1
        self.epoch = EpochState(0)
        gh = C.c_void_p()
        _lib.check(self._lib.hkv_table_gate(h, C.byref(gh)))
        self.gate = RoleGate(event_hook=gate_event_hook, _handle=gh)  # the table's native gate (hkv_gate.cu)
        self.events = None  # record_events: event logs are a CPU-reference debug feature
        self.validate_keys = True

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._lib.hkv_destroy(h)
            except Exception:
                pass
            self._h = None

    # ----- plumbing -------------------------------------------------------
    def _stream(self):
        return torch.cuda.current_stream(self.device)

    def _sp(self):
        return C.c_void_p(self._stream().cuda_stream)

    def _keys_in(self, keys):
        """-> (device u64-as-int64 tensor, io mode).  io mode is True for numpy
        inputs (outputs returned as numpy, like the reference), "host" for CPU
        torch tensors (outputs returned as CPU tensors), False for tensors on the
        table's device.  Host inputs are validated on the host exactly as
        table.py:164-170; device inputs on the device (error latch)."""
        if isinstance(keys, torch.Tensor):
            if keys.dim() != 1:
                raise ValueError("keys must be one-dimensional")
            if keys.dtype not in (torch.int64, torch.uint64):
                raise ValueError("keys must be uint64 (or bit-identical int64)")
            mode = False
            if keys.device != self.device:
                if keys.device.type == "cpu":
                    self._host_key_check(keys.view(torch.int64).numpy().view(np.uint64))
                    mode = "host"
                keys = keys.to(self.device, non_blocking=True)
            return keys.contiguous().view(torch.int64), mode
        k = np.ascontiguousarray(keys, dtype=np.uint64)
        if k.ndim != 1:
            raise ValueError("keys must be one-dimensional")
        self._host_key_check(k)
        return torch.from_numpy(k.view(np.int64)).to(self.device, non_blocking=False), True

    @staticmethod
    def _host_key_check(k: np.ndarray):
        if len(k) and (k >= _LOCKED).any():
            raise ValueError("keys must not equal a reserved sentinel value")

    def _values_in(self, values, n: int, numpy_mode: bool):
        if isinstance(values, torch.Tensor):
            if tuple(values.shape) != (n, self.config.value_dim) or values.dtype != torch.float32:
                raise ValueError("values must have shape (len(keys), value_dim)")
            return values.to(self.device).contiguous()
        v = np.ascontiguousarray(values, dtype=np.float32)
        if v.shape != (n, self.config.value_dim):
            raise ValueError("values must have shape (len(keys), value_dim)")
        return torch.from_numpy(v).to(self.device)

    def _scores_in(self, scores, n: int):
        # table.py:178-188
        if scores is None:
            if self.config.score_policy is PolicyId.kCustomized:
                raise ValueError("kCustomized requires explicit scores")
            return None
        if self.config.score_policy is not PolicyId.kCustomized:
            raise ValueError("explicit scores require the kCustomized policy")
        if isinstance(scores, torch.Tensor):
            if tuple(scores.shape) != (n,):
                raise ValueError("scores must have shape (len(keys),)")
            return scores.to(self.device).contiguous().view(torch.int64)
        s = np.ascontiguousarray(scores, dtype=np.uint64)
        if s.shape != (n,):
            raise ValueError("scores must have shape (len(keys),)")
        return torch.from_numpy(s.view(np.int64)).to(self.device)

    def _check_device_error(self):
        if not self.validate_keys:
            return
        bits = C.c_int32()
        _lib.check(self._lib.hkv_device_error(self._h, C.byref(bits), self._sp()))
        if bits.value & 2:
            raise RuntimeError("a mutation kernel ran outside an inserter/updater group (role gate violated)")
        if bits.value & 1:
            raise ValueError("keys must not equal a reserved sentinel value")

    def _out(self, t: torch.Tensor, mode, dtype=None):
        if mode is True:
            a = t.cpu().numpy()
            return a if dtype is None else a.view(dtype)
        if mode == "host":
            h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            h.copy_(t, non_blocking=True)
            self._stream().synchronize()
            return h if dtype is None else h.view(dtype)
        return t if dtype is None else t.view(dtype)

    # ----- reader operations (table.py:304-372) ------------------------------
    def find(self, keys, out=None):
        """Batched lookup copying values; returns (found, values).  Misses leave
        the output row untouched (table.py:304-323)."""
        if self._host_call(keys, out):
            return self._find_host(keys, out)
        k, np_mode = self._keys_in(keys)
        n = k.numel()
        dim = self.config.value_dim
        host_out = None
        zero_misses = 0
        if out is None:
            out_d = torch.empty((n, dim), dtype=torch.float32, device=self.device)
            zero_misses = 1  # the kernel zero-fills miss rows (== reference's np.zeros out)
        elif isinstance(out, torch.Tensor):
            if tuple(out.shape) != (n, dim) or out.dtype != torch.float32:
                raise ValueError("out must be float32 with shape (len(keys), value_dim)")
            out_d = out if (out.device == self.device and out.is_contiguous()) else out.to(self.device).contiguous()
        else:
            if out.shape != (n, dim) or out.dtype != np.float32:
                raise ValueError("out must be float32 with shape (len(keys), value_dim)")
            host_out = out
            out_d = torch.from_numpy(np.ascontiguousarray(out)).to(self.device)
        _t0 = time.perf_counter() if _TRACE else 0.0
        found = torch.empty(n, dtype=torch.bool, device=self.device)
        _t1 = time.perf_counter() if _TRACE else 0.0
        st = self._stream()
        with self.gate.scope(Role.Reader, st):
            _t2 = time.perf_counter() if _TRACE else 0.0
            _lib.check(self._lib.hkv_find(self._h, _ptr(k), n, _ptr(out_d), _ptr(found), zero_misses, self._sp()))
            _t3 = time.perf_counter() if _TRACE else 0.0
        if _TRACE:
            _t4 = time.perf_counter()
            if _t4 - _t0 > 5e-4:
                print(f"[trace find] empty {1e3*(_t1-_t0):.3f} acquire {1e3*(_t2-_t1):.3f} hkv_find "
                      f"{1e3*(_t3-_t2):.3f} release {1e3*(_t4-_t3):.3f} ms", file=sys.stderr)
        if not np_mode or np_mode == "host":
            self._check_device_error()
            if isinstance(out, torch.Tensor) and out_d is not out:
                out.copy_(out_d)
                return self._out(found, np_mode), out
            if np_mode == "host":
                fh = torch.empty(found.shape, dtype=found.dtype, pin_memory=True)
                vh = torch.empty(out_d.shape, dtype=out_d.dtype, pin_memory=True)
                fh.copy_(found, non_blocking=True)
                vh.copy_(out_d, non_blocking=True)
                self._stream().synchronize()
                return fh, vh
            return found, out_d
        f = found.cpu().numpy()
        if host_out is not None:
            host_out[...] = out_d.cpu().numpy()
            return f, host_out
        return f, out_d.cpu().numpy()

    # ----- host buffers (pinned CPU tensors): hkv_find_host / hkv_upsert_host --
    @staticmethod
    def _host_call(keys, *others) -> bool:
        """CPU torch tensors in and out: the library pipelines the PCIe copies
        with the kernels (include/hkv_b200.h, host-buffer entry points)."""
        if not (isinstance(keys, torch.Tensor) and keys.device.type == "cpu"):
            return False
        return all(o is None or (isinstance(o, torch.Tensor) and o.device.type == "cpu") for o in others)

    def _host_keys(self, keys: torch.Tensor) -> torch.Tensor:
        # table.py:164-170; the reserved-sentinel test runs on the device
        # (error latch, no mutation) and surfaces through _check_device_error
        if keys.dim() != 1:
            raise ValueError("keys must be one-dimensional")
        if keys.dtype not in (torch.int64, torch.uint64):
            raise ValueError("keys must be uint64 (or bit-identical int64)")
        return keys.contiguous().view(torch.int64)

    def _find_host(self, keys, out):
        k = self._host_keys(keys)
        n = k.numel()
        dim = self.config.value_dim
        zero_misses = 0
        if out is None:
            out = torch.empty((n, dim), dtype=torch.float32, pin_memory=True)
            zero_misses = 1
        elif tuple(out.shape) != (n, dim) or out.dtype != torch.float32 or not out.is_contiguous():
            raise ValueError("out must be float32 with shape (len(keys), value_dim)")
        found = torch.empty(n, dtype=torch.bool, pin_memory=True)
        with self.gate.scope(Role.Reader, self._stream()):
            _lib.check(self._lib.hkv_find_host(self._h, _ptr(k), n, _ptr(out), _ptr(found), zero_misses,
                                               self._sp()))
        self._check_device_error()
        return found, out

    def _upsert_host(self, op: int, keys, values, scores, clock_advance: int):
        k = self._host_keys(keys)
        n = k.numel()
        dim = self.config.value_dim
        if op == 1:
            if tuple(values.shape) != (n, dim) or values.dtype != torch.float32 or not values.is_contiguous():
                raise ValueError("values_inout must be a C-contiguous float32 array of shape (n, value_dim)")
        elif tuple(values.shape) != (n, dim) or values.dtype != torch.float32:
            raise ValueError("values must have shape (len(keys), value_dim)")
        v = values.contiguous()
        s = None  # table.py:178-188
        if self.config.score_policy is PolicyId.kCustomized:
            if scores is None:
                raise ValueError("kCustomized requires explicit scores")
            if tuple(scores.shape) != (n,):
                raise ValueError("scores must have shape (len(keys),)")
            s = scores.contiguous().view(torch.int64)
        elif scores is not None:
            raise ValueError("explicit scores require the kCustomized policy")
        outcomes = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        with self.gate.scope(Role.Inserter, self._stream()):
            _lib.check(self._lib.hkv_upsert_host(self._h, op, _ptr(k), _ptr(v), _ptr(s), n, _ptr(outcomes), None,
                                                 int(clock_advance), self._sp()))
        self._check_device_error()
        return outcomes

    # ----- sharded find over peer memory (sharded.py) -------------------------
    def _set_peers_local(self, shards):
        """Shards of one process (same device, or P2P-capable devices) as the
        peer set of a sharded table; shard r owns global buckets
        [r * B, (r + 1) * B)."""
        arr = (C.c_void_p * len(shards))(*[s._h.value for s in shards])
        _lib.check(self._lib.hkv_set_peers_local(self._h, len(shards), arr))

    def _find_peer(self, keys: torch.Tensor, out=None):
        k = keys.contiguous().view(torch.int64)
        n = k.numel()
        dim = self.config.value_dim
        zero = 1 if out is None else 0
        if out is None:
            out = torch.empty((n, dim), dtype=torch.float32, device=self.device)
        found = torch.empty(n, dtype=torch.bool, device=self.device)
        with self.gate.scope(Role.Reader, self._stream()):
            _lib.check(self._lib.hkv_find_peer(self._h, _ptr(k), n, _ptr(out), _ptr(found), zero, self._sp()))
        self._check_device_error()
        return found, out

    def contains(self, keys):
        k, np_mode = self._keys_in(keys)
        n = k.numel()
        found = torch.empty(n, dtype=torch.bool, device=self.device)
        with self.gate.scope(Role.Reader, self._stream()):
            _lib.check(self._lib.hkv_contains(self._h, _ptr(k), n, _ptr(found), self._sp()))
        if not np_mode:
            self._check_device_error()
        return self._out(found, np_mode)

    def find_ptr(self, keys):
        """(found, tier, offset) without value copies (table.py:325-342)."""
        k, np_mode = self._keys_in(keys)
        n = k.numel()
        found = torch.empty(n, dtype=torch.bool, device=self.device)
        tier = torch.empty(n, dtype=torch.uint8, device=self.device)
        off = torch.empty(n, dtype=torch.int64, device=self.device)
        with self.gate.scope(Role.Reader, self._stream()):
            _lib.check(self._lib.hkv_find_ptr(self._h, _ptr(k), n, _ptr(found), _ptr(tier), _ptr(off), self._sp()))
        if not np_mode:
            self._check_device_error()
        return self._out(found, np_mode), self._out(tier, np_mode), self._out(off, np_mode)

    def export_batch_if(self, predicate, cursor, max_count: int):
        """Stream entries matching predicate in slot order; returns (keys,
        values, scores, next_cursor) (table.py:374-434).  `predicate` may be
        None, a number (native device predicate `score >= min_score`, the
        service's only use, service.py:263-268) or a Python callable on numpy
        (keys, scores) chunks, evaluated like the reference on 64-bucket
        chunks copied to the host."""
        if cursor is None:
            cursor = 0
        if not (0 <= cursor < self.config.capacity):
            raise ValueError("cursor out of range")
        if max_count < 1:
            raise ValueError("max_count must be >= 1")
        cap = self.config.capacity
        m = min(int(max_count), cap - cursor)
        dim = self.config.value_dim
        ok = torch.empty(m, dtype=torch.int64, device=self.device)
        ov = torch.empty((m, dim), dtype=torch.float32, device=self.device)
        osc = torch.empty(m, dtype=torch.int64, device=self.device)
        cnt = C.c_int64()
        nxt = C.c_int64()
        with self.gate.scope(Role.Reader, self._stream()):
            if predicate is None or isinstance(predicate, (int, np.integer)):
                has = predicate is not None
                _lib.check(self._lib.hkv_export(self._h, cursor, m, int(has), int(predicate) if has else 0, None, 0,
                                                _ptr(ok), _ptr(ov), _ptr(osc), C.byref(cnt), C.byref(nxt),
                                                self._sp()))
                taken, next_cursor = cnt.value, nxt.value
            else:
                taken, next_cursor = self._export_callable(predicate, cursor, m, ok, ov, osc)
        keys = ok[:taken].cpu().numpy().view(np.uint64)
        vals = ov[:taken].cpu().numpy()
        scores = osc[:taken].cpu().numpy().view(np.uint64)
        return keys, vals, scores, (None if next_cursor < 0 else int(next_cursor))

    def _export_callable(self, predicate, cursor, m, ok, ov, osc):
        chunk = 64 * BUCKET_SLOTS * 64  # rows per host round trip (a multiple of the reference's 64-bucket chunk)
        cap = self.config.capacity
        taken = 0
        pos = cursor
        next_cursor = -1
        kbuf = np.empty(chunk, dtype=np.uint64)
        sbuf = np.empty(chunk, dtype=np.uint64)
        while pos < cap and taken < m:
            hi = min(pos + chunk, cap)
            # only this chunk's keys and scores cross PCIe (hkv_read_rows)
            kc, sc = kbuf[: hi - pos], sbuf[: hi - pos]
            _lib.check(self._lib.hkv_read_rows(self._h, pos, hi - pos, kc.ctypes.data_as(C.c_void_p),
                                               sc.ctypes.data_as(C.c_void_p), self._sp()))
            # reference evaluates the predicate per 64-bucket chunk (table.py:402-409)
            mask = np.zeros(hi - pos, dtype=bool)
            sub = 64 * BUCKET_SLOTS
            for a in range(0, hi - pos, sub):
                b = min(a + sub, hi - pos)
                mask[a:b] = np.asarray(predicate(kc[a:b].copy(), sc[a:b].copy()), dtype=bool)
            md = torch.from_numpy(mask.view(np.uint8)).to(self.device)
            cnt = C.c_int64()
            nxt = C.c_int64()
            _lib.check(self._lib.hkv_export(self._h, pos, m - taken, 0, 0, _ptr(md), hi - pos,
                                            C.c_void_p(ok.data_ptr() + 8 * taken),
                                            C.c_void_p(ov.data_ptr() + 4 * taken * self.config.value_dim),
                                            C.c_void_p(osc.data_ptr() + 8 * taken), C.byref(cnt), C.byref(nxt),
                                            self._sp()))
            taken += cnt.value
            if taken >= m:
                next_cursor = nxt.value
                break
            pos = hi
        return taken, next_cursor

    # ----- updater operations (table.py:438-506) -----------------------------
    def assign(self, keys, values):
        k, np_mode = self._keys_in(keys)
        v = self._values_in(values, k.numel(), np_mode)
        return self._assign_impl(k, v, None, False, np_mode)

    def assign_scores(self, keys, scores=None, *, ticks=None, clock_advance: int = 0):
        k, np_mode = self._keys_in(keys)
        s = self._scores_in(scores, k.numel())
        return self._assign_impl(k, None, s, scores is None, np_mode, ticks, clock_advance)

    def _assign_impl(self, k, v, s, refresh, np_mode, ticks=None, clock_advance=0):
        n = k.numel()
        outcomes = torch.empty(n, dtype=torch.uint8, device=self.device)
        tk = None if ticks is None else ticks.to(self.device).contiguous()
        with self.gate.scope(Role.Updater, self._stream()):
            _lib.check(self._lib.hkv_assign(self._h, _ptr(k), _ptr(v), _ptr(s), int(refresh), n, _ptr(outcomes),
                                            _ptr(tk), int(clock_advance), self._sp()))
        self._check_device_error()
        return self._out(outcomes, np_mode)

    # ----- inserter operations (table.py:515-558) ----------------------------
    def insert_or_assign(self, keys, values, scores=None, *, ticks=None, clock_advance: int = 0):
        if ticks is None and self._host_call(keys, values, scores):
            return self._upsert_host(0, keys, values, scores, clock_advance)
        k, np_mode = self._keys_in(keys)
        n = k.numel()
        v = self._values_in(values, n, np_mode)
        s = self._scores_in(scores, n)
        outcomes = torch.empty(n, dtype=torch.uint8, device=self.device)
        tk = None if ticks is None else ticks.to(self.device).contiguous()
        with self.gate.scope(Role.Inserter, self._stream()):
            _lib.check(self._lib.hkv_upsert(self._h, 0, _ptr(k), _ptr(v), _ptr(s), n, _ptr(outcomes), None, None,
                                            None, None, _ptr(tk), int(clock_advance), self._sp()))
        self._check_device_error()
        return self._out(outcomes, np_mode)

    def insert_and_evict(self, keys, values, scores=None, *, ticks=None, clock_advance: int = 0):
        """Upsert and return (outcomes, evicted_keys, evicted_values,
        evicted_scores), evicted entries in batch order (table.py:525-533)."""
        k, np_mode = self._keys_in(keys)
        n = k.numel()
        dim = self.config.value_dim
        v = self._values_in(values, n, np_mode)
        s = self._scores_in(scores, n)
        outcomes = torch.empty(n, dtype=torch.uint8, device=self.device)
        ek = torch.empty(n, dtype=torch.int64, device=self.device)
        ev = torch.empty((n, dim), dtype=torch.float32, device=self.device)
        es = torch.empty(n, dtype=torch.int64, device=self.device)
        ne = torch.zeros(1, dtype=torch.int64, device=self.device)
        tk = None if ticks is None else ticks.to(self.device).contiguous()
        with self.gate.scope(Role.Inserter, self._stream()):
            _lib.check(self._lib.hkv_upsert(self._h, 0, _ptr(k), _ptr(v), _ptr(s), n, _ptr(outcomes), _ptr(ek),
                                            _ptr(ev), _ptr(es), _ptr(ne), _ptr(tk), int(clock_advance), self._sp()))
        self._check_device_error()
        e = int(ne.item())
        if np_mode is True:
            return (outcomes.cpu().numpy(), ek[:e].cpu().numpy().view(np.uint64), ev[:e].cpu().numpy(),
                    es[:e].cpu().numpy().view(np.uint64))
        if np_mode == "host":
            return (self._out(outcomes, "host"), self._out(ek[:e], "host", torch.uint64),
                    self._out(ev[:e], "host"), self._out(es[:e], "host", torch.uint64))
        return outcomes, ek[:e].view(torch.uint64), ev[:e], es[:e].view(torch.uint64)

    def find_or_insert(self, keys, values_inout, scores=None, *, ticks=None, clock_advance: int = 0):
        """Present keys: copy the stored value out and refresh the score;
        absent keys: upsert the caller's value (table.py:535-551)."""
        if ticks is None and self._host_call(keys, values_inout, scores):
            return self._upsert_host(1, keys, values_inout, scores, clock_advance)
        k, np_mode = self._keys_in(keys)
        n = k.numel()
        dim = self.config.value_dim
        if isinstance(values_inout, torch.Tensor):
            if (values_inout.dtype != torch.float32 or tuple(values_inout.shape) != (n, dim)
                    or not values_inout.is_contiguous() or values_inout.device != self.device):
                raise ValueError(
                    "values_inout must be a C-contiguous float32 array of shape (n, value_dim)")
            vd = values_inout
        else:
            v = values_inout
            if (not isinstance(v, np.ndarray) or v.dtype != np.float32 or v.shape != (n, dim)
                    or not v.flags.c_contiguous):
                raise ValueError(
                    "values_inout must be a C-contiguous float32 array of shape (n, value_dim)")
            vd = torch.from_numpy(v).to(self.device)
        s = self._scores_in(scores, n)
        outcomes = torch.empty(n, dtype=torch.uint8, device=self.device)
        tk = None if ticks is None else ticks.to(self.device).contiguous()
        with self.gate.scope(Role.Inserter, self._stream()):
            _lib.check(self._lib.hkv_upsert(self._h, 1, _ptr(k), _ptr(vd), _ptr(s), n, _ptr(outcomes), None, None,
                                            None, None, _ptr(tk), int(clock_advance), self._sp()))
        self._check_device_error()
        if not isinstance(values_inout, torch.Tensor):
            values_inout[...] = vd.cpu().numpy()
        return self._out(outcomes, np_mode)

    def erase(self, keys):
        k, np_mode = self._keys_in(keys)
        n = k.numel()
        outcomes = torch.empty(n, dtype=torch.uint8, device=self.device)
        with self.gate.scope(Role.Inserter, self._stream()):
            _lib.check(self._lib.hkv_erase(self._h, _ptr(k), n, _ptr(outcomes), self._sp()))
        self._check_device_error()
        return self._out(outcomes, np_mode)

    # ----- single-key API (table.py:562-620) ---------------------------------
    def value_address(self, bucket_index: int, slot_index: int) -> ValueHandle:
        """(bucket, slot) -> (tier, element offset) (store.py:84-94)."""
        if not (0 <= bucket_index < self.config.bucket_count):
            raise ValueError("bucket index out of range")
        if not (0 <= slot_index < BUCKET_SLOTS):
            raise ValueError("slot index out of range")
        dim, budget = self.config.value_dim, self.config.fast_tier_budget
        off = (bucket_index * BUCKET_SLOTS + slot_index) * dim
        if bucket_index < budget:
            return ValueHandle(Tier.Fast, off)
        return ValueHandle(Tier.Overflow, off - budget * BUCKET_SLOTS * dim)

    def _lookup_result(self, r: "_OneResult") -> LookupResult:
        if r.kind != int(Outcome.Found):
            return LookupResult(False)
        return LookupResult(True, int(r.bucket), int(r.slot), self.value_address(int(r.bucket), int(r.slot)))

    def lookup(self, key: int) -> LookupResult:
        """Single-key find returning slot coordinates and a value handle."""
        r = _OneResult()
        with self.gate.scope(Role.Reader, self._stream()):
            _lib.check(self._lib.hkv_lookup(self._h, int(key) & EMPTY_KEY, C.byref(r), self._sp()))
        return self._lookup_result(r)

    def find_in_bucket(self, bucket_index: int, key: int) -> LookupResult:
        """Digest-accelerated probe of one bucket; a miss is definitive for
        this bucket."""
        b = int(bucket_index)
        if not (0 <= b < self.config.bucket_count):
            raise IndexError("bucket index out of range")
        r = _OneResult()
        with self.gate.scope(Role.Reader, self._stream()):
            _lib.check(self._lib.hkv_find_in_bucket(self._h, b, int(key) & EMPTY_KEY, C.byref(r), self._sp()))
        return self._lookup_result(r)

    def _upsert_one(self, fn, key, value, score) -> UpsertResult:
        key = int(key)
        if key >= LOCKED_KEY:
            raise ValueError("keys must not equal a reserved sentinel value")
        v = np.ascontiguousarray(value, dtype=np.float32).reshape(-1)
        if v.shape != (self.config.value_dim,):
            raise ValueError("value must have value_dim elements")
        r = _OneResult()
        with self.gate.scope(Role.Inserter, self._stream()):
            _lib.check(fn(self._h, key, v.ctypes.data_as(C.c_void_p), int(score is not None),
                          0 if score is None else int(score), C.byref(r), self._sp()))
        kind = Outcome(int(r.kind))
        if kind is Outcome.Evicted:
            return UpsertResult(kind, int(r.evicted_key), int(r.evicted_score))
        return UpsertResult(kind)

    def upsert_single(self, key: int, value, score: Optional[int] = None) -> UpsertResult:
        """One-key single-bucket upsert (update / insert / reject / evict)
        in bucket h1 -- also on a dual-mode table (table.py:584-599)."""
        return self._upsert_one(self._lib.hkv_upsert_single, key, value, score)

    def upsert_dual(self, key: int, value, score: Optional[int] = None) -> UpsertResult:
        """One-key dual-bucket upsert: fill the less-occupied candidate while
        space remains, then evict in the bucket with the lower minimum score
        (ties rejected unless unified) (table.py:601-620)."""
        if self.config.mode is not Mode.dual:
            raise ValueError("upsert_dual requires dual mode")
        return self._upsert_one(self._lib.hkv_upsert_dual, key, value, score)

    def read_value(self, handle: ValueHandle, out_buffer: Optional[np.ndarray] = None) -> np.ndarray:
        """The value row a handle addresses (store.py:96-100)."""
        dim, budget = self.config.value_dim, self.config.fast_tier_budget
        row = handle.offset // dim + (0 if handle.tier is Tier.Fast else budget * BUCKET_SLOTS)
        out = np.empty(dim, dtype=np.float32) if out_buffer is None else out_buffer
        if out.shape != (dim,):
            raise ValueError("buffer length must equal value_dim")
        _lib.check(self._lib.hkv_read_value_rows(self._h, row, 1, out.ctypes.data_as(C.c_void_p), self._sp()))
        return out

    # ----- size / clock / epoch (table.py:192-215) ---------------------------
    def size(self) -> int:
        v = C.c_int64()
        with self.gate.scope(Role.Reader, self._stream()):
            _lib.check(self._lib.hkv_size(self._h, C.byref(v), self._sp()))
        return int(v.value)

    def load_factor(self) -> float:
        return self.size() / self.config.capacity

    def set_workers(self, workers: int) -> None:
        """Switch the upsert engine (TableConfig.workers semantics): 1 =
        serial batch order, > 1 = concurrent slot CAS (hkv_set_workers)."""
        if workers < 1:
            raise ValueError("workers must be >= 1")
        _lib.check(self._lib.hkv_set_workers(self._h, int(workers)))
        self.config.workers = int(workers)

    def set_epoch(self, epoch: int) -> None:
        self.epoch.advance_to(epoch)
        _lib.check(self._lib.hkv_set_epoch(self._h, int(epoch)))

    @property
    def _size(self) -> int:
        v = C.c_int64()
        _lib.check(self._lib.hkv_size(self._h, C.byref(v), self._sp()))
        return int(v.value)

    @property
    def _clock(self) -> int:
        v = C.c_uint64()
        _lib.check(self._lib.hkv_clock(self._h, C.byref(v), self._sp()))
        return int(v.value)

    @property
    def first_eviction_lambda(self) -> Optional[float]:
        s = C.c_int32()
        v = C.c_double()
        _lib.check(self._lib.hkv_first_eviction_lambda(self._h, C.byref(s), C.byref(v), self._sp()))
        return float(v.value) if s.value else None

    @property
    def counters(self) -> TxnCounters:
        """Live device counters (metrics.py:14-39): reset() / snapshot() /
        field reads go to the device."""
        c = self.__dict__.get("_counters")
        if c is None:
            c = self.__dict__["_counters"] = DeviceTxnCounters(self)
        return c

    def _device_counters(self) -> dict:
        arr = (C.c_int64 * 6)()
        _lib.check(self._lib.hkv_counters(self._h, arr, self._sp()))
        return dict(zip(("digest_line_loads", "full_key_compares", "score_scans", "slot_lock_retries",
                         "value_copies_fast", "value_copies_overflow"), (int(x) for x in arr)))

    def reset_counters(self) -> None:
        _lib.check(self._lib.hkv_reset_counters(self._h, self._sp()))

    # ----- checkpoint (the reference streams export_batch_if
    # "for checkpointing", but has no restore) --
    CHECKPOINT_VERSION = 1

    def save_checkpoint(self, path) -> None:
        """Write the table's exact state (slot positions, stale erased
        entries, scores, values, size, logical clock, epoch, first-eviction
        lambda) to one uncompressed .npz file; load_checkpoint restores it
        bit-for-bit, so every later op behaves as on the original table.
        TxnCounters are not part of the state."""
        st = self.export_state()
        c = self.config
        header = {"version": self.CHECKPOINT_VERSION, "capacity": c.capacity, "value_dim": c.value_dim,
                  "mode": c.mode.value, "score_policy": c.score_policy.value,
                  "fast_tier_budget": c.fast_tier_budget, "digest_filter": bool(c.digest_filter),
                  "admit_ties_unified": bool(c.admit_ties_unified), "epoch": int(self.epoch.current_epoch),
                  "clock": int(st["clock"]), "size": int(st["size"]),
                  "first_eviction_lambda": st["fel"]}
        import json

        with open(path, "wb") as f:
            np.savez(f, header=np.frombuffer(json.dumps(header).encode(), dtype=np.uint8), keys=st["keys"],
                     digests=st["digests"], scores=st["scores"], values=st["values"])

    @classmethod
    def load_checkpoint(cls, path, device: Optional[int] = None, overflow_in_hbm: bool = False) -> "CacheTable":
        """Create a table from save_checkpoint's file (same configuration,
        same bytes)."""
        import json

        with np.load(path) as z:
            h = json.loads(bytes(z["header"]).decode())
            if h.get("version") != cls.CHECKPOINT_VERSION:
                raise ValueError("unsupported checkpoint version")
            cfg = TableConfig(capacity=h["capacity"], value_dim=h["value_dim"], mode=h["mode"],
                              score_policy=h["score_policy"], fast_tier_budget=h["fast_tier_budget"],
                              digest_filter=h["digest_filter"], admit_ties_unified=h["admit_ties_unified"],
                              device=device, overflow_in_hbm=overflow_in_hbm)
            t = cls(cfg)
            t.import_state(z["keys"], z["digests"], z["scores"], z["values"], clock=h["clock"],
                           first_eviction_lambda=h["first_eviction_lambda"])
        if h["epoch"]:
            t.set_epoch(h["epoch"])
        if t.size() != h["size"]:
            raise ValueError("checkpoint size does not match its keys")
        return t

    # ----- raw state (test / checkpoint support) -----------------------------
    def export_state(self) -> dict:
        """Host copy of the raw arrays in the reference layout (table.py:143-146)."""
        cap, dim, bc = self.config.capacity, self.config.value_dim, self.config.bucket_count
        keys = np.empty((bc, BUCKET_SLOTS), dtype=np.uint64)
        dig = np.empty((bc, BUCKET_SLOTS), dtype=np.uint8)
        sc = np.empty((bc, BUCKET_SLOTS), dtype=np.uint64)
        vals = np.empty((cap, dim), dtype=np.float32)
        occ = np.empty(bc, dtype=np.int64)
        _lib.check(self._lib.hkv_export_state(self._h, keys.ctypes.data_as(C.c_void_p), dig.ctypes.data_as(C.c_void_p),
                                              sc.ctypes.data_as(C.c_void_p), vals.ctypes.data_as(C.c_void_p),
                                              occ.ctypes.data_as(C.c_void_p)))
        return {"keys": keys, "digests": dig, "scores": sc, "values": vals, "occupancy": occ,
                "size": self._size, "clock": self._clock, "fel": self.first_eviction_lambda}

    def import_state(self, keys, digests, scores, values, clock: int = 0, first_eviction_lambda=None) -> None:
        k = np.ascontiguousarray(keys, dtype=np.uint64)
        d = np.ascontiguousarray(digests, dtype=np.uint8)
        s = np.ascontiguousarray(scores, dtype=np.uint64)
        v = np.ascontiguousarray(values, dtype=np.float32)
        cap = self.config.capacity
        if k.size != cap or d.size != cap or s.size != cap or v.size != cap * self.config.value_dim:
            raise ValueError("state arrays do not match the table shape")
        fel = first_eviction_lambda
        _lib.check(self._lib.hkv_import_state(self._h, k.ctypes.data_as(C.c_void_p), d.ctypes.data_as(C.c_void_p),
                                              s.ctypes.data_as(C.c_void_p), v.ctypes.data_as(C.c_void_p),
                                              int(clock), int(fel is not None), 0.0 if fel is None else float(fel)))

    def snapshot(self) -> None:
        _lib.check(self._lib.hkv_snapshot(self._h, self._sp()))

    def restore(self) -> None:
        _lib.check(self._lib.hkv_restore(self._h, self._sp()))

    def check_consistency(self) -> bool:
        """Device full scan (table.py:1284-1299)."""
        ok = C.c_int32()
        with self.gate.scope(Role.Reader, self._stream()):
            _lib.check(self._lib.hkv_check_consistency(self._h, C.byref(ok), self._sp()))
        if not ok.value:
            raise ConsistencyError("occupancy / size / digest disagree with bucket contents")
        return True

    def occupied_keys(self) -> np.ndarray:
        """All user keys currently stored, slot order (table.py:1301-1305)."""
        flat = self._dev_keys_flat().cpu().numpy().view(np.uint64)
        return flat[flat < _LOCKED].copy()

    # lazily materialised private views used by reference callers (bench.py)
    def _dev_keys_flat(self) -> torch.Tensor:
        st = self.export_state_arrays(("keys",))
        return torch.from_numpy(st["keys"].reshape(-1).view(np.int64))

    def _dev_scores_flat(self) -> torch.Tensor:
        st = self.export_state_arrays(("scores",))
        return torch.from_numpy(st["scores"].reshape(-1).view(np.int64))

    def export_state_arrays(self, names) -> dict:
        bc = self.config.bucket_count
        out = {}
        keys = np.empty((bc, BUCKET_SLOTS), dtype=np.uint64) if "keys" in names else None
        dig = np.empty((bc, BUCKET_SLOTS), dtype=np.uint8) if "digests" in names else None
        sc = np.empty((bc, BUCKET_SLOTS), dtype=np.uint64) if "scores" in names else None
        occ = np.empty(bc, dtype=np.int64) if "occupancy" in names else None
        vp = lambda a: None if a is None else a.ctypes.data_as(C.c_void_p)  # noqa: E731
        _lib.check(self._lib.hkv_export_state(self._h, vp(keys), vp(dig), vp(sc), None, vp(occ)))
        for name, a in (("keys", keys), ("digests", dig), ("scores", sc), ("occupancy", occ)):
            if a is not None:
                out[name] = a
        return out

    @property
    def _keys(self) -> np.ndarray:
        return self.export_state_arrays(("keys",))["keys"]

    @property
    def _digests(self) -> np.ndarray:
        return self.export_state_arrays(("digests",))["digests"]

    @property
    def _scores(self) -> np.ndarray:
        return self.export_state_arrays(("scores",))["scores"]

    @property
    def _occupancy(self) -> np.ndarray:
        return self.export_state_arrays(("occupancy",))["occupancy"]
