"""Hash-sharded CacheTable across the GPUs of one box.

The reference leaves sharding to the application;
this is the B200 build's multi-GPU layer.  One process per GPU.

Layout: contiguous bucket ranges.  A key's global bucket is
gb = fmix64(key) & (B_global - 1); rank = gb >> log2(B_local); the local bucket
is gb & (B_local - 1) = fmix64(key) & (B_local - 1), which is exactly what the
rank's local CacheTable computes.  The sharded table is therefore
bucket-for-bucket identical to one global table of the same capacity, and
the CPU oracle at the global capacity checks it bit-exactly.

Global batch order is rank-major (rank 0's batch, then rank 1's, ...).  Each
op travels to its owner in one all-to-all (keys + values + scores + explicit
LRU ticks = clock + global index + 1, packed into one int32 row per op); a
shard receives the segments in source rank order, each in source batch order,
so applying them in received order is the global serial order restricted to
the shard.  Results return in a second all-to-all and are scattered back
through the inverse routing permutation.  The split sizes and every rank's
batch size travel in one all_gather: one host synchronisation per op.
Every rank advances its clock by the global batch size, so all shards share
one logical clock.  size() is an all-reduce.

Dual mode: keys route by the owner of their FIRST
bucket, and each shard is a dual-mode table of capacity / G whose second
bucket is drawn inside the shard (second_hash(h) & (B_local - 1)).  The
sharded dual table is therefore exactly G independent reference dual tables,
each fed its routed sub-batch in global order (checked shard by shard
against the oracle); it differs from ONE global dual table only in where a
key's second candidate may live -- a global second bucket on another GPU
would need a cross-GPU two-bucket critical section per op.  Dual shards use
the routed find (the peer find probes single-mode shards).
"""

from __future__ import annotations

import ctypes as C
import dataclasses
from typing import Callable, Optional

import numpy as np
import torch
import torch.distributed as dist

from .table import CacheTable, Mode, Outcome, TableConfig

_EVICTED = int(Outcome.Evicted)
_UPDATED = int(Outcome.Updated)


def cuda_router(keys: torch.Tensor, global_buckets: int, world: int):
    """Stable grouping of keys by owner rank on the GPU (hkv_route kernel)."""
    from . import _lib

    lib = _lib.load()
    n = keys.numel()
    perm = torch.empty(n, dtype=torch.int32, device=keys.device)
    counts = torch.empty(world, dtype=torch.int64, device=keys.device)
    _lib.check(lib.hkv_route(C.c_void_p(keys.data_ptr()), n, global_buckets, world, C.c_void_p(perm.data_ptr()),
                             C.c_void_p(counts.data_ptr()),
                             C.c_void_p(torch.cuda.current_stream(keys.device).cuda_stream)))
    return perm, counts


class ShardedCacheTable:
    def __init__(self, config: TableConfig, group=None, local_factory: Optional[Callable] = None,
                 router: Optional[Callable] = None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.config = config
        bg = config.bucket_count
        if self.world & (self.world - 1) or bg % self.world:
            raise ValueError("world size must be a power of two dividing the bucket count")
        self.global_buckets = bg
        bl = bg // self.world
        lo = self.rank * bl
        budget = min(max(config.fast_tier_budget - lo, 0), bl)
        local_cfg = dataclasses.replace(config, capacity=config.capacity // self.world, fast_tier_budget=budget)
        self.local = (local_factory or CacheTable)(local_cfg)
        self.router = router or cuda_router
        self.clock = 0  # the global logical clock; every rank holds the same value
        self._fence_t = None

    # ----- exchange plumbing ----------------------------------------------------
    # One host synchronisation per op: the routing counts of every rank and
    # every rank's batch size travel in ONE all_gather (the all-to-all split
    # sizes must be host integers); the op's columns (key, tick, score, value
    # row ...) travel packed as int32 words in ONE all_to_all each way.
    def _plan(self, keys: torch.Tensor):
        """-> perm (routed order), send splits, recv splits, batch sizes of every rank."""
        perm, counts = self.router(keys, self.global_buckets, self.world)
        meta = torch.cat([counts.to(torch.int64),
                          torch.tensor([keys.numel()], dtype=torch.int64, device=counts.device)])
        allm = torch.empty(self.world * (self.world + 1), dtype=torch.int64, device=meta.device)
        dist.all_gather_into_tensor(allm, meta, group=self.group)
        m = allm.view(self.world, self.world + 1).tolist()  # the op's one host sync
        send = m[self.rank][: self.world]
        recv = [m[q][self.rank] for q in range(self.world)]
        sizes = [m[q][self.world] for q in range(self.world)]
        return perm, send, recv, sizes

    @staticmethod
    def _words(x: torch.Tensor) -> torch.Tensor:
        """(n, k) int32 view of a 1-D 64-bit / 8-bit-bool / 2-D 32-bit column."""
        n = x.shape[0]
        if x.numel() == 0:
            per = x.element_size() // 4 if x.element_size() >= 4 else 1
            k = per * (x.shape[1] if x.dim() == 2 else 1)
            return torch.empty((n, k), dtype=torch.int32, device=x.device)
        if x.dtype in (torch.int64, torch.uint64, torch.float64):
            return x.contiguous().view(torch.int32).view(n, -1)
        if x.dtype in (torch.bool, torch.uint8):
            return x.to(torch.int32).view(n, 1)
        return x.contiguous().view(torch.int32).view(n, -1)

    def _a2a_packed(self, cols, send, recv):
        """Pack columns into (n, W) int32 rows, exchange them in one
        all_to_all, return the received (m, W) block."""
        x = torch.cat([self._words(c) for c in cols], dim=1) if len(cols) > 1 else self._words(cols[0])
        w = x.shape[1]
        out = torch.empty((sum(recv), w), dtype=torch.int32, device=x.device)
        dist.all_to_all_single(out, x.contiguous(), recv, send, group=self.group)
        return out

    @staticmethod
    def _col64(block, a):
        return block[:, a:a + 2].contiguous().view(torch.int64).view(-1)

    def _sp(self, t: torch.Tensor):
        return C.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)

    def _gather_send(self, perm, keys, values, scores, tick_base):
        """Routed-order send columns in one pass: meta rows (key, tick
        [, score]) as int64 and the value rows (hkv_route_gather on the
        device; torch indexing for the CPU tensors of the host-logic tests)."""
        n = keys.numel()
        w = 3 if scores is not None else 2
        d = self.config.value_dim
        if keys.is_cuda:
            from . import _lib

            p32 = perm if perm.dtype == torch.int32 else perm.to(torch.int32)
            meta = torch.empty((n, w), dtype=torch.int64, device=keys.device)
            vrows = torch.empty((n, d), dtype=torch.float32, device=keys.device) if values is not None else None
            rc = _lib.load().hkv_route_gather(
                C.c_void_p(p32.data_ptr()), n, C.c_void_p(keys.data_ptr()),
                None if scores is None else C.c_void_p(scores.contiguous().data_ptr()),
                None if values is None else C.c_void_p(values.contiguous().data_ptr()), d,
                int(tick_base) & 0xFFFFFFFFFFFFFFFF, C.c_void_p(meta.data_ptr()),
                None if vrows is None else C.c_void_p(vrows.data_ptr()), self._sp(keys))
            if rc:
                raise RuntimeError("hkv_route_gather failed")
            return meta, vrows
        cols = [keys[perm].view(torch.int64), perm.to(torch.int64) + (tick_base + 1)]
        if scores is not None:
            cols.append(scores[perm].view(torch.int64))
        return torch.stack(cols, dim=1), (values[perm] if values is not None else None)

    def _scatter_back(self, routed: torch.Tensor, perm: torch.Tensor):
        """out[perm[j]] = routed[j] (hkv_scatter_rows on the device)."""
        if not routed.is_cuda:
            return self._unpermute(routed, perm)
        from . import _lib

        out = torch.empty_like(routed)
        n = routed.shape[0]
        rb = routed.element_size() * (routed[0].numel() if n else 1)
        p32 = perm if perm.dtype == torch.int32 else perm.to(torch.int32)
        rc = _lib.load().hkv_scatter_rows(C.c_void_p(p32.data_ptr()), n, C.c_void_p(routed.contiguous().data_ptr()),
                                          C.c_void_p(out.data_ptr()), rb, self._sp(routed))
        if rc:
            raise RuntimeError("hkv_scatter_rows failed")
        return out

    def _splits(self, counts: torch.Tensor):
        recv = torch.empty_like(counts)
        dist.all_to_all_single(recv, counts, group=self.group)
        return counts.tolist(), recv.tolist()

    def _a2a(self, x: torch.Tensor, send_splits, recv_splits):
        out = torch.empty((sum(recv_splits),) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        dist.all_to_all_single(out, x.contiguous(), recv_splits, send_splits, group=self.group)
        return out

    def _unpermute(self, routed_back: torch.Tensor, perm: torch.Tensor):
        out = torch.empty_like(routed_back)
        out[perm] = routed_back
        return out

    @staticmethod
    def _u8(x: torch.Tensor):
        return x.to(torch.uint8) if x.dtype == torch.bool else x

    def _fence(self):
        """Stream-ordered barrier: a one-element all_reduce on the compute
        stream.  No rank's kernels after it start before every rank's kernels
        before it finished (no host synchronisation with NCCL)."""
        if self._fence_t is None or self._fence_t.device != self.local.device:
            self._fence_t = torch.zeros(1, dtype=torch.int32, device=getattr(self.local, "device", "cpu"))
        dist.all_reduce(self._fence_t, group=self.group)

    # ----- reader ops -----------------------------------------------------------
    def enable_peer_find(self):
        """Collective: exchange CUDA IPC handles of every shard's keys,
        digests and value arena, so find() reads the owner shard over NVLink
        instead of routing keys and rows through two all-to-alls
        (hkv_find_peer; every value row must be in HBM)."""
        from . import _lib

        lib = self.local._lib
        buf = (C.c_char * 192)()
        _lib.check(lib.hkv_ipc_handles(self.local._h, buf, 192))
        allh = [None] * self.world
        dist.all_gather_object(allh, bytes(buf), group=self.group)
        blob = b"".join(allh)
        _lib.check(lib.hkv_set_peers(self.local._h, self.world, self.rank,
                                     (C.c_char * len(blob)).from_buffer_copy(blob)))
        self._peer = True

    def find(self, keys: torch.Tensor):
        if getattr(self, "_peer", False):
            # every shard's previous mutations are complete before any rank
            # reads it, and no rank mutates its shard before every peer read
            # finished: two stream-ordered fences, no host barrier
            self._fence()
            f, v = self.local._find_peer(keys)
            self._fence()
            return f, v
        if self.world == 1:  # one shard: nothing to route
            return self.local.find(keys)
        perm, send, recv, _ = self._plan(keys)
        rk = self._a2a(keys[perm], send, recv)
        f, v = self.local.find(rk)
        vb = self._a2a(v, recv, send)
        fb = self._a2a(self._u8(f), recv, send)
        return self._scatter_back(fb, perm).bool(), self._scatter_back(vb, perm)

    def contains(self, keys: torch.Tensor):
        if self.world == 1:
            return self.local.contains(keys)
        perm, send, recv, _ = self._plan(keys)
        rk = self._a2a(keys[perm], send, recv)
        f = self.local.contains(rk)
        return self._unpermute(self._a2a(self._u8(f), recv, send), perm).bool()

    def size(self) -> int:
        s = torch.tensor([self.local.size()], dtype=torch.int64,
                         device=getattr(self.local, "device", torch.device("cpu")))
        dist.all_reduce(s, group=self.group)
        return int(s.item())

    def load_factor(self) -> float:
        return self.size() / self.config.capacity

    # ----- inserter ops ---------------------------------------------------------
    def _upsert(self, op: str, keys, values, scores):
        n = keys.numel()
        if self.world == 1:
            # one shard holds every bucket: the local op with the global ticks
            ticks = torch.arange(n, dtype=torch.int64, device=keys.device) + (self.clock + 1)
            fn = getattr(self.local, op)
            r = fn(keys, values, scores, ticks=ticks, clock_advance=n)
            self.clock += n
            return r
        perm, send, recv, sizes = self._plan(keys)
        off, total = sum(sizes[: self.rank]), sum(sizes)
        d = self.config.value_dim
        meta, vrows = self._gather_send(perm, keys.view(torch.int64), values,
                                        None if scores is None else scores.view(torch.int64), self.clock + off)
        # two exchanges: the packed (key, tick[, score]) rows and the value rows
        rmeta = self._a2a(meta, send, recv)
        rv = self._a2a(vrows, send, recv)
        rk = rmeta[:, 0].contiguous()
        rt = rmeta[:, 1].contiguous()
        rs = rmeta[:, 2].contiguous() if scores is not None else None
        res = None
        if op == "insert_or_assign":
            o = self.local.insert_or_assign(rk, rv, rs, ticks=rt, clock_advance=total)
            ob = self._a2a(o, recv, send)
        elif op == "find_or_insert":
            o = self.local.find_or_insert(rk, rv, rs, ticks=rt, clock_advance=total)
            ob = self._a2a(o, recv, send)
            values.copy_(self._scatter_back(self._a2a(rv, recv, send), perm))
        else:  # insert_and_evict
            o, ek, ev, es = self.local.insert_and_evict(rk, rv, rs, ticks=rt, clock_advance=total)
            ob = self._a2a(o, recv, send)
            # evicted tuples per source rank, in received (= source batch) order
            is_ev = (o == _EVICTED)
            seg = torch.repeat_interleave(torch.arange(self.world, device=o.device),
                                          torch.tensor(recv, device=o.device), output_size=o.numel())
            ev_send = torch.bincount(seg[is_ev], minlength=self.world).to(torch.int64)
            es_split, er_split = self._splits(ev_send)
            back = self._a2a_packed([ek.view(torch.int64), es.view(torch.int64), ev], es_split, er_split)
            res = (self._col64(back, 0), back[:, 4:].contiguous().view(torch.float32), self._col64(back, 2))
        self.clock += total
        outcomes = self._scatter_back(ob, perm)
        if res is None:
            return outcomes
        # entries arrive grouped by shard in routed order; restore batch order
        routed_ev = torch.nonzero(ob == _EVICTED).flatten()
        order = torch.argsort(perm[routed_ev])
        bk, bv, bs = res
        return outcomes, bk[order].view(torch.uint64), bv[order], bs[order].view(torch.uint64)

    def insert_or_assign(self, keys, values, scores=None):
        return self._upsert("insert_or_assign", keys, values, scores)

    def insert_and_evict(self, keys, values, scores=None):
        return self._upsert("insert_and_evict", keys, values, scores)

    def find_or_insert(self, keys, values_inout, scores=None):
        return self._upsert("find_or_insert", keys, values_inout, scores)

    def erase(self, keys):
        if self.world == 1:
            return self.local.erase(keys)
        perm, send, recv, _ = self._plan(keys)
        rk = self._a2a(keys[perm], send, recv)
        o = self.local.erase(rk)
        return self._unpermute(self._a2a(o, recv, send), perm)

    # ----- updater ops ----------------------------------------------------------
    def assign(self, keys, values):
        if self.world == 1:
            return self.local.assign(keys, values)
        perm, send, recv, _ = self._plan(keys)
        meta, vrows = self._gather_send(perm, keys.view(torch.int64), values, None, 0)
        rk = self._a2a(meta, send, recv)[:, 0].contiguous()
        o = self.local.assign(rk, self._a2a(vrows, send, recv))
        return self._scatter_back(self._a2a(o, recv, send), perm)

    def assign_scores(self, keys, scores=None):
        if self.world == 1:
            if scores is not None:
                return self.local.assign_scores(keys, scores)
            o = self.local.assign_scores(keys)
            self.clock += int((o == _UPDATED).sum().item())
            return o
        perm, send, recv, _ = self._plan(keys)
        if scores is not None:
            blk = self._a2a_packed([keys[perm].view(torch.int64), scores[perm].view(torch.int64)], send, recv)
            o = self.local.assign_scores(self._col64(blk, 0), self._col64(blk, 2))
            return self._unpermute(self._a2a(o, recv, send), perm)
        rk = self._a2a(keys[perm], send, recv)
        # refresh: ticks follow the GLOBAL found order (table.py:481-483)
        f = self._unpermute(self._a2a(self._u8(self.local.contains(rk)), recv, send), perm).bool()
        nf = int(f.sum().item())
        off, total = self._global_offsets(nf, keys.device)
        rank_in_batch = torch.cumsum(f.to(torch.int64), 0) - 1
        ticks = rank_in_batch + (self.clock + off + 1)
        rt = self._a2a(ticks[perm], send, recv)
        o = self.local.assign_scores(rk, None, ticks=rt, clock_advance=total)
        self.clock += total
        return self._unpermute(self._a2a(o, recv, send), perm)

    def _global_offsets(self, n: int, device):
        t = torch.tensor([n], dtype=torch.int64, device=device)
        allv = torch.empty(self.world, dtype=torch.int64, device=device)
        dist.all_gather_into_tensor(allv, t, group=self.group)
        sizes = allv.tolist()
        return sum(sizes[: self.rank]), sum(sizes)

    # ----- export (global rows are rank-major) ----------------------------------
    def export_batch_if(self, min_score, cursor, max_count: int):
        """Global export_batch_if over rank-major rows (table.py:374-434).
        Ranks answer in order, each with the room the previous ones left."""
        cap_l = self.config.capacity // self.world
        cursor = 0 if cursor is None else cursor
        if not (0 <= cursor < self.config.capacity):
            raise ValueError("cursor out of range")
        if max_count < 1:
            raise ValueError("max_count must be >= 1")
        ks, vs, ss = [], [], []
        taken = 0
        nxt = None
        for r in range(self.world):
            lo = r * cap_l
            if cursor >= lo + cap_l:
                continue
            payload = None
            if self.rank == r:
                k, v, s, n = self.local.export_batch_if(min_score, max(cursor - lo, 0), max_count - taken)
                payload = (np.asarray(k), np.asarray(v), np.asarray(s), None if n is None else n + lo)
            box = [payload]
            # src is a GLOBAL rank even when the table lives on a subgroup
            src = r if self.group is None else dist.get_global_rank(self.group, r)
            dist.broadcast_object_list(box, src=src, group=self.group)
            k, v, s, n = box[0]
            ks.append(k)
            vs.append(v)
            ss.append(s)
            taken += len(k)
            if taken >= max_count:
                if n is not None:
                    nxt = n
                elif r + 1 < self.world:
                    nxt = (r + 1) * cap_l  # the last taken row closed rank r's range
                break
        dim = self.config.value_dim
        keys = np.concatenate(ks) if ks else np.zeros(0, np.uint64)
        vals = np.concatenate(vs) if vs else np.zeros((0, dim), np.float32)
        scs = np.concatenate(ss) if ss else np.zeros(0, np.uint64)
        return keys, vals, scs, nxt
