"""Multi-process (gloo, world_size 2, CPU) test of the sharded table's host
logic: routing, all-to-all exchanges, global tick order, evicted-tuple
reordering, global export.  Each shard's local table is the C oracle (test
infrastructure) behind a torch adapter; the whole sharded table must be
bit-identical to ONE global oracle table fed the rank-major concatenated
batches."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.oracle import OracleTable, fmix64_array

WORLD = 2
CAP = 128 * 64
DIM = 4


class OracleShard:
    """torch-tensor adapter with the CacheTable signature over an OracleTable."""

    def __init__(self, cfg):
        self.config = cfg
        self.t = OracleTable(cfg.capacity, cfg.value_dim, cfg.mode.value, cfg.score_policy.value,
                             cfg.fast_tier_budget)
        self.device = torch.device("cpu")

    @staticmethod
    def _k(k):
        return k.view(torch.int64).numpy().view(np.uint64)

    @staticmethod
    def _s(s):
        return None if s is None else s.view(torch.int64).numpy().view(np.uint64)

    def find(self, k):
        f, v = self.t.find(self._k(k))
        return torch.from_numpy(f), torch.from_numpy(v)

    def contains(self, k):
        return torch.from_numpy(self.t.contains(self._k(k)))

    def insert_or_assign(self, k, v, s=None, ticks=None, clock_advance=0):
        return torch.from_numpy(self.t.insert_or_assign(self._k(k), v.numpy(), self._s(s), self._s(ticks),
                                                        clock_advance))

    def insert_and_evict(self, k, v, s=None, ticks=None, clock_advance=0):
        o, ek, ev, es = self.t.insert_and_evict(self._k(k), v.numpy(), self._s(s), self._s(ticks), clock_advance)
        return (torch.from_numpy(o), torch.from_numpy(ek.view(np.int64)).view(torch.uint64), torch.from_numpy(ev),
                torch.from_numpy(es.view(np.int64)).view(torch.uint64))

    def find_or_insert(self, k, v, s=None, ticks=None, clock_advance=0):
        a = v.numpy()
        o = self.t.find_or_insert(self._k(k), a, self._s(s), self._s(ticks), clock_advance)
        return torch.from_numpy(o)

    def erase(self, k):
        return torch.from_numpy(self.t.erase(self._k(k)))

    def assign(self, k, v):
        return torch.from_numpy(self.t.assign(self._k(k), v.numpy()))

    def assign_scores(self, k, s=None, ticks=None, clock_advance=0):
        return torch.from_numpy(self.t.assign_scores(self._k(k), self._s(s), self._s(ticks), clock_advance))

    def size(self):
        return self.t.size()

    def export_batch_if(self, min_score, cursor, max_count):
        return self.t.export_batch_if(min_score, cursor, max_count)


def numpy_router(keys, global_buckets, world):
    k = keys.view(torch.int64).numpy().view(np.uint64)
    gb = fmix64_array(k) & np.uint64(global_buckets - 1)
    shift = int(np.log2(global_buckets // world))
    dest = (gb >> np.uint64(shift)).astype(np.int64)
    perm = np.argsort(dest, kind="stable")
    counts = np.bincount(dest, minlength=world).astype(np.int64)
    return torch.from_numpy(perm), torch.from_numpy(counts)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _batches(step, policy):
    """Deterministic per-rank batches; every rank can rebuild all of them."""
    out = []
    for r in range(WORLD):
        rng = np.random.default_rng(1000 * step + r)
        n = int(rng.integers(200, 900))
        keys = rng.integers(1, 3 * CAP, size=n).astype(np.uint64)
        vals = rng.standard_normal((n, DIM)).astype(np.float32)
        sc = rng.integers(0, 40, size=n).astype(np.uint64) if policy == "kCustomized" else None
        out.append((keys, vals, sc))
    return out


def _worker(rank, port, policy, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        import paper_2603_17168_b200 as hkv
        from paper_2603_17168_b200.sharded import ShardedCacheTable

        cfg = hkv.TableConfig(capacity=CAP, value_dim=DIM, score_policy=policy)
        st = ShardedCacheTable(cfg, local_factory=OracleShard, router=numpy_router)
        g = OracleTable(CAP, DIM, "single", policy)
        ops = ["insert_or_assign", "insert_and_evict", "find", "find_or_insert", "erase", "assign", "assign_scores",
               "contains", "insert_and_evict", "export"] * 3
        for step, op in enumerate(ops):
            bs = _batches(step, policy)
            gk = np.concatenate([b[0] for b in bs])
            gv = np.concatenate([b[1] for b in bs])
            gs = None if policy != "kCustomized" else np.concatenate([b[2] for b in bs])
            off = sum(len(b[0]) for b in bs[:rank])
            k, v, s = bs[rank]
            n = len(k)
            kt = torch.from_numpy(k.view(np.int64))
            vt = torch.from_numpy(v.copy())
            stt = None if s is None else torch.from_numpy(s.view(np.int64))
            sl = slice(off, off + n)
            if op == "insert_or_assign":
                a = st.insert_or_assign(kt, vt, stt).numpy()
                b = g.insert_or_assign(gk, gv, gs)[sl]
                assert np.array_equal(a, b), op
            elif op == "insert_and_evict":
                o, ek, ev, es = st.insert_and_evict(kt, vt, stt)
                go, gek, gev, ges = g.insert_and_evict(gk, gv, gs)
                assert np.array_equal(o.numpy(), go[sl]), op
                evicted_idx = np.flatnonzero(go == 3)
                mine = (evicted_idx >= off) & (evicted_idx < off + n)
                assert np.array_equal(ek.view(torch.int64).numpy().view(np.uint64), gek[mine])
                assert ev.numpy().tobytes() == gev[mine].tobytes()
                assert np.array_equal(es.view(torch.int64).numpy().view(np.uint64), ges[mine])
            elif op == "find":
                f, vv = st.find(kt)
                gf, gvv = g.find(gk)
                assert np.array_equal(f.numpy(), gf[sl]) and vv.numpy().tobytes() == gvv[sl].tobytes()
            elif op == "contains":
                assert np.array_equal(st.contains(kt).numpy(), g.contains(gk)[sl])
            elif op == "find_or_insert":
                o = st.find_or_insert(kt, vt, stt)
                gvv = gv.copy()
                go = g.find_or_insert(gk, gvv, gs)
                assert np.array_equal(o.numpy(), go[sl]) and vt.numpy().tobytes() == gvv[sl].tobytes()
            elif op == "erase":
                assert np.array_equal(st.erase(kt).numpy(), g.erase(gk)[sl])
            elif op == "assign":
                assert np.array_equal(st.assign(kt, vt).numpy(), g.assign(gk, gv)[sl])
            elif op == "assign_scores":
                if policy == "kCustomized":
                    a = st.assign_scores(kt, stt).numpy()
                    b = g.assign_scores(gk, gs)[sl]
                else:
                    a = st.assign_scores(kt).numpy()
                    b = g.assign_scores(gk)[sl]
                assert np.array_equal(a, b), op
            elif op == "export":
                for cursor, mc, ms in ((0, 10**9, None), (CAP // 2 - 5, 300, 3), (17, 4000, None)):
                    a = st.export_batch_if(ms, cursor, mc)
                    b = g.export_batch_if(ms, cursor, mc)
                    assert a[3] == b[3], (cursor, mc, a[3], b[3])
                    assert all(x.tobytes() == y.tobytes() for x, y in zip(a[:3], b[:3]))
        # final state: this shard == the global table's bucket range
        bl = (CAP // 128) // WORLD
        lo, hi = rank * bl, (rank + 1) * bl
        loc = st.local.t
        assert loc.keys.tobytes() == g.keys[lo:hi].tobytes()
        assert loc.scores.tobytes() == g.scores[lo:hi].tobytes()
        assert loc.digests.tobytes() == g.digests[lo:hi].tobytes()
        assert loc.values.tobytes() == g.values[lo * 128:hi * 128].tobytes()
        assert st.size() == g.size()
        assert loc.clock == g.clock and st.clock == g.clock
        results[rank] = "ok"
    except Exception as e:  # surface the failure to the parent
        import traceback

        results[rank] = traceback.format_exc()
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("policy", ["kLru", "kLfu", "kCustomized"])
def test_sharded_table_equals_global_table(policy):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, policy, results)) for r in range(WORLD)]
    [p.start() for p in procs]
    [p.join(240) for p in procs]
    for p in procs:
        if p.is_alive():
            p.kill()
    for r in range(WORLD):
        assert results.get(r) == "ok", results.get(r)


def _dual_worker(rank, port, policy, results):
    """Dual-mode sharding: every shard equals an oracle DUAL table of
    capacity / world fed the rank-major global batch restricted to the keys
    whose first bucket it owns, with the global ticks."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        import paper_2603_17168_b200 as hkv
        from paper_2603_17168_b200.sharded import ShardedCacheTable

        cfg = hkv.TableConfig(capacity=CAP, value_dim=DIM, score_policy=policy, mode="dual")
        st = ShardedCacheTable(cfg, local_factory=OracleShard, router=numpy_router)
        ref = OracleTable(CAP // WORLD, DIM, "dual", policy)  # this shard's reference
        bl = (CAP // 128) // WORLD
        clock = 0
        for step in range(10):
            bs = _batches(step, policy)
            gk = np.concatenate([b[0] for b in bs])
            gv = np.concatenate([b[1] for b in bs])
            gs = None if policy != "kCustomized" else np.concatenate([b[2] for b in bs])
            owner = ((fmix64_array(gk) & np.uint64(bl * WORLD - 1)) // np.uint64(bl)).astype(np.int64)
            mine = np.flatnonzero(owner == rank)
            ticks = (clock + 1 + mine).astype(np.uint64)
            k, v, s = bs[rank]
            kt = torch.from_numpy(k.view(np.int64))
            vt = torch.from_numpy(v.copy())
            stt = None if s is None else torch.from_numpy(s.view(np.int64))
            st.insert_or_assign(kt, vt, stt)
            ref.insert_or_assign(gk[mine], gv[mine], None if gs is None else gs[mine], ticks=ticks,
                                 clock_advance=len(gk))
            clock += len(gk)
            f, vv = st.find(kt)
            off = sum(len(b[0]) for b in bs[:rank])
            assert f.numpy().sum() > 0 or step == 0
        loc = st.local.t
        assert loc.keys.tobytes() == ref.keys.tobytes()
        assert loc.scores.tobytes() == ref.scores.tobytes()
        assert loc.values.tobytes() == ref.values.tobytes()
        assert loc.clock == ref.clock == st.clock
        results[rank] = "ok"
    except Exception:
        import traceback

        results[rank] = traceback.format_exc()
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("policy", ["kLru", "kCustomized"])
def test_sharded_dual_mode_equals_per_shard_dual_tables(policy):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_dual_worker, args=(r, port, policy, results)) for r in range(WORLD)]
    [p.start() for p in procs]
    [p.join(240) for p in procs]
    for p in procs:
        if p.is_alive():
            p.kill()
    for r in range(WORLD):
        assert results.get(r) == "ok", results.get(r)
