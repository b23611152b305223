"""GPU side of the sharded table on the one GPU this run has:

* hkv_route (hash + stable grouping by owner rank) against a numpy router for
  world sizes 2 / 4 / 8;
* ShardedCacheTable over a 1-rank NCCL process group: real CUDA local table,
  real all_to_all_single, explicit global LRU ticks and clock_advance through
  the kernels — bit-exact against one global oracle table.

The multi-rank exchange logic itself is covered on CPU by
tests/test_sharded_gloo.py (world size 2, gloo).
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402

from oracle.oracle import OracleTable  # noqa: E402
from test_sharded_gloo import numpy_router  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 4, 8])
def test_route_kernel_matches_numpy(world):
    from paper_2603_17168_b200.sharded import cuda_router

    rng = np.random.default_rng(world)
    keys = rng.integers(1, 2**63, size=100_003, dtype=np.uint64)
    kd = torch.from_numpy(keys.view(np.int64)).cuda()
    gb = 1 << 16
    perm_d, counts_d = cuda_router(kd, gb, world)
    perm_h, counts_h = numpy_router(torch.from_numpy(keys.view(np.int64)), gb, world)
    assert np.array_equal(counts_d.cpu().numpy(), counts_h.numpy())
    assert np.array_equal(perm_d.cpu().numpy(), perm_h.numpy())


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("policy", ["kLru", "kLfu", "kCustomized"])
def test_sharded_one_rank_nccl_equals_oracle(policy):
    import paper_2603_17168_b200 as hkv
    from paper_2603_17168_b200.sharded import ShardedCacheTable

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        cap, dim = 128 * 64, 8
        st = ShardedCacheTable(hkv.TableConfig(capacity=cap, value_dim=dim, score_policy=policy))
        g = OracleTable(cap, dim, "single", policy)
        rng = np.random.default_rng(7)
        ops = ["insert_or_assign", "insert_and_evict", "find", "find_or_insert", "erase", "assign", "assign_scores",
               "contains", "insert_and_evict"] * 3
        for step, op in enumerate(ops):
            n = int(rng.integers(500, 3000))
            k = rng.integers(1, 3 * cap, size=n).astype(np.uint64)
            v = rng.standard_normal((n, dim)).astype(np.float32)
            s = rng.integers(0, 40, size=n).astype(np.uint64) if policy == "kCustomized" else None
            kt = torch.from_numpy(k.view(np.int64)).cuda()
            vt = torch.from_numpy(v.copy()).cuda()
            stt = None if s is None else torch.from_numpy(s.view(np.int64)).cuda()
            if op == "insert_or_assign":
                assert np.array_equal(st.insert_or_assign(kt, vt, stt).cpu().numpy(), g.insert_or_assign(k, v, s))
            elif op == "insert_and_evict":
                o, ek, ev, es = st.insert_and_evict(kt, vt, stt)
                go, gek, gev, ges = g.insert_and_evict(k, v, s)
                assert np.array_equal(o.cpu().numpy(), go)
                assert np.array_equal(ek.view(torch.int64).cpu().numpy().view(np.uint64), gek)
                assert ev.cpu().numpy().tobytes() == gev.tobytes()
                assert np.array_equal(es.view(torch.int64).cpu().numpy().view(np.uint64), ges)
            elif op == "find":
                f, vv = st.find(kt)
                gf, gvv = g.find(k)
                assert np.array_equal(f.cpu().numpy(), gf) and vv.cpu().numpy().tobytes() == gvv.tobytes()
            elif op == "contains":
                assert np.array_equal(st.contains(kt).cpu().numpy(), g.contains(k))
            elif op == "find_or_insert":
                o = st.find_or_insert(kt, vt, stt)
                gv = v.copy()
                go = g.find_or_insert(k, gv, s)
                assert np.array_equal(o.cpu().numpy(), go) and vt.cpu().numpy().tobytes() == gv.tobytes()
            elif op == "erase":
                assert np.array_equal(st.erase(kt).cpu().numpy(), g.erase(k))
            elif op == "assign":
                assert np.array_equal(st.assign(kt, vt).cpu().numpy(), g.assign(k, v))
            elif op == "assign_scores":
                a = st.assign_scores(kt, stt) if policy == "kCustomized" else st.assign_scores(kt)
                b = g.assign_scores(k, s) if policy == "kCustomized" else g.assign_scores(k)
                assert np.array_equal(a.cpu().numpy(), b), op
        assert st.size() == g.size()
        state = st.local.export_state()
        assert state["keys"].tobytes() == g.keys.tobytes()
        assert state["scores"].tobytes() == g.scores.tobytes()
        assert state["values"].tobytes() == g.values.tobytes()
        assert state["clock"] == g.clock and st.clock == g.clock
    finally:
        dist.destroy_process_group()


def _peer_ipc_worker(rank, world, port, cap_l, dim, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2603_17168_b200 as hkv
        from paper_2603_17168_b200.sharded import ShardedCacheTable
        from paper_2603_17168_b200.workloads import fmix64_array

        st = ShardedCacheTable(hkv.TableConfig(capacity=cap_l * world, value_dim=dim))
        o = OracleTable(cap_l * world, dim)
        rng = np.random.default_rng(3)  # same stream on every rank
        bl = cap_l // 128
        keys = rng.integers(1, 2**60, size=30_000, dtype=np.uint64)
        vals = rng.standard_normal((len(keys), dim)).astype(np.float32)
        o.insert_or_assign(keys, vals)
        owner = ((fmix64_array(keys) & np.uint64(bl * world - 1)) // np.uint64(bl)).astype(np.int64)
        sel = owner == rank
        st.local.insert_or_assign(keys[sel], vals[sel])
        st.enable_peer_find()  # IPC handles over the gloo group, opened across processes
        q = np.concatenate([keys[rank::2], rng.integers(2**61, 2**62, size=3000, dtype=np.uint64)])
        f, v = st.find(torch.from_numpy(q.view(np.int64)).cuda())
        fo, vo = o.find(q)
        ok = np.array_equal(f.cpu().numpy(), fo) and v.cpu().numpy().tobytes() == vo.tobytes()
        ret[rank] = 1 if ok else 0
        dist.barrier()  # keep every shard alive until all peers finished reading it
    finally:
        dist.destroy_process_group()


def test_peer_find_ipc_two_processes():
    """hkv_find_peer across PROCESSES: two ranks (gloo plumbing) each own a
    shard on this GPU, exchange CUDA IPC handles and find over the other
    process's memory — the multi-GPU NVLink path with both ends on one
    device.  Bit-exact against the global oracle table."""
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    ret = ctx.Array("i", [0, 0])
    procs = [ctx.Process(target=_peer_ipc_worker, args=(r, 2, port, 128 * 128, 8, ret)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert list(ret) == [1, 1]


@pytest.mark.parametrize("dim,custom", [(64, False), (7, True), (128, True)])
def test_route_gather_and_scatter_kernels(dim, custom):
    """hkv_route_gather / hkv_scatter_rows (the routed exchange's device
    passes) equal torch indexing."""
    import types

    from paper_2603_17168_b200.sharded import ShardedCacheTable

    torch.cuda.set_device(0)
    n = 100_003
    g = torch.Generator(device="cuda").manual_seed(1)
    keys = torch.randint(1, 2**62, (n,), device="cuda", generator=g)
    vals = torch.randn((n, dim), device="cuda", generator=g)
    sc = torch.randint(0, 2**40, (n,), device="cuda", generator=g) if custom else None
    perm = torch.randperm(n, device="cuda", generator=g).to(torch.int32)
    fake = types.SimpleNamespace(config=types.SimpleNamespace(value_dim=dim))
    fake._sp = lambda t: ShardedCacheTable._sp(fake, t)
    meta, rows = ShardedCacheTable._gather_send(fake, perm, keys, vals, sc, 1000)
    p = perm.long()
    assert torch.equal(meta[:, 0], keys[p]) and torch.equal(meta[:, 1], p + 1001)
    if custom:
        assert torch.equal(meta[:, 2], sc[p])
    assert torch.equal(rows, vals[p])
    fake._unpermute = ShardedCacheTable._unpermute
    back = ShardedCacheTable._scatter_back(fake, rows, perm)
    assert torch.equal(back, vals)
    flags = (torch.arange(n, device="cuda") % 3 == 0).to(torch.uint8)
    fb = ShardedCacheTable._scatter_back(fake, flags[p], perm)
    assert torch.equal(fb, flags)
