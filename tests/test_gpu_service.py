"""The service front-end over a B200 table: the reference service's JSON
routes and the binary tensor routes give the oracle's results.

Run on a B200: python -m pytest tests -m gpu"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytest.importorskip("fastapi")
from fastapi.testclient import TestClient  # noqa: E402

from oracle.oracle import OracleTable  # noqa: E402

pytestmark = pytest.mark.gpu
NAMES = {0: "Inserted", 1: "Updated", 2: "Rejected", 3: "Evicted", 4: "Found", 5: "NotFound", 6: "Erased"}


@pytest.fixture
def client():
    if not torch.cuda.is_available():
        pytest.fail("gpu test ran without a CUDA device")
    from paper_2603_17168_b200.service import create_app

    return TestClient(create_app())


@pytest.mark.parametrize("policy", ["kLru", "kCustomized"])
def test_json_routes_match_oracle(client, policy):
    cap, dim = 128 * 16, 3
    r = client.post("/tables", json={"name": "t", "capacity": cap, "value_dim": dim, "score_policy": policy})
    assert r.status_code == 201, r.text
    assert client.post("/tables", json={"name": "t", "capacity": cap, "value_dim": dim}).status_code == 409
    o = OracleTable(cap, dim, "single", policy)
    rng = np.random.default_rng(4)
    custom = policy == "kCustomized"
    for step in range(8):
        k = rng.integers(1, 4 * cap, size=700, dtype=np.uint64)
        v = rng.standard_normal((700, dim)).astype(np.float32)
        s = rng.integers(0, 50, size=700, dtype=np.uint64) if custom else None
        body = {"keys": k.tolist(), "values": v.tolist(), "scores": None if s is None else s.tolist(),
                "return_evicted": step % 2 == 1}
        got = client.post("/tables/t/insert", json=body).json()
        if step % 2:
            oo, ek, ev, es = o.insert_and_evict(k, v, s)
            assert got["evicted_keys"] == ek.tolist() and got["evicted_scores"] == es.tolist()
            assert np.array_equal(np.asarray(got["evicted_values"], np.float32).reshape(-1, dim), ev)
        else:
            oo = o.insert_or_assign(k, v, s)
        assert got["outcomes"] == [NAMES[x] for x in oo.tolist()]
        q = rng.integers(1, 4 * cap, size=500, dtype=np.uint64)
        f = client.post("/tables/t/find", json={"keys": q.tolist()}).json()
        fo, vo = o.find(q)
        assert f["found"] == fo.tolist()
        assert all((row is None) == (not hit) for row, hit in zip(f["values"], fo))
        assert all(np.array_equal(np.asarray(row, np.float32), vo[i]) for i, row in enumerate(f["values"]) if row)
        assert client.post("/tables/t/contains", json={"keys": q.tolist()}).json()["present"] == o.contains(q).tolist()
        fp = client.post("/tables/t/find-ptr", json={"keys": q.tolist()}).json()
        ofp = o.find_ptr(q)
        assert fp["found"] == ofp[0].tolist() and fp["offset"] == ofp[2].tolist()
        a = client.post("/tables/t/assign", json={"keys": q.tolist(), "values": None,
                                                  "scores": (q % 40).tolist() if custom else None}).json()
        oa = o.assign_scores(q, (q % 40).astype(np.uint64)) if custom else o.assign_scores(q)
        assert a["outcomes"] == [NAMES[x] for x in oa.tolist()]
        e = client.post("/tables/t/erase", json={"keys": q[:50].tolist()}).json()
        assert e["outcomes"] == [NAMES[x] for x in o.erase(q[:50]).tolist()]
    info = client.get("/tables/t").json()
    assert info["size"] == o.size() and info["first_eviction_lambda"] == o.first_eviction_lambda
    ex = client.post("/tables/t/export", json={"cursor": 0, "max_count": 500, "min_score": 5}).json()
    ok, ov, osc, onx = o.export_batch_if(5, 0, 500)
    assert ex["keys"] == ok.tolist() and ex["scores"] == osc.tolist() and ex["next_cursor"] == onx
    c0 = client.get("/tables/t/counters").json()
    assert c0 == o.counters
    assert client.post("/tables/t/counters/reset").json() == c0
    assert client.get("/tables/t/counters").json()["digest_line_loads"] == 0
    assert client.delete("/tables/t").status_code == 204
    assert client.get("/tables/t").status_code == 404


def test_binary_routes_match_oracle(client):
    cap, dim = 128 * 64, 16
    assert client.post("/tables", json={"name": "b", "capacity": cap, "value_dim": dim}).status_code == 201
    o = OracleTable(cap, dim)
    rng = np.random.default_rng(5)
    for step in range(4):
        k = rng.integers(1, 3 * cap, size=20_000, dtype=np.uint64)
        v = rng.standard_normal((len(k), dim)).astype(np.float32)
        ev_flag = step % 2 == 1
        r = client.post(f"/tables/b/insert.bin?n={len(k)}&return_evicted={str(ev_flag).lower()}",
                        content=k.tobytes() + v.tobytes(), headers={"content-type": "application/octet-stream"})
        assert r.status_code == 200, r.text
        buf = r.content
        if ev_flag:
            oo, ek, evv, es = o.insert_and_evict(k, v)
            n = len(k)
            assert np.frombuffer(buf[:n], np.uint8).tolist() == oo.tolist()
            e = int(np.frombuffer(buf[n:n + 8], np.int64)[0])
            assert e == len(ek)
            off = n + 8
            assert np.array_equal(np.frombuffer(buf[off:off + 8 * e], np.uint64), ek)
            off += 8 * e
            assert np.array_equal(np.frombuffer(buf[off:off + 4 * e * dim], np.float32).reshape(e, dim), evv)
            off += 4 * e * dim
            assert np.array_equal(np.frombuffer(buf[off:], np.uint64), es)
        else:
            assert np.array_equal(np.frombuffer(buf, np.uint8), o.insert_or_assign(k, v))
        q = rng.integers(1, 3 * cap, size=30_000, dtype=np.uint64)
        r = client.post(f"/tables/b/find.bin?n={len(q)}", content=q.tobytes(),
                        headers={"content-type": "application/octet-stream"})
        fo, vo = o.find(q)
        assert np.array_equal(np.frombuffer(r.content[: len(q)], np.uint8).astype(bool), fo)
        vals = np.frombuffer(r.content[len(q):], np.float32).reshape(len(q), dim)
        assert np.array_equal(vals[fo], vo[fo])
    bad = client.post("/tables/b/find.bin?n=10", content=b"\x00" * 7)
    assert bad.status_code == 422
