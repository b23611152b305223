"""Service front-end (paper_2603_17168_b200/service.py) on CPU: the routes of
the reference service exist with its status codes (service.py:156-290); a
table cannot be created without a CUDA device (503, no CPU fallback)."""

import pytest

pytest.importorskip("fastapi")
from fastapi.testclient import TestClient  # noqa: E402

from paper_2603_17168_b200.service import create_app  # noqa: E402

REF_ROUTES = {
    ("POST", "/tables"), ("GET", "/tables"), ("GET", "/tables/{name}"), ("DELETE", "/tables/{name}"),
    ("POST", "/tables/{name}/insert"), ("POST", "/tables/{name}/find-or-insert"), ("POST", "/tables/{name}/find"),
    ("POST", "/tables/{name}/find-ptr"), ("POST", "/tables/{name}/contains"), ("POST", "/tables/{name}/assign"),
    ("POST", "/tables/{name}/erase"), ("POST", "/tables/{name}/export"), ("GET", "/tables/{name}/counters"),
    ("POST", "/tables/{name}/counters/reset"),
}


def test_reference_routes_present():
    app = create_app()
    have = {(m, r.path) for r in app.routes for m in getattr(r, "methods", ())}
    assert REF_ROUTES <= have
    assert ("POST", "/tables/{name}/find.bin") in have and ("POST", "/tables/{name}/insert.bin") in have


def test_unknown_table_and_validation_without_gpu():
    import torch

    c = TestClient(create_app())
    assert c.get("/tables").json() == []
    assert c.get("/tables/nope").status_code == 404
    assert c.post("/tables/nope/find", json={"keys": [1]}).status_code == 404
    # invalid config -> 422 before any device work (table.py:108-127)
    r = c.post("/tables", json={"name": "t", "capacity": 100, "value_dim": 4})
    assert r.status_code == 422 and "multiple of 128" in r.json()["detail"]
    r = c.post("/tables", json={"name": "t", "capacity": 1024, "value_dim": 4})
    assert r.status_code == (201 if torch.cuda.is_available() else 503)
