"""Replay a golden fixture (tests/golden/*.npz, recorded from the reference by
tests/golden/make_golden.py) against any table with the CacheTable batch API
and report the first divergence."""

from __future__ import annotations

import glob
import os

import numpy as np

from refdiff import outputs_equal, run_impl

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASE_FILES = sorted(p for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz")) if not p.endswith("hash_kat.npz"))


def load_case(path):
    z = np.load(path, allow_pickle=False)
    meta = {
        "capacity": int(z["meta_capacity"]), "dim": int(z["meta_dim"]), "mode": str(z["meta_mode"]),
        "policy": str(z["meta_policy"]), "budget": None if int(z["meta_budget"]) < 0 else int(z["meta_budget"]),
        "unified": bool(int(z["meta_unified"])) if "meta_unified" in z else False,
    }
    ops = []
    for j in range(int(z["meta_nops"])):
        name = str(z[f"op{j}_name"])
        args = {}
        for key in ("keys", "values", "scores", "epoch", "cursor", "max_count", "min_score"):
            f = f"op{j}_in_{key}"
            if f in z:
                v = z[f]
                args[key] = v if v.ndim else v.item()
            else:
                args[key] = None
        outs = []
        m = 0
        while f"op{j}_out{m}" in z:
            outs.append(z[f"op{j}_out{m}"])
            m += 1
        ops.append((name, args, tuple(outs)))
    state = {k[len("state_"):]: z[k] for k in z.files if k.startswith("state_")}
    ctr = {k[len("ctr_"):]: int(z[k]) for k in z.files if k.startswith("ctr_")}
    return meta, ops, state, ctr


def replay(table, ops):
    """Returns None when every op matches, else a description of the first mismatch."""
    for j, (name, args, expect) in enumerate(ops):
        got = run_impl(table, name, args)
        if not outputs_equal(expect, got):
            return f"op {j} ({name}) output differs"
    return None
