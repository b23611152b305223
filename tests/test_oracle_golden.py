"""Pin the C oracle (oracle/hkv_oracle.c) to fixtures recorded from the
reference (tests/golden/make_golden.py).  CPU only."""

import os

import numpy as np
import pytest

from golden_replay import CASE_FILES, GOLDEN_DIR, load_case, replay
from oracle.oracle import OracleTable, fmix64, fmix64_array


def test_fixtures_present():
    assert len(CASE_FILES) >= 10


@pytest.mark.parametrize("path", CASE_FILES, ids=[os.path.basename(p)[:-4] for p in CASE_FILES])
def test_oracle_replays_reference_fixture(path):
    meta, ops, state, ctr = load_case(path)
    t = OracleTable(meta["capacity"], meta["dim"], meta["mode"], meta["policy"], meta["budget"],
                    admit_ties_unified=meta["unified"])
    assert replay(t, ops) is None
    assert t.keys.tobytes() == state["keys"].tobytes()
    assert t.digests.tobytes() == state["digests"].tobytes()
    assert t.scores.tobytes() == state["scores"].tobytes()
    assert t.occupancy.tobytes() == state["occupancy"].tobytes()
    assert t.values.tobytes() == state["values"].tobytes()
    assert t.size() == int(state["size"])
    assert t.clock == int(state["clock"])
    fel = t.first_eviction_lambda
    assert (-1.0 if fel is None else fel) == float(state["fel"])
    assert t.counters == ctr
    assert t.check_consistency()


def test_hash_kat():
    z = np.load(os.path.join(GOLDEN_DIR, "hash_kat.npz"))
    assert np.array_equal(fmix64_array(z["keys"]), z["h1"])
    h2 = fmix64_array(z["h1"] ^ np.uint64(0x9E3779B97F4A7C15))
    assert np.array_equal(h2, z["h2"])
    # pkg/tests/test_hashing.py:53-57
    h = 0xAABBCCDD_11223344
    assert (h >> 32) & 0xFF == 0xDD and h & (2**32 - 1) == 0x11223344
    assert fmix64(0) == 0
