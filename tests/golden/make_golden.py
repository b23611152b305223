"""Generate golden fixtures from the REFERENCE implementation itself.

Run in the build container (needs /root/reference; not on the GPU box):

    python tests/golden/make_golden.py

For each (mode, policy, tier budget) case it replays a seeded op script
(tests/refdiff.py:make_script) on `cachekv.CacheTable` (workers=1, imported
from /root/reference/pkg/src) and records every op's inputs and outputs plus
the final raw state (keys, digests, scores, occupancy, values, size, clock,
first_eviction_lambda, TxnCounters).  tests/test_oracle_golden.py pins the C
oracle to these files; tests/test_gpu_parity.py pins the B200 table to them.

Also writes hashing known-answer vectors (hashing.py:21-75) and the reference
test KAT h=0xAABBCCDD_11223344 (pkg/tests/test_hashing.py:53-57).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")

from refdiff import make_script, ref_state, run_reference  # noqa: E402

CASES = [
    # name, mode, policy, budget, capacity, dim, seed, n_batches, batch, universe_scale
    ("single_lru", "single", "kLru", None, 2048, 3, 11, 24, 400, 1.5),
    ("single_lfu", "single", "kLfu", None, 2048, 4, 12, 24, 400, 3.0),
    ("single_epochlru", "single", "kEpochLru", None, 2048, 2, 13, 24, 400, 3.0),
    ("single_epochlfu", "single", "kEpochLfu", 4, 2048, 3, 14, 24, 400, 2.0),
    ("single_custom", "single", "kCustomized", 8, 2048, 5, 15, 24, 400, 3.0),
    ("single_lru_crowded", "single", "kLru", None, 256, 8, 16, 20, 900, 4.0),
    ("dual_lru", "dual", "kLru", None, 2048, 3, 21, 24, 400, 4.0),
    ("dual_lfu", "dual", "kLfu", None, 2048, 2, 22, 24, 400, 4.0),
    ("dual_custom", "dual", "kCustomized", 4, 2048, 3, 23, 24, 400, 4.0),
    ("dual_epochlfu", "dual", "kEpochLfu", None, 1024, 4, 24, 24, 400, 4.0),
    ("dual_lru_unified", "dual", "kLru", None, 1024, 2, 25, 20, 400, 4.0),
]


def main():
    from cachekv import CacheTable, TableConfig
    from cachekv.hashing import fmix64, second_hash

    for name, mode, pol, budget, cap, dim, seed, nb, bs, us in CASES:
        unified = name.endswith("_unified")
        t = CacheTable(TableConfig(capacity=cap, value_dim=dim, mode=mode, score_policy=pol,
                                   fast_tier_budget=budget, admit_ties_unified=unified))
        ops = make_script(seed, cap, dim, pol, n_batches=nb, batch=bs, universe_scale=us)
        rec = {"meta_capacity": np.int64(cap), "meta_dim": np.int64(dim), "meta_mode": np.array(mode),
               "meta_policy": np.array(pol), "meta_budget": np.int64(-1 if budget is None else budget),
               "meta_nops": np.int64(len(ops)),
               "meta_unified": np.int64(unified)}
        for j, (op, a) in enumerate(ops):
            rec[f"op{j}_name"] = np.array(op)
            for k, v in a.items():
                if v is None:
                    continue
                rec[f"op{j}_in_{k}"] = np.asarray(v)
            outs = run_reference(t, op, a)
            for m, o in enumerate(outs):
                o = np.asarray(o)
                rec[f"op{j}_out{m}"] = o.astype(np.uint8) if o.dtype == bool else o
        st = ref_state(t)
        for k, v in st.items():
            rec[f"state_{k}"] = v
        for k, v in t.counters.as_dict().items():
            rec[f"ctr_{k}"] = np.int64(v)
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **rec)
        print(f"{name}: {len(ops)} ops, size={t._size}, fel={t.first_eviction_lambda} -> {path}")

    rng = np.random.default_rng(7)
    keys = np.concatenate([np.array([0, 1, 42, 2**63, 2**64 - 3, 0xAABBCCDD11223344], dtype=np.uint64),
                           rng.integers(0, 2**64 - 2, size=4090, dtype=np.uint64)])
    h1 = np.array([fmix64(int(k)) for k in keys], dtype=np.uint64)
    h2 = np.array([second_hash(int(h)) for h in h1], dtype=np.uint64)
    np.savez_compressed(os.path.join(HERE, "hash_kat.npz"), keys=keys, h1=h1, h2=h2)
    print("hash_kat: 4096 vectors")


if __name__ == "__main__":
    main()
