"""Deterministic key streams used by the parity tests and bench.py — a
restatement of the reference generator (workloads.py:45-127) so the GPU box,
which has no /root/reference, produces byte-identical inputs.  Pinned to the
reference by tests/test_host.py::test_workloads_match_reference."""

from __future__ import annotations

import numpy as np

LOCKED_KEY = 0xFFFFFFFFFFFFFFFE
_SEED_SALT = 0x517CC1B727220A95


def fmix64_array(x: np.ndarray) -> np.ndarray:
    k = np.asarray(x, dtype=np.uint64).copy()
    with np.errstate(over="ignore"):
        k ^= k >> np.uint64(33)
        k *= np.uint64(0xFF51AFD7ED558CCD)
        k ^= k >> np.uint64(33)
        k *= np.uint64(0xC4CEB9FE1A85EC53)
        k ^= k >> np.uint64(33)
    return k


def fmix64(x: int) -> int:
    return int(fmix64_array(np.array([x & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))[0])


def mix_to_keys(x: np.ndarray) -> np.ndarray:
    """hashing.py:82-94: bijective map of distinct inputs to distinct user keys."""
    keys = fmix64_array(x)
    bad = keys >= np.uint64(LOCKED_KEY)
    while bad.any():
        keys[bad] = fmix64_array(keys[bad])
        bad = keys >= np.uint64(LOCKED_KEY)
    return keys


def _seed_mix(seed: int) -> int:
    return fmix64((seed & 0xFFFFFFFFFFFFFFFF) ^ _SEED_SALT)


def uniform_distinct_keys(count: int, seed: int, stream_offset: int = 0) -> np.ndarray:
    """workloads.py:91-95."""
    base = (_seed_mix(seed) + stream_offset) & 0xFFFFFFFFFFFFFFFF
    with np.errstate(over="ignore"):
        x = np.arange(count, dtype=np.uint64) + np.uint64(base)
    return mix_to_keys(x)


class ZipfSampler:
    """Rejection-inversion sampler, P(r) ~ r^-alpha over 1..n (workloads.py:45-84)."""

    def __init__(self, n: int, alpha: float, rng: np.random.Generator):
        self.n = n
        self.alpha = alpha
        self.rng = rng
        self._h_x1 = self._h_integral(1.5) - 1.0
        self._h_n = self._h_integral(n + 0.5)
        self._s = 2.0 - self._h_integral_inv(self._h_integral(2.5) - self._h(2.0))

    def _h(self, x):
        return np.power(x, -self.alpha)

    def _h_integral(self, x):
        if self.alpha == 1.0:
            return np.log(x)
        return (np.power(x, 1.0 - self.alpha) - 1.0) / (1.0 - self.alpha)

    def _h_integral_inv(self, u):
        if self.alpha == 1.0:
            return np.exp(u)
        return np.power(1.0 + u * (1.0 - self.alpha), 1.0 / (1.0 - self.alpha))

    def sample(self, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.int64)
        filled = 0
        while filled < count:
            want = count - filled
            u = self._h_n + self.rng.random(want) * (self._h_x1 - self._h_n)
            x = self._h_integral_inv(u)
            k = np.clip(np.rint(x), 1, self.n)
            accept = (k - x <= self._s) | (u >= self._h_integral(k + 0.5) - self._h(k))
            good = k[accept].astype(np.int64)
            take = min(len(good), want)
            out[filled: filled + take] = good[:take]
            filled += take
        return out


def zipf_ranks(count: int, universe: int, alpha: float, seed: int) -> np.ndarray:
    rng = np.random.default_rng(np.random.PCG64(seed))
    return ZipfSampler(universe, alpha, rng).sample(count)


def rank_to_key(ranks: np.ndarray, seed: int) -> np.ndarray:
    base = np.uint64(_seed_mix(seed ^ 0xD6E8FEB86659FD93))
    with np.errstate(over="ignore"):
        return mix_to_keys(ranks.astype(np.uint64) + base)


def zipf_keys(count: int, universe: int, alpha: float, seed: int) -> np.ndarray:
    """workloads.py:109-110."""
    return rank_to_key(zipf_ranks(count, universe, alpha, seed), seed)


# ---- device-side generation (torch int64 carries the uint64 bit pattern) ----
_C1_S = 0xFF51AFD7ED558CCD - (1 << 64)
_C2_S = 0xC4CEB9FE1A85EC53 - (1 << 64)
_M31 = (1 << 31) - 1


def _to_i64(v: int) -> int:
    v &= 0xFFFFFFFFFFFFFFFF
    return v - (1 << 64) if v >= (1 << 63) else v


def fmix64_torch(x):
    """fmix64 on an int64 tensor holding uint64 bit patterns (logical shifts
    emulated with arithmetic shift + mask; multiplies wrap mod 2^64)."""
    x = x ^ ((x >> 33) & _M31)
    x = x * _C1_S
    x = x ^ ((x >> 33) & _M31)
    x = x * _C2_S
    x = x ^ ((x >> 33) & _M31)
    return x


def uniform_distinct_keys_torch(count: int, seed: int, stream_offset: int = 0, device="cuda"):
    """Byte-identical to uniform_distinct_keys, generated on `device` (int64 view)."""
    import torch

    base = _to_i64(_seed_mix(seed) + stream_offset)
    x = torch.arange(count, dtype=torch.int64, device=device) + base
    k = fmix64_torch(x)
    bad = (k == -1) | (k == -2)  # >= LOCKED as uint64
    while bool(bad.any()):
        k = torch.where(bad, fmix64_torch(k), k)
        bad = (k == -1) | (k == -2)
    return k
