"""The reference's seeded synthetic database generator (datasets.py:66-142),
restated: geometric item weights skew**i, per-transaction length around
avg_len, distinct items by Gumbel-top-k sampling, all randomness from a
counter-based SplitMix64 stream so equal specs give identical databases —
the same databases as the reference's generator (same streams, same float
formulas, same stable ordering).  Host-side input tooling for the CLI's
``generate``; the BASELINE configs use workloads.py's generators."""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .bitmap import BitDatabase
from .exceptions import SpecError

DEFAULT_SKEW = 0.90
GEN_MAX_ITEMS = 64  # the generator emits single-word masks, as the reference's
_BLOCK = 16384

_G = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _splitmix_finalize(x: np.ndarray) -> np.ndarray:
    x = (x ^ (x >> np.uint64(30))) * _M1
    x = (x ^ (x >> np.uint64(27))) * _M2
    return x ^ (x >> np.uint64(31))


def _stream_key(seed: int, tag: int) -> np.uint64:
    return _splitmix_finalize(np.array([(seed & (2**64 - 1)) ^ tag], dtype=np.uint64))[0]


def _uniforms(key: np.uint64, first: int, count: int) -> np.ndarray:
    """Floats in (0, 1) from stream counters first+1 .. first+count."""
    ctr = np.arange(first + 1, first + count + 1, dtype=np.uint64)
    return ((_splitmix_finalize(key + ctr * _G) >> np.uint64(11)).astype(np.float64) + 0.5) * 2.0**-53


@dataclass(frozen=True)
class DatasetSpec:
    """Shape of a synthetic transaction database (skew: decay of item weights)."""

    n: int
    m: int
    avg_len: float
    seed: int
    skew: float = DEFAULT_SKEW

    def validate(self) -> None:
        if self.n < 1:
            raise SpecError(f"n must be >= 1, got {self.n}")
        if not 1 <= self.m <= GEN_MAX_ITEMS:
            raise SpecError(f"m must lie in [1, {GEN_MAX_ITEMS}], got {self.m}")
        if not 1 <= self.avg_len <= self.m:
            raise SpecError(f"avg_len must lie in [1, m={self.m}], got {self.avg_len}")
        if not 0.0 < self.skew <= 1.0:
            raise SpecError(f"skew must lie in (0, 1], got {self.skew}")


def generate_synthetic(spec: DatasetSpec) -> BitDatabase:
    spec.validate()
    n, m = spec.n, spec.m
    k_len = _stream_key(spec.seed, 0x6C656E)
    k_key = _stream_key(spec.seed, 0x6B6579)
    lo = int(math.floor(spec.avg_len))
    frac = spec.avg_len - lo
    jit = max(min(2, lo - 1, m - lo - (1 if frac > 0 else 0)), 0)
    log_w = np.arange(m, dtype=np.float64) * math.log(spec.skew)
    pos = np.arange(m, dtype=np.int64)[None, :]
    out = np.empty(n, dtype=np.uint64)
    for r0 in range(0, n, _BLOCK):
        r = min(_BLOCK, n - r0)
        u = _uniforms(k_len, 2 * r0, 2 * r).reshape(r, 2)
        length = np.full(r, lo, dtype=np.int64)
        if frac > 0:
            length += (u[:, 0] < frac).astype(np.int64)
        if jit > 0:
            length += (u[:, 1] * (2 * jit + 1)).astype(np.int64) - jit
        g = log_w - np.log(-np.log(_uniforms(k_key, r0 * m, r * m).reshape(r, m)))
        rank = np.argsort(-g, axis=1, kind="stable")
        picked = np.where(pos < length[:, None], np.uint64(1) << rank.astype(np.uint64), np.uint64(0))
        out[r0:r0 + r] = np.bitwise_or.reduce(picked, axis=1)
    return BitDatabase(out, m=m)
