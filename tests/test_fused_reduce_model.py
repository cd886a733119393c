"""Host model of the fused per-stop reduction (csrc/engine.cu,
fused_reduce_kernel / fused_slices / fused_zero) for several world sizes.

Only one GPU is available to this build, and ranks whose kernels wait on one
another must not share it, so the N > 1 behaviour is checked here on the
kernel's own index arithmetic:
  * the G x P slices (CTA b of rank r owns slice q = b*P + r, rows
    [n*q/S, n*(q+1)/S), S = G*P) tile [0, n) exactly once;
  * CTA b's zeroing range after the second barrier is exactly the union of the
    slices (b, *) that the peers' CTA b read before it;
  * with the barriers as phase boundaries, every rank's sum buffer ends as the
    element-wise sum of all partials and every partial ends zero.
"""

from __future__ import annotations

import numpy as np
import pytest


def slice_bounds(n: int, G: int, P: int, b: int, r: int) -> tuple[int, int]:
    S = G * P
    q = b * P + r
    return n * q // S, n * (q + 1) // S


def zero_bounds(n: int, G: int, P: int, b: int) -> tuple[int, int]:
    S = G * P
    return n * (b * P) // S, n * (b * P + P) // S


@pytest.mark.parametrize("P", [1, 2, 3, 8])
@pytest.mark.parametrize("n", [0, 1, 255, 256, 499_500, 1_000_003])
def test_slices_tile_the_live_range(n, P):
    G = 256  # kFusedCtas
    cover = np.zeros(n, dtype=np.int64)
    for b in range(G):
        zlo, zhi = zero_bounds(n, G, P, b)
        owned = []
        for r in range(P):
            lo, hi = slice_bounds(n, G, P, b, r)
            assert 0 <= lo <= hi <= n
            cover[lo:hi] += 1
            owned.append((lo, hi))
        # the slices (b, 0..P-1) are contiguous and are exactly CTA b's zero range
        assert owned[0][0] == zlo and owned[-1][1] == zhi
        assert all(owned[i][1] == owned[i + 1][0] for i in range(P - 1))
    assert np.all(cover == 1)


@pytest.mark.parametrize("P", [2, 3, 8])
def test_phases_sum_and_rezero(P):
    rng = np.random.default_rng(P)
    G, n = 16, 10_007
    partial = [rng.integers(0, 1000, size=n, dtype=np.uint64) for _ in range(P)]
    want = np.sum(partial, axis=0, dtype=np.uint64)
    total = [np.full(n, 0xDEAD, dtype=np.uint64) for _ in range(P)]  # stale sums from an earlier stop
    # phase 2 (after barrier 1): owner (b, r) sums its slice over every peer's
    # partial and stores the sum into every peer's sum buffer
    for r in range(P):
        for b in range(G):
            lo, hi = slice_bounds(n, G, P, b, r)
            v = np.zeros(hi - lo, dtype=np.uint64)
            for p in range(P):
                v += partial[p][lo:hi]
            for p in range(P):
                total[p][lo:hi] = v
    # phase 3 (after barrier 2): CTA b of every rank re-zeroes its own partial's slices (b, *)
    for r in range(P):
        for b in range(G):
            zlo, zhi = zero_bounds(n, G, P, b)
            partial[r][zlo:zhi] = 0
    for p in range(P):
        assert np.array_equal(total[p], want)
        assert not partial[p].any()
