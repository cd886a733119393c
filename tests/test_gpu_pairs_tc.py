"""The dense pair triangle on the tensor cores (csrc/pairs_mma.cu) against the
AND/POPC kernel and a NumPy Gram matrix: bit-exact integer counts for every
pair a < b, on universes that are not multiples of the 128 x 256 tile, chunks
with unaligned ends, tiny chunks (fewer 4-word stages than K slices), dense
and sparse rows, and through the engine (cfg4-shaped run vs the oracle).
The count is first_pass's pair wave (engine.py:165-168) per chunk."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_1812_10959_b200 as dic
from oracle import oracle as O
from paper_1812_10959_b200 import device as D
from paper_1812_10959_b200.workloads import CONFIGS, generate_csr, scaled

pytestmark = pytest.mark.gpu


def _rows(rng, n, m, density):
    W = (m + 63) // 64
    bits = rng.random((n, m)) < density
    rows = np.zeros((n, W), dtype=np.uint64)
    for i in range(m):
        rows[:, i >> 6] |= bits[:, i].astype(np.uint64) << np.uint64(i & 63)
    return rows, bits


class _Mode:
    def __init__(self, mode: int):
        self.mode = mode

    def __enter__(self):
        self.prev = D.pair_kernel_select(self.mode)

    def __exit__(self, *exc):
        D.pair_kernel_select(self.prev)


@pytest.mark.parametrize("m,n,density,first,last", [
    (1000, 100_000, 0.02, 0, 99_999),      # the cfg4 chunk shape
    (1000, 30_000, 0.3, 7, 29_950),        # dense, unaligned ends
    (842, 20_000, 0.05, 31, 19_999),       # cfg2's |L1|, TW = 16
    (700, 20_000, 0.08, 1, 18_000),        # TW = 32
    (128, 5_000, 0.5, 0, 4_999),           # one A block
    (129, 4_000, 0.4, 33, 3_100),          # one item into a second block
    (300, 70, 0.5, 3, 66),                 # 3 words: fewer stages than slices
    (257, 1_000, 0.9, 500, 500),           # a single row
])
def test_tensor_triangle_matches_numpy_and_lop3(m, n, density, first, last):
    rng = np.random.default_rng(m * 7 + n)
    rows, bits = _rows(rng, n, m, density)
    tids = D.rows_to_tids(torch.from_numpy(rows.view(np.int64)).cuda(), n, m)
    with _Mode(2):
        tc = D.count_pairs(tids, n, m, first, last).cpu().numpy()
    with _Mode(1):
        lop = D.count_pairs(tids, n, m, first, last).cpu().numpy()
    blk = bits[first:last + 1].astype(np.float64)
    gram = (blk.T @ blk)[np.triu_indices(m, k=1)].astype(np.int64)
    assert np.array_equal(tc, gram)
    assert np.array_equal(lop, gram)


def test_tensor_triangle_accumulates():
    rng = np.random.default_rng(5)
    m, n = 500, 9_000
    rows, bits = _rows(rng, n, m, 0.1)
    tids = D.rows_to_tids(torch.from_numpy(rows.view(np.int64)).cuda(), n, m)
    with _Mode(2):
        tri = torch.full((m * (m - 1) // 2,), 3, dtype=torch.int64, device="cuda")
        D.count_pairs(tids, n, m, 0, 4_000, tri)
        D.count_pairs(tids, n, m, 4_001, n - 1, tri)
    b = bits.astype(np.float64)
    want = (b.T @ b)[np.triu_indices(m, k=1)].astype(np.int64) + 3
    assert np.array_equal(tri.cpu().numpy(), want)


@pytest.mark.parametrize("mode", [1, 2])
def test_engine_pair_wave_either_kernel_matches_oracle(mode):
    """A cfg4-shaped mining run (1000 frequent items: a 499,500-pair wave)
    through the engine's graphs with each pair kernel, against the oracle."""
    cfg = scaled(CONFIGS[4], 60_000, interval=6_000)
    indptr, indices = generate_csr(cfg)
    db = dic.BitDatabase.from_csr(indptr, indices, cfg.m)
    params = dic.MiningParams.create(cfg.n, cfg.minsup, interval=cfg.interval)
    with _Mode(mode):
        res = dic.mine_parallel(db, params)
    want = O.mine(db.rows, cfg.m, cfg.minsup, interval=cfg.interval, threads=8)
    assert [(f.mask, f.size, f.support) for f in res.frequent] == want.frequent
    s = res.stats
    assert (s.db_passes, s.peak_dashed, s.candidates_generated, s.candidates_pruned, s.interval_counts) == (
        want.db_passes, want.peak_dashed, want.candidates_generated, want.candidates_pruned, want.interval_counts)
