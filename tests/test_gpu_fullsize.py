"""Parity at BASELINE.json's full sizes through size-independent properties
(the CPU oracle cannot mine 10M rows in a test's time): cfg4 (10M x 1000,
the bench workload) and cfg5 (50M x 512, the kernel microbenchmark).

Every check compares the bit-sliced hot kernels against an independent
kernel or an identity that holds for any correct result:
  * supports recounted by the literal (T & I) == I row-form kernel
    (dic_count_support_rows, count.cu) on the uint64 row bitmap;
  * singleton supports == the column popcounts of first_pass;
  * the frequent set is downward closed and supports are anti-monotone
    (engine.py:165-168/:320-369 admit a candidate only when every immediate
    subset is frequent; support(I) <= support(J) for J in I);
  * linearity over rows: counting [0, h) and [h, n) adds up to [0, n);
  * the dense pair triangle of a whole chunk equals per-pair recounts.
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_1812_10959_b200 as dic
from paper_1812_10959_b200 import bits
from paper_1812_10959_b200.workloads import CONFIGS, generate_csr

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _masks_to_device(masks: list[int], W: int):
    arr = np.zeros((len(masks), W), dtype=np.uint64)
    for i, mk in enumerate(masks):
        for w in range(W):
            arr[i, w] = (mk >> (64 * w)) & 0xFFFFFFFFFFFFFFFF
    return torch.from_numpy(arr.view(np.int64)).cuda()


@pytest.fixture(scope="module")
def cfg4_run():
    from paper_1812_10959_b200 import device as D

    D.require_cuda()
    cfg = CONFIGS[4]
    indptr, indices = generate_csr(cfg)
    db = dic.BitDatabase.from_csr(indptr, indices, cfg.m)
    params = dic.MiningParams.create(cfg.n, cfg.minsup, interval=cfg.interval)
    res = dic.mine_parallel(db, params)
    yield cfg, db, params, res
    torch.cuda.empty_cache()


def test_cfg4_frequent_set_is_downward_closed_and_antimonotone(cfg4_run):
    cfg, db, params, res = cfg4_run
    need = params.min_support_count
    sup = {f.mask: f.support for f in res.frequent}
    assert len(sup) == len(res.frequent) > 1000
    for f in res.frequent:
        assert f.support >= need
        assert f.size == bin(f.mask).count("1")
        if f.size < 2:
            continue
        m = f.mask
        while m:
            low = m & -m
            sub = f.mask ^ low
            assert sub in sup, f"subset {sub:#x} of frequent {f.mask:#x} missing"
            assert sup[sub] >= f.support
            m ^= low
    # canonical order: (size, mask)
    keys = [(f.size, f.mask) for f in res.frequent]
    assert keys == sorted(keys)


def test_cfg4_singletons_equal_column_counts(cfg4_run):
    from paper_1812_10959_b200 import device as D

    cfg, db, params, res = cfg4_run
    counts = D.item_support(db.device_tids(), cfg.n, cfg.m, 0, cfg.n - 1).cpu().numpy()
    singles = {f.mask.bit_length() - 1: f.support for f in res.frequent if f.size == 1}
    for item, s in singles.items():
        assert counts[item] == s
    assert set(singles) == {i for i in range(cfg.m) if counts[i] >= params.min_support_count}


def test_cfg4_supports_recounted_by_row_kernel(cfg4_run):
    from paper_1812_10959_b200 import device as D

    cfg, db, params, res = cfg4_run
    rng = np.random.default_rng(4)
    by_size: dict[int, list] = {}
    for f in res.frequent:
        by_size.setdefault(f.size, []).append(f)
    sample = []
    for k, fs in sorted(by_size.items()):
        idx = rng.choice(len(fs), size=min(len(fs), 150), replace=False)
        sample += [fs[i] for i in idx]
    W = bits.words_for(cfg.m)
    rows = D.tids_to_rows(db.device_tids(), cfg.n, cfg.m)
    got = D.count_support_rows(rows, 0, cfg.n - 1, _masks_to_device([f.mask for f in sample], W)).cpu().numpy()
    assert [int(x) for x in got] == [f.support for f in sample]


def test_cfg4_dense_pair_chunk_equals_row_recount(cfg4_run):
    """The pair kernel (hybrid static/dynamic schedule, grain counters
    re-armed per launch) over one full M-row chunk, twice, against the row
    kernel on a sample of pairs."""
    from paper_1812_10959_b200 import device as D

    cfg, db, params, res = cfg4_run
    first, last = 3 * cfg.interval, 4 * cfg.interval - 1
    tids = db.device_tids()
    tri1 = D.count_pairs(tids, cfg.n, cfg.m, first, last).cpu().numpy()
    tri2 = D.count_pairs(tids, cfg.n, cfg.m, first, last).cpu().numpy()
    assert np.array_equal(tri1, tri2)
    rng = np.random.default_rng(5)
    ab = []
    while len(ab) < 2000:
        a, b = sorted(rng.choice(cfg.m, 2, replace=False).tolist())
        ab.append((a, b))
    W = bits.words_for(cfg.m)
    rows = D.tids_to_rows(tids, cfg.n, cfg.m)
    got = D.count_support_rows(rows, first, last, _masks_to_device([(1 << a) | (1 << b) for a, b in ab], W))
    m = cfg.m
    idx = [a * m - a * (a + 1) // 2 + (b - a - 1) for a, b in ab]
    assert [int(x) for x in got.cpu().numpy()] == [int(tri1[i]) for i in idx]
    assert int(tri1.sum()) > 0


@pytest.fixture(scope="module")
def cfg5_bitmap():
    from paper_1812_10959_b200 import device as D

    D.require_cuda()
    cfg = CONFIGS[5]
    n, m = cfg.n, cfg.m
    rows = D.bernoulli_rows(n, m, cfg.params["p"], cfg.seed)
    tids = D.rows_to_tids(rows, n, m)
    ks, items = D.synth_candidates(cfg.params["candidates"], m, cfg.params["kmin"], cfg.params["kmax"], cfg.seed)
    yield cfg, rows, tids, ks, items
    del rows, tids
    torch.cuda.empty_cache()


@pytest.mark.parametrize("k", [2, 3, 6])
def test_cfg5_bit_sliced_count_equals_row_count_and_is_linear(cfg5_bitmap, k):
    from paper_1812_10959_b200 import device as D

    cfg, rows, tids, ks, items = cfg5_bitmap
    n, m = cfg.n, cfg.m
    sel = items[ks == k][:, :k][:1500]
    sel = sel[np.lexsort(sel.T[::-1])]
    it = torch.from_numpy(np.ascontiguousarray(sel).view(np.int16)).cuda()
    full = D.count_support(tids, n, m, 0, n - 1, it).cpu().numpy()
    h = 31_415_927  # an unaligned split (not a multiple of 32 or of a tile)
    halves = (D.count_support(tids, n, m, 0, h - 1, it) + D.count_support(tids, n, m, h, n - 1, it)).cpu().numpy()
    assert np.array_equal(full, halves)
    masks = [sum(1 << int(i) for i in row) for row in sel[:300]]
    got = D.count_support_rows(rows, 0, n - 1, _masks_to_device(masks, bits.words_for(m))).cpu().numpy()
    assert np.array_equal(got, full[:300])
    if k <= 3:  # i.i.d. Bernoulli(0.05): E[support] = n * 0.05^k (tight for small k)
        assert abs(full.mean() / (n * 0.05 ** k) - 1) < 0.05


# ------------------------------------------------ full-size oracle goldens
# tests/golden/cfg4.npz: the C oracle mined all 10M rows (make_golden_cfg4.py,
# 51 min on 7 host threads); tests/golden/cfg5.npz: the support of all 100k
# cfg5 candidates over all 50M rows (make_golden_cfg5.py).  The oracle itself
# is pinned to the reference in tests/test_oracle_golden.py.
from tests.golden_util import csr_digest, load_config_golden  # noqa: E402


def _golden_stats(g) -> tuple:
    st = g.stats
    return (st["db_passes"], st["peak_dashed"], st["candidates_generated"], st["candidates_pruned"],
            st["interval_counts"])


def _stats(s) -> tuple:
    return (s.db_passes, s.peak_dashed, s.candidates_generated, s.candidates_pruned, s.interval_counts)


def test_cfg4_full_equals_oracle_golden(cfg4_run):
    """Bench workload, one GPU: every frequent itemset, its support and every
    MiningStats counter equal the oracle's full-size run."""
    cfg, db, params, res = cfg4_run
    g = load_config_golden(4)
    indptr, indices = generate_csr(cfg)
    assert csr_digest(indptr, indices) == g.meta["csr_sha256"], "generator drift"
    assert [(f.mask, f.support) for f in res.frequent] == g.pairs
    assert [f.size for f in res.frequent] == g.sizes.tolist()
    assert _stats(res.stats) == _golden_stats(g)


@pytest.mark.parametrize("world", [2, 8])
def test_cfg4_full_sharded_lockstep_equals_oracle_golden(world):
    """The sharded trajectory at full size: `world` engines over the
    chunk-sliced shards of all 10M rows, counts summed slot by slot per stop
    (lockstep.py), against the same golden — frequent set, supports, stats."""
    from paper_1812_10959_b200.lockstep import mine_lockstep

    cfg = CONFIGS[4]
    g = load_config_golden(4)
    params = dic.MiningParams.create(cfg.n, cfg.minsup, interval=cfg.interval)
    shards = []
    for r in range(world):
        plan = dic.ShardPlan.for_params(params, world, r)
        ip, ix = generate_csr(cfg, ranges=plan.ranges())
        shards.append(dic.BitDatabase.from_csr(ip, ix, cfg.m))
    res, info = mine_lockstep(shards, params, check_layout=world == 2, max_size=6)
    assert [(f.mask, f.support) for f in res.frequent] == g.pairs
    assert _stats(res.stats) == _golden_stats(g)
    assert info.stops == g.meta["stops"]
    del shards
    torch.cuda.empty_cache()


def test_cfg5_device_generator_matches_host_restatement(cfg5_bitmap):
    from oracle import oracle as O

    cfg, rows, tids, ks, items = cfg5_bitmap
    for r0 in (0, 31_415_926, cfg.n - 2000):
        host = O.bernoulli_rows(r0, 2000, cfg.m, cfg.params["p"], cfg.seed)
        dev = rows[r0:r0 + 2000].cpu().numpy().view(np.uint64)
        assert np.array_equal(host, dev)


def test_cfg5_all_candidates_equal_oracle_golden(cfg5_bitmap):
    """All 100,000 cfg5 candidates over all 50M rows through the product
    count kernel (dic_count_support, one launch per size bucket) against the
    oracle's column count; plus first_pass's column popcounts."""
    import hashlib

    from paper_1812_10959_b200 import device as D

    z = np.load(GOLD5)
    import json

    meta = json.loads(str(z["meta"]))
    cfg, rows, tids, ks, items = cfg5_bitmap
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(ks, dtype=np.int32).tobytes())
    h.update(np.ascontiguousarray(items, dtype=np.uint16).tobytes())
    assert h.hexdigest() == meta["cand_sha256"]
    n, m = cfg.n, cfg.m
    counts = torch.zeros(m, dtype=torch.int64, device="cuda")
    D.item_support(tids, n, m, 0, n - 1, counts)
    assert np.array_equal(counts.cpu().numpy(), z["item_counts"].astype(np.int64))
    got = np.zeros(len(ks), dtype=np.int64)
    for k in range(cfg.params["kmin"], cfg.params["kmax"] + 1):
        idx = np.nonzero(ks == k)[0]
        it = torch.from_numpy(np.ascontiguousarray(items[idx, :k]).view(np.int16)).cuda()
        got[idx] = D.count_support(tids, n, m, 0, n - 1, it).cpu().numpy()
    want = z["supports"].astype(np.int64)
    assert np.array_equal(got, want)
    assert int(got.sum()) == meta["support_checksum"]


GOLD5 = __import__("pathlib").Path(__file__).resolve().parent / "golden" / "cfg5.npz"
