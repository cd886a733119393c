"""Pin the C oracle (oracle/dic_oracle.c) to golden vectors produced by the
reference itself (tests/golden/make_golden.py).  CPU only."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O

GOLD = Path(__file__).resolve().parent / "golden"


def stats_tuple(run: O.OracleRun) -> dict:
    return {"db_passes": run.db_passes, "peak_dashed": run.peak_dashed,
            "candidates_generated": run.candidates_generated, "candidates_pruned": run.candidates_pruned,
            "interval_counts": run.interval_counts}


def test_phase_kats():
    g = json.loads((GOLD / "phases.json").read_text())
    c = g["count_3j1_61"]
    rows = O.rows_from_ints(c["masks"], 64)
    for mask, support, _ in c["result"]:
        assert O.count_block(rows, c["first"], c["last"], mask) == support
    c = g["count_7j_97"]
    assert O.count_block(O.rows_from_ints(c["masks"], 64), c["first"], c["last"], 0x9) == c["support"]
    # first_pass KAT: supports of the singletons
    fp = g["first_pass_1_3_7"]
    assert O.item_support(O.rows_from_ints([0x1, 0x3, 0x7], 3), 3).tolist() == [s for _, s, _ in fp["solid"]]
    # worked example (tiny_db) end to end
    run = O.mine(O.rows_from_ints([0x3, 0x3, 0x1], 2), 2, 0.5, interval=2)
    assert [[m, s] for m, _, s in run.frequent] == g["tiny_db"]
    assert O.absolute_support(0.1, 512) == g["absolute_support_0.1_512"] == 52
    assert O.absolute_support(0.07, 100) == g["absolute_support_0.07_100"] == 8


def test_corpus_matches_reference():
    cases = json.loads((GOLD / "corpus.json").read_text())
    assert len(cases) >= 200
    for c in cases:
        run = O.mine(O.rows_from_ints(c["masks"], c["m"]), c["m"], c["minsup"], interval=c["interval"])
        assert [[m, s] for m, _, s in run.frequent] == c["frequent"]
        assert stats_tuple(run) == c["stats"]


def test_wide_matches_reference():
    cases = json.loads((GOLD / "wide.json").read_text())
    for c in cases:
        masks = [int(x, 16) for x in c["masks"]]
        run = O.mine(O.rows_from_ints(masks, c["m"]), c["m"], c["minsup"], interval=c["interval"])
        assert [[hex(m), s] for m, _, s in run.frequent] == c["frequent"]
        assert stats_tuple(run) == c["stats"]


def test_oracle_threads_do_not_change_counts():
    rng = np.random.default_rng(3)
    rows = rng.integers(0, 2**63, size=(5000, 3), dtype=np.uint64) & rng.integers(0, 2**63, size=(5000, 3),
                                                                                  dtype=np.uint64)
    masks = np.zeros((40, 3), dtype=np.uint64)
    for c in range(40):
        for it in rng.choice(192, size=2, replace=False):
            masks[c, it // 64] |= np.uint64(1) << np.uint64(it % 64)
    a = O.count_many(rows, 17, 4990, masks, threads=1)
    b = O.count_many(rows, 17, 4990, masks, threads=7)
    assert np.array_equal(a, b)
    assert a[0] == O.count_block(rows, 17, 4990, O.mask_from_words(masks[0]))


@pytest.mark.parametrize("idx", [1, 3])
def test_config_goldens(idx):
    from paper_1812_10959_b200.workloads import CONFIGS, generate_csr
    from tests.golden_util import load_config_golden, rows_from_csr

    g = load_config_golden(idx)
    cfg = CONFIGS[idx]
    indptr, indices = generate_csr(cfg)
    assert g.digest_ok(indptr, indices), "generator output drifted from the golden's input"
    rows = rows_from_csr(indptr, indices, cfg.m)
    run = O.mine(rows, cfg.m, cfg.minsup, interval=cfg.interval, threads=8)
    assert [(m, s) for m, _, s in run.frequent] == g.pairs
    assert stats_tuple(run) == g.stats


# ------------------------------------------------ full-size goldens (cfg4 / cfg5)
def test_cfg5_column_count_equals_row_count():
    """oracle/cfg5.c's column-form count (used for the cfg5 golden) equals
    the row-form restatement of _count_block, and its column bitmap is the
    row bitmap transposed."""
    n, m, p, seed = 20_000, 512, 0.05, 5
    rows = O.bernoulli_rows(0, n, m, p, seed)
    cols = O.bernoulli_cols(n, m, p, seed, threads=4)
    back = np.zeros_like(rows)
    for i in range(m):
        bitsv = np.unpackbits(cols[i].view(np.uint8), bitorder="little")[:n].astype(np.uint64)
        back[:, i >> 6] |= bitsv << np.uint64(i & 63)
    assert np.array_equal(rows, back)
    rng = np.random.default_rng(1)
    ks = rng.integers(1, 7, size=300).astype(np.int32)
    items = np.full((300, 6), 0xFFFF, np.uint16)
    masks = np.zeros((300, 8), np.uint64)
    for c in range(300):
        items[c, :ks[c]] = np.sort(rng.choice(m, ks[c], replace=False))
        for it in items[c, :ks[c]]:
            masks[c, it >> 6] |= np.uint64(1) << np.uint64(it & 63)
    assert np.array_equal(O.count_cols(cols, items, ks, threads=4), O.count_many(rows, 0, n - 1, masks, threads=4))


def test_cfg5_golden_candidates_and_checksum():
    import hashlib

    from oracle import synth as S
    from paper_1812_10959_b200.workloads import CONFIGS

    z = np.load(GOLD / "cfg5.npz")
    meta = json.loads(str(z["meta"]))
    cfg = CONFIGS[5]
    ks, items = S.candidates(cfg.params["candidates"], cfg.m, cfg.params["kmin"], cfg.params["kmax"], cfg.seed)
    h = hashlib.sha256()
    h.update(ks.astype(np.int32).tobytes())
    h.update(items.astype(np.uint16).tobytes())
    assert h.hexdigest() == meta["cand_sha256"]
    sup = z["supports"].astype(np.int64)
    assert int(sup.sum()) == meta["support_checksum"] and len(sup) == cfg.params["candidates"]
    assert (z["ks"].astype(np.int32) == ks).all()
    # i.i.d. Bernoulli(0.05): E[support] = n 0.05^k
    for k in (2, 3):
        assert abs(sup[ks == k].mean() / (cfg.n * 0.05 ** k) - 1) < 0.02
    assert abs(z["item_counts"].mean() / (cfg.n * 0.05) - 1) < 0.001


def test_cfg4_golden_consistent_and_recounted():
    """The cfg4 golden (oracle over all 10M rows): the generator still makes
    the same CSR (sha256), the frequent set is downward closed with
    anti-monotone supports, and 24 sampled supports recount exactly from the
    CSR with an independent NumPy intersection of item row lists."""
    from oracle import synth as S
    from paper_1812_10959_b200.workloads import CONFIGS
    from tests.golden_util import csr_digest, load_config_golden

    g = load_config_golden(4)
    assert g.stats["candidates_generated"] == 509_227 and len(g.sizes) == 8_523
    sup = dict(g.pairs)
    for mask, s in g.pairs:
        assert s >= 10_000
        x = mask
        while x:
            b = x & -x
            x ^= b
            if mask ^ b:
                assert sup[mask ^ b] >= s
    cfg = CONFIGS[4]
    indptr, indices = S.generate_csr(cfg)
    assert csr_digest(indptr, indices) == g.meta["csr_sha256"]
    rng = np.random.default_rng(4)
    multi = [p for p in g.pairs if bin(p[0]).count("1") >= 2]
    pick = [multi[i] for i in rng.choice(len(multi), 24, replace=False)]
    need = sorted({b for mk, _ in pick for b in range(cfg.m) if mk >> b & 1})
    sel = np.isin(indices, need)
    row_of = np.repeat(np.arange(cfg.n, dtype=np.int64), np.diff(indptr))[sel]
    it_of = indices[sel]
    order = np.argsort(it_of, kind="stable")
    it_sorted, rows_sorted = it_of[order], row_of[order]
    bounds = np.searchsorted(it_sorted, need + [cfg.m])
    lists = {it: np.unique(rows_sorted[bounds[j]:bounds[j + 1]]) for j, it in enumerate(need)}
    for mk, s in pick:
        its = [b for b in range(cfg.m) if mk >> b & 1]
        acc = lists[its[0]]
        for it in its[1:]:
            acc = np.intersect1d(acc, lists[it], assume_unique=True)
        assert len(acc) == s
