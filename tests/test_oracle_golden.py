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
