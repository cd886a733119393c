"""GPU parity of the drop-in API and the device engine against the reference's
golden vectors and the CPU oracle: frequent itemsets, supports and every
MiningStats counter must be identical (bit-exact integer work)."""

from __future__ import annotations

import json
import random
from pathlib import Path

import numpy as np
import pytest

import paper_1812_10959_b200 as dic
from oracle import oracle as O
from paper_1812_10959_b200.workloads import CONFIGS, generate_csr, scaled
from tests.golden_util import has_config_golden, load_config_golden

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


def pairs(res) -> list[list[int]]:
    return [[f.mask, f.support] for f in res.frequent]


def stats(res) -> dict:
    s = res.stats
    return {"db_passes": s.db_passes, "peak_dashed": s.peak_dashed, "candidates_generated": s.candidates_generated,
            "candidates_pruned": s.candidates_pruned, "interval_counts": s.interval_counts}


# ---------------------------------------------------------------- phase KATs
def record(mask, shape, support=0, intervals=0):
    r = dic.CountedItemset.fresh(mask)
    r.shape, r.support, r.intervals_counted = shape, support, intervals
    return r


def catalog(dashed=(), solid=()):
    cat = dic.ItemsetCatalog()
    for r in dashed:
        cat.dashed.append(r)
        cat.known[r.mask] = r
    for r in solid:
        cat.solid.append(r)
        cat.known[r.mask] = r
    return cat


S = dic.Shape


def test_first_pass_kat():
    g = json.loads((GOLD / "phases.json").read_text())["first_pass_1_3_7"]
    db = dic.BitDatabase([0x1, 0x3, 0x7])
    cat = dic.ItemsetCatalog()
    lvl = dic.first_pass(cat, db, dic.MiningParams.create(3, 0.5))
    assert [[r.mask, r.support, r.shape.value] for r in cat.solid] == g["solid"]
    assert lvl == g["level1"] and [r.mask for r in cat.dashed] == g["dashed"]


def test_first_pass_nothing_frequent_and_single_row():
    cat = dic.ItemsetCatalog()
    assert dic.first_pass(cat, dic.BitDatabase([0x1, 0x2]), dic.MiningParams.create(2, 1.0)) == []
    assert cat.dashed == [] and all(r.shape is S.SOLID_CIRCLE for r in cat.solid)
    cat = dic.ItemsetCatalog()
    assert dic.first_pass(cat, dic.BitDatabase([0x3]), dic.MiningParams.create(1, 1.0)) == [0x1, 0x2]
    assert [r.mask for r in cat.dashed] == [0x3]


def test_count_support_interval_kats():
    g = json.loads((GOLD / "phases.json").read_text())
    db = dic.BitDatabase([0x5, 0x7, 0x6, 0x4])
    cat = catalog(dashed=[record(0x4, S.DASHED_CIRCLE)])
    dic.count_support_interval(cat, db, 0, 3)
    assert (cat.dashed[0].support, cat.dashed[0].intervals_counted) == (4, 1)
    cat = catalog(dashed=[record(0x3, S.DASHED_CIRCLE, 2, 1)])
    dic.count_support_interval(cat, dic.BitDatabase([0x1, 0x2]), 0, 1)
    assert (cat.dashed[0].support, cat.dashed[0].intervals_counted) == (2, 2)
    dic.count_support_interval(catalog(), dic.BitDatabase([0x1]), 0, 0)  # empty: no-op
    with pytest.raises(ValueError):
        dic.count_support_interval(catalog(dashed=[record(1, S.DASHED_CIRCLE)]), dic.BitDatabase([1, 2]), 0, 2)
    c = g["count_3j1_61"]
    for threads in (1, 2, 5, 16):
        cat = catalog(dashed=[record(q, S.DASHED_CIRCLE) for q in (0x1, 0x3, 0x8, 0x15)])
        dic.count_support_interval(cat, dic.BitDatabase(c["masks"]), c["first"], c["last"], threads)
        assert [[r.mask, r.support, r.intervals_counted] for r in cat.dashed] == c["result"]
    c = g["count_7j_97"]
    cat = catalog(dashed=[record(0x9, S.DASHED_CIRCLE)])
    dic.count_support_interval(cat, dic.BitDatabase(c["masks"]), c["first"], c["last"], kernel="python")
    assert cat.dashed[0].support == c["support"]


def test_prune_kats():
    p = dic.MiningParams.create(50, 0.8, interval=10)  # need 40, 5 chunks
    cat = catalog(dashed=[record(0x3, S.DASHED_CIRCLE, 3, 2)])
    st = dic.MiningStats()
    dic.prune(cat, p, stats=st)
    assert cat.dashed == [] and st.candidates_pruned == 1
    cat = catalog(dashed=[record(0x3, S.DASHED_CIRCLE, 40, 2)])
    assert [r.mask for r in dic.prune(cat, p)] == [0x3] and cat.dashed[0].shape is S.DASHED_BOX
    cat = catalog(dashed=[record(0x3, S.DASHED_CIRCLE, 3, 2), record(0x7, S.DASHED_CIRCLE, 2, 1),
                          record(0x18, S.DASHED_CIRCLE, 39, 4)])
    st = dic.MiningStats()
    dic.prune(cat, p, stats=st)
    assert [r.mask for r in cat.dashed] == [0x18] and st.candidates_pruned == 2  # superset branch
    cat = catalog(dashed=[record(0x3, S.DASHED_CIRCLE, 3, 2)])
    dic.prune(cat, p, bound_enabled=False)
    assert [r.mask for r in cat.dashed] == [0x3]
    cat = catalog(dashed=[record(0x3, S.DASHED_CIRCLE, 3, 5)])
    dic.prune(cat, p)
    assert [r.mask for r in cat.dashed] == [0x3]


def _lattice(pair_shapes):
    solid = [record(0x1, S.SOLID_BOX, 9), record(0x2, S.SOLID_BOX, 9), record(0x4, S.SOLID_BOX, 9)]
    return catalog(solid=solid, dashed=[record(mk, sh, 5, 1) for mk, sh in pair_shapes])


def test_make_candidates_kats():
    p = dic.MiningParams.create(10, 0.2)
    assert dic.make_candidates(_lattice([(0x3, S.DASHED_BOX), (0x6, S.DASHED_BOX), (0x5, S.DASHED_CIRCLE)]), p) == 0
    cat = catalog(solid=[record(0x1, S.SOLID_BOX, 9), record(0x2, S.SOLID_BOX, 9), record(0x4, S.SOLID_CIRCLE)],
                  dashed=[record(0x3, S.DASHED_BOX, 5, 1)])
    assert dic.make_candidates(cat, p) == 0
    cat = _lattice([(0x3, S.DASHED_BOX), (0x5, S.DASHED_BOX), (0x6, S.DASHED_BOX)])
    st = dic.MiningStats()
    assert dic.make_candidates(cat, p, stats=st) == 1 and st.candidates_generated == 1
    new = [r for r in cat.dashed if r.mask == 0x7]
    assert len(new) == 1 and new[0].shape is S.DASHED_CIRCLE and new[0].support == 0
    assert dic.make_candidates(cat, p) == 0  # dedup index blocks regeneration
    assert dic.make_candidates(catalog(solid=[record(0x1, S.SOLID_CIRCLE)],
                                       dashed=[record(0x3, S.DASHED_CIRCLE)]), p) == 0
    full = _lattice([(0x3, S.DASHED_BOX), (0x5, S.DASHED_BOX), (0x6, S.DASHED_BOX)])
    dic.make_candidates(full, p)
    front = _lattice([(0x3, S.DASHED_BOX), (0x5, S.DASHED_BOX), (0x6, S.DASHED_BOX)])
    dic.make_candidates(front, p, frontier=[front.known[0x6]])
    assert {r.mask for r in full.dashed} == {r.mask for r in front.dashed}


def test_check_full_pass_kats():
    p = dic.MiningParams.create(20, 0.5, interval=5)
    cat = catalog(dashed=[record(0x3, S.DASHED_BOX, 12, 4)])
    dic.check_full_pass(cat, p)
    assert cat.dashed == [] and cat.solid[0].shape is S.SOLID_BOX
    cat = catalog(dashed=[record(0x3, S.DASHED_CIRCLE, 4, 4)])
    dic.check_full_pass(cat, p)
    assert cat.solid[0].shape is S.SOLID_CIRCLE
    cat = catalog(dashed=[record(0x3, S.DASHED_BOX, 12, 3)])
    dic.check_full_pass(cat, p)
    assert [r.mask for r in cat.dashed] == [0x3] and cat.solid == []


# ------------------------------------------------------------ end to end
def test_worked_examples():
    g = json.loads((GOLD / "phases.json").read_text())
    tiny = dic.BitDatabase([0x3, 0x3, 0x1])
    assert pairs(dic.mine_serial(tiny, dic.MiningParams.create(3, 0.5, interval=2))) == g["tiny_db"]
    assert pairs(dic.mine_parallel(tiny, dic.MiningParams.create(3, 0.5, interval=2, threads=4))) == g["tiny_db"]
    assert pairs(dic.mine_serial(dic.BitDatabase([0x1]), dic.MiningParams.create(1, 1.0))) == [[0x1, 1]]
    with pytest.raises(ValueError):
        dic.mine_serial(tiny, dic.MiningParams.create(7, 0.5))
    keys = [(f.size, f.mask) for f in dic.mine_serial(dic.BitDatabase([0x7, 0x7, 0x7, 0x6]),
                                                        dic.MiningParams.create(4, 0.5)).frequent]
    assert keys == sorted(keys)


def test_corpus_engine_matches_reference():
    for c in json.loads((GOLD / "corpus.json").read_text()):
        db = dic.BitDatabase(c["masks"], m=c["m"])
        res = dic.mine_parallel(db, dic.MiningParams.create(c["n"], c["minsup"], interval=c["interval"]))
        assert pairs(res) == c["frequent"], (c["n"], c["m"], c["minsup"], c["interval"])
        assert stats(res) == c["stats"]


def test_wide_engine_matches_reference():
    for c in json.loads((GOLD / "wide.json").read_text()):
        masks = [int(x, 16) for x in c["masks"]]
        db = dic.BitDatabase(masks, m=c["m"])
        res = dic.mine_parallel(db, dic.MiningParams.create(c["n"], c["minsup"], interval=c["interval"]))
        assert [[hex(m), s] for m, s in pairs(res)] == c["frequent"]
        assert stats(res) == c["stats"]


def test_audit_mode_is_legal_and_equal():
    rng = random.Random(5150)
    for _ in range(6):
        n, m = rng.randint(4, 120), rng.randint(2, 10)
        masks = [sum(1 << i for i in range(m) if rng.random() < 0.4) for _ in range(n)]
        db = dic.BitDatabase(masks, m=m)
        p = dic.MiningParams.create(n, 0.25, interval=max(1, n // 4))
        audit = dic.TransitionAudit()
        a = dic.mine_parallel(db, p, audit=audit)
        b = dic.mine_parallel(db, p)
        assert audit.illegal() == [] and pairs(a) == pairs(b) and stats(a) == stats(b)
        assert {(o, nw) for _, o, nw in audit.transitions} <= dic.LEGAL_TRANSITIONS


@pytest.mark.parametrize("seed,m_fixed", [(s, None) for s in range(8)] + [(100, 1100), (101, 1600)])
def test_random_wide_engine_matches_oracle(seed, m_fixed):
    """m_fixed > 1024: masks of more than 16 words take the generic (mask
    view) candidate evaluation; at 1600 items a double-buffered tile no
    longer fits shared memory and the counts take the unstaged path."""
    rng = np.random.default_rng(seed)
    m = m_fixed or int(rng.choice([65, 130, 257, 700, 1000, 1200]))
    n = int(rng.integers(200, 6000))
    hot = rng.choice(m, size=8, replace=False)
    W = (m + 63) // 64
    rows = np.zeros((n, W), dtype=np.uint64)
    for it in hot:
        on = rng.random(n) < 0.5
        rows[on, it // 64] |= np.uint64(1) << np.uint64(it % 64)
    noise = rng.integers(0, m, size=(n, 5))
    for j in range(5):
        np.bitwise_or.at(rows, (np.arange(n), noise[:, j] // 64), np.uint64(1) << (noise[:, j] % 64).astype(np.uint64))
    minsup = float(rng.choice([0.03, 0.1, 0.3]))
    interval = int(rng.integers(1, n + 1))
    db = dic.BitDatabase(rows, m=m)
    res = dic.mine_parallel(db, dic.MiningParams.create(n, minsup, interval=interval))
    want = O.mine(rows, m, minsup, interval=interval, threads=4)
    assert [(f.mask, f.size, f.support) for f in res.frequent] == want.frequent
    assert stats(res) == {"db_passes": want.db_passes, "peak_dashed": want.peak_dashed,
                          "candidates_generated": want.candidates_generated,
                          "candidates_pruned": want.candidates_pruned, "interval_counts": want.interval_counts}


def test_prune_bound_fires_and_is_safe():
    cfg = scaled(CONFIGS[3], 40_000, interval=2_000)  # dense: the bound prunes many candidates
    indptr, indices = generate_csr(cfg)
    db = dic.BitDatabase.from_csr(indptr, indices, cfg.m)
    on = dic.mine_parallel(db, dic.MiningParams.create(cfg.n, cfg.minsup, interval=cfg.interval))
    off = dic.mine_parallel(db, dic.MiningParams.create(cfg.n, cfg.minsup, interval=cfg.interval), prune_bound=False)
    assert pairs(on) == pairs(off)
    assert on.stats.candidates_pruned > 0
    assert on.stats.interval_counts <= off.stats.interval_counts
    want = O.mine(db.rows, cfg.m, cfg.minsup, interval=cfg.interval, threads=8)
    assert [(f.mask, f.size, f.support) for f in on.frequent] == want.frequent
    assert on.stats.candidates_pruned == want.candidates_pruned


@pytest.mark.parametrize("idx", [1, 2, 3])
def test_config_goldens_on_gpu(idx):
    if not has_config_golden(idx):
        pytest.skip(f"cfg{idx} golden not generated")
    g = load_config_golden(idx)
    cfg = CONFIGS[idx]
    indptr, indices = generate_csr(cfg)
    assert g.digest_ok(indptr, indices)
    db = dic.BitDatabase.from_csr(indptr, indices, cfg.m)
    res = dic.mine_parallel(db, dic.MiningParams.create(cfg.n, cfg.minsup, interval=cfg.interval))
    assert [(f.mask, f.support) for f in res.frequent] == g.pairs
    assert stats(res) == g.stats


def test_encoder_rejects_out_of_range_items():
    with pytest.raises(dic.ItemOutOfRange) as ei:
        dic.BitDatabase.from_csr(np.array([0, 2, 4]), np.array([1, 3, 5, 64]), 64)
    assert ei.value.item == 64 and ei.value.line == 1
    with pytest.raises(dic.ItemOutOfRange):
        dic.database_from_transactions([[0, 1], [-1]])
    db = dic.database_from_transactions([[2, 2, 0], [], [1]])
    assert db.m == 3 and db.as_int_list() == [0x5, 0x0, 0x2]
    with pytest.raises(dic.EmptyDatabase):
        dic.database_from_transactions([])


def test_stop_graphs_match_direct_launches():
    """The Python pipelined loop (graph launches for scheduled chunks) and the
    native loop agree with the oracle; an unscheduled loop (direct launches)
    too, and the graphs are captured a handful of times, not per stop."""
    from paper_1812_10959_b200.miner import DeviceEngine, run_engine

    cfg = scaled(CONFIGS[2], 30_000, interval=1_500)
    indptr, indices = generate_csr(cfg)
    db = dic.BitDatabase.from_csr(indptr, indices, cfg.m)
    p = dic.MiningParams.create(cfg.n, cfg.minsup, interval=cfg.interval)
    seen = {}

    class Recording(DeviceEngine):
        def close(self):
            if self.h:
                seen[self.tag] = self.graph_stats()
            super().close()

    class Graphed(Recording):
        tag = "graphed"

    class Direct(Recording):
        tag = "direct"

        def set_schedule(self, lfirst, llast):  # never declared: every count launches directly
            pass

    tids = db.device_tids()
    native = run_engine(tids, db.n, db.m, p)
    graphed = run_engine(tids, db.n, db.m, p, engine_factory=Graphed)
    direct = run_engine(tids, db.n, db.m, p, engine_factory=Direct)
    want = O.mine(db.rows, cfg.m, cfg.minsup, interval=cfg.interval, threads=8)
    for res in (native, graphed, direct):
        assert [(f.mask, f.size, f.support) for f in res.frequent] == want.frequent
        assert stats(res) == stats(native)
    cap, launches = seen["graphed"]
    assert 2 <= cap <= 40 and launches > 4 * cap
    cap_d, launches_d = seen["direct"]
    assert launches_d > 0  # the checkpoint half is a graph either way
