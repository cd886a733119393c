"""The replicated state machine really is replicated.

A sharded run reduces every stop's counts SLOT BY SLOT across ranks
(DESIGN.md §9), so every rank must give the same itemset the same bucket
slot.  Two properties are checked on one GPU:

1. Layout determinism: the same run with different grid sizes for the
   checkpoint kernel (DIC_CKPT_CTAS) — i.e. a different work split and
   different thread timing in every atomic — leaves byte-identical buckets
   (record ids and item lists) after every stop.
2. Lockstep emulation of G ranks (lockstep.py): G engines over the
   chunk-sliced shards of one database, their delta buffers and pair
   triangles summed slot by slot between the count and checkpoint halves,
   exactly the arithmetic of the NCCL / fused reductions.  Every stop's
   status and every bucket must agree across the engines, and the result
   (frequent itemsets, supports, every MiningStats counter) must equal the
   CPU oracle's.  This is the reference's per-record reduction
   (engine.py:268-270) made slot-wise.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

import paper_1812_10959_b200 as dic
from oracle import oracle as O
from paper_1812_10959_b200.lockstep import mine_lockstep
from paper_1812_10959_b200.miner import DeviceEngine
from paper_1812_10959_b200.workloads import CONFIGS, generate_csr, scaled
from tests.golden_util import load_config_golden

pytestmark = pytest.mark.gpu
THREADS = os.cpu_count() or 1


def _stats(s) -> tuple:
    return (s.db_passes, s.peak_dashed, s.candidates_generated, s.candidates_pruned, s.interval_counts)


def _oracle_tuple(o) -> tuple:
    return (o.db_passes, o.peak_dashed, o.candidates_generated, o.candidates_pruned, o.interval_counts)


def _step_dumps(db, params, kmax: int = 10) -> list:
    """Drive one engine stop by stop; bucket dumps after every stop."""
    eng = DeviceEngine(db.device_tids(), db.n, db.m, params, True)
    dumps = []
    try:
        eng.seed(eng.item_counts())
        live, stop = 1, 0
        while live:
            stop = stop + 1 if stop < params.intervals_per_pass else 1
            eng.issue_count(*params.chunk_bounds(stop))
            st, _ = eng.poll(eng.issue_checkpoint())
            dumps.append([eng.bucket(k) for k in range(2, kmax + 1)])
            live = st.dashed_at_end
    finally:
        eng.close()
    return dumps


@pytest.mark.parametrize("idx,n,interval", [(1, 10_000, 1_000), (3, 100_000, 10_000), (4, 40_000, 400)])
def test_layout_independent_of_grid(monkeypatch, idx, n, interval):
    cfg = scaled(CONFIGS[idx], n, interval=interval)
    indptr, indices = generate_csr(cfg)
    db = dic.BitDatabase.from_csr(indptr, indices, cfg.m)
    params = dic.MiningParams.create(cfg.n, cfg.minsup, interval=cfg.interval)
    runs = []
    for grid in ("7", "148", "61"):
        monkeypatch.setenv("DIC_CKPT_CTAS", grid)
        runs.append(_step_dumps(db, params))
    assert len(runs[0]) == len(runs[1]) == len(runs[2])
    new = 0
    for s, (a, b, c) in enumerate(zip(*runs)):
        for k, ((ra, ia), (rb, ib), (rc, ic)) in enumerate(zip(a, b, c), start=2):
            assert np.array_equal(ra, rb) and np.array_equal(ra, rc), f"stop {s} bucket {k}: record ids differ"
            assert np.array_equal(ia, ib) and np.array_equal(ia, ic), f"stop {s} bucket {k}: items differ"
            if k >= 3:
                new = max(new, len(ra))
    assert new > 0, "the run must create join candidates for the check to mean anything"


def test_new_candidates_in_canonical_order():
    """Within a stop, joins are committed in (size, items ascending) order."""
    cfg = scaled(CONFIGS[1], 10_000, interval=1_000)
    indptr, indices = generate_csr(cfg)
    db = dic.BitDatabase.from_csr(indptr, indices, cfg.m)
    params = dic.MiningParams.create(cfg.n, cfg.minsup, interval=cfg.interval)
    seen = -1
    checked = 0
    for dump in _step_dumps(db, params):
        # records created at this stop: ids above every id seen before; all
        # of them are live (just inserted), so all are in the buckets
        fresh = sorted((rid, k, tuple(it)) for k, (rec, items) in enumerate(dump, start=2)
                       for rid, it in zip(rec.tolist(), items.tolist()) if rid > seen)
        keys = [(k, it) for _, k, it in fresh]
        assert keys == sorted(keys), "new candidates not numbered in (size, items) order"
        if fresh:
            assert [r for r, _, _ in fresh] == list(range(fresh[0][0], fresh[0][0] + len(fresh)))
            seen = fresh[-1][0]
            checked += len(fresh)
    assert checked > 1000


def _shards(cfg, params, world: int):
    out = []
    for r in range(world):
        plan = dic.ShardPlan.for_params(params, world, r)
        ip, ix = generate_csr(cfg, ranges=plan.ranges())
        out.append(dic.BitDatabase.from_csr(ip, ix, cfg.m))
    return out


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("idx,n,interval", [(1, 10_000, 1_000), (3, 100_000, 10_000), (4, 40_000, 400)])
def test_lockstep_matches_oracle(idx, n, interval, world):
    cfg = scaled(CONFIGS[idx], n, interval=interval)
    params = dic.MiningParams.create(cfg.n, cfg.minsup, interval=cfg.interval)
    res, info = mine_lockstep(_shards(cfg, params, world), params)
    assert info.layouts_checked == info.stops > 0
    ip, ix = generate_csr(cfg)
    from tests.golden_util import rows_from_csr

    want = O.mine(rows_from_csr(ip, ix, cfg.m), cfg.m, cfg.minsup, interval=cfg.interval, threads=THREADS)
    assert [(f.mask, f.size, f.support) for f in res.frequent] == want.frequent
    assert _stats(res.stats) == _oracle_tuple(want)


def test_lockstep_cfg2_full_matches_reference_golden():
    """BASELINE cfg2 at full size (100k x 1000, 354k seeded pairs) over 4
    lockstep ranks against the fixture the reference itself produced."""
    cfg = CONFIGS[2]
    g = load_config_golden(2)
    params = dic.MiningParams.create(cfg.n, cfg.minsup, interval=cfg.interval)
    res, info = mine_lockstep(_shards(cfg, params, 4), params, check_layout=False)
    assert [(f.mask, f.support) for f in res.frequent] == g.pairs
    st = g.stats
    assert _stats(res.stats) == (st["db_passes"], st["peak_dashed"], st["candidates_generated"],
                                 st["candidates_pruned"], st["interval_counts"])


def test_large_stop_multi_run_commit_is_canonical_and_exact(monkeypatch):
    """A dense database whose stops admit more than one sort run (2,048) of
    new candidates at once: the run-merging commit path, under two grid
    sizes and over 2 lockstep ranks, against the oracle."""
    rng = np.random.default_rng(11)
    n, m = 3000, 24
    rows = np.zeros((n, 1), dtype=np.uint64)
    bits = rng.random((n, m)) < 0.6
    for i in range(m):
        rows[:, 0] |= bits[:, i].astype(np.uint64) << np.uint64(i)
    params = dic.MiningParams.create(n, 0.15, interval=300)
    ints = [int(x) for x in rows[:, 0]]
    shards = []
    for r in range(2):
        plan = dic.ShardPlan.for_params(params, 2, r)
        shards.append(dic.BitDatabase([ints[b + j] for b, ln in plan.ranges() for j in range(ln)], m=m))
    res, info = mine_lockstep(shards, params)
    assert max(st["inserted"] for st in info.statuses) > 2048
    want = O.mine(rows, m, 0.15, interval=300, threads=THREADS)
    assert [(f.mask, f.size, f.support) for f in res.frequent] == want.frequent
    assert _stats(res.stats) == _oracle_tuple(want)
    db = dic.BitDatabase(ints, m=m)
    runs = []
    for grid in ("3", "148"):
        monkeypatch.setenv("DIC_CKPT_CTAS", grid)
        runs.append(_step_dumps(db, params, kmax=8))
    for a, b in zip(*runs):
        for (ra, ia), (rb, ib) in zip(a, b):
            assert np.array_equal(ra, rb) and np.array_equal(ia, ib)
