"""Paths of the cooperative checkpoint kernel (csrc/engine.cu) that the config
goldens reach rarely or not at all, each against the CPU oracle (itemsets,
supports, every MiningStats counter):

* the overflow recovery: a stop whose joins do not fit raises the abort flag
  AFTER its joins claimed temporary hash entries; the host must rebuild the
  index, replay the candidate step and re-issue the skipped stops;
* itemsets of more than 8 items: the mask-only join path, the item lists that
  stop at 8 ids, and the result order sorted on the host;
* stops that run on one CTA and stops that call the grid in, under several grid
  sizes;
* a bucket compacted by the whole grid that is not the pair bucket.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

import paper_1812_10959_b200 as dic
from oracle import oracle as O
from paper_1812_10959_b200.miner import StopTrace, run_engine

pytestmark = pytest.mark.gpu
THREADS = os.cpu_count() or 1


def _rows(bits: np.ndarray) -> np.ndarray:
    n, m = bits.shape
    W = (m + 63) // 64
    rows = np.zeros((n, W), dtype=np.uint64)
    for i in range(m):
        rows[:, i >> 6] |= bits[:, i].astype(np.uint64) << np.uint64(i & 63)
    return rows


def _check(rows: np.ndarray, m: int, minsup: float, interval: int, depth: int = 4) -> StopTrace:
    n = rows.shape[0]
    W = rows.shape[1]
    ints = [sum(int(rows[j, w]) << (64 * w) for w in range(W)) for j in range(n)]
    db = dic.BitDatabase(ints, m=m)
    params = dic.MiningParams.create(n, minsup, interval=interval)
    trace = StopTrace()
    res = run_engine(db.device_tids(), n, m, params, trace=trace, depth=depth)
    want = O.mine(rows, m, minsup, interval=interval, threads=THREADS)
    assert [(f.mask, f.size, f.support) for f in res.frequent] == want.frequent
    s = res.stats
    assert (s.db_passes, s.peak_dashed, s.candidates_generated, s.candidates_pruned, s.interval_counts) == (
        want.db_passes, want.peak_dashed, want.candidates_generated, want.candidates_pruned, want.interval_counts)
    return trace


def test_overflow_replay_with_claimed_entries():
    """Dense rows: stops admit tens of thousands of joins of a new size at
    once, more than the buckets' headroom — the run must replay stops (and
    still equal the oracle: the aborted stops' temporary entries are gone)."""
    rng = np.random.default_rng(5)
    bits = rng.random((4000, 26)) < 0.5
    trace = _check(_rows(bits), 26, 0.04, 400)
    assert trace.native["replays"] > 0, trace.native
    assert max(st["dashed_at_start"] for st in trace.stops) > 32768


@pytest.mark.parametrize("m,group", [(20, 11), (150, 10)])
def test_itemsets_of_more_than_eight_items(m, group):
    """A planted group of 10-11 items present together in most rows: every one
    of its subsets is frequent, up to the whole group (sizes 9+ take the
    mask-only paths; m = 150 makes the masks three words wide)."""
    rng = np.random.default_rng(m)
    n = 2500
    bits = rng.random((n, m)) < 0.03
    planted = rng.choice(m, group, replace=False)
    on = rng.random(n) < 0.7
    bits[np.ix_(on, planted)] = True
    trace = _check(_rows(bits), m, 0.6, 250)
    assert len(trace.stops) > 0


@pytest.mark.parametrize("ctas", ["2", "5", "148"])
def test_single_cta_stops_and_join_in(monkeypatch, ctas):
    """Few live itemsets (every stop below the single-CTA limit) with bursts of
    promotions that need the grid for the joins, under three grid sizes."""
    monkeypatch.setenv("DIC_CKPT_CTAS", ctas)
    rng = np.random.default_rng(17)
    n, m = 6000, 60
    p = rng.beta(2, 5, size=m)
    bits = rng.random((n, m)) < p
    for g in range(6):
        items = rng.choice(m, 5, replace=False)
        on = rng.random(n) < 0.25
        bits[np.ix_(on, items)] = True
    _check(_rows(bits), m, 0.2, 500)


def test_grid_compaction_of_a_large_triple_bucket():
    """More than 16k 3-item candidates die together (the bound prunes them):
    bucket 3 is compacted by the whole grid, not just the pair bucket."""
    rng = np.random.default_rng(23)
    n, m = 12000, 64
    bits = rng.random((n, m)) < 0.33
    # the first rows are much denser: pairs look frequent early, triples are
    # admitted in bulk and most of them fall behind later
    bits[:1500] |= rng.random((1500, m)) < 0.5
    trace = _check(_rows(bits), m, 0.13, 500)
    assert max(st["dashed_at_start"] for st in trace.stops) > 16384


@pytest.mark.parametrize("batch", ["0", "3", "8"])
def test_batches_of_quiet_stops(monkeypatch, batch):
    """The tail of a run goes out in batches of stops (one count launch over the
    next chunks, one single-CTA kernel for their checkpoints); a batch ends
    early when a stop inserts candidates.  Same result for every batch size,
    and batches really are used."""
    monkeypatch.setenv("DIC_BATCH_STOPS", batch)
    rng = np.random.default_rng(29)
    n, m = 20000, 48
    p = rng.beta(2, 6, size=m)
    bits = rng.random((n, m)) < p
    # groups planted in the second half only: their itemsets are promoted (and
    # their supersets inserted) late, in the middle of otherwise quiet stops
    for g in range(5):
        items = rng.choice(m, 4, replace=False)
        on = np.zeros(n, dtype=bool)
        on[n // 2:] = rng.random(n - n // 2) < 0.5
        bits[np.ix_(on, items)] = True
    trace = _check(_rows(bits), m, 0.12, 250)
    if batch == "0":
        assert trace.native["batches"] == 0
    else:
        assert trace.native["batches"] > 0 and trace.native["batched_stops"] > trace.native["batches"]
