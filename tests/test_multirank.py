"""World-size-2 gloo tests of the multi-GPU path on CPU.

The sharded driver (miner.run_engine with a ShardPlan) runs on two gloo
ranks with a CPU stand-in engine whose counts come from the oracle over the
rank's LOCAL rows; the per-stop count deltas travel through a real
torch.distributed all_reduce.  The result and every stat must equal the
single-process oracle run: this pins the chunk-sliced partition, the local
chunk bounds and the delta-allreduce protocol (allreducing supports instead
of deltas would multiply earlier chunks by G)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_1812_10959_b200 import _abi, bits
from paper_1812_10959_b200.catalog import ItemsetCatalog, Shape
from paper_1812_10959_b200.config import MiningParams
from paper_1812_10959_b200.sharding import ShardPlan


class CpuStandInEngine:
    """Host re-statement of the device engine's contract (test only)."""

    rows: np.ndarray = None  # local rows, set per rank

    def __init__(self, tids, n_local, m, params, prune_bound):
        self.m, self.p, self.bound = m, params, prune_bound
        self.cat = ItemsetCatalog()
        self.level1: list[int] = []
        self._delta = None

    def close(self):
        pass

    def item_counts(self):
        return torch.from_numpy(O.item_support(self.rows, self.m))

    def seed(self, counts):
        need, full = self.p.min_support_count, self.p.intervals_per_pass
        for i, c in enumerate(counts.tolist()):
            rec = self.cat.add_candidate(1 << i)
            self.cat.dashed.pop()
            rec.support, rec.intervals_counted = c, full
            rec.shape = Shape.SOLID_BOX if c >= need else Shape.SOLID_CIRCLE
            self.cat.solid.append(rec)
            if c >= need:
                self.level1.append(i)
        for a, x in enumerate(self.level1):
            for y in self.level1[a + 1:]:
                self.cat.add_candidate((1 << x) | (1 << y))
        return len(self.level1), len(self.cat.dashed)

    def count(self, lfirst, llast):
        W = self.rows.shape[1]
        masks = bits.masks_to_array([r.mask for r in self.cat.dashed], W)
        inc = O.count_many(self.rows, lfirst, llast, masks) if llast >= lfirst else np.zeros(len(masks), np.int64)
        self._delta = torch.from_numpy(inc)

    def delta(self):
        return self._delta

    def pair_counts(self):
        return torch.empty(0, dtype=torch.int64)

    def checkpoint(self):
        st = _abi.StopStatus()
        st.dashed_at_start = len(self.cat.dashed)
        for rec, d in zip(self.cat.dashed, self._delta.tolist()):
            rec.support += d
            rec.intervals_counted += 1
        need, full, M = self.p.min_support_count, self.p.intervals_per_pass, self.p.interval
        front = []
        for rec in self.cat.dashed:
            if rec.shape is Shape.DASHED_CIRCLE:
                if rec.support >= need:
                    rec.shape = Shape.DASHED_BOX
                    front.append(rec)
                elif self.bound and rec.intervals_counted < full and rec.support + M * (full - rec.intervals_counted) < need:
                    rec.shape = Shape.NIL
                    st.pruned += 1
        self.cat.compact_dashed()
        for src in front:
            for one in self.level1:
                cand = src.mask | (1 << one)
                if cand == src.mask or cand in self.cat.known:
                    continue
                subs = [self.cat.known.get(cand ^ (1 << it)) for it in bits.items_of(cand)]
                if all(r is not None and r.shape.is_box for r in subs):
                    self.cat.add_candidate(cand)
                    st.inserted += 1
        st.promoted = len(front)
        st.dashed_peak = len(self.cat.dashed)
        for rec in self.cat.dashed:
            if rec.intervals_counted == full:
                rec.shape = Shape.SOLID_BOX if rec.support >= need else Shape.SOLID_CIRCLE
                self.cat.solid.append(rec)
                st.finalized += 1
        self.cat.compact_dashed()
        st.dashed_at_end = len(self.cat.dashed)
        return st

    # pipelined protocol of DeviceEngine (statuses are ready immediately here)
    def issue_count(self, lfirst, llast):
        self.count(lfirst, llast)

    def issue_checkpoint(self):
        self._done = getattr(self, "_done", [])
        self._done.append(self.checkpoint())
        return len(self._done) - 1

    def poll(self, seq):
        return self._done[seq], False

    def frequent(self):
        recs = [r for r in self.cat.solid if r.shape is Shape.SOLID_BOX]
        W = bits.words_for(self.m)
        return (bits.masks_to_array([r.mask for r in recs], W), np.array([r.size for r in recs], np.int32),
                np.array([r.support for r in recs], np.int64))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, rows, m, minsup, interval, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1812_10959_b200.miner import run_engine

        params = MiningParams.create(rows.shape[0], minsup, interval=interval)
        plan = ShardPlan.for_params(params, world, rank)
        local = np.concatenate([rows[b:b + ln] for b, ln in plan.ranges()]) if plan.local_rows() else rows[:0]
        CpuStandInEngine.rows = np.ascontiguousarray(local)
        res = run_engine(None, local.shape[0], m, params, plan=plan, group=dist.group.WORLD,
                         engine_factory=CpuStandInEngine)
        s = res.stats
        q.put((rank, [(f.mask, f.size, f.support) for f in res.frequent],
               (s.db_passes, s.peak_dashed, s.candidates_generated, s.candidates_pruned, s.interval_counts)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,m,interval,minsup", [(2, 1500, 40, 170, 0.05), (2, 997, 130, 97, 0.1),
                                                       (3, 640, 24, 64, 0.2)])
def test_sharded_driver_matches_single_process(world, n, m, interval, minsup):
    rng = np.random.default_rng(n)
    W = bits.words_for(m)
    hot = rng.choice(m, size=7, replace=False)
    rows = np.zeros((n, W), dtype=np.uint64)
    for it in hot:
        on = rng.random(n) < 0.45
        rows[on, it // 64] |= np.uint64(1) << np.uint64(it % 64)
    want = O.mine(rows, m, minsup, interval=interval)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, rows, m, minsup, interval, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    for _, freq, st in got:
        assert freq == want.frequent
        assert st == (want.db_passes, want.peak_dashed, want.candidates_generated, want.candidates_pruned,
                      want.interval_counts)
