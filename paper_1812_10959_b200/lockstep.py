"""Several sharded engines driven in lockstep inside ONE process on ONE GPU.

A sharded run keeps one device engine per
rank, each over its chunk-sliced local rows (sharding.py), and sums every
stop's slot-indexed counts across ranks between the count and checkpoint
halves.  That sum is only right if every rank holds the SAME slot layout —
the replicated state machine must really be replicated (the reference reduces
per record, engine.py:268-270).  This driver runs G engines side by side on
one device and does the cross-rank sum itself (device adds of their delta
buffers and pair triangles), so the sharded trajectory — slot layouts,
per-stop statuses, final results — can be checked bit-exactly against the
oracle without G GPUs.  No collective library is involved: it is the
reduction's arithmetic, not its transport, that is under test here.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from .config import MiningParams
from .miner import DeviceEngine, sorted_frequent
from .phases import MiningResult, MiningStats
from .sharding import ShardPlan


@dataclass
class LockstepInfo:
    world: int
    stops: int = 0
    replays: int = 0
    layouts_checked: int = 0
    statuses: list[dict] = field(default_factory=list)


def local_csr(indptr: np.ndarray, indices: np.ndarray, ranges: list[tuple[int, int]]) -> tuple[np.ndarray, np.ndarray]:
    """CSR of the global rows [b, b + len) of every range, concatenated (a rank's local rows)."""
    indptr = np.asarray(indptr, dtype=np.int64)
    parts, lens = [], []
    for b, ln in ranges:
        p0, p1 = int(indptr[b]), int(indptr[b + ln])
        parts.append(indices[p0:p1])
        lens.append(np.diff(indptr[b:b + ln + 1]))
    lp = np.concatenate([np.zeros(1, np.int64)] + [np.asarray(x, np.int64) for x in lens])
    return np.cumsum(lp), (np.concatenate(parts) if parts else indices[:0])


def _bucket_dump(eng: DeviceEngine, kmax: int) -> list[tuple[np.ndarray, np.ndarray]]:
    return [eng.bucket(k) for k in range(2, kmax + 1)]


def mine_lockstep(shards, params: MiningParams, *, prune_bound: bool = True, check_layout: bool = True,
                  max_size: int = 12) -> tuple[MiningResult, LockstepInfo]:
    """DIC over G local shards (BitDatabases of chunk-sliced rows, rank order)
    with G engines in lockstep; raises AssertionError at the first stop where
    two engines disagree (status, or — with ``check_layout`` — any bucket's
    record ids / item lists)."""
    import torch

    G = len(shards)
    t0 = time.perf_counter()
    info = LockstepInfo(world=G)
    plans = [ShardPlan.for_params(params, G, r) for r in range(G)]
    chunks = [p.local_chunks() for p in plans]
    for r, db in enumerate(shards):
        if db.n != plans[r].local_rows():
            raise ValueError(f"shard {r} holds {db.n} rows, the plan gives it {plans[r].local_rows()}")
    engs = [DeviceEngine(db.device_tids(), db.n, db.m, params, prune_bound) for db in shards]
    try:
        counts = [e.item_counts() for e in engs]
        total = torch.stack(counts).sum(0)
        seeds = [e.seed(total) for e in engs]
        assert all(s == seeds[0] for s in seeds), f"seeding differs across ranks: {seeds}"
        stats = MiningStats()
        stats.candidates_generated = stats.peak_dashed = seeds[0][1]
        scanned = params.n
        live = seeds[0][1]
        stop = 0
        while live:
            stop = stop + 1 if stop < params.intervals_per_pass else 1
            first, last = params.chunk_bounds(stop)
            for r, e in enumerate(engs):
                e.issue_count(*chunks[r][stop - 1])
            # the cross-rank reduction: slot-indexed sums
            for view in ("delta", "pair_counts"):
                bufs = [getattr(e, view)() for e in engs]
                lens = {int(b.numel()) for b in bufs}
                assert len(lens) == 1, f"{view} lengths differ across ranks: {lens}"
                if bufs[0].numel():
                    s = torch.stack(bufs).sum(0)
                    for b in bufs:
                        b.copy_(s)
            seqs = [e.issue_checkpoint() for e in engs]
            polled = [e.poll(q) for e, q in zip(engs, seqs)]
            sts = [{f: getattr(st, f) for f, _ in type(st)._fields_} for st, _ in polled]
            reps = {rep for _, rep in polled}
            assert all(s == sts[0] for s in sts), f"stop {info.stops}: statuses differ across ranks: {sts}"
            assert len(reps) == 1, f"stop {info.stops}: replay decisions differ"
            info.replays += int(polled[0][1])
            if check_layout:
                dumps = [_bucket_dump(e, max_size) for e in engs]
                for r in range(1, G):
                    for k, ((ra, ia), (rb, ib)) in enumerate(zip(dumps[0], dumps[r]), start=2):
                        assert np.array_equal(ra, rb) and np.array_equal(ia, ib), \
                            f"stop {info.stops}: bucket {k} layout differs between rank 0 and rank {r}"
                info.layouts_checked += 1
            st = sts[0]
            info.statuses.append(st)
            info.stops += 1
            stats.interval_counts += st["dashed_at_start"]
            scanned += last - first + 1
            stats.candidates_pruned += st["pruned"]
            stats.candidates_generated += st["inserted"]
            stats.peak_dashed = max(stats.peak_dashed, st["dashed_peak"])
            live = st["dashed_at_end"]
        results = [e.frequent() for e in engs]
        for r in range(1, G):
            for a, b in zip(results[0], results[r]):
                assert np.array_equal(a, b), f"final results differ between rank 0 and rank {r}"
        frequent = sorted_frequent(*results[0], presorted=True)
    finally:
        for e in engs:
            e.close()
    torch.cuda.synchronize()
    stats.db_passes = scanned / params.n
    stats.wall_time_s = time.perf_counter() - t0
    return MiningResult(frequent=frequent, stats=stats), info
