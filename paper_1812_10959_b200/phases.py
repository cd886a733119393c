"""The DIC stop-boundary phases on a host ItemsetCatalog.

Same names, signatures, state transitions, stats and error behaviour as the
reference's phase functions (/root/reference/pkg/src/dicmine/engine.py:
105-390).  The arithmetic runs on the GPU: singleton counts through
dic_item_support, every dashed itemset's chunk count through
dic_count_support (one launch per itemset size), and make_candidates' join
+ immediate-subset test through dic_candidate_admission.  The host keeps the
catalog (Python records, the reference's API objects) and applies the
transitions in the reference's order, so an audit trail matches it
transition for transition.  ``threads`` / ``pool`` / ``kernel`` are
accepted for signature compatibility; there is one (GPU) kernel.
"""

from __future__ import annotations

from collections import defaultdict
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

from . import bits
from .bitmap import BitDatabase
from .catalog import CountedItemset, ItemsetCatalog, Shape, TransitionAudit
from .config import MiningParams


class FrequentItemset(NamedTuple):
    mask: int
    size: int
    support: int


@dataclass
class MiningStats:
    """Run counters (engine.py:76-85); identical for every engine and GPU count."""

    db_passes: float = 0.0
    peak_dashed: int = 0
    candidates_generated: int = 0
    candidates_pruned: int = 0
    interval_counts: int = 0
    wall_time_s: float = 0.0


@dataclass(frozen=True)
class MiningResult:
    frequent: tuple[FrequentItemset, ...]
    stats: MiningStats

    def as_dict(self) -> dict[int, int]:
        return {f.mask: f.support for f in self.frequent}


def _torch():
    import torch

    return torch


def _counts_over(db: BitDatabase, first: int, last: int, masks: list[int]) -> list[int]:
    """Exact chunk counts of ``masks`` (any sizes) via dic_count_support."""
    from . import device as D

    torch = _torch()
    by_size: dict[int, list[int]] = defaultdict(list)
    for pos, mk in enumerate(masks):
        by_size[int(mk).bit_count()].append(pos)
    out = [0] * len(masks)
    tids = db.device_tids()
    for k, positions in by_size.items():
        if k == 0:
            # the empty itemset is contained in every row of the chunk
            for p in positions:
                out[p] = last - first + 1
            continue
        items = bits.masks_to_items([masks[p] for p in positions], k)
        dev = torch.from_numpy(items.view(np.int16)).cuda()
        got = D.count_support(tids, db.n, db.m, first, last, dev).cpu().numpy()
        for p, c in zip(positions, got.tolist()):
            out[p] = c
    return out


def first_pass(catalog: ItemsetCatalog, db: BitDatabase, params: MiningParams, *, kernel: str = "numpy",
               pool=None, threads: int = 1, audit: TransitionAudit | None = None,
               stats: MiningStats | None = None) -> list[int]:
    """Count every singleton over the whole database, finalize them, seed all
    frequent pairs as dashed circles.  Returns the frequent singleton masks."""
    from . import device as D

    singles = [CountedItemset.fresh(1 << i) for i in range(db.m)]
    for rec in singles:
        if audit is not None:
            audit.record(rec.mask, None, Shape.DASHED_CIRCLE)
        catalog.register(rec)
    counts = D.item_support(db.device_tids(), db.n, db.m, 0, db.n - 1).cpu().numpy()
    need = params.min_support_count
    for rec, c in zip(singles, counts.tolist()):
        rec.support = c
        rec.intervals_counted = params.intervals_per_pass
        if c >= need:
            catalog.transition(rec, Shape.DASHED_BOX, audit)
            catalog.transition(rec, Shape.SOLID_BOX, audit)
        else:
            catalog.transition(rec, Shape.SOLID_CIRCLE, audit)
        catalog.solid.append(rec)
    level1 = [rec.mask for rec in singles if rec.shape is Shape.SOLID_BOX]
    for a, x in enumerate(level1):
        for y in level1[a + 1:]:
            catalog.add_candidate(x | y, audit)
    if stats is not None:
        stats.candidates_generated += len(catalog.dashed)
        stats.peak_dashed = max(stats.peak_dashed, len(catalog.dashed))
    return level1


def count_support_interval(catalog: ItemsetCatalog, db: BitDatabase, first: int, last: int, threads: int = 1, *,
                           pool=None, kernel: str = "numpy") -> None:
    """support += exact count over rows [first, last]; intervals_counted += 1."""
    if not (0 <= first <= last < db.n):
        raise ValueError(f"chunk [{first}, {last}] outside database of {db.n} rows")
    recs = catalog.dashed
    if not recs:
        return
    inc = _counts_over(db, first, last, [r.mask for r in recs])
    for rec, c in zip(recs, inc):
        rec.support += c
        rec.intervals_counted += 1


def prune(catalog: ItemsetCatalog, params: MiningParams, *, bound_enabled: bool = True,
          audit: TransitionAudit | None = None, stats: MiningStats | None = None) -> list[CountedItemset]:
    """Promote circles that reached the threshold; discard (with their circle
    supersets) circles that can no longer reach it.  Returns the promoted."""
    need = params.min_support_count
    full = params.intervals_per_pass
    promoted: list[CountedItemset] = []
    for rec in catalog.dashed:
        if rec.shape is not Shape.DASHED_CIRCLE:
            continue
        if rec.support >= need:
            catalog.transition(rec, Shape.DASHED_BOX, audit)
            promoted.append(rec)
            continue
        if not bound_enabled or rec.intervals_counted >= full:
            continue  # fully counted circles belong to check_full_pass
        best_case = rec.support + params.interval * (full - rec.intervals_counted)
        if best_case >= need:
            continue
        catalog.transition(rec, Shape.NIL, audit)
        if stats is not None:
            stats.candidates_pruned += 1
        for other in catalog.dashed:
            if other.shape is Shape.DASHED_CIRCLE and bits.contains(rec.mask, other.mask):
                catalog.transition(other, Shape.NIL, audit)
                if stats is not None:
                    stats.candidates_pruned += 1
    catalog.compact_dashed()
    return promoted


def make_candidates(catalog: ItemsetCatalog, params: MiningParams, *,
                    frontier: list[CountedItemset] | None = None, level1: list[int] | None = None,
                    audit: TransitionAudit | None = None, stats: MiningStats | None = None) -> int:
    """Join box sources with frequent items; admit a join when it is new and
    every immediate subset is a box.  The join/subset test runs on the GPU;
    insertion follows the reference's (source, item) order with
    first-occurrence dedup.  Returns the number of candidates inserted."""
    from . import device as D

    torch = _torch()
    if level1 is None:
        level1 = sorted(r.mask for r in catalog.known.values() if r.size == 1 and r.shape.is_box)
    if frontier is None:
        sources = [r for r in list(catalog.dashed) + catalog.solid if r.shape.is_box]
    else:
        sources = [r for r in frontier if r.shape.is_box]
    inserted = 0
    if sources and level1:
        one_items = []
        for one in level1:
            if int(one).bit_count() != 1:
                raise ValueError(f"level1 entry {one:#x} is not a single item")
            one_items.append(int(one).bit_length() - 1)
        known = list(catalog.known.keys())
        boxes = [mk for mk, r in catalog.known.items() if r.shape.is_box]
        width = max([mk.bit_length() for mk in known] + [s.mask.bit_length() for s in sources] + one_items + [1])
        W = bits.words_for(max(width, max(one_items) + 1))
        dev = lambda arr: torch.from_numpy(np.ascontiguousarray(arr)).cuda()  # noqa: E731
        admit = D.candidate_admission(
            dev(bits.masks_to_array([s.mask for s in sources], W)),
            dev(np.asarray(one_items, dtype=np.int32)),
            dev(bits.masks_to_array(known, W)),
            dev(bits.masks_to_array(boxes, W)),
        ).cpu().numpy()
        rows, cols = np.nonzero(admit)
        for s, l in zip(rows.tolist(), cols.tolist()):
            cand = sources[s].mask | level1[l]
            if cand in catalog.known:  # an earlier join of this call made it
                continue
            catalog.add_candidate(cand, audit)
            inserted += 1
    if stats is not None:
        stats.candidates_generated += inserted
    return inserted


def check_full_pass(catalog: ItemsetCatalog, params: MiningParams, *, audit: TransitionAudit | None = None,
                    stats: MiningStats | None = None) -> int:
    """Dashed itemsets counted over a full pass become solid boxes / circles."""
    done = 0
    need = params.min_support_count
    for rec in catalog.dashed:
        if rec.shape.is_dashed and rec.intervals_counted == params.intervals_per_pass:
            catalog.transition(rec, Shape.SOLID_BOX if rec.support >= need else Shape.SOLID_CIRCLE, audit)
            catalog.solid.append(rec)
            done += 1
    catalog.compact_dashed()
    return done
