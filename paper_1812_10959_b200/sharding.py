"""Chunk-sliced row sharding for multi-GPU DIC.

Rank g of G holds the g-th contiguous 1/G slice of EVERY chunk
[first_s, last_s] (params.py:67-75); its local rows are those slices
concatenated in chunk order.  Local chunk s is therefore one contiguous row
range, the union over ranks of local chunk s is exactly global chunk s, and
the per-stop sum-allreduce of the local counts equals the single-GPU count —
so the state machine (replicated on every rank) and all stats follow the
single-GPU trajectory exactly.  Pure host arithmetic: tested on CPU with
gloo ranks.
"""

from __future__ import annotations

from dataclasses import dataclass

from .config import MiningParams


@dataclass(frozen=True)
class ShardPlan:
    n: int
    interval: int
    world: int
    rank: int

    @classmethod
    def for_params(cls, params: MiningParams, world: int, rank: int) -> "ShardPlan":
        if not 0 <= rank < world:
            raise ValueError(f"rank {rank} outside world of {world}")
        return cls(params.n, params.interval, world, rank)

    @property
    def stop_max(self) -> int:
        return -(-self.n // self.interval)

    def global_chunk(self, stop: int) -> tuple[int, int]:
        lo = (stop - 1) * self.interval
        return lo, min(lo + self.interval, self.n) - 1

    def slice_of(self, stop: int, rank: int | None = None) -> tuple[int, int]:
        """Global rows [begin, begin + length) of chunk ``stop`` held by ``rank``."""
        r = self.rank if rank is None else rank
        first, last = self.global_chunk(stop)
        span = last - first + 1
        b = first + span * r // self.world
        e = first + span * (r + 1) // self.world
        return b, e - b

    def ranges(self, rank: int | None = None) -> list[tuple[int, int]]:
        """Global (begin, length) ranges of this rank's local rows, in local order."""
        return [self.slice_of(s, rank) for s in range(1, self.stop_max + 1)]

    def local_rows(self, rank: int | None = None) -> int:
        return sum(length for _, length in self.ranges(rank))

    def local_chunk(self, stop: int) -> tuple[int, int]:
        """Local inclusive range of chunk ``stop`` (last < first when empty)."""
        off = 0
        for s in range(1, stop):
            off += self.slice_of(s)[1]
        length = self.slice_of(stop)[1]
        return off, off + length - 1

    def local_chunks(self) -> list[tuple[int, int]]:
        out, off = [], 0
        for _, length in self.ranges():
            out.append((off, off + length - 1))
            off += length
        return out
