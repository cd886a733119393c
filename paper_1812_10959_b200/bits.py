"""Itemset masks as Python ints (any width) and their W-word device form.

The public helpers keep the signatures of the reference's bitops.py
(/root/reference/pkg/src/dicmine/bitops.py:24-74): bit p of a mask <=> item
p.  Differences: masks are not capped at 64 bits (the reference's MAX_ITEMS,
bitops.py:18) — the universe bound is enforced by BitDatabase — so
encode_transaction only rejects negative ids.  The word helpers convert to
and from the device layout (W little-endian uint64 words, LSW first).
"""

from __future__ import annotations

from typing import Iterable, Iterator

import numpy as np

from .exceptions import ItemOutOfRange

WORD = 64
_WMASK = (1 << WORD) - 1


def encode_transaction(items: Iterable[int]) -> int:
    """OR of 1 << item over the ids (duplicates collapse)."""
    out = 0
    for it in items:
        it = int(it)
        if it < 0:
            raise ItemOutOfRange(it)
        out |= 1 << it
    return out


def contains(itemset: int, transaction: int) -> bool:
    """Subset test: every item of ``itemset`` is in ``transaction``."""
    return itemset & ~transaction == 0


def join(a: int, b: int) -> int:
    return a | b


def cardinality(mask: int) -> int:
    return int(mask).bit_count()


def items_of(mask: int) -> Iterator[int]:
    """Item ids of ``mask``, ascending."""
    x = int(mask)
    while x:
        low = x & -x
        yield low.bit_length() - 1
        x ^= low


def immediate_subsets(mask: int) -> Iterator[int]:
    """Masks with exactly one item of ``mask`` removed (lowest item first)."""
    for it in items_of(mask):
        yield mask ^ (1 << it)


def popcounts(masks: np.ndarray) -> np.ndarray:
    arr = np.asarray(masks, dtype=np.uint64)
    out = np.bitwise_count(arr)
    return out if arr.ndim == 1 else out.sum(axis=-1)


def words_for(m: int) -> int:
    return max(1, (int(m) + WORD - 1) // WORD)


def to_words(mask: int, W: int) -> list[int]:
    return [(mask >> (WORD * w)) & _WMASK for w in range(W)]


def from_words(words) -> int:
    out = 0
    for w, v in enumerate(words):
        out |= int(v) << (WORD * w)
    return out


def masks_to_array(masks: Iterable[int], W: int) -> np.ndarray:
    """Python-int masks -> uint64 [len][W]."""
    ms = [int(x) for x in masks]
    out = np.zeros((len(ms), W), dtype=np.uint64)
    if W == 1:
        out[:, 0] = np.array(ms, dtype=np.uint64) if ms else out[:, 0]
        return out
    for w in range(W):
        out[:, w] = np.array([(x >> (WORD * w)) & _WMASK for x in ms], dtype=np.uint64)
    return out


def array_to_masks(arr: np.ndarray) -> list[int]:
    """uint64 [len][W] (LSW first) -> Python ints."""
    a = np.asarray(arr, dtype=np.uint64)
    if a.ndim == 1:
        return a.tolist()
    if a.shape[1] == 1:
        return a[:, 0].tolist()
    raw = np.ascontiguousarray(a, dtype="<u8").tobytes()
    step = a.shape[1] * 8
    fb = int.from_bytes
    return [fb(raw[i:i + step], "little") for i in range(0, len(raw), step)]


def masks_to_items(masks: list[int], k: int) -> np.ndarray:
    """Size-k masks -> uint16 [len][k] ascending item ids (count-kernel input)."""
    out = np.empty((len(masks), k), dtype=np.uint16)
    for c, mk in enumerate(masks):
        its = list(items_of(mk))
        if len(its) != k:
            raise ValueError(f"mask {mk:#x} has {len(its)} items, expected {k}")
        out[c] = its
    return out
