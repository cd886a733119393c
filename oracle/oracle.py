"""TEST INFRASTRUCTURE ONLY — ctypes front end of the C oracle (dic_oracle.c).

A CPU restatement of the reference `dicmine` engine (see dic_oracle.c for
file:line citations), generalised to W-word masks.  Only tests/, the
smoke() check and bench.py's cpu_baseline / --impl reference leg may use it;
the product package never imports it.
"""

from __future__ import annotations

import ctypes as C
import math
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "liboracle.so"

_lib: C.CDLL | None = None


class OrcStats(C.Structure):
    _fields_ = [
        ("scanned", C.c_int64),
        ("peak_dashed", C.c_int64),
        ("candidates_generated", C.c_int64),
        ("candidates_pruned", C.c_int64),
        ("interval_counts", C.c_int64),
        ("stops", C.c_int64),
    ]


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE), "all"], check=True)
    return LIB


def load() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        lib = C.CDLL(str(LIB))
        vp, i64 = C.c_void_p, C.c_int64
        lib.orc_count_block.restype = i64
        lib.orc_count_block.argtypes = [vp, C.c_int, i64, i64, vp]
        lib.orc_count_many.restype = None
        lib.orc_count_many.argtypes = [vp, C.c_int, i64, i64, vp, i64, vp, C.c_int]
        lib.orc_item_support.restype = None
        lib.orc_item_support.argtypes = [vp, i64, C.c_int, C.c_int, vp]
        lib.orc_mine.restype = vp
        lib.orc_mine.argtypes = [vp, i64, C.c_int, C.c_int, i64, i64, C.c_int, C.c_int, i64, C.POINTER(OrcStats)]
        lib.orc_result_count.restype = i64
        lib.orc_result_count.argtypes = [vp]
        lib.orc_result_get.restype = None
        lib.orc_result_get.argtypes = [vp, vp, vp, vp]
        lib.orc_result_free.restype = None
        lib.orc_result_free.argtypes = [vp]
        lib.orc_bernoulli_rows.restype = None
        lib.orc_bernoulli_rows.argtypes = [i64, i64, C.c_int, C.c_double, C.c_uint64, vp]
        lib.orc_bernoulli_cols.restype = C.c_int
        lib.orc_bernoulli_cols.argtypes = [i64, C.c_int, C.c_double, C.c_uint64, vp, C.c_int]
        lib.orc_count_cols.restype = C.c_int
        lib.orc_count_cols.argtypes = [vp, i64, vp, vp, i64, C.c_int, vp, C.c_int]
        _lib = lib
    return _lib


def rows_from_ints(masks, m: int | None = None) -> np.ndarray:
    """Python-int masks -> uint64 [n][W] (LSW first)."""
    masks = [int(x) for x in masks]
    if m is None:
        m = max(max((x.bit_length() for x in masks), default=1), 1)
    W = (m + 63) // 64
    out = np.zeros((len(masks), W), dtype=np.uint64)
    for j, x in enumerate(masks):
        for w in range(W):
            out[j, w] = (x >> (64 * w)) & 0xFFFFFFFFFFFFFFFF
    return out


def mask_from_words(words) -> int:
    x = 0
    for w, v in enumerate(words):
        x |= int(v) << (64 * w)
    return x


def words_from_mask(mask: int, W: int) -> np.ndarray:
    return np.array([(mask >> (64 * w)) & 0xFFFFFFFFFFFFFFFF for w in range(W)], dtype=np.uint64)


def absolute_support(minsup: float, n: int) -> int:
    """params.py:17-19 — the float ceil is part of the semantics."""
    return math.ceil(minsup * n)


def count_block(rows: np.ndarray, first: int, last: int, mask: int) -> int:
    rows = np.ascontiguousarray(rows, dtype=np.uint64)
    W = rows.shape[1]
    mk = words_from_mask(mask, W)
    return int(load().orc_count_block(rows.ctypes.data, W, first, last, mk.ctypes.data))


def count_many(rows: np.ndarray, first: int, last: int, masks: np.ndarray, threads: int = 1) -> np.ndarray:
    rows = np.ascontiguousarray(rows, dtype=np.uint64)
    masks = np.ascontiguousarray(masks, dtype=np.uint64)
    out = np.zeros(masks.shape[0], dtype=np.int64)
    load().orc_count_many(rows.ctypes.data, rows.shape[1], first, last, masks.ctypes.data, masks.shape[0],
                          out.ctypes.data, threads)
    return out


def item_support(rows: np.ndarray, m: int) -> np.ndarray:
    rows = np.ascontiguousarray(rows, dtype=np.uint64)
    out = np.zeros(m, dtype=np.int64)
    load().orc_item_support(rows.ctypes.data, rows.shape[0], rows.shape[1], m, out.ctypes.data)
    return out


@dataclass
class OracleRun:
    frequent: list[tuple[int, int, int]]  # (mask, size, support) in (size, mask) order
    db_passes: float
    peak_dashed: int
    candidates_generated: int
    candidates_pruned: int
    interval_counts: int
    stops: int

    def pairs(self) -> dict[int, int]:
        return {m: s for m, _, s in self.frequent}


def mine(rows: np.ndarray, m: int, minsup: float, interval: int | None = None, prune_bound: bool = True,
         threads: int = 1, max_stops: int = -1, need: int | None = None) -> OracleRun:
    """DIC over rows uint64 [n][W] with the reference's defaults
    (interval = ceil(n/2), params.py:9-14)."""
    rows = np.ascontiguousarray(rows, dtype=np.uint64)
    n, W = rows.shape
    if interval is None:
        interval = n if n < 2 else (n + 1) // 2
    if need is None:
        need = absolute_support(minsup, n)
    st = OrcStats()
    lib = load()
    h = lib.orc_mine(rows.ctypes.data, n, W, m, need, interval, 1 if prune_bound else 0, threads, max_stops,
                     C.byref(st))
    if not h:
        raise MemoryError("oracle out of memory")
    try:
        F = lib.orc_result_count(h)
        masks = np.zeros((max(F, 1), W), dtype=np.uint64)
        sizes = np.zeros(max(F, 1), dtype=np.int32)
        sups = np.zeros(max(F, 1), dtype=np.int64)
        lib.orc_result_get(h, masks.ctypes.data, sizes.ctypes.data, sups.ctypes.data)
    finally:
        lib.orc_result_free(h)
    freq = [(mask_from_words(masks[i]), int(sizes[i]), int(sups[i])) for i in range(F)]
    return OracleRun(freq, st.scanned / n, st.peak_dashed, st.candidates_generated, st.candidates_pruned,
                     st.interval_counts, st.stops)


# ---------------------------------------------------------------- cfg5 (cfg5.c)
def bernoulli_rows(r0: int, nrows: int, m: int, p: float, seed: int) -> np.ndarray:
    """Rows [r0, r0 + nrows) of the cfg5 bitmap, uint64 [nrows][W] (the device
    generator's hash restated on the host)."""
    W = (m + 63) // 64
    out = np.zeros((nrows, W), dtype=np.uint64)
    load().orc_bernoulli_rows(r0, nrows, m, p, seed, out.ctypes.data)
    return out


def bernoulli_cols(n: int, m: int, p: float, seed: int, threads: int = 1) -> np.ndarray:
    """The whole cfg5 bitmap column-wise: uint64 [m][ceil(n/64)], item i's bits of rows 64w..64w+63 in word w."""
    cols = np.empty((m, (n + 63) // 64), dtype=np.uint64)
    if load().orc_bernoulli_cols(n, m, p, seed, cols.ctypes.data, threads) != 0:
        raise ValueError("orc_bernoulli_cols: bad arguments")
    return cols


def count_cols(cols: np.ndarray, items: np.ndarray, ks: np.ndarray, threads: int = 1) -> np.ndarray:
    """Support of every candidate (items[c][:ks[c]]) over a column bitmap."""
    cols = np.ascontiguousarray(cols, dtype=np.uint64)
    items = np.ascontiguousarray(items, dtype=np.uint16)
    ks = np.ascontiguousarray(ks, dtype=np.int32)
    out = np.zeros(len(ks), dtype=np.int64)
    load().orc_count_cols(cols.ctypes.data, cols.shape[1], items.ctypes.data, ks.ctypes.data, len(ks),
                          items.shape[1], out.ctypes.data, threads)
    return out
