"""Option B of INTEGRATION.md: keep the reference `dicmine` package and bind
its counting seam to the B200 C ABI (include/dic_b200.h) with ctypes — the
module a dicmine maintainer would add as `dicmine/_b200.py`.

    import dicmine.engine
    from integration import dicmine_b200 as b200
    b200.install(dicmine.engine)      # engine._count_block + engine.count_support_interval

`_run` resolves `count_support_interval` (engine.py:429) and `first_pass`
resolves `_count_block` (engine.py:146) as module globals at call time, so the
reference's own checkpoint loop then counts on the GPU while everything else
(catalog, prune, make_candidates, check_full_pass, stats) stays the
reference's.  Masks wider than 64 bits work when the database exposes
`masks` as uint64 [n][W] (the reference itself stops at 64 items).

No torch: device buffers come from the library's own allocator calls
(cudart via ctypes), so the binding needs only the .so and numpy.
"""

from __future__ import annotations

import ctypes as C
import os
from collections import defaultdict
from pathlib import Path

import numpy as np

_LIB = Path(os.environ.get("DIC_LIB") or Path(__file__).resolve().parent.parent / "paper_1812_10959_b200" / "lib" /
            "libdicb200.so")
_lib = None
_cudart = None


def _load():
    global _lib, _cudart
    if _lib is None:
        lib = C.CDLL(str(_LIB))
        vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        lib.dic_last_error.restype = C.c_char_p
        lib.dic_tids_words.restype = i64
        lib.dic_tids_words.argtypes = [i64, i32]
        lib.dic_rows_to_tids.argtypes = [vp, i64, i32, vp, vp]
        lib.dic_count_support.argtypes = [vp, i64, i32, i64, i64, vp, i32, i64, vp, vp]
        lib.dic_launch_count.restype = i64
        _lib = lib
        # the CUDA runtime the library itself links (for cudaMalloc / memcpy)
        for name in ("libcudart.so.12", "libcudart.so"):
            try:
                _cudart = C.CDLL(name)
                break
            except OSError:
                continue
        if _cudart is None:
            raise OSError("libcudart not found")
    return _lib


def _check(rc: int) -> None:
    if rc < 0:
        raise RuntimeError(_lib.dic_last_error().decode())


class _Dev:
    """A device buffer (cudaMalloc / cudaFree)."""

    def __init__(self, nbytes: int):
        self.p = C.c_void_p()
        if _cudart.cudaMalloc(C.byref(self.p), C.c_size_t(max(nbytes, 1))) != 0:
            raise MemoryError("cudaMalloc failed")

    def upload(self, a: np.ndarray) -> "_Dev":
        a = np.ascontiguousarray(a)
        if _cudart.cudaMemcpy(self.p, a.ctypes.data_as(C.c_void_p), C.c_size_t(a.nbytes), 1) != 0:  # H2D
            raise RuntimeError("cudaMemcpy H2D failed")
        return self

    def download(self, a: np.ndarray) -> np.ndarray:
        if _cudart.cudaMemcpy(a.ctypes.data_as(C.c_void_p), self.p, C.c_size_t(a.nbytes), 2) != 0:  # D2H
            raise RuntimeError("cudaMemcpy D2H failed")
        return a

    def __del__(self):
        if self.p and _cudart is not None:
            _cudart.cudaFree(self.p)


_TIDS: dict = {}


def device_tids(arr: np.ndarray, m: int):
    """The bit-sliced copy of a mask array (uint64 [n] or [n][W]), built once on the device."""
    lib = _load()
    key = (id(arr), arr.shape, m)
    hit = _TIDS.get(key)
    if hit is not None and hit[0] is arr:
        return hit[1]
    n = arr.shape[0]
    rows = _Dev(arr.nbytes).upload(arr.reshape(n, -1).astype(np.uint64, copy=False))
    tids = _Dev(4 * int(lib.dic_tids_words(n, m)))
    _check(lib.dic_rows_to_tids(rows.p, n, m, tids.p, None))
    _TIDS.clear()
    _TIDS[key] = (arr, tids)
    return tids


def _universe(arr: np.ndarray) -> int:
    return 64 * (arr.shape[1] if arr.ndim == 2 else 1)


def _count(arr: np.ndarray, first: int, last: int, items: np.ndarray, k: int) -> np.ndarray:
    lib = _load()
    m = _universe(arr)
    tids = device_tids(arr, m)
    C_ = items.shape[0]
    dit = _Dev(items.nbytes).upload(items.astype(np.uint16))
    out = _Dev(8 * C_).upload(np.zeros(C_, dtype=np.int64))
    _check(lib.dic_count_support(tids.p, arr.shape[0], m, first, last, dit.p, k, C_, out.p, None))
    return out.download(np.zeros(C_, dtype=np.int64))


def _items(mask: int) -> list[int]:
    out, b = [], 0
    while mask:
        if mask & 1:
            out.append(b)
        mask >>= 1
        b += 1
    return out


def count_block(arr: np.ndarray, first: int, last: int, mask: int) -> int:
    """_count_block (engine.py:43-58) on the GPU: rows in [first, last] holding every item of mask."""
    its = _items(int(mask))
    if not its:
        return last - first + 1
    return int(_count(arr, first, last, np.array([its], dtype=np.uint16), len(its))[0])


def count_support_interval(catalog, db, first: int, last: int, threads: int = 1, *, pool=None,
                           kernel: str = "numpy") -> None:
    """count_support_interval (engine.py:176-223): every dashed itemset's
    support over [first, last], one dic_count_support launch per itemset size."""
    if not 0 <= first <= last < db.n:
        raise ValueError(f"chunk [{first}, {last}] outside database of {db.n} rows")
    if not catalog.dashed:
        return
    by_k = defaultdict(list)
    for it in catalog.dashed:
        by_k[it.size].append(it)
    arr = db.masks
    for k, recs in by_k.items():
        items = np.array([_items(it.mask) for it in recs], dtype=np.uint16)
        for it, c in zip(recs, _count(arr, first, last, items, k).tolist()):
            it.support += c
            it.intervals_counted += 1


def install(engine_module) -> None:
    """Point the reference engine's counting seam at the GPU."""
    engine_module._count_block = count_block
    engine_module.count_support_interval = count_support_interval


def launches() -> int:
    return int(_load().dic_launch_count())
