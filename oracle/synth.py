"""TEST / BASELINE INFRASTRUCTURE — the seeded input generators of the five
configs (csrc/synth.cpp) through their own build, oracle/_build/libsynth.so.

bench.py's CPU reference arm (`--impl reference`) generates its workload with
this module, so no product library (libdicb200.so) is mapped in that process:
the arm runs only the oracle port over these rows.  Same generator source,
so the rows are identical to workloads.generate_csr's (tests check the
digest).
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "libsynth.so"
_lib: C.CDLL | None = None


def load() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists():
            from . import oracle as O

            O.build()
        lib = C.CDLL(str(LIB))
        vp, i32, i64, dbl, u64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double, C.c_uint64
        P = C.POINTER
        lib.dic_synth_zipf.argtypes = [vp, vp, C.c_int, i32, dbl, dbl, u64, C.c_int, P(vp)]
        lib.dic_synth_quest.argtypes = [vp, vp, C.c_int, i32, i32, dbl, dbl, u64, C.c_int, P(vp)]
        lib.dic_synth_dense.argtypes = [vp, vp, C.c_int, i32, i32, i32, dbl, u64, C.c_int, P(vp)]
        lib.dic_csr_info.argtypes = [vp, P(i64), P(i64)]
        lib.dic_csr_export.argtypes = [vp, vp, vp]
        lib.dic_csr_free.argtypes = [vp]
        lib.dic_csr_free.restype = None
        lib.dic_synth_candidates.argtypes = [i64, i32, i32, i32, u64, vp, vp]
        _lib = lib
    return _lib


def _check(rc: int, what: str) -> None:
    if rc != 0:
        raise RuntimeError(f"{what} failed ({rc})")


def generate_csr(cfg, ranges=None, threads: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """CSR of a workloads.Config's rows (all rows, or the given global (begin, len) ranges)."""
    lib = load()
    ranges = [(0, cfg.n)] if ranges is None else ranges
    rb = np.ascontiguousarray([r[0] for r in ranges], dtype=np.int64)
    rl = np.ascontiguousarray([r[1] for r in ranges], dtype=np.int64)
    h = C.c_void_p()
    kw = cfg.params
    if cfg.kind == "zipf":
        _check(lib.dic_synth_zipf(rb.ctypes.data, rl.ctypes.data, len(rb), cfg.m, kw["s"], kw["mean_len"], cfg.seed,
                                  threads, C.byref(h)), "dic_synth_zipf")
    elif cfg.kind == "quest":
        _check(lib.dic_synth_quest(rb.ctypes.data, rl.ctypes.data, len(rb), cfg.m, kw["n_patterns"],
                                   kw["pattern_len"], kw["mean_len"], cfg.seed, threads, C.byref(h)), "dic_synth_quest")
    elif cfg.kind == "dense":
        _check(lib.dic_synth_dense(rb.ctypes.data, rl.ctypes.data, len(rb), cfg.m, kw["groups"], kw["group_size"],
                                   kw["group_p"], cfg.seed, threads, C.byref(h)), "dic_synth_dense")
    else:
        raise ValueError(f"no CSR generator for {cfg.kind!r}")
    n, nnz = C.c_int64(), C.c_int64()
    try:
        _check(lib.dic_csr_info(h, C.byref(n), C.byref(nnz)), "dic_csr_info")
        indptr = np.empty(n.value + 1, dtype=np.int64)
        indices = np.empty(max(nnz.value, 1), dtype=np.int32)
        _check(lib.dic_csr_export(h, indptr.ctypes.data, indices.ctypes.data), "dic_csr_export")
    finally:
        lib.dic_csr_free(h)
    return indptr, indices[: nnz.value]


def candidates(C_: int, m: int, kmin: int, kmax: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """cfg5's random candidate itemsets: ks [C], items [C][kmax] (0xFFFF past k)."""
    ks = np.empty(C_, dtype=np.int32)
    items = np.empty((C_, kmax), dtype=np.uint16)
    _check(load().dic_synth_candidates(C_, m, kmin, kmax, seed, ks.ctypes.data, items.ctypes.data),
           "dic_synth_candidates")
    return ks, items
