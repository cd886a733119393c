"""Thin tensor-level wrappers over the C ABI (torch only allocates device
buffers and supplies the current CUDA stream).

Every function here launches sm_100a kernels from libdicb200.so; there is no
CPU path.  Shapes and dtypes follow the layouts in include/dic_b200.h.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _abi


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1812_10959_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    _abi.load()
    return torch.device("cuda", torch.cuda.current_device())


def words_for(m: int) -> int:
    return (m + 63) // 64


def tids_words(n: int, m: int) -> int:
    return int(_abi.load().dic_tids_words(n, m))


def tile_groups(m: int) -> int:
    return int(_abi.load().dic_tids_tile_groups(m))


def encode_csr(indptr: torch.Tensor, indices: torch.Tensor, n: int, m: int) -> tuple[torch.Tensor, torch.Tensor]:
    """CSR (device int64 indptr[n+1], int32 indices[nnz]) -> rows uint64 [n][W].

    Returns (rows, status) with status = int64[4] (dedup, bad_pos, bad_row, 0),
    still on the device (read it after the stream syncs)."""
    W = words_for(m)
    rows = torch.empty((max(n, 1), W), dtype=torch.uint64, device=indptr.device)
    status = torch.empty(4, dtype=torch.int64, device=indptr.device)
    _abi.call("dic_encode_csr", _ptr(indptr), _ptr(indices), n, m, _ptr(rows), _ptr(status), _stream())
    return rows[:n], status


def encode_status_init(status: torch.Tensor) -> None:
    _abi.call("dic_encode_status_init", _ptr(status), _stream())


def encode_csr_tids(indptr: torch.Tensor, indices: torch.Tensor, n: int, m: int, row_begin: int, row_end: int,
                    tids: torch.Tensor, status: torch.Tensor) -> None:
    """Rows [row_begin, row_end) of a device CSR (int64 indptr[n+1], uint16 or
    int32 indices) straight into the bit-sliced tiles ``tids``."""
    ib = 2 if indices.dtype in (torch.uint16, torch.int16) else 4
    if ib == 4 and indices.dtype != torch.int32:
        raise TypeError(f"indices must be uint16 or int32, got {indices.dtype}")
    _abi.call("dic_encode_csr_tids", _ptr(indptr), _ptr(indices) if indices.numel() else None, ib, n, m,
              row_begin, row_end, _ptr(tids), _ptr(status), _stream())


def encode_status_finish(indptr: torch.Tensor, n: int, status: torch.Tensor) -> None:
    _abi.call("dic_encode_status_finish", _ptr(indptr), n, _ptr(status), _stream())


def tids_to_rows(tids: torch.Tensor, n: int, m: int) -> torch.Tensor:
    """Bit-sliced tiles -> row bitmap uint64 [n][W] (the inverse transform)."""
    rows = torch.empty((max(n, 1), words_for(m)), dtype=torch.uint64, device=tids.device)
    _abi.call("dic_tids_to_rows", _ptr(tids), n, m, _ptr(rows), _stream())
    return rows[:n]


def patterns_to_device(masks) -> tuple[torch.Tensor, torch.Tensor]:
    """Python-int masks -> (uint16 items, int64 offsets[P+1]) on the device,
    each pattern's ids ascending (the containment kernel's input)."""
    from .bits import items_of

    lens, flat = [], []
    for mk in masks:
        its = list(items_of(int(mk)))
        lens.append(len(its))
        flat.extend(its)
    offs = np.zeros(len(lens) + 1, dtype=np.int64)
    np.cumsum(lens, out=offs[1:])
    items = np.asarray(flat if flat else [0], dtype=np.uint16)
    return torch.from_numpy(items).cuda(), torch.from_numpy(offs).cuda()


def containment(tids: torch.Tensor, n: int, m: int, items: torch.Tensor, offs: torch.Tensor,
                packed: bool = False) -> torch.Tensor:
    """Pattern containment over the bit-sliced rows: bool [n][P] (or the
    packed uint32 [ceil(n/32)][P] bit matrix)."""
    P = int(offs.numel()) - 1
    if packed:
        out = torch.empty(((n + 31) // 32, max(P, 1)), dtype=torch.int32, device=tids.device)
        _abi.call("dic_containment_packed", _ptr(tids), n, m, _ptr(items), _ptr(offs), P, _ptr(out), _stream())
        return out[:, :P]
    out = torch.empty((n, max(P, 1)), dtype=torch.uint8, device=tids.device)
    _abi.call("dic_containment", _ptr(tids), n, m, _ptr(items), _ptr(offs), P, _ptr(out), _stream())
    return out[:, :P].view(torch.bool)


def rows_to_tids(rows: torch.Tensor, n: int, m: int) -> torch.Tensor:
    """Row bitmap -> the tiled bit-sliced layout (int32 words, see dic_b200.h)."""
    tids = torch.empty(max(tids_words(n, m), 1), dtype=torch.int32, device=rows.device)
    _abi.call("dic_rows_to_tids", _ptr(rows), n, m, _ptr(tids), _stream())
    return tids


def item_support(tids: torch.Tensor, n: int, m: int, first: int, last: int,
                 counts: torch.Tensor | None = None) -> torch.Tensor:
    if counts is None:
        counts = torch.zeros(m, dtype=torch.int64, device=tids.device)
    _abi.call("dic_item_support", _ptr(tids), n, m, first, last, _ptr(counts), _stream())
    return counts


def count_support(tids: torch.Tensor, n: int, m: int, first: int, last: int, items: torch.Tensor,
                  out: torch.Tensor | None = None) -> torch.Tensor:
    """items: device uint16/int16 [C][k] ascending item ids; out += counts (int64 [C])."""
    Cn, k = items.shape
    if out is None:
        out = torch.zeros(Cn, dtype=torch.int64, device=tids.device)
    if Cn:
        _abi.call("dic_count_support", _ptr(tids), n, m, first, last, _ptr(items), k, Cn, _ptr(out), _stream())
    return out


def pair_kernel_select(mode: int) -> int:
    """Process-wide pair-triangle kernel: -1 env, 0 auto, 1 AND/POPC, 2 tensor cores; returns the previous mode."""
    prev = C.c_int32()
    _abi.call("dic_pair_kernel_select", mode, C.byref(prev))
    return prev.value


def count_pairs(tids: torch.Tensor, n: int, m: int, first: int, last: int,
                tri: torch.Tensor | None = None) -> torch.Tensor:
    """Counts of all pairs a < b < m over rows [first, last], a-major triangle (int64)."""
    if tri is None:
        tri = torch.zeros(m * (m - 1) // 2, dtype=torch.int64, device=tids.device)
    _abi.call("dic_count_pairs", _ptr(tids), n, m, first, last, _ptr(tri), _stream())
    return tri


def tids_select(tids: torch.Tensor, n: int, m: int, items: torch.Tensor) -> torch.Tensor:
    L = items.numel()
    out = torch.empty(max(tids_words(n, L), 1), dtype=torch.int32, device=tids.device)
    _abi.call("dic_tids_select", _ptr(tids), n, m, _ptr(items), L, _ptr(out), _stream())
    return out


def count_support_rows(rows: torch.Tensor, first: int, last: int, masks: torch.Tensor,
                       out: torch.Tensor | None = None) -> torch.Tensor:
    Cn, W = masks.shape
    if out is None:
        out = torch.zeros(Cn, dtype=torch.int64, device=rows.device)
    if Cn:
        _abi.call("dic_count_support_rows", _ptr(rows), W, first, last, _ptr(masks), Cn, _ptr(out), _stream())
    return out


def candidate_admission(src_masks: torch.Tensor, level1: torch.Tensor, known_masks: torch.Tensor,
                        box_masks: torch.Tensor) -> torch.Tensor:
    S, W = src_masks.shape
    L = level1.numel()
    admit = torch.zeros(S * L, dtype=torch.uint8, device=src_masks.device)
    _abi.call("dic_candidate_admission", _ptr(src_masks), S, _ptr(level1), L, W, _ptr(known_masks),
              known_masks.shape[0], _ptr(box_masks), box_masks.shape[0], _ptr(admit), _stream())
    return admit.view(S, L)


def bernoulli_rows(n: int, m: int, p: float, seed: int, device=None) -> torch.Tensor:
    W = words_for(m)
    rows = torch.empty((n, W), dtype=torch.uint64, device=device or "cuda")
    _abi.call("dic_synth_bernoulli_rows", n, m, p, seed, _ptr(rows), _stream())
    return rows


def probe_int_pipe(op: int, blocks: int, threads: int, iters: int) -> tuple[float, float]:
    """Returns (lane_ops, milliseconds) of the op's chain (0 LOP3, 1 POPC, 2 IADD)."""
    sink = torch.zeros(1, dtype=torch.int32, device="cuda")
    lane_ops, ms = C.c_double(), C.c_float()
    _abi.call("dic_probe_int_pipe", op, blocks, threads, iters, _ptr(sink), C.byref(lane_ops), C.byref(ms),
              _stream())
    return lane_ops.value, ms.value


# ---------------------------------------------------------------------------
# host generators (CSR as numpy arrays)
# ---------------------------------------------------------------------------
def _ranges(ranges):
    rb = np.ascontiguousarray([r[0] for r in ranges], dtype=np.int64)
    rl = np.ascontiguousarray([r[1] for r in ranges], dtype=np.int64)
    return rb, rl


def _export(h: C.c_void_p) -> tuple[np.ndarray, np.ndarray]:
    lib = _abi.load()
    n, nnz = C.c_int64(), C.c_int64()
    try:
        _abi.call("dic_csr_info", h, C.byref(n), C.byref(nnz))
        indptr = np.empty(n.value + 1, dtype=np.int64)
        indices = np.empty(max(nnz.value, 1), dtype=np.int32)
        _abi.call("dic_csr_export", h, indptr.ctypes.data, indices.ctypes.data)
    finally:
        lib.dic_csr_free(h)
    return indptr, indices[: nnz.value]


def synth(kind: str, ranges, m: int, seed: int, threads: int = 0, **kw) -> tuple[np.ndarray, np.ndarray]:
    """Generate CSR rows for the global row ranges [(begin, len), ...]."""
    rb, rl = _ranges(ranges)
    h = C.c_void_p()
    if kind == "zipf":
        _abi.call("dic_synth_zipf", rb.ctypes.data, rl.ctypes.data, len(rb), m, kw["s"], kw["mean_len"], seed,
                  threads, C.byref(h))
    elif kind == "quest":
        _abi.call("dic_synth_quest", rb.ctypes.data, rl.ctypes.data, len(rb), m, kw["n_patterns"],
                  kw["pattern_len"], kw["mean_len"], seed, threads, C.byref(h))
    elif kind == "dense":
        _abi.call("dic_synth_dense", rb.ctypes.data, rl.ctypes.data, len(rb), m, kw["groups"], kw["group_size"],
                  kw["group_p"], seed, threads, C.byref(h))
    else:
        raise ValueError(f"unknown generator {kind!r}")
    return _export(h)


def synth_candidates(C_: int, m: int, kmin: int, kmax: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
    ks = np.empty(C_, dtype=np.int32)
    items = np.empty((C_, kmax), dtype=np.uint16)
    _abi.call("dic_synth_candidates", C_, m, kmin, kmax, seed, ks.ctypes.data, items.ctypes.data)
    return ks, items
