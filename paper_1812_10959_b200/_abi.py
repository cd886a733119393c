"""ctypes binding of libdicb200.so (the C ABI declared in include/dic_b200.h).

There is no CPU fallback: importing a compute entry point without the built
library raises immediately, and every call checks the return code.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

# DIC_LIB: an alternative build of the same library (A/B timing of kernel variants)
_LIB_PATH = Path(os.environ.get("DIC_LIB") or Path(__file__).resolve().parent / "lib" / "libdicb200.so")

DIC_OK, DIC_EINVAL, DIC_ECUDA, DIC_ENOMEM, DIC_EDATA, DIC_ESTATE = 0, -1, -2, -3, -4, -5

i32, i64, u64, dbl, vp = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_void_p
P = C.POINTER


class StopStatus(C.Structure):
    _fields_ = [
        ("dashed_at_start", i64),
        ("promoted", i64),
        ("pruned", i64),
        ("inserted", i64),
        ("dashed_peak", i64),
        ("finalized", i64),
        ("dashed_at_end", i64),
        ("records", i64),
    ]


class ParseStatus(C.Structure):
    _fields_ = [("kind", i32), ("reserved", i32), ("line", i64), ("offset", i64), ("length", i64)]


class RunStats(C.Structure):
    _fields_ = [
        ("stops", i64),
        ("scanned", i64),
        ("interval_counts", i64),
        ("candidates_generated", i64),
        ("candidates_pruned", i64),
        ("peak_dashed", i64),
        ("replays", i64),
        ("issue_us", dbl),
        ("poll_us", dbl),
        ("graphs_captured", i64),
        ("batches", i64),
        ("batched_stops", i64),
    ]


# name -> (restype, argtypes); kept in the order of include/dic_b200.h
SIGNATURES: dict[str, tuple] = {
    "dic_abi_version": (C.c_int, []),
    "dic_last_error": (C.c_char_p, []),
    "dic_device_sm_count": (C.c_int, []),
    "dic_launch_count": (i64, []),
    "dic_encode_csr": (C.c_int, [vp, vp, i64, i32, vp, vp, vp]),
    "dic_rows_to_tids": (C.c_int, [vp, i64, i32, vp, vp]),
    "dic_tids_words": (i64, [i64, i32]),
    "dic_tids_tile_groups": (C.c_int, [i32]),
    "dic_tids_index": (i64, [i32, i32, i64]),
    "dic_item_support": (C.c_int, [vp, i64, i32, i64, i64, vp, vp]),
    "dic_count_support": (C.c_int, [vp, i64, i32, i64, i64, vp, i32, i64, vp, vp]),
    "dic_count_pairs": (C.c_int, [vp, i64, i32, i64, i64, vp, vp]),
    "dic_pair_kernel_select": (C.c_int, [i32, P(i32)]),
    "dic_tids_select": (C.c_int, [vp, i64, i32, vp, i32, vp, vp]),
    "dic_count_support_rows": (C.c_int, [vp, i32, i64, i64, vp, i64, vp, vp]),
    "dic_candidate_admission": (C.c_int, [vp, i64, vp, i64, i32, vp, i64, vp, i64, vp, vp]),
    "dic_engine_create": (C.c_int, [vp, i64, i32, i64, i64, i64, i32, vp, P(vp)]),
    "dic_engine_destroy": (C.c_int, [vp]),
    "dic_engine_item_counts": (C.c_int, [vp, vp]),
    "dic_engine_seed": (C.c_int, [vp, vp, P(i64), P(i64)]),
    "dic_engine_count": (C.c_int, [vp, i64, i64]),
    "dic_engine_delta": (C.c_int, [vp, P(vp), P(i64)]),
    "dic_engine_checkpoint": (C.c_int, [vp, P(StopStatus)]),
    "dic_engine_issue_count": (C.c_int, [vp, i64, i64]),
    "dic_nccl_unique_id": (C.c_int, [vp]),
    "dic_nccl_comm_init": (C.c_int, [vp, i32, i32, P(vp)]),
    "dic_nccl_comm_destroy": (C.c_int, [vp]),
    "dic_engine_set_comm": (C.c_int, [vp, vp]),
    "dic_engine_collective_mode": (C.c_int, [vp]),
    "dic_containment": (C.c_int, [vp, i64, i32, vp, vp, i64, vp, vp]),
    "dic_containment_packed": (C.c_int, [vp, i64, i32, vp, vp, i64, vp, vp]),
    "dic_encode_status_init": (C.c_int, [vp, vp]),
    "dic_encode_csr_tids": (C.c_int, [vp, vp, i32, i64, i32, i64, i64, vp, vp, vp]),
    "dic_encode_status_finish": (C.c_int, [vp, i64, vp, vp]),
    "dic_tids_to_rows": (C.c_int, [vp, i64, i32, vp, vp]),
    "dic_engine_set_schedule": (C.c_int, [vp, vp, vp, i64]),
    "dic_engine_graph_stats": (C.c_int, [vp, P(i64), P(i64)]),
    "dic_engine_pair_counts": (C.c_int, [vp, P(vp), P(i64)]),
    "dic_engine_issue_checkpoint": (C.c_int, [vp, P(i64)]),
    "dic_engine_poll": (C.c_int, [vp, i64, P(StopStatus), P(i32)]),
    "dic_engine_run": (C.c_int, [vp, vp, vp, vp, i64, i32, P(RunStats), vp, vp, i64]),
    "dic_engine_num_frequent": (C.c_int, [vp, P(i64)]),
    "dic_engine_frequent": (C.c_int, [vp, vp, vp, vp, i64]),
    "dic_engine_words": (C.c_int, [vp]),
    "dic_engine_bucket": (C.c_int, [vp, i32, vp, vp, i64, P(i64)]),
    "dic_synth_zipf": (C.c_int, [vp, vp, C.c_int, i32, dbl, dbl, u64, C.c_int, P(vp)]),
    "dic_synth_quest": (C.c_int, [vp, vp, C.c_int, i32, i32, dbl, dbl, u64, C.c_int, P(vp)]),
    "dic_synth_dense": (C.c_int, [vp, vp, C.c_int, i32, i32, i32, dbl, u64, C.c_int, P(vp)]),
    "dic_csr_info": (C.c_int, [vp, P(i64), P(i64)]),
    "dic_csr_export": (C.c_int, [vp, vp, vp]),
    "dic_csr_free": (None, [vp]),
    "dic_parse_transactions": (C.c_int, [vp, i64, i32, i32, P(vp), P(ParseStatus)]),
    "dic_format_transactions": (C.c_int, [vp, i64, i32, i32, P(vp), P(i64)]),
    "dic_free_buffer": (None, [vp]),
    "dic_synth_bernoulli_rows": (C.c_int, [i64, i32, dbl, u64, vp, vp]),
    "dic_synth_candidates": (C.c_int, [i64, i32, i32, i32, u64, vp, vp]),
    "dic_probe_int_pipe": (C.c_int, [C.c_int, C.c_int, C.c_int, i64, vp, P(dbl), P(C.c_float), vp]),
}


class DicError(RuntimeError):
    """A C-ABI call returned an error code."""

    def __init__(self, fn: str, code: int, msg: str):
        self.fn, self.code, self.msg = fn, code, msg
        super().__init__(f"{fn} failed ({code}): {msg}")


_lib: C.CDLL | None = None


def lib_path() -> Path:
    return _LIB_PATH


def load() -> C.CDLL:
    """Load libdicb200.so, raising if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        raise ImportError(
            f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the DIC hot path)"
        )
    lib = C.CDLL(str(_LIB_PATH), mode=os.RTLD_NOW | os.RTLD_LOCAL)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def call(name: str, *args) -> int:
    """Call an int-returning entry point and raise DicError on failure."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc is not None and rc < 0:
        msg = lib.dic_last_error().decode(errors="replace")
        raise DicError(name, rc, msg)
    return rc
