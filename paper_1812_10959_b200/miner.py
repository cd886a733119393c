"""DIC entry points: mine_parallel / mine_serial and the device-engine driver.

Same signatures, results (frequent itemsets in (size, mask) order with exact
supports) and MiningStats as the reference's engines (/root/reference/pkg/
src/dicmine/engine.py:398-496).  The checkpoint loop of _run (:422-441) runs
here on the host, one iteration per stop, driving the device-resident state
machine in libdicb200.so (csrc/engine.cu):

    dic_engine_count        count every dashed candidate over the local chunk
    [all_reduce of deltas]  only when sharded over several GPUs
    dic_engine_checkpoint   apply + prune + make_candidates + check_full_pass

One small synchronous status read per stop drives the loop test, exactly the
``while catalog.dashed`` of the reference.  With an ``audit`` recorder the
run instead goes through the phase-level API (phases.py) so every
transition is recorded in the reference's order.
"""

from __future__ import annotations

import ctypes as C
import gc
import time
from pathlib import Path
from collections import deque
from functools import partial
from dataclasses import dataclass, field

import numpy as np

from . import _abi, bits
from .bitmap import BitDatabase
from .catalog import ItemsetCatalog, Shape, TransitionAudit
from .config import MiningParams
from .phases import (FrequentItemset, MiningResult, MiningStats, check_full_pass, count_support_interval,
                     first_pass, make_candidates, prune)
from .sharding import ShardPlan


@dataclass
class StopTrace:
    """Per-stop engine status (for tests and the bench's accounting)."""

    stops: list[dict] = field(default_factory=list)
    native: dict | None = None  # host-side diagnostics of the native loop
    phases: dict = field(default_factory=dict)  # host wall ms per run_engine phase


class DeviceEngine:
    """RAII handle over dic_engine (one per rank)."""

    presorted = True  # dic_engine_frequent returns the canonical (size, mask) order

    def __init__(self, tids, n_local: int, m: int, params: MiningParams, prune_bound: bool):
        import torch

        self._torch = torch
        self.tids = tids  # keep the buffer alive as long as the engine
        self.m = m
        h = C.c_void_p()
        _abi.call("dic_engine_create", tids.data_ptr() if n_local > 0 else None, n_local, m,
                  params.min_support_count, params.interval, params.intervals_per_pass, 1 if prune_bound else 0,
                  torch.cuda.current_stream().cuda_stream, C.byref(h))
        self.h = h

    def close(self) -> None:
        if self.h:
            _abi.call("dic_engine_destroy", self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def item_counts(self):
        counts = self._torch.empty(self.m, dtype=self._torch.int64, device="cuda")
        _abi.call("dic_engine_item_counts", self.h, counts.data_ptr())
        return counts

    def seed(self, counts) -> tuple[int, int]:
        L, P = C.c_int64(), C.c_int64()
        _abi.call("dic_engine_seed", self.h, counts.data_ptr(), C.byref(L), C.byref(P))
        return L.value, P.value

    def issue_count(self, lfirst: int, llast: int) -> None:
        _abi.call("dic_engine_issue_count", self.h, lfirst, llast)

    def set_comm(self, comm) -> None:
        """Attach a native NCCL communicator (native_comm): the engine then
        allreduces the item counts and every stop's counts itself."""
        _abi.call("dic_engine_set_comm", self.h, comm)

    def collective_mode(self) -> str:
        """'none', 'nccl' (per-stop ncclAllReduce) or 'fused' (peer-memory reduction kernel)."""
        return ("none", "nccl", "fused")[_abi.call("dic_engine_collective_mode", self.h)]

    def set_schedule(self, lfirst: np.ndarray, llast: np.ndarray) -> None:
        """The chunk cycle of the coming stops (matching counts run as graphs)."""
        lf = np.ascontiguousarray(lfirst, dtype=np.int64)
        ll = np.ascontiguousarray(llast, dtype=np.int64)
        _abi.call("dic_engine_set_schedule", self.h, lf.ctypes.data, ll.ctypes.data, len(lf))

    def graph_stats(self) -> tuple[int, int]:
        cap, lau = C.c_int64(), C.c_int64()
        _abi.call("dic_engine_graph_stats", self.h, C.byref(cap), C.byref(lau))
        return cap.value, lau.value

    def _device_view(self, fn: str):
        ptr, ln = C.c_void_p(), C.c_int64()
        _abi.call(fn, self.h, C.byref(ptr), C.byref(ln))
        n = ln.value
        if n == 0:
            return self._torch.empty(0, dtype=self._torch.int64, device="cuda")

        class _View:
            __cuda_array_interface__ = {"shape": (n,), "typestr": "<i8", "data": (ptr.value, False), "version": 3,
                                        "strides": None}

        return self._torch.as_tensor(_View(), device="cuda")

    def delta(self):
        """The per-stop count deltas as a (non-owning) int64 CUDA tensor."""
        return self._device_view("dic_engine_delta")

    def pair_counts(self):
        """The per-stop dense pair-triangle counts (empty if none)."""
        return self._device_view("dic_engine_pair_counts")

    def bucket(self, k: int) -> tuple[np.ndarray, np.ndarray]:
        """Bucket k as the device holds it now: record ids [n] and item lists [n][k]
        (live and dead slots; diagnostics, synchronising)."""
        n = C.c_int64()
        _abi.call("dic_engine_bucket", self.h, k, None, None, 0, C.byref(n))
        rec = np.zeros(max(n.value, 1), dtype=np.int32)
        items = np.zeros((max(n.value, 1), k), dtype=np.uint16)
        if n.value:
            _abi.call("dic_engine_bucket", self.h, k, rec.ctypes.data, items.ctypes.data, n.value, C.byref(n))
        return rec[: n.value], items[: n.value]

    def issue_checkpoint(self) -> int:
        seq = C.c_int64()
        _abi.call("dic_engine_issue_checkpoint", self.h, C.byref(seq))
        return seq.value

    def poll(self, seq: int) -> tuple[_abi.StopStatus, bool]:
        st, rep = _abi.StopStatus(), C.c_int32()
        _abi.call("dic_engine_poll", self.h, seq, C.byref(st), C.byref(rep))
        return st, bool(rep.value)

    def run(self, lfirst: np.ndarray, llast: np.ndarray, rows: np.ndarray, stop_max: int, depth: int,
            timed: bool, max_stops: int = 1 << 16) -> tuple[_abi.RunStats, np.ndarray | None, np.ndarray]:
        """The whole checkpoint loop natively (dic_engine_run)."""
        out = _abi.RunStats()
        count_ms = np.zeros(max_stops, dtype=np.float32) if timed else None
        dashed = np.zeros(max_stops, dtype=np.int64)
        _abi.call("dic_engine_run", self.h, lfirst.ctypes.data, llast.ctypes.data, rows.ctypes.data, stop_max, depth,
                  C.byref(out), count_ms.ctypes.data if timed else None, dashed.ctypes.data, max_stops)
        k = min(out.stops, max_stops)
        return out, (count_ms[:k] if timed else None), dashed[:k]

    def frequent(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        F = C.c_int64()
        _abi.call("dic_engine_num_frequent", self.h, C.byref(F))
        W = bits.words_for(self.m)
        masks = np.zeros((max(F.value, 1), W), dtype=np.uint64)
        sizes = np.zeros(max(F.value, 1), dtype=np.int32)
        sups = np.zeros(max(F.value, 1), dtype=np.int64)
        _abi.call("dic_engine_frequent", self.h, masks.ctypes.data, sizes.ctypes.data, sups.ctypes.data, F.value)
        return masks[: F.value], sizes[: F.value], sups[: F.value]


_new_frequent = partial(tuple.__new__, FrequentItemset)


_COMMS: dict = {}


def native_comm(group=None) -> C.c_void_p:
    """An NCCL communicator over the ranks of a torch.distributed group, built
    by the library (dic_nccl_comm_init; rank 0's unique id is broadcast once
    through the group) and cached per group.  Engines that use it run the
    whole sharded checkpoint loop natively (dic_engine_run)."""
    import torch
    import torch.distributed as dist

    key = id(group)
    if key in _COMMS:
        return _COMMS[key]
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    uid = (C.c_uint8 * 128)()
    if rank == 0:
        _abi.call("dic_nccl_unique_id", uid)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor(list(bytes(uid)), dtype=torch.uint8, device=dev)
    dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    ids = (C.c_uint8 * 128)(*t.cpu().tolist())
    comm = C.c_void_p()
    _abi.call("dic_nccl_comm_init", ids, world, rank, C.byref(comm))
    _COMMS[key] = comm
    return comm


def sorted_frequent(masks: np.ndarray, sizes: np.ndarray, sups: np.ndarray,
                    presorted: bool = False) -> tuple[FrequentItemset, ...]:
    """Canonical (size, mask) order (engine.py:446-455) with masks compared as
    Python ints, i.e. most significant word first (dic_engine_frequent
    already returns that order: presorted)."""
    if len(sizes) == 0:
        return ()
    if not presorted:
        W = masks.shape[1]
        order = np.lexsort(tuple(masks[:, w] for w in range(W)) + (sizes,))
        masks, sizes, sups = masks[order], sizes[order], sups[order]
    # the tuple of FrequentItemset built in C (csrc/pyresults.c)
    m64 = np.ascontiguousarray(masks, dtype=np.uint64)
    if m64.ndim == 1:
        m64 = m64.reshape(-1, 1)
    # thousands of fresh tuples would trigger generation-0 collections
    enabled = gc.isenabled()
    gc.disable()
    try:
        return _dicpy().frequent_tuple(FrequentItemset, m64.tobytes(), m64.shape[1],
                                       np.ascontiguousarray(sizes, dtype=np.int32).tobytes(),
                                       np.ascontiguousarray(sups, dtype=np.int64).tobytes())
    finally:
        if enabled:
            gc.enable()


_DICPY = None


def _dicpy():
    """The result-builder extension built next to libdicb200.so."""
    global _DICPY
    if _DICPY is None:
        import importlib.util
        import sysconfig

        PY_EXT = Path(__file__).resolve().parent / "lib" / ("_dicpy" + (sysconfig.get_config_var("EXT_SUFFIX") or ".so"))
        if not PY_EXT.exists():
            raise ImportError(f"{PY_EXT} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        spec = importlib.util.spec_from_file_location("_dicpy", PY_EXT)
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _DICPY = mod
    return _DICPY


def run_engine(tids, n_local: int, m: int, params: MiningParams, *, prune_bound: bool = True,
               plan: ShardPlan | None = None, group=None, trace: StopTrace | None = None,
               t0: float | None = None, count_events: list | None = None,
               engine_factory=None, depth: int = 4, collective: bool | str | None = None) -> MiningResult:
    """The checkpoint loop of _run over one rank's local rows.

    ``plan``/``group``: chunk-sliced sharding (sharding.py) with a
    torch.distributed process group; counts are sum-allreduced per stop.
    ``count_events``: if a list, [start, end, word_popcounts, rows] entries
    are appended around every count launch (the bench's roofline figures).
    ``depth``: stops in flight (1 = the reference's strictly sequential loop).
    ``engine_factory``: test seam (a CPU stand-in engine for the gloo
    multi-rank tests); the product always uses DeviceEngine.
    ``collective="native"``: the per-stop allreduces run inside the library on
    its own NCCL communicator (native_comm) and the whole loop is
    dic_engine_run; ``True``: torch.distributed all_reduce from this loop."""
    import torch
    import torch.distributed as dist

    t0 = time.perf_counter() if t0 is None else t0
    # per-stop collectives: whenever sharded (collective=True forces the
    # collective loop even for one rank, e.g. to test the NCCL path on one GPU)
    sharded = (plan is not None and plan.world > 1) if collective is None else bool(collective)
    native = collective == "native" and engine_factory is None
    local_chunks = plan.local_chunks() if plan is not None else None
    tp = [time.perf_counter()]

    def phase(name: str) -> None:
        tp.append(time.perf_counter())
        if trace is not None:
            trace.phases[name] = (tp[-1] - tp[-2]) * 1e3

    eng = (engine_factory or DeviceEngine)(tids, n_local, m, params, prune_bound)
    if native:
        eng.set_comm(native_comm(group))
    phase("create")
    try:
        stats = MiningStats()
        counts = eng.item_counts()
        if sharded and not native:
            dist.all_reduce(counts, group=group)
        _, npairs = eng.seed(counts)
        phase("first_pass")
        stats.candidates_generated = npairs
        stats.peak_dashed = npairs
        scanned = params.n
        if engine_factory is None and (not sharded or native):
            # the whole loop natively: no Python on the per-stop path
            nst = params.intervals_per_pass
            bounds = [params.chunk_bounds(s) for s in range(1, nst + 1)]
            rows = np.array([b[1] - b[0] + 1 for b in bounds], dtype=np.int64)  # global rows per stop
            if local_chunks is not None:
                bounds = local_chunks  # this rank's slice of each chunk
            lf = np.array([b[0] for b in bounds], dtype=np.int64)
            ll = np.array([b[1] for b in bounds], dtype=np.int64)
            out, cms, dashed = eng.run(lf, ll, rows, nst, depth, count_events is not None)
            phase("loop")
            if trace is not None:
                trace.native = {"stops": out.stops, "replays": out.replays, "issue_ms": out.issue_us / 1e3,
                                "poll_ms": out.poll_us / 1e3, "graphs_captured": out.graphs_captured,
                                "batches": out.batches, "batched_stops": out.batched_stops,
                                "collective": eng.collective_mode() if hasattr(eng, "collective_mode") else "none"}
            stats.interval_counts += out.interval_counts
            stats.candidates_pruned += out.candidates_pruned
            stats.candidates_generated += out.candidates_generated
            stats.peak_dashed = max(stats.peak_dashed, out.peak_dashed)
            scanned += out.scanned
            for i in range(len(dashed)):
                stop_no = i % nst + 1
                if trace is not None:
                    trace.stops.append({"stop": stop_no, "dashed_at_start": int(dashed[i])})
                if count_events is not None:
                    count_events.append(("native", float(cms[i]), int(dashed[i]) * (-(-int(rows[stop_no - 1]) // 32)),
                                         int(rows[stop_no - 1])))
            fr = eng.frequent()
            phase("collect")
            frequent = sorted_frequent(*fr, presorted=getattr(eng, "presorted", False))
            phase("build")
            eng.close()
            eng = None
            phase("close")
        # Pipelined checkpoint loop: stops are enqueued up to `depth` ahead
        # and their statuses consumed in order (the reference's loop test
        # `while catalog.dashed` is evaluated on the polled status; stops
        # enqueued after the last live one are no-ops and are not counted).
        inflight: deque = deque()
        stop = 0
        live = npairs
        done = live == 0 or eng is None
        if not done and hasattr(eng, "set_schedule"):
            # the stops cycle through fixed chunks: declare them so each count
            # is one graph launch
            nst = params.intervals_per_pass
            sched = [local_chunks[s] if local_chunks is not None else params.chunk_bounds(s + 1) for s in range(nst)]
            eng.set_schedule(np.array([c[0] for c in sched], dtype=np.int64),
                             np.array([c[1] for c in sched], dtype=np.int64))
        while True:
            while not done and len(inflight) < depth:
                stop = stop + 1 if stop < params.intervals_per_pass else 1
                first, last = params.chunk_bounds(stop)
                lfirst, llast = local_chunks[stop - 1] if local_chunks is not None else (first, last)
                if count_events is not None:
                    ev0 = torch.cuda.Event(enable_timing=True)
                    ev1 = torch.cuda.Event(enable_timing=True)
                    ev0.record()
                    eng.issue_count(lfirst, llast)
                    ev1.record()
                    count_events.append([ev0, ev1, 0, llast - lfirst + 1])
                else:
                    eng.issue_count(lfirst, llast)
                if sharded:
                    dist.all_reduce(eng.delta(), group=group)
                    tri = eng.pair_counts()
                    if tri.numel():
                        dist.all_reduce(tri, group=group)
                inflight.append((eng.issue_checkpoint(), stop, first, last))
            if not inflight:
                break
            seq, s_stop, first, last = inflight.popleft()
            st, replayed = eng.poll(seq)
            if done:
                continue  # a no-op stop issued after the last live one
            if count_events is not None:
                # word-popcount work of this stop's count launch
                ev = count_events[len(count_events) - len(inflight) - 1]
                ev[2] = st.dashed_at_start * (-(-max(ev[3], 0) // 32))
            stats.interval_counts += st.dashed_at_start
            scanned += last - first + 1
            stats.candidates_pruned += st.pruned
            stats.candidates_generated += st.inserted
            stats.peak_dashed = max(stats.peak_dashed, st.dashed_peak)
            live = st.dashed_at_end
            if trace is not None:
                trace.stops.append({f: getattr(st, f) for f, _ in _abi.StopStatus._fields_} | {"stop": s_stop})
            if replayed:
                # stops after seq were skipped on the device: re-issue them
                if count_events is not None:
                    del count_events[len(count_events) - len(inflight):]
                inflight.clear()
                stop = s_stop
            if live == 0:
                done = True
        if eng is not None:
            frequent = sorted_frequent(*eng.frequent(), presorted=getattr(eng, "presorted", False))
    finally:
        if eng is not None:
            eng.close()
    if torch.cuda.is_available():
        torch.cuda.synchronize()
    stats.db_passes = scanned / params.n
    stats.wall_time_s = time.perf_counter() - t0
    return MiningResult(frequent=frequent, stats=stats)


def _run_phases(db: BitDatabase, params: MiningParams, prune_bound: bool,
                audit: TransitionAudit | None) -> MiningResult:
    """Phase-level loop (audit mode): host catalog, GPU counting/admission."""
    t0 = time.perf_counter()
    stats = MiningStats()
    catalog = ItemsetCatalog()
    level1 = first_pass(catalog, db, params, audit=audit, stats=stats)
    scanned = db.n
    stop = 0
    while catalog.dashed:
        stop = stop + 1 if stop < params.intervals_per_pass else 1
        first, last = params.chunk_bounds(stop)
        stats.interval_counts += len(catalog.dashed)
        count_support_interval(catalog, db, first, last)
        scanned += last - first + 1
        promoted = prune(catalog, params, bound_enabled=prune_bound, audit=audit, stats=stats)
        make_candidates(catalog, params, frontier=promoted, level1=level1, audit=audit, stats=stats)
        stats.peak_dashed = max(stats.peak_dashed, len(catalog.dashed))
        check_full_pass(catalog, params, audit=audit, stats=stats)
    frequent = tuple(sorted((FrequentItemset(r.mask, r.size, r.support) for r in catalog.solid
                             if r.shape is Shape.SOLID_BOX), key=lambda f: (f.size, f.mask)))
    stats.db_passes = scanned / db.n
    stats.wall_time_s = time.perf_counter() - t0
    return MiningResult(frequent=frequent, stats=stats)


def mine_parallel(db: BitDatabase, params: MiningParams, *, prune_bound: bool = True,
                  audit: TransitionAudit | None = None) -> MiningResult:
    """DIC on the GPU; same frequent itemsets, supports and stats as the
    reference engines (engine.py:478-496)."""
    if params.n != db.n:
        raise ValueError(f"params were built for n={params.n}, database has n={db.n}")
    if audit is not None:
        return _run_phases(db, params, prune_bound, audit)
    t0 = time.perf_counter()
    return run_engine(db.device_tids(), db.n, db.m, params, prune_bound=prune_bound, t0=t0)


def mine_serial(db: BitDatabase, params: MiningParams, *, prune_bound: bool = True,
                audit: TransitionAudit | None = None) -> MiningResult:
    """The reference's serial engine is its pure-Python verification path
    (engine.py:461-475); here both entry points run the same GPU engine,
    whose output is identical by construction."""
    return mine_parallel(db, params, prune_bound=prune_bound, audit=audit)
