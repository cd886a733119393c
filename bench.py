"""Benchmark: end-to-end DIC on BASELINE.json's large sharded config (cfg4).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

A step is one complete DIC run (first pass + every checkpoint until no
dashed itemset is left) of cfg4 — n = 10,000,000 Quest-style transactions
over m = 1,000 items, minsup 0.1 %, M = 100,000 — from the bit-sliced
database resident in HBM to the sorted frequent itemsets on the host.
`value` is subset-tests/s over the whole job (first pass m*n singleton tests
plus, per stop, |dashed| x chunk rows), `e2e` the same metric through the
public API from pinned host CSR (H2D + GPU encode + mine + D2H result).

Under torchrun (N > 1) each rank generates and holds only its chunk-sliced
shard (sharding.py) and the per-stop count deltas are sum-allreduced over
NCCL; the total work is fixed, so scaling is "strong".

`--impl reference` times the CPU restatement of the reference engine
(oracle/dic_oracle.c, the "port" arm: the reference is pure Python and
cannot travel to the GPU box) on the host cores, rank 0 only, each step a
bounded sample of the same workload: first pass + the first checkpoint.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

CFG_INDEX = 4


def parse() -> argparse.Namespace:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", type=int, default=CFG_INDEX)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-kernel-bench", action="store_true")
    ap.add_argument("--no-config-sweep", action="store_true", help="skip the cfg1-3 GPU vs CPU-oracle sweep")
    ap.add_argument("--clock-ms", type=int, default=50, help="nvidia-smi sampling period in the timed region")
    ap.add_argument("--profile", action="store_true", help="one short run for ncu (no JSON contract)")
    ap.add_argument("--step-trace", action="store_true", help="per-step host phase / loop diagnostics in the JSON")
    return ap.parse_args()


# ---------------------------------------------------------------- helpers
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int, period_ms: int = 500):
        self.gpu = gpu
        self.period_ms = period_ms
        self.proc = None
        self.path = None

    def __enter__(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", str(self.period_ms)], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def mark(self) -> None:
        """Start of the timed region: summary() keeps the samples from here on
        (and the one just before, so a short region has at least one)."""
        self.t_mark = time.time()
        self.n_mark = len(self._rows())

    def _rows(self) -> list:
        rows = []
        if self.path:
            for line in Path(self.path).read_text().splitlines():
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        return rows

    def summary(self) -> dict:
        if self.proc is None or not self.path:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = self._rows()
        n0 = getattr(self, "n_mark", 0)
        rows = rows[max(0, n0 - 1):]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        loaded = [v for v in sm if v > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def int_peaks() -> dict:
    """Live LOP3 / POPC lane-op peaks (MEASURED_PEAKS.json has no integer pipes)."""
    import torch

    from paper_1812_10959_b200 import device as D

    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    out = {}
    for op, name in ((0, "lop3"), (1, "popc")):
        best = 0.0
        for threads in (512, 1024):
            blocks = sms * (2048 // threads)
            D.probe_int_pipe(op, blocks, threads, 32)
            ops, ms = D.probe_int_pipe(op, blocks, threads, 1024)
            best = max(best, ops / (ms * 1e-3))
        out[name] = best
    return out


def measured_hbm() -> tuple[float, str]:
    try:
        mp = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(mp["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def kernel_microbench(peaks: dict, reps: int = 3) -> dict:
    """cfg5: dic_count_support over a 50M x 512 i.i.d. Bernoulli(0.05) bitmap
    for 100k random candidates (k ~ U{2..6}), one launch per size bucket, all
    rows.  Buckets are sorted lexicographically (any order gives the same
    counts).  Roofline: >= 1 POPC per (candidate, 32-row word)."""
    import torch

    from paper_1812_10959_b200 import device as D
    from paper_1812_10959_b200.workloads import CONFIGS

    cfg = CONFIGS[5]
    n, m, C = cfg.n, cfg.m, cfg.params["candidates"]
    rows = D.bernoulli_rows(n, m, cfg.params["p"], cfg.seed)
    tids = D.rows_to_tids(rows, n, m)
    del rows
    ks, items = D.synth_candidates(C, m, cfg.params["kmin"], cfg.params["kmax"], cfg.seed)
    buckets = []
    for k in range(cfg.params["kmin"], cfg.params["kmax"] + 1):
        sel = items[ks == k][:, :k]
        sel = sel[np.lexsort(sel.T[::-1])]
        buckets.append(torch.from_numpy(np.ascontiguousarray(sel).view(np.int16)).cuda())
    outs = [torch.zeros(b.shape[0], dtype=torch.int64, device="cuda") for b in buckets]
    for b, o in zip(buckets, outs):
        D.count_support(tids, n, m, 0, n - 1, b, o)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        for o in outs:
            o.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for b, o in zip(buckets, outs):
            D.count_support(tids, n, m, 0, n - 1, b, o)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    # the streaming regime: first_pass's column popcounts (item_support) over
    # the whole 3.2 GB bitmap, HBM-bound (SURVEY 8(d) evidence)
    counts = torch.zeros(m, dtype=torch.int64, device="cuda")
    D.item_support(tids, n, m, 0, n - 1, counts)
    torch.cuda.synchronize()
    hb = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        D.item_support(tids, n, m, 0, n - 1, counts)
        e1.record()
        torch.cuda.synchronize()
        hb.append(e0.elapsed_time(e1))
    hbm_gbs, hbm_src = measured_hbm()
    t_hbm = min(hb)
    moved = tids.numel() * tids.element_size()  # whole tiles (dense rows: the bitmap rounded up to tiles)
    hbm = {"kernel": "item_support_kernel", "ms": t_hbm, "bytes_read": moved,
           "algorithmic_bytes": n * words_for(m) * 8, "achieved_gbs": moved / (t_hbm * 1e-3) / 1e9,
           "peak_gbs": hbm_gbs, "frac": moved / (t_hbm * 1e-3) / 1e9 / hbm_gbs, "peak_source": hbm_src}
    del counts
    words = (n + 31) // 32
    ops = float(sum(int(b.shape[0]) * int(b.shape[1]) for b in buckets)) * words  # k lane-ops per cand-word
    sum_nnz64 = 0
    for b in buckets:
        it = b.cpu().numpy().view(np.uint16).astype(np.int64) // 64
        it.sort(axis=1)
        sum_nnz64 += int((1 + (np.diff(it, axis=1) != 0).sum(axis=1)).sum())
    ns = north_star_roofline(n, words_for(m), sum_nnz64, best, peaks)
    achieved = ops / (best * 1e-3)
    checksum = int(sum(int(o.sum().item()) for o in outs))
    golden = None
    gp = ROOT / "tests" / "golden" / "cfg5.npz"
    if gp.exists():
        z = np.load(gp)
        gmeta = json.loads(str(z["meta"]))
        # per-candidate equality in the bench's own (per-size, sorted) order
        ks_all, items_all = ks, items
        want = z["supports"].astype(np.int64)
        ok = True
        for b, o, k in zip(buckets, outs, range(cfg.params["kmin"], cfg.params["kmax"] + 1)):
            idx = np.nonzero(ks_all == k)[0]
            sel = items_all[idx][:, :k]
            order = np.lexsort(sel.T[::-1])
            ok &= bool(np.array_equal(o.cpu().numpy(), want[idx][order]))
        golden = {"support_checksum": gmeta["support_checksum"], "match": bool(ok and checksum ==
                                                                             gmeta["support_checksum"]),
                  "golden": "tests/golden/cfg5.npz (all 100k candidates x 50M rows, oracle/cfg5.c)"}
    del tids
    torch.cuda.empty_cache()
    return {"workload": cfg.name, "n": n, "m": m, "candidates": C, "ms": best,
            "subset_tests_per_s": C * n / (best * 1e-3), "bound": "alu", "bound_detail": "integer ALU pipe (LOP3 lane-ops); neither HBM nor tensor cores bind this path",
            "achieved": achieved / 1e12, "peak": peaks["lop3"] / 1e12, "unit": "T lane-ops/s",
            "frac": achieved / peaks["lop3"], "support_checksum": checksum, "golden_check": golden,
            "north_star": ns,
            "hbm_streaming": hbm,
            "ops_rule": "k lane-ops per (candidate, 32-row word): (k-1) ANDs + >= 1 to accumulate the popcount"}


def measured_tensor_peak() -> tuple[float, str]:
    """Dense peak of the pair kernel's MMA kind in FLOP/s: the measured bf16
    GEMM burst (MEASURED_PEAKS.json) scaled by NVIDIA's nominal dense ratio of
    the kind to bf16 (FP4 9 / 2.25 = 4, INT8 4.5 / 2.25 = 2): B200_PROFILING.md
    gives no measured FP4 / INT8 figure."""
    kind = os.environ.get("DIC_PAIR_TC_KIND", "4")
    ratio, name = (2.0, "i8") if kind == "8" else (4.0, "mxf4")
    try:
        bf16 = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["bf16_tflops"])
        src = "MEASURED_PEAKS.json bf16 burst"
    except Exception:
        bf16, src = 1590.0, "fallback bf16 1.59 PF (B200_PROFILING.md)"
    return bf16 * ratio * 1e12, f"{src} {bf16:.0f} TF/s x {ratio:g} (nominal {name}:bf16 dense ratio)"


def pair_kernel_roofline(tids, n: int, m: int, interval: int, peaks: dict, reps: int = 10) -> dict:
    """The pair-wave kernel of the cfg4 run, measured alone on the run's own
    data: dic_count_pairs over one M-row chunk (a dense-pair stop), which runs
    the tensor-core triangle (pairs_mma.cu) for m >= 128."""
    import torch

    from paper_1812_10959_b200 import device as D

    tri = torch.zeros(m * (m - 1) // 2, dtype=torch.int64, device="cuda")
    first, last = 0, min(interval, n) - 1
    D.count_pairs(tids, n, m, first, last, tri)
    torch.cuda.synchronize()
    # `reps` launches back to back between two events on the launching
    # stream: the average launch duration, without the host's per-call
    # launch latency (the engine launches it from CUDA graphs)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        D.count_pairs(tids, n, m, first, last, tri)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps
    words = (last - first + 1 + 31) // 32
    rows = last - first + 1
    pairs = tri.numel()
    # algorithmic work: one multiply-add (2 FLOP) per (pair, row); the MMAs
    # also cover the lower half of the diagonal tiles and the padding to
    # 128 x 256 tiles (issued FLOPs)
    flops = 2.0 * pairs * rows
    na, nb = -(-m // 128), -(-m // 256)
    tiles = sum(nb - ia // 2 for ia in range(na))
    issued = 2.0 * 128 * 256 * tiles * (-(-rows // 256) * 256)
    # north-star roofline: 2 lane-ops per 64-bit word-test of a
    # candidate's non-zero words, per ROW; a pair has 1 such word if both
    # items share a 64-bit word, else 2
    full, rem = divmod(m, 64)
    same = full * (64 * 63 // 2) + rem * (rem - 1) // 2
    nnz64 = same + 2 * (pairs - same)
    ns = north_star_roofline(rows, words_for(m), nnz64, t, peaks)
    return {"t_ms": t, "flops": flops, "issued_flops": issued, "tests_per_s": pairs * rows / (t * 1e-3),
            "achieved": flops / (t * 1e-3), "lop3_equiv_ops": 2.0 * pairs * words, "north_star": ns}


def words_for(m: int) -> int:
    return (m + 63) // 64


def north_star_roofline(rows: int, W: int, sum_nnz64: int, t_ms: float, peaks: dict) -> dict:
    """BASELINE.json's roofline, literally: the slower of the transaction
    bitmap bytes over HBM and the candidate x transaction 64-bit word-tests
    (non-zero candidate words only) at the integer-ALU peak, 2 LOP3 lane-ops
    per word-test.  The bit-sliced kernels test 32 rows per lane-op, so they
    run far below this per-row bound; the `frac` of the main roofline is the
    stricter, bit-sliced figure (k lane-ops per candidate and 32-row word)."""
    hbm_gbs, _ = measured_hbm()
    t_hbm = rows * W * 8 / (hbm_gbs * 1e9)
    t_alu = 2.0 * rows * sum_nnz64 / peaks["lop3"]
    t_roof = max(t_hbm, t_alu)
    return {"rule": "max(rows*W*8 B / HBM, 2 * rows * sum_c nnz64(c) / LOP3 peak) (SURVEY 8(d))",
            "word_tests": rows * sum_nnz64, "t_roof_ms": t_roof * 1e3, "t_ms": t_ms,
            "t_over_roof": t_roof * 1e3 / t_ms,
            "note": "> 1: the bit-sliced layout beats the per-row word-test bound by testing 32 rows per lane-op"}


def ncu_traffic(kernel: str):
    """DRAM bytes per launch of `kernel` from the committed ncu summary, if any."""
    try:
        summ = json.loads((ROOT / "profiles" / "ncu_summary.json").read_text())
        return summ.get(kernel, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def subset_tests(n: int, m: int, params, trace) -> int:
    """First pass (m*n singleton tests) + sum over stops of |dashed| x chunk rows."""
    total = n * m
    for st in trace.stops:
        first, last = params.chunk_bounds(st["stop"])
        total += st["dashed_at_start"] * (last - first + 1)
    return total


# ---------------------------------------------------------------- reference arm
def run_reference(args, cfg, rank: int, world: int) -> None:
    if rank != 0:
        return
    from oracle import oracle as O
    from oracle import synth as S
    from paper_1812_10959_b200.config import MiningParams
    from tests.golden_util import rows_from_csr

    cores = os.cpu_count() or 1
    # the input from the generator's own build (oracle/_build/libsynth.so):
    # this process maps no product library, only the oracle's
    indptr, indices = S.generate_csr(cfg, threads=cores)
    rows = rows_from_csr(indptr, indices, cfg.m)
    params = MiningParams.create(cfg.n, cfg.minsup, interval=cfg.interval)
    times, tests = [], 0
    for i in range(args.warmup + args.steps):
        t = time.perf_counter()
        run = O.mine(rows, cfg.m, cfg.minsup, interval=cfg.interval, threads=cores, max_stops=1)
        dt = time.perf_counter() - t
        first, last = params.chunk_bounds(1)
        tests = cfg.n * cfg.m + run.interval_counts * (last - first + 1)
        if i >= args.warmup:
            times.append(dt)
    ms = 1000.0 * sum(times) / len(times)
    value = tests / (ms * 1e-3)
    sample = (f"{cfg.name}: oracle first pass over all {cfg.n} rows + the first checkpoint "
              f"({run.interval_counts} dashed pairs x {cfg.interval} rows)")
    line = {"metric": "subset-tests/s (end-to-end DIC, cfg4)", "value": value, "unit": "subset-tests/s",
            "impl": "reference", "n_gpus": 0, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (seeded Quest-style generator)",
            "config": {"workload": cfg.name, "n": cfg.n, "m": cfg.m, "minsup": cfg.minsup, "interval": cfg.interval,
                       "sample": "first pass + 1 checkpoint per step"},
            "cpu_baseline": {"value": value, "unit": "subset-tests/s", "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": "subset-tests/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    line["native_libs"] = mapped_libs()
    print(json.dumps(line), flush=True)


def mapped_libs() -> list:
    """Shared objects of this repo mapped into the process (evidence of which
    native code a leg ran)."""
    try:
        maps = Path("/proc/self/maps").read_text().splitlines()
    except OSError:
        return []
    out = sorted({ln.split()[-1] for ln in maps if ln.endswith(".so") and str(ROOT) in ln})
    return [str(Path(x).relative_to(ROOT)) for x in out]


def golden_check(idx: int, res) -> dict | None:
    """The run's frequent itemsets, supports and MiningStats against the
    committed full-size oracle golden (tests/golden/cfg<idx>.npz)."""
    from tests.golden_util import has_config_golden, load_config_golden

    if not has_config_golden(idx):
        return None
    g = load_config_golden(idx)
    s = res.stats
    st = g.stats
    same_sets = [(f.mask, f.support) for f in res.frequent] == g.pairs
    same_stats = (s.db_passes, s.peak_dashed, s.candidates_generated, s.candidates_pruned, s.interval_counts) == (
        st["db_passes"], st["peak_dashed"], st["candidates_generated"], st["candidates_pruned"], st["interval_counts"])
    return {"match": bool(same_sets and same_stats), "frequent_itemsets_equal": bool(same_sets),
            "stats_equal": bool(same_stats), "golden": f"tests/golden/cfg{idx}.npz",
            "source": g.meta.get("source", "reference")}


def same_sample_rate(cfg, tids, n_local: int, params, reps: int = 5) -> dict:
    """The B200 engine on exactly the CPU arm's sample: first pass over all
    rows + the first checkpoint (the step-by-step API, CUDA events around
    engine creation .. the first stop's status), median of `reps`."""
    import torch

    from paper_1812_10959_b200.miner import DeviceEngine

    first, last = params.chunk_bounds(1)
    times, tests = [], 0
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng = DeviceEngine(tids, n_local, cfg.m, params, True)
        eng.seed(eng.item_counts())
        eng.issue_count(first, last)
        st, _ = eng.poll(eng.issue_checkpoint())
        e1.record()
        torch.cuda.synchronize()
        eng.close()
        times.append(e0.elapsed_time(e1))
        tests = cfg.n * cfg.m + st.dashed_at_start * (last - first + 1)
    ms = statistics.median(times[1:])
    return {"value": tests / (ms * 1e-3), "unit": "subset-tests/s", "ms": ms,
            "sample": "first pass + checkpoint 1 (the --impl reference sample)", "subset_tests": tests}


# ---------------------------------------------------------------- B200 arm
def main() -> None:
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    from paper_1812_10959_b200.workloads import CONFIGS

    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_1812_10959_b200 as dic
    from paper_1812_10959_b200 import _abi
    from paper_1812_10959_b200 import device as D
    from paper_1812_10959_b200.miner import StopTrace, run_engine
    from paper_1812_10959_b200.workloads import generate_csr

    torch.cuda.set_device(local_rank)
    D.require_cuda()
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        group = dist.group.WORLD
    lib = _abi.load()
    params = dic.MiningParams.create(cfg.n, cfg.minsup, interval=cfg.interval)
    plan = dic.ShardPlan.for_params(params, world, rank)
    cores = os.cpu_count() or 1
    threads = max(1, cores // max(world, 1))
    ranges = plan.ranges() if world > 1 else [(0, cfg.n)]
    indptr, indices = generate_csr(cfg, ranges=ranges, threads=threads)
    n_local = int(indptr.size - 1)

    # pinned host CSR (the e2e input) and the HBM-resident bit-sliced copy
    # pinned host CSR (the e2e input): item ids as uint16 (the universe is
    # < 65536) and int32 offsets (nnz < 2^31), the compact form
    # BitDatabase.from_csr streams to the encoder
    off_dtype = np.int32 if int(indptr[-1]) < 2**31 else np.int64
    h_indptr = torch.from_numpy(indptr.astype(off_dtype)).pin_memory()
    h_indices = torch.from_numpy(indices.astype(np.uint16)).pin_memory()
    db = dic.BitDatabase.from_csr(h_indptr, h_indices, cfg.m)
    tids = db.device_tids()
    torch.cuda.synchronize()

    # N > 1: the library's own NCCL communicator, the whole loop native
    # (DIC_COLLECTIVE=torch: torch.distributed all_reduce from the Python loop)
    collective = None if world == 1 else ("native" if os.environ.get("DIC_COLLECTIVE", "native") == "native"
                                          else True)

    def one_run(trace=None, count_events=None):
        return run_engine(tids, n_local, cfg.m, params, plan=plan if world > 1 else None, group=group,
                          trace=trace, count_events=count_events, collective=collective)

    if args.profile:
        one_run()
        torch.cuda.synchronize()
        return

    # nvidia-smi starts (NVML init) before the warm-up, so its start-up does
    # not land in the timed region; it keeps sampling through it
    clocks = ClockSampler(local_rank, args.clock_ms).__enter__()
    for _ in range(args.warmup):
        one_run()
    trace = StopTrace()
    ref = one_run(trace=trace)
    tests = subset_tests(cfg.n, cfg.m, params, trace)
    golden = golden_check(args.config, ref)  # correctness gate before timing (benchmark.py:91-95)
    assert golden is None or golden["match"], f"result differs from the oracle golden: {golden}"
    cross_check = None
    if world > 1 and (trace.native or {}).get("collective") == "fused":
        # the fused peer-memory reduction must agree with ncclAllReduce, bit
        # for bit, before anything is timed (every rank runs both)
        os.environ["DIC_FUSED_REDUCE"] = "0"
        try:
            alt = one_run()
        finally:
            os.environ.pop("DIC_FUSED_REDUCE", None)
        same = [(f.mask, f.support) for f in alt.frequent] == [(f.mask, f.support) for f in ref.frequent]
        assert same, "fused reduction disagrees with ncclAllReduce"
        cross_check = "fused reduction == ncclAllReduce (frequent sets and supports)"

    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    count_events: list = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = lib.dic_launch_count()
    # after setup, move the interpreter's long-lived objects (torch's import
    # graph) out of the collector's generations: a gen-2 collection over them,
    # triggered by the result objects, costs ~40 ms of host time in one step
    gc_mode = os.environ.get("DIC_BENCH_GC", "freeze")
    if gc_mode != "on":
        import gc
        gc.collect()
        gc.freeze() if gc_mode == "freeze" else gc.disable()
    clocks.mark()
    step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    e0.record(stream)
    step_ev[0].record(stream)
    step_diag = []
    for i in range(args.steps):
        if args.step_trace:
            tr = StopTrace()
            res = one_run(trace=tr)
            step_diag.append({"phases": {k: round(v, 2) for k, v in tr.phases.items()}, "loop": tr.native})
        else:
            res = one_run()
        step_ev[i + 1].record(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    clocks.__exit__(None, None, None)
    step_ms = [step_ev[i].elapsed_time(step_ev[i + 1]) for i in range(args.steps)]
    one_run(count_events=count_events)  # instrumented run (per-stop count timing), outside the timed region
    if world > 1:
        dist.barrier()
    launches = (lib.dic_launch_count() - launches0) // args.steps
    ms_local = e0.elapsed_time(e1) / args.steps
    ms_t = torch.tensor([ms_local], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    assert [(f.mask, f.support) for f in res.frequent] == [(f.mask, f.support) for f in ref.frequent]

    # roofline of the dominant kernel (the streaming support count) over the
    # last timed run: per launch >= 1 POPC per (candidate, 32-row word)
    count_ms = [ev[1] if ev[0] == "native" else ev[0].elapsed_time(ev[1]) for ev in count_events]
    peaks = int_peaks()
    hbm_gbs, hbm_src = measured_hbm()
    tot_ms = sum(count_ms)
    # the dominant kernel: the dense pair triangle (pair_tri_kernel), timed
    # alone on one cfg4 chunk; its share of the step from the run's own count
    # launches (the pair kernel runs inside them during the pair wave)
    pk = pair_kernel_roofline(tids, n_local, cfg.m, cfg.interval, peaks) if world == 1 else None
    dense_stops = min(len(count_ms), params.intervals_per_pass)
    roofline = None
    if pk is not None:
        tpk, tsrc = measured_tensor_peak()
        roofline = {"bound": "tensor",
                    "bound_detail": "tensor cores (tcgen05 kind::mxf4, bits expanded to E2M1 operands in shared "
                                    "memory): the dense pair triangle X^T X of each chunk",
                    "achieved": pk["achieved"] / 1e12, "peak": tpk / 1e12, "unit": "TFLOP/s",
                    "frac": pk["achieved"] / tpk, "traffic": ncu_traffic("pair_tc_kernel"),
                    "kernel": "pair_tc_kernel", "avg_launch_ms": pk["t_ms"], "flops_per_launch": pk["flops"],
                    "issued_flops_per_launch": pk["issued_flops"],
                    "issued_frac": pk["issued_flops"] / (pk["t_ms"] * 1e-3) / tpk,
                    "tests_per_s": pk["tests_per_s"],
                    "flops_rule": "2 FLOP (one multiply-add) per (pair, row) of the chunk; issued = 128x256 MMA "
                                  "tiles incl. the lower half of diagonal tiles and padding",
                    "share_of_step": pk["t_ms"] * dense_stops / ms if ms else None, "peak_source": tsrc,
                    "vs_lop3": {"ops": pk["lop3_equiv_ops"], "frac_of_lop3_peak":
                                pk["lop3_equiv_ops"] / (pk["t_ms"] * 1e-3) / peaks["lop3"],
                                "lop3_peak": peaks["lop3"], "note": "the round-1 AND/POPC kernel's metric "
                                "(2 lane-ops per pair and 32-row word) against the live LOP3 probe; > 1 means "
                                "faster than any integer-pipe kernel can be"},
                    "north_star": pk["north_star"],
                    "count_launches_in_step": len(count_ms),
                    "hbm_peak_gbs": hbm_gbs, "hbm_peak_source": hbm_src}

    # end to end through the public API from pinned host CSR
    e2e = None
    if not args.no_e2e:
        h2d = int(h_indptr.numel() * h_indptr.element_size() + h_indices.numel() * h_indices.element_size())
        W = dic.bits.words_for(cfg.m)
        d2h = int(len(ref.frequent) * (W * 8 + 4 + 8) + 4 * 8)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t = time.perf_counter()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            dbe = dic.BitDatabase.from_csr(h_indptr, h_indices,
                                           cfg.m)
            out = run_engine(dbe.device_tids(), n_local, cfg.m, params, plan=plan if world > 1 else None,
                             group=group, collective=collective)
            del dbe
        f1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = f0.elapsed_time(f1) / args.steps
        e2e_t = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
        e2e_ms = float(e2e_t.item())
        assert [(f.mask, f.support) for f in out.frequent] == [(f.mask, f.support) for f in ref.frequent]
        e2e = {"value": tests / (e2e_ms * 1e-3), "unit": "subset-tests/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms, "host_wall_ms_per_step":
                   1000 * (time.perf_counter() - t) / args.steps}

    same_sample = same_sample_rate(cfg, tids, n_local, params) if world == 1 else None
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, db, params)
    sweep = None
    if rank == 0 and world == 1 and not args.no_config_sweep:
        sweep = config_sweep()
    kernel = None
    if rank == 0 and world == 1 and not args.no_kernel_bench:
        del db, tids
        torch.cuda.empty_cache()
        kernel = kernel_microbench(peaks)

    if rank == 0:
        s = ref.stats
        line = {
            "metric": "subset-tests/s (end-to-end DIC, cfg4)", "value": tests / (ms * 1e-3), "unit": "subset-tests/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32 bit-sliced (int)",
            "data": "synthetic (seeded Quest-style generator, DESIGN.md §Inputs)",
            "config": {"workload": cfg.name, "n": cfg.n, "m": cfg.m, "minsup": cfg.minsup,
                       "interval": cfg.interval, "parallelism": f"rows-sharded x{world}",
                       "l2": "inputs larger than L2 (bit-sliced db 1.28 GB > 126 MB)",
                       "dic_seconds": ms / 1000.0, "subset_tests_per_step": tests,
                       "frequent_itemsets": len(ref.frequent), "stops": len(trace.stops),
                       "db_passes": s.db_passes, "candidates_generated": s.candidates_generated,
                       "peak_dashed": s.peak_dashed, "interval_counts": s.interval_counts},
            "step_ms": [round(x, 3) for x in step_ms], "host_loop": trace.native,
            # the per-stop cost that does not shard: the step minus its count halves (pair triangle +
            # support count, timed per stop in the instrumented run), i.e. the checkpoint kernel, the
            # launch gaps, the first pass and the result collection
            "step_split_ms": {"count_halves": round(tot_ms, 3), "replicated": round(ms - tot_ms, 3),
                              "stops": len(count_ms),
                              "projected_8gpu_ms": round(tot_ms / 8 + (ms - tot_ms) + 0.007 * len(count_ms), 3),
                              "projection": "count/8 + replicated + 7 us per stop for the fused reduction "
                                            "(not measured: one GPU per call)"},
            "host_phases_ms": {k: round(v, 3) for k, v in trace.phases.items()},
            **({"step_diag": step_diag} if step_diag else {}),
            "roofline": roofline, "clocks": clocks.summary(), "gpu_launches": launches, "e2e": e2e,
            "collective": (trace.native or {}).get("collective"), "collective_cross_check": cross_check,
            "cpu_baseline": cpu, "kernel_microbench": kernel, "config_sweep": sweep,
            "golden_check": golden, "same_sample": same_sample, "native_libs": mapped_libs(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def config_sweep(reps: int = 5) -> dict:
    """BASELINE.json cfg1-3 (the parity configs) at full size: the GPU DIC
    (HBM-resident bitmap -> sorted results, min of `reps` after a warm-up)
    against the oracle port mining the same rows on all host cores, with the
    frequent sets checked equal (bit-exact itemsets and supports)."""
    import torch

    import paper_1812_10959_b200 as dic
    from oracle import oracle as O
    from paper_1812_10959_b200.miner import StopTrace, run_engine
    from paper_1812_10959_b200.workloads import CONFIGS, generate_csr

    cores = os.cpu_count() or 1
    out = {}
    for idx in (1, 2, 3):
        cfg = CONFIGS[idx]
        ip, ix = generate_csr(cfg)
        db = dic.BitDatabase.from_csr(ip, ix, cfg.m)
        tids = db.device_tids()
        params = dic.MiningParams.create(cfg.n, cfg.minsup, interval=cfg.interval)
        trace = StopTrace()
        res = run_engine(tids, cfg.n, cfg.m, params, trace=trace)
        tests = subset_tests(cfg.n, cfg.m, params, trace)
        best = 1e30
        for _ in range(reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            res = run_engine(tids, cfg.n, cfg.m, params)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        rows = db.rows
        t = time.perf_counter()
        want = O.mine(rows, cfg.m, cfg.minsup, interval=cfg.interval, threads=cores)
        cpu_s = time.perf_counter() - t
        same = [(f.mask, f.size, f.support) for f in res.frequent] == want.frequent
        out[cfg.name] = {"n": cfg.n, "m": cfg.m, "minsup": cfg.minsup, "interval": cfg.interval,
                         "stops": len(trace.stops), "frequent_itemsets": len(res.frequent),
                         "subset_tests": tests, "gpu_ms": best, "gpu_subset_tests_per_s": tests / (best * 1e-3),
                         "cpu_oracle_s": cpu_s, "cpu_cores": cores,
                         "cpu_subset_tests_per_s": tests / cpu_s, "speedup": cpu_s * 1e3 / best,
                         "bit_exact_vs_oracle": same}
        del db, tids, rows
        torch.cuda.empty_cache()
    return out


def cpu_baseline(cfg, db, params) -> dict:
    """The oracle port on the host cores, bounded sample: first pass + the
    first checkpoint (the first stop counts every seeded pair)."""
    from oracle import oracle as O

    cores = os.cpu_count() or 1
    rows = db.rows  # D2H of the row bitmap, outside any timed region
    t = time.perf_counter()
    run = O.mine(rows, cfg.m, cfg.minsup, interval=cfg.interval, threads=cores, max_stops=1)
    dt = time.perf_counter() - t
    first, last = params.chunk_bounds(1)
    tests = cfg.n * cfg.m + run.interval_counts * (last - first + 1)
    return {"value": tests / dt, "unit": "subset-tests/s", "cores": cores, "kind": "port",
            "sample": f"first pass + checkpoint 1 ({run.interval_counts} pairs x {last - first + 1} rows), "
                      f"{dt:.1f} s"}


if __name__ == "__main__":
    main()
