"""Per-kernel breakdown of one DIC run (torch.profiler / CUPTI; no nsys
needed): kernel name, launches, total and mean device time, and the share of
the run's wall time the GPU was busy.  Prints a table and writes JSON."""

from __future__ import annotations

import json
import sys
import time
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1812_10959_b200 as dic  # noqa: E402
from paper_1812_10959_b200 import device as D  # noqa: E402
from paper_1812_10959_b200.miner import StopTrace, run_engine  # noqa: E402
from paper_1812_10959_b200.workloads import CONFIGS, generate_csr  # noqa: E402


def main() -> None:
    idx = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    depth = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    out_json = sys.argv[3] if len(sys.argv) > 3 else None
    cfg = CONFIGS[idx]
    D.require_cuda()
    ip, ix = generate_csr(cfg)
    db = dic.BitDatabase.from_csr(ip, ix, cfg.m)
    tids = db.device_tids()
    params = dic.MiningParams.create(cfg.n, cfg.minsup, interval=cfg.interval)
    run_engine(tids, cfg.n, cfg.m, params, depth=depth)  # warm-up
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        t = time.perf_counter()
        trace = StopTrace()
        res = run_engine(tids, cfg.n, cfg.m, params, depth=depth, trace=trace)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t
    agg = defaultdict(lambda: [0, 0.0])
    busy = 0.0
    for ev in prof.events():
        if ev.device_type.name != "CUDA":
            continue
        a = agg[ev.name[:90]]
        a[0] += 1
        a[1] += ev.device_time_total / 1000.0  # us -> ms
        busy += ev.device_time_total / 1000.0
    rows = sorted(agg.items(), key=lambda kv: -kv[1][1])
    # timeline: idle gaps between consecutive device activities
    acts = sorted((ev.time_range.start, ev.time_range.end, ev.name[:40]) for ev in prof.events()
                  if ev.device_type.name == "CUDA")
    gaps = []
    for (s0, e0, n0), (s1, e1, n1) in zip(acts, acts[1:]):
        if s1 > e0:
            gaps.append((s1 - e0, n0, n1))
    span = (acts[-1][1] - acts[0][0]) / 1000.0 if acts else 0.0
    idle = sum(g for g, _, _ in gaps) / 1000.0
    print(f"device span {span:.1f} ms, idle inside the span {idle:.1f} ms over {len(gaps)} gaps")
    hist = defaultdict(lambda: [0, 0.0])
    for g, n0, n1 in gaps:
        key = (n0.split("(")[0][-28:], n1.split("(")[0][-28:])
        hist[key][0] += 1
        hist[key][1] += g / 1000.0
    for (n0, n1), (c, ms) in sorted(hist.items(), key=lambda kv: -kv[1][1])[:12]:
        print(f"  gap {ms:7.3f} ms {c:5d} x {ms / c * 1000:8.2f} us  {n0} -> {n1}")
    # per-launch duration series of the per-stop kernels (stop order)
    series = defaultdict(list)
    for s0, e0, n0 in acts:
        for key in ("count_dev", "eval_cand", "apply_prune", "pair_tri", "pair_tc", "dedup", "commit_status", "checkpoint_kernel",
                    "compact", "status_kernel", "checkpoint_batch"):
            if key in n0:
                series[key].append(round(e0 - s0, 1))
    for key, v in series.items():
        chunks = [v[i:i + 25] for i in range(0, len(v), 25)]
        print(f"  {key:12s} us per 25-stop window (mean):", [round(sum(c) / len(c), 1) for c in chunks])
    d = [st["dashed_at_start"] for st in trace.stops]
    print("  dashed       per 25-stop window (mean):", [round(sum(d[i:i + 25]) / len(d[i:i + 25])) for i in range(0, len(d), 25)])
    top = sorted(gaps, reverse=True)[:8]
    print("  largest:", [(round(g / 1000.0, 3), a.split("(")[0][-24:], b.split("(")[0][-24:]) for g, a, b in top])
    print(f"{cfg.name}: wall {wall * 1000:.1f} ms, GPU busy {busy:.1f} ms, frequent {len(res.frequent)}")
    for name, (n, ms) in rows[:25]:
        print(f"{ms:9.3f} ms {n:6d} x {ms / n * 1000:9.2f} us  {name}")
    if out_json:
        Path(out_json).write_text(json.dumps({"config": cfg.name, "depth": depth, "wall_ms": wall * 1000,
                                              "gpu_busy_ms": busy, "series_us": series,
                                              "dashed": d,
                                              "kernels": [{"name": k, "launches": n, "total_ms": ms}
                                                          for k, (n, ms) in rows]}, indent=1))


if __name__ == "__main__":
    main()
