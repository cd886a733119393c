"""One dic_count_pairs launch on a cfg4-shaped chunk (m = 1000 items, 100k
rows of the Quest data) — the target for `ncu -k regex:pair_tri`.  Also
prints its CUDA-event time and rate."""

from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1812_10959_b200 import device as D  # noqa: E402
from paper_1812_10959_b200.workloads import CONFIGS, generate_csr, scaled  # noqa: E402


def main() -> None:
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    cfg = scaled(CONFIGS[4], 1_000_000)
    ip, ix = generate_csr(cfg)
    rows, _ = D.encode_csr(torch.from_numpy(ip).cuda(), torch.from_numpy(ix).cuda(), cfg.n, cfg.m)
    tids = D.rows_to_tids(rows, cfg.n, cfg.m)
    tri = torch.zeros(cfg.m * (cfg.m - 1) // 2, dtype=torch.int64, device="cuda")
    first, last = 0, 99_999
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        D.count_pairs(tids, cfg.n, cfg.m, first, last, tri)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    tests = tri.numel() * (last - first + 1)
    print(f"pairs {tri.numel()} x {last - first + 1} rows: {best:.3f} ms, {tests / (best * 1e-3):.3e} tests/s")


if __name__ == "__main__":
    main()
