"""One dic_count_pairs launch on a cfg4-shaped chunk (m = 1000 items, 100k
rows of the Quest data) — the target for `ncu -k regex:pair_`.  Prints the
CUDA-event time and rate of each pair kernel (tensor cores, AND/POPC), timed
over back-to-back launches.

    python tools/pair_kernel_probe.py [reps] [modes: 2,1]
"""

from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1812_10959_b200 import device as D  # noqa: E402
from paper_1812_10959_b200.workloads import CONFIGS, generate_csr, scaled  # noqa: E402


def main() -> None:
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    modes = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [2, 1]
    cfg = scaled(CONFIGS[4], 1_000_000)
    ip, ix = generate_csr(cfg)
    rows, _ = D.encode_csr(torch.from_numpy(ip).cuda(), torch.from_numpy(ix).cuda(), cfg.n, cfg.m)
    tids = D.rows_to_tids(rows, cfg.n, cfg.m)
    first, last = 0, 99_999
    ref = None
    for mode in modes:
        D.pair_kernel_select(mode)
        tri = torch.zeros(cfg.m * (cfg.m - 1) // 2, dtype=torch.int64, device="cuda")
        D.count_pairs(tids, cfg.n, cfg.m, first, last, tri)
        torch.cuda.synchronize()
        if ref is None:
            ref = tri.clone()
        same = bool(torch.equal(ref, tri))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            D.count_pairs(tids, cfg.n, cfg.m, first, last, tri)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        tests = tri.numel() * (last - first + 1)
        name = {1: "and_popc", 2: "tensor"}.get(mode, str(mode))
        print(f"{name:9s} pairs {tri.numel()} x {last - first + 1} rows: {ms * 1e3:.1f} us/launch, "
              f"{tests / (ms * 1e-3):.3e} tests/s, equal_to_first={same}", flush=True)
    D.pair_kernel_select(-1)


if __name__ == "__main__":
    main()
