"""dic_count_support on one cfg4-shaped chunk (m = 1000, TW = 16) for a
mid-size candidate set (the engine's stops 100-200 count ~9.5k candidates of
sizes 3-4): is the row-lane unit slow at TW = 16, or the engine's grid?"""

from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1812_10959_b200 import device as D  # noqa: E402
from paper_1812_10959_b200.workloads import CONFIGS, generate_csr, scaled  # noqa: E402


def main() -> None:
    cfg = scaled(CONFIGS[4], 1_000_000)
    ip, ix = generate_csr(cfg)
    rows, _ = D.encode_csr(torch.from_numpy(ip).cuda(), torch.from_numpy(ix).cuda(), cfg.n, cfg.m)
    tids = D.rows_to_tids(rows, cfg.n, cfg.m)
    rng = np.random.default_rng(3)
    for k, C, srt in [(3, 3000, True), (3, 9400, True), (3, 9400, False), (4, 9400, True), (4, 9400, False)]:
        sel = np.sort(np.array([rng.choice(cfg.m, k, replace=False) for _ in range(C)]), axis=1)
        if srt:
            sel = sel[np.lexsort(sel.T[::-1])]
        sel = sel.astype(np.uint16)
        it = torch.from_numpy(np.ascontiguousarray(sel).view(np.int16)).cuda()
        out = torch.zeros(C, dtype=torch.int64, device="cuda")
        for first, last in [(0, 511), (0, 99_999), (0, 399_999)]:
            D.count_support(tids, cfg.n, cfg.m, first, last, it, out)
            torch.cuda.synchronize()
            best = 1e30
            reps = 20  # back to back: the host launch overhead hides behind the GPU
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(reps):
                    D.count_support(tids, cfg.n, cfg.m, first, last, it, out)
                e1.record()
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1) / reps)
            frac = C * k * ((last - first + 1) / 32) / (best * 1e-3) / 1.851e13
            print(f"k={k} C={C} sorted={srt} chunk [{first},{last}]: {best * 1e3:.1f} us  frac {frac:.3f}")


if __name__ == "__main__":
    main()
