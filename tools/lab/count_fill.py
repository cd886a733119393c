"""dic_count_support on cfg4-shaped chunks (m = 1000, TW = 16) as a function of
the candidate count of ONE block (<= 3,584 candidates of 3 items): what does a
tile cost when the block is nearly empty (the tile's arrival, barriers) and
what does each candidate add?  Sizes the row splits of small buckets."""

from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1812_10959_b200 import device as D  # noqa: E402
from paper_1812_10959_b200.workloads import CONFIGS, generate_csr, scaled  # noqa: E402


def main() -> None:
    cfg = scaled(CONFIGS[4], 4_000_000)
    ip, ix = generate_csr(cfg)
    rows, _ = D.encode_csr(torch.from_numpy(ip).cuda(), torch.from_numpy(ix).cuda(), cfg.n, cfg.m)
    tids = D.rows_to_tids(rows, cfg.n, cfg.m)
    rng = np.random.default_rng(3)
    k = 3
    for C in (16, 300, 1000, 2000, 3584):
        sel = np.sort(np.array([rng.choice(cfg.m, k, replace=False) for _ in range(C)]), axis=1)
        sel = sel[np.lexsort(sel.T[::-1])].astype(np.uint16)
        it = torch.from_numpy(np.ascontiguousarray(sel).view(np.int16)).cuda()
        out = torch.zeros(C, dtype=torch.int64, device="cuda")
        res = []
        # one block -> 148 row splits: tiles per CTA = rows / 512 / 148
        for last in (75_775, 757_759, 3_031_039):  # 1, 10, 40 tiles per CTA
            D.count_support(tids, cfg.n, cfg.m, 0, last, it, out)
            torch.cuda.synchronize()
            best = 1e30
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(10):
                    D.count_support(tids, cfg.n, cfg.m, 0, last, it, out)
                e1.record()
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1) / 10)
            res.append(best * 1e3)
        per_tile = (res[2] - res[1]) / 30
        print(f"C={C:5d}: 1 tile/CTA {res[0]:.1f} us, 10 tiles {res[1]:.1f} us, 40 tiles {res[2]:.1f} us"
              f"  -> {per_tile:.2f} us per tile, fixed {res[1] - 10 * per_tile:.1f} us")


if __name__ == "__main__":
    main()
