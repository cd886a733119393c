"""Quick throughput probe of dic_count_support on a cfg5-shaped workload
(i.i.d. Bernoulli(0.05) bitmap, random k in [2, 6] candidates)."""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1812_10959_b200 import device as D  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8_000_000)
    ap.add_argument("--m", type=int, default=512)
    ap.add_argument("--C", type=int, default=20_000)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    D.require_cuda()
    rows = D.bernoulli_rows(a.n, a.m, 0.05, 5)
    tids = D.rows_to_tids(rows, a.n, a.m)
    ks, items = D.synth_candidates(a.C, a.m, 2, 6, 5)
    res = {}
    total_t = 0.0
    for k in range(2, 7):
        sel = items[ks == k][:, :k]
        it = torch.from_numpy(np.ascontiguousarray(sel).view(np.int16)).cuda()
        out = torch.zeros(sel.shape[0], dtype=torch.int64, device="cuda")
        D.count_support(tids, a.n, a.m, 0, a.n - 1, it, out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e30
        for _ in range(a.reps):
            out.zero_()
            e0.record()
            D.count_support(tids, a.n, a.m, 0, a.n - 1, it, out)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        total_t += best
        res[f"k{k}"] = {"C": int(sel.shape[0]), "ms": best, "tests_per_s": sel.shape[0] * a.n / (best * 1e-3)}
    res["all"] = {"C": a.C, "ms": total_t, "tests_per_s": a.C * a.n / (total_t * 1e-3)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
