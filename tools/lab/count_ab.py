"""A/B timing of dic_count_support on cfg5-shaped data (i.i.d. Bernoulli(0.05)
bits, random k in [2, 6] candidates, buckets sorted as bench.py sorts them),
per size and in total.  Select the library build with DIC_LIB=... ."""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1812_10959_b200 import device as D  # noqa: E402


def main() -> None:
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
    C = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
    m = 512
    rows = D.bernoulli_rows(n, m, 0.05, 5)
    tids = D.rows_to_tids(rows, n, m)
    del rows
    ks, items = D.synth_candidates(C, m, 2, 6, 5)
    res, tot, chk = {}, 0.0, 0
    for k in range(2, 7):
        sel = items[ks == k][:, :k]
        sel = sel[np.lexsort(sel.T[::-1])]
        it = torch.from_numpy(np.ascontiguousarray(sel).view(np.int16)).cuda()
        out = torch.zeros(sel.shape[0], dtype=torch.int64, device="cuda")
        D.count_support(tids, n, m, 0, n - 1, it, out)
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(3):
            out.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            D.count_support(tids, n, m, 0, n - 1, it, out)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        chk += int(out.sum().item())
        tot += best
        frac = sel.shape[0] * k * (n / 32) / (best * 1e-3) / 1.851e13
        res[f"k{k}"] = round(best, 3), round(frac, 3)
    words = n / 32
    ops = sum(int((ks == k).sum()) * k for k in range(2, 7)) * words
    print(json.dumps({"lib": os.environ.get("DIC_LIB", "main"), "stages": os.environ.get("DIC_COUNT_STAGES", "3"),
                      "per_k_ms_frac": res, "total_ms": round(tot, 3), "frac": round(ops / (tot * 1e-3) / 1.851e13, 4),
                      "checksum": chk}))


if __name__ == "__main__":
    main()
