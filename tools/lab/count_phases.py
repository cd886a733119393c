"""Per-CTA phase timeline of dic_count_support (lab build with
-DDIC_LAB_TIMING, DIC_LIB=tools/lab/libs/lib_TIMING.so): where does a
mid-size count on one cfg4 chunk spend its time?"""

from __future__ import annotations

import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1812_10959_b200 import _abi, device as D  # noqa: E402
from paper_1812_10959_b200.workloads import CONFIGS, generate_csr, scaled  # noqa: E402


def main() -> None:
    cfg = scaled(CONFIGS[4], 1_000_000)
    ip, ix = generate_csr(cfg)
    rows, _ = D.encode_csr(torch.from_numpy(ip).cuda(), torch.from_numpy(ix).cuda(), cfg.n, cfg.m)
    tids = D.rows_to_tids(rows, cfg.n, cfg.m)
    lib = _abi.load()
    rng = np.random.default_rng(3)
    for k, Cn in [(3, 9400), (3, 3000)]:
        sel = np.sort(np.array([rng.choice(cfg.m, k, replace=False) for _ in range(Cn)]), axis=1)
        sel = sel[np.lexsort(sel.T[::-1])].astype(np.uint16)
        it = torch.from_numpy(np.ascontiguousarray(sel).view(np.int16)).cuda()
        out = torch.zeros(Cn, dtype=torch.int64, device="cuda")
        for _ in range(3):
            D.count_support(tids, cfg.n, cfg.m, 0, 99_999, it, out)
        torch.cuda.synchronize()
        buf = (C.c_ulonglong * (4096 * 6))()
        lib.dic_lab_stamps(buf, 4096)
        a = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 6).astype(np.int64)
        a = a[a[:, 0] > 0]
        t0 = a[:, 0].min()
        rel = (a[:, :5] - t0) / 1e3
        print(f"k={k} C={Cn}: {len(a)} CTAs")
        names = ["start", "ids", "first tile", "tiles done", "end"]
        for j, nm in enumerate(names):
            col = rel[:, j]
            print(f"  {nm:11s} min {col.min():7.2f}  p50 {np.median(col):7.2f}  max {col.max():7.2f} us")


if __name__ == "__main__":
    main()
