"""Per-CTA phase timeline of the tensor-core pair kernel on one cfg4 chunk
(lab build: python tools/lab/build_variant.py TIMING -DDIC_LAB_TIMING, then
DIC_LIB=tools/lab/libs/lib_TIMING.so python tools/lab/tc_phases.py)."""

from __future__ import annotations

import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1812_10959_b200 import _abi  # noqa: E402
from paper_1812_10959_b200 import device as D  # noqa: E402
from paper_1812_10959_b200.workloads import CONFIGS, generate_csr, scaled  # noqa: E402


def main() -> None:
    cfg = scaled(CONFIGS[4], 1_000_000)
    ip, ix = generate_csr(cfg)
    rows, _ = D.encode_csr(torch.from_numpy(ip).cuda(), torch.from_numpy(ix).cuda(), cfg.n, cfg.m)
    tids = D.rows_to_tids(rows, cfg.n, cfg.m)
    tri = torch.zeros(cfg.m * (cfg.m - 1) // 2, dtype=torch.int64, device="cuda")
    for _ in range(3):
        D.count_pairs(tids, cfg.n, cfg.m, 0, 99_999, tri)
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * (1024 * 6))()
    _abi.load().dic_lab_tc_stamps(buf)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 6).astype(np.int64)
    a = a[a[:, 0] > 0]
    t0 = a[:, 0].min()
    rel = (a - t0) / 1e3
    names = ["start", "tmem ready", "first MMA", "loop done", "epilogue done", "exit"]
    print(f"{len(a)} CTAs")
    for j, nm in enumerate(names):
        col = rel[:, j]
        col = col[a[:, j] > 0]
        if len(col):
            print(f"  {nm:14s} min {col.min():7.2f}  p50 {np.median(col):7.2f}  max {col.max():7.2f} us")


if __name__ == "__main__":
    main()
