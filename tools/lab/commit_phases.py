"""Phase timeline of the per-stop checkpoint kernel (CTA 0) over a cfg4 run (lab
build: python tools/lab/build_variant.py TIMING -DDIC_LAB_TIMING, then
DIC_LIB=tools/lab/libs/lib_TIMING.so python tools/lab/commit_phases.py)."""

from __future__ import annotations

import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))

import numpy as np  # noqa: E402

import paper_1812_10959_b200 as dic  # noqa: E402
from paper_1812_10959_b200 import _abi  # noqa: E402
from paper_1812_10959_b200.miner import run_engine  # noqa: E402
from paper_1812_10959_b200.workloads import CONFIGS, generate_csr  # noqa: E402


def main() -> None:
    cfg = CONFIGS[4]
    ip, ix = generate_csr(cfg)
    db = dic.BitDatabase.from_csr(ip, ix, cfg.m)
    params = dic.MiningParams.create(cfg.n, cfg.minsup, interval=cfg.interval)
    run_engine(db.device_tids(), cfg.n, cfg.m, params)
    buf = (C.c_ulonglong * (512 * 12))()
    _abi.load().dic_lab_commit_stamps(buf)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(512, 12).astype(np.int64)
    # stamps of CTA 0: 0 start, 1 after apply (+ barrier), 2 after compaction / joins (+ barrier),
    # 3 after the commit, 4 last CTA out (before the status), 5 after the status; [6] = mode
    # (0 grid, 1 small stop that called the grid in, 2 CTA 0 alone).  4 and 5 exist only when CTA 0 left last.
    names = ["apply", "joins", "commit", "last-out", "status"]
    tot = np.zeros(3)
    modes = [0, 0, 0]
    for s in range(326):
        r = a[s].copy()
        if r[0] == 0:
            continue
        if r[2] < r[1]:
            r[2] = r[1]
        d = np.diff(r[:4]) / 1e3
        tot += d
        tail = np.diff(r[3:6]) / 1e3 if r[4] > r[3] and r[5] > r[4] else None
        if tail is not None:
            modes[int(r[6])] += 1
        if s % 10 == 0 or s in (101, 102, 103, 104, 105):
            extra = " ".join(f"{n}={x:.1f}" for n, x in zip(names[3:], tail)) + f" mode={r[6]}" if tail is not None else ""
            ev = (f"(pre-eval {(r[11] - r[1]) / 1e3:.1f}, eval cta0 {(r[7] - r[11]) / 1e3:.1f}, last cta {(r[9] - r[1]) / 1e3:.1f}, {r[10]} claims, "
                  f"slowest {r[8] / 1e3:.1f})") if a[s][7] > r[1] else ""
            print(s, " ".join(f"{n}={x:.1f}" for n, x in zip(names, d)), ev, extra, f"sum={d.sum():.1f} us")
    print("totals ms:", " ".join(f"{n}={x / 1e3:.2f}" for n, x in zip(names, tot)), f"sum={tot.sum() / 1e3:.2f}",
          "stops seen to the end by CTA 0 per mode:", modes)


if __name__ == "__main__":
    main()
