"""Phase timeline of the per-stop commit_status kernel over a cfg4 run (lab
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
    buf = (C.c_ulonglong * (512 * 8))()
    _abi.load().dic_lab_commit_stamps(buf)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(512, 8).astype(np.int64)
    names = ["scan", "rank+commit", "last-out"]
    for s in list(range(60, 100, 3)) + [100, 101, 150]:
        r = a[s]
        if r[0] == 0:
            continue
        if r[1] == 0:
            print(s, "no commit")
            continue
        d = np.diff(r[:4]) / 1e3
        print(s, " ".join(f"{n}={x:.1f}" for n, x in zip(names, d)), "us")


if __name__ == "__main__":
    main()
