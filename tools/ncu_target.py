"""The ncu target: ONE DIC run of cfg4 (the bench's step) on the engine, then
item_support once more — nothing else launches kernels after the encode.

    python tools/ncu_target.py            # plain run first (the profiling recipe requires it), then e.g.
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
        python tools/ncu_target.py
    ncu --set full --clock-control none --import-source on -k regex:checkpoint_kernel -s 150 -c 1 \
        -o gpurun_out/ckpt python tools/ncu_target.py
"""

from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_1812_10959_b200 as dic  # noqa: E402
from paper_1812_10959_b200 import device as D  # noqa: E402
from paper_1812_10959_b200.miner import run_engine  # noqa: E402
from paper_1812_10959_b200.workloads import CONFIGS, generate_csr  # noqa: E402


def main() -> None:
    cfg = CONFIGS[4]
    D.require_cuda()
    ip, ix = generate_csr(cfg)
    db = dic.BitDatabase.from_csr(ip, ix, cfg.m)
    tids = db.device_tids()
    params = dic.MiningParams.create(cfg.n, cfg.minsup, interval=cfg.interval)
    res = run_engine(tids, cfg.n, cfg.m, params)
    torch.cuda.synchronize()
    print(f"{cfg.name}: {len(res.frequent)} frequent itemsets, {res.stats.db_passes} passes")


if __name__ == "__main__":
    main()
