"""DicMiner.transform's containment kernel on BASELINE shapes: cfg2 (100k rows
x its 850 frequent itemsets, dense bool output) and a 2M-row slice of cfg4 x
its 8,523 frequent itemsets (packed bit output).  Reports time, rows x
patterns / s and the output-write bandwidth against the measured HBM peak."""

from __future__ import annotations

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_1812_10959_b200 as dic  # noqa: E402
from paper_1812_10959_b200 import device as D  # noqa: E402
from paper_1812_10959_b200.workloads import CONFIGS, generate_csr, scaled  # noqa: E402


def timed(fn, reps=5):
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def case(cfg, packed: bool) -> dict:
    ip, ix = generate_csr(cfg)
    db = dic.BitDatabase.from_csr(ip, ix, cfg.m)
    p = dic.MiningParams.create(cfg.n, cfg.minsup, interval=cfg.interval)
    res = dic.mine_parallel(db, p)
    items, offs = D.patterns_to_device(f.mask for f in res.frequent)
    P = len(res.frequent)
    tids = db.device_tids()
    ms = timed(lambda: D.containment(tids, db.n, db.m, items, offs, packed=packed))
    out_bytes = ((db.n + 31) // 32) * P * 4 if packed else db.n * P
    return {"config": cfg.name, "n": db.n, "m": db.m, "patterns": P, "output": "packed" if packed else "dense",
            "ms": ms, "row_patterns_per_s": db.n * P / (ms * 1e-3), "out_GBps": out_bytes / (ms * 1e-3) / 1e9}


def main() -> None:
    D.require_cuda()
    out = [case(CONFIGS[2], False), case(scaled(CONFIGS[4], 2_000_000, interval=20_000), True)]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
