"""Time the pieces of the end-to-end path on cfg4 (H2D, encode, bit-slice
transform, DIC run, result D2H) with CUDA events; prints one JSON line."""

from __future__ import annotations

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_1812_10959_b200 as dic  # noqa: E402
from paper_1812_10959_b200 import device as D  # noqa: E402
from paper_1812_10959_b200.miner import run_engine  # noqa: E402
from paper_1812_10959_b200.workloads import CONFIGS, generate_csr  # noqa: E402


def timed(fn, reps=3):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    best = 1e30
    out = None
    for _ in range(reps):
        torch.cuda.synchronize()
        ev[0].record()
        out = fn()
        ev[1].record()
        torch.cuda.synchronize()
        best = min(best, ev[0].elapsed_time(ev[1]))
    return best, out


def main() -> None:
    idx = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    cfg = CONFIGS[idx]
    D.require_cuda()
    ip, ix = generate_csr(cfg)
    hip, hix = torch.from_numpy(ip).pin_memory(), torch.from_numpy(ix).pin_memory()
    res = {"config": cfg.name, "n": cfg.n, "nnz": int(ix.size)}
    res["h2d_ms"], (dip, dix) = timed(lambda: (hip.cuda(non_blocking=True), hix.cuda(non_blocking=True)))
    res["encode_ms"], (rows, st) = timed(lambda: D.encode_csr(dip, dix, cfg.n, cfg.m))
    res["transform_ms"], tids = timed(lambda: D.rows_to_tids(rows, cfg.n, cfg.m))
    params = dic.MiningParams.create(cfg.n, cfg.minsup, interval=cfg.interval)
    res["item_support_ms"], _ = timed(lambda: D.item_support(tids, cfg.n, cfg.m, 0, cfg.n - 1))
    res["dic_ms"], out = timed(lambda: run_engine(tids, cfg.n, cfg.m, params))
    res["frequent"] = len(out.frequent)
    res["from_csr_i32_ms"], _ = timed(lambda: dic.BitDatabase.from_csr(hip, hix, cfg.m).device_tids())
    hix16 = torch.from_numpy(ix.astype("uint16")).pin_memory()
    res["h2d_u16_ms"], _ = timed(lambda: (hip.cuda(non_blocking=True), hix16.cuda(non_blocking=True)))
    res["from_csr_u16_ms"], _ = timed(lambda: dic.BitDatabase.from_csr(hip, hix16, cfg.m).device_tids())
    print(json.dumps(res))


if __name__ == "__main__":
    main()
