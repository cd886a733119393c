"""Small end-to-end runs for compute-sanitizer (memcheck / racecheck):
encoder straight to tiles, the engine on cfg1 and a shrunken cfg4 (the
tensor-core pair triangle, graphs, compaction, replay growth), containment,
row-form count, two lockstep engines (sharded trajectory), and a dense
database whose stops commit thousands of joins at once."""

from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1812_10959_b200 as dic  # noqa: E402
from paper_1812_10959_b200 import device as D  # noqa: E402
from paper_1812_10959_b200.workloads import CONFIGS, generate_csr, scaled  # noqa: E402


def main() -> None:
    for cfg in (CONFIGS[1], scaled(CONFIGS[4], 20_000, interval=2_000), scaled(CONFIGS[3], 8_000, interval=1_000)):
        ip, ix = generate_csr(cfg)
        db = dic.BitDatabase.from_csr(ip, ix.astype(np.uint16), cfg.m, slabs=3)
        res = dic.mine_parallel(db, dic.MiningParams.create(cfg.n, cfg.minsup, interval=cfg.interval))
        items, offs = D.patterns_to_device(f.mask for f in res.frequent[:200])
        D.containment(db.device_tids(), db.n, db.m, items, offs)
        D.containment(db.device_tids(), db.n, db.m, items, offs, packed=True)
        masks = torch.from_numpy(dic.bits.masks_to_array([f.mask for f in res.frequent[:64]], db.words)).cuda()
        D.count_support_rows(db.device_rows(), 0, db.n - 1, masks)
        torch.cuda.synchronize()
        print(cfg.name, len(res.frequent))
    # two lockstep engines over the chunk-sliced shards of a shrunken cfg4
    from paper_1812_10959_b200.lockstep import mine_lockstep

    cfg = scaled(CONFIGS[4], 20_000, interval=2_000)
    params = dic.MiningParams.create(cfg.n, cfg.minsup, interval=cfg.interval)
    shards = []
    for r in range(2):
        plan = dic.ShardPlan.for_params(params, 2, r)
        ip, ix = generate_csr(cfg, ranges=plan.ranges())
        shards.append(dic.BitDatabase.from_csr(ip, ix, cfg.m))
    res, info = mine_lockstep(shards, params)
    print("lockstep x2", len(res.frequent), info.stops)
    # a dense database: stops that admit thousands of new candidates
    rng = np.random.default_rng(11)
    bits = rng.random((3000, 24)) < 0.6
    ints = [int(sum(1 << i for i in range(24) if row[i])) for row in bits]
    res = dic.mine_parallel(dic.BitDatabase(ints, m=24), dic.MiningParams.create(3000, 0.15, interval=300))
    torch.cuda.synchronize()
    print("dense", len(res.frequent))


if __name__ == "__main__":
    main()
