"""How much shared-prefix reuse do the engine's count buckets offer?  Runs
cfg4 stop by stop to stop S, dumps buckets 3..6 and counts item-row loads per
candidate-tile for a thread owning R consecutive candidates: (a) reusing only
the first item's row (the current count unit), (b) reusing the AND of the
longest prefix shared with the previous candidate."""

from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))

import numpy as np  # noqa: E402

import paper_1812_10959_b200 as dic  # noqa: E402
from paper_1812_10959_b200.miner import DeviceEngine  # noqa: E402
from paper_1812_10959_b200.workloads import CONFIGS, generate_csr  # noqa: E402


def loads(items: np.ndarray, R: int) -> tuple[float, float]:
    a = b = 0
    n, k = items.shape
    for s in range(0, n, R):
        prev = None
        for row in items[s:s + R]:
            if prev is None:
                a += k
                b += k
            else:
                a += k - (1 if row[0] == prev[0] else 0)
                p = 0
                while p < k - 1 and row[p] == prev[p]:
                    p += 1
                b += k - p
            prev = row
    return a / max(n, 1), b / max(n, 1)


def main() -> None:
    stops = [int(x) for x in sys.argv[1:]] or [120, 150, 180]
    cfg = CONFIGS[4]
    ip, ix = generate_csr(cfg)
    db = dic.BitDatabase.from_csr(ip, ix, cfg.m)
    params = dic.MiningParams.create(cfg.n, cfg.minsup, interval=cfg.interval)
    eng = DeviceEngine(db.device_tids(), db.n, db.m, params, True)
    eng.seed(eng.item_counts())
    stop = 0
    for s in range(1, max(stops) + 1):
        stop = stop + 1 if stop < params.intervals_per_pass else 1
        eng.issue_count(*params.chunk_bounds(stop))
        eng.poll(eng.issue_checkpoint())
        if s in stops:
            for k in range(3, 7):
                rec, items = eng.bucket(k)
                live = items  # dead slots included (the kernel counts them too)
                if len(live):
                    fa, fb = loads(live.astype(np.int32), 28)
                    print(f"stop {s} k={k} slots {len(live)}: loads/cand first-item {fa:.2f}, prefix {fb:.2f}")
    eng.close()


if __name__ == "__main__":
    main()
