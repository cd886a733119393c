"""Generate tests/golden/cfg4.npz: BASELINE config 4 at FULL size (10M x 1000),
mined by the C oracle (oracle/dic_oracle.c) on all host cores.

The reference would need ~8 h here ("Full-size cfg4/5
goldens"), so the golden comes from the oracle restatement of engine.py:105-458,
which is itself pinned to the unmodified reference on the phase KATs, the
240-run corpus, the wide databases and cfg1-3 (tests/test_oracle_golden.py).
This is the route SURVEY §8(c) prescribes for the full-size configs.

    python tests/golden/make_golden_cfg4.py [--threads 8]

Writes masks / sizes / supports of every frequent itemset in (size, mask)
order, the oracle's MiningStats and the sha256 of the generated CSR, so
generator drift is caught before any comparison. ~45 min on 8 vCPU.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_1812_10959_b200.workloads import CONFIGS, generate_csr  # noqa: E402
from tests.golden_util import csr_digest, rows_from_csr  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--out", type=str, default=str(HERE / "cfg4.npz"))
    a = ap.parse_args()
    cfg = CONFIGS[4]
    t0 = time.perf_counter()
    indptr, indices = generate_csr(cfg)
    digest = csr_digest(indptr, indices)
    rows = rows_from_csr(indptr, indices, cfg.m)
    del indices
    print(f"cfg4: generated + encoded in {time.perf_counter() - t0:.1f}s, sha256 {digest}", flush=True)
    t1 = time.perf_counter()
    run = O.mine(rows, cfg.m, cfg.minsup, interval=cfg.interval, threads=a.threads)
    wall = time.perf_counter() - t1
    W = rows.shape[1]
    fm = np.stack([O.words_from_mask(mk, W) for mk, _, _ in run.frequent]) if run.frequent else \
        np.zeros((0, W), np.uint64)
    stats = {"db_passes": run.db_passes, "peak_dashed": run.peak_dashed,
             "candidates_generated": run.candidates_generated, "candidates_pruned": run.candidates_pruned,
             "interval_counts": run.interval_counts}
    np.savez_compressed(a.out, masks=fm, sizes=np.array([s for _, s, _ in run.frequent], dtype=np.int64),
                        supports=np.array([s for _, _, s in run.frequent], dtype=np.int64),
                        meta=json.dumps({"config": 4, "n": cfg.n, "m": cfg.m, "minsup": cfg.minsup,
                                         "interval": cfg.interval, "csr_sha256": digest, "stats": stats,
                                         "stops": run.stops, "source": "oracle/dic_oracle.c (C port)",
                                         "oracle_threads": a.threads, "oracle_wall_s": wall}))
    print(f"cfg4: {len(run.frequent)} frequent, stops {run.stops}, stats {stats}, oracle {wall:.0f}s", flush=True)


if __name__ == "__main__":
    main()
