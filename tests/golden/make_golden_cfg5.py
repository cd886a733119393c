"""Generate tests/golden/cfg5.npz: BASELINE config 5 at FULL size — the
support of every one of the 100,000 random candidates over all 50,000,000
rows of the i.i.d. Bernoulli(0.05) 512-item bitmap.

The bitmap is regenerated on the host by oracle/cfg5.c (a restatement of the
device generator's hash, pinned row-for-row against the device in
tests/test_gpu_fullsize.py) and counted column-wise by the same file's
restatement of the reference's support count (_count_block,
engine.py:43-58), which tests/test_oracle_golden.py cross-checks against the
row-form oracle.  The reference itself would need ~6 h here.

    python tests/golden/make_golden_cfg5.py [--threads 8]     (~1-2 min, 3.3 GB RAM)
"""

from __future__ import annotations

import argparse
import hashlib
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
from oracle import synth as S  # noqa: E402
from paper_1812_10959_b200.workloads import CONFIGS  # noqa: E402


def cand_digest(ks: np.ndarray, items: np.ndarray) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(ks, dtype=np.int32).tobytes())
    h.update(np.ascontiguousarray(items, dtype=np.uint16).tobytes())
    return h.hexdigest()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    cfg = CONFIGS[5]
    n, m, p = cfg.n, cfg.m, cfg.params["p"]
    t0 = time.perf_counter()
    cols = O.bernoulli_cols(n, m, p, cfg.seed, threads=a.threads)
    t1 = time.perf_counter()
    ks, items = S.candidates(cfg.params["candidates"], m, cfg.params["kmin"], cfg.params["kmax"], cfg.seed)
    item_counts = O.count_cols(cols, np.arange(m, dtype=np.uint16).reshape(-1, 1), np.ones(m, np.int32),
                               threads=a.threads)
    sup = O.count_cols(cols, items, ks, threads=a.threads)
    t2 = time.perf_counter()
    assert sup.max() < 2**31
    np.savez_compressed(HERE / "cfg5.npz", supports=sup.astype(np.int32), item_counts=item_counts.astype(np.int32),
                        ks=ks.astype(np.int8),
                        meta=json.dumps({"config": 5, "n": n, "m": m, "p": p, "seed": cfg.seed,
                                         "candidates": int(len(ks)), "cand_sha256": cand_digest(ks, items),
                                         "support_checksum": int(sup.sum()),
                                         "source": "oracle/cfg5.c (host restatement of the generator + column count)",
                                         "gen_s": t1 - t0, "count_s": t2 - t1, "threads": a.threads}))
    print(f"cfg5: {len(ks)} candidates, checksum {int(sup.sum())}, gen {t1 - t0:.1f}s count {t2 - t1:.1f}s",
          flush=True)


if __name__ == "__main__":
    main()
