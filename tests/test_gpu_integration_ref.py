"""INTEGRATION.md Option B, executed: the UNMODIFIED reference package
(`dicmine`, installed into baseline/_ref by tools/install_reference.sh) runs
its own `mine_parallel` with only its counting seam — `engine._count_block`
(engine.py:43-58, resolved at :146) and `engine.count_support_interval`
(engine.py:176-223, resolved at :429) — bound to libdicb200.so through the
ctypes stub integration/dicmine_b200.py.  Results and MiningStats must equal
the goldens the reference produced on its own CPU path."""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O
from paper_1812_10959_b200.workloads import CONFIGS, generate_csr, scaled
from tests.golden_util import load_config_golden, rows_from_csr

pytestmark = pytest.mark.gpu
REF = Path(__file__).resolve().parent.parent / "baseline" / "_ref"


@pytest.fixture(scope="module")
def dicmine():
    if not (REF / "dicmine" / "engine.py").exists():
        pytest.skip("baseline/_ref has no dicmine: run tools/install_reference.sh")
    sys.path.insert(0, str(REF))
    import dicmine as dm
    import dicmine.engine as eng

    from integration import dicmine_b200 as b200

    saved = (eng._count_block, eng.count_support_interval)
    b200.install(eng)
    yield dm, b200
    eng._count_block, eng.count_support_interval = saved
    sys.path.remove(str(REF))


def _stats(s) -> tuple:
    return (s.db_passes, s.peak_dashed, s.candidates_generated, s.candidates_pruned, s.interval_counts)


def test_reference_mine_parallel_cfg1_on_gpu_seam(dicmine):
    dm, b200 = dicmine
    assert "baseline/_ref" in dm.__file__
    cfg = CONFIGS[1]
    ip, ix = generate_csr(cfg)
    rows = rows_from_csr(ip, ix, cfg.m)
    db = dm.BitDatabase([int(x) for x in rows[:, 0]], m=cfg.m)
    params = dm.MiningParams.create(cfg.n, cfg.minsup, interval=cfg.interval)
    l0 = b200.launches()
    res = dm.mine_parallel(db, params)
    assert b200.launches() - l0 > cfg.m  # every singleton + every stop counted on the GPU
    g = load_config_golden(1)  # the reference's own (CPU) run
    assert [(f.mask, f.support) for f in res.frequent] == g.pairs
    st = g.stats
    assert _stats(res.stats) == (st["db_passes"], st["peak_dashed"], st["candidates_generated"],
                                 st["candidates_pruned"], st["interval_counts"])


class _WideDB:
    """The attributes the reference engine touches, with masks uint64 [n][W]
    (the reference's BitDatabase stops at 64 items; SURVEY 8(c) route 2)."""

    def __init__(self, rows: np.ndarray, m: int):
        self.masks, self.n, self.m = rows, rows.shape[0], m

    def as_int_list(self):
        return [sum(int(v) << (64 * w) for w, v in enumerate(r)) for r in self.masks]


@pytest.mark.parametrize("idx,n,interval", [(3, 100_000, 10_000), (2, 30_000, 3_000)])
def test_reference_mine_parallel_wide_on_gpu_seam(dicmine, idx, n, interval):
    dm, b200 = dicmine
    cfg = scaled(CONFIGS[idx], n, interval=interval)
    ip, ix = generate_csr(cfg)
    rows = rows_from_csr(ip, ix, cfg.m)
    params = dm.MiningParams.create(cfg.n, cfg.minsup, interval=cfg.interval)
    res = dm.mine_parallel(_WideDB(rows, cfg.m), params)
    want = O.mine(rows, cfg.m, cfg.minsup, interval=cfg.interval, threads=os.cpu_count() or 1)
    assert [(f.mask, f.size, f.support) for f in res.frequent] == want.frequent
    assert _stats(res.stats) == (want.db_passes, want.peak_dashed, want.candidates_generated,
                                 want.candidates_pruned, want.interval_counts)
