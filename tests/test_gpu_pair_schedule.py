"""The dense pair kernel's unit schedule (csrc/pairs.cu) is a tuning knob,
not a semantic one: every split between the static share and the claimed
grains must give the same triangle, bit for bit, and the grain counters must
re-arm between launches.  The knobs are read once per process, so each
setting runs in its own interpreter."""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent

SNIPPET = r"""
import hashlib, sys
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_1812_10959_b200 import device as D
n, m = 300_000, 1000
rows = D.bernoulli_rows(n, m, 0.03, 11)
tids = D.rows_to_tids(rows, n, m)
h = hashlib.sha256()
for first, last in [(0, n - 1), (12_345, 212_344), (99_999, 100_030)]:
    for _ in range(2):  # twice: the grain counters must be re-armed by the kernel
        tri = D.count_pairs(tids, n, m, first, last).cpu().numpy()
        h.update(tri.tobytes())
print(h.hexdigest())
"""


def _digest(env: dict) -> str:
    e = dict(os.environ)
    e.update(env)
    out = subprocess.run([sys.executable, "-c", SNIPPET, str(ROOT)], env=e, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    return out.stdout.strip().splitlines()[-1]


def test_pair_schedule_variants_agree():
    ref = _digest({})
    for env in ({"DIC_PAIR_STATIC_PCT": "100"}, {"DIC_PAIR_STATIC_PCT": "0", "DIC_PAIR_GRAIN": "1"},
                {"DIC_PAIR_STATIC_PCT": "30", "DIC_PAIR_GRAIN": "64"}, {"DIC_PAIR_MINB": "4"}):
        assert _digest(env) == ref, env
