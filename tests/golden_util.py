"""Helpers shared by the golden-fixture tests (no reference import)."""

from __future__ import annotations

import hashlib
import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np

GOLD = Path(__file__).resolve().parent / "golden"


def csr_digest(indptr: np.ndarray, indices: np.ndarray) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(indptr, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(indices, dtype=np.int32).tobytes())
    return h.hexdigest()


def rows_from_csr(indptr: np.ndarray, indices: np.ndarray, m: int) -> np.ndarray:
    """Host restatement of the encoder (test side): uint64 [n][W]."""
    n = indptr.size - 1
    W = (m + 63) // 64
    rows = np.zeros((n, W), dtype=np.uint64)
    rid = np.repeat(np.arange(n), np.diff(indptr))
    idx = indices.astype(np.int64)
    np.bitwise_or.at(rows, (rid, idx // 64), np.left_shift(np.uint64(1), (idx % 64).astype(np.uint64)))
    return rows


@dataclass
class ConfigGolden:
    meta: dict
    masks: np.ndarray
    sizes: np.ndarray
    supports: np.ndarray

    @property
    def stats(self) -> dict:
        return self.meta["stats"]

    @property
    def pairs(self) -> list[tuple[int, int]]:
        out = []
        for row, s in zip(self.masks, self.supports.tolist()):
            x = 0
            for w, v in enumerate(row.tolist()):
                x |= int(v) << (64 * w)
            out.append((x, s))
        return out

    def digest_ok(self, indptr, indices) -> bool:
        return csr_digest(indptr, indices) == self.meta["csr_sha256"]


def load_config_golden(idx: int) -> ConfigGolden:
    z = np.load(GOLD / f"cfg{idx}.npz")
    return ConfigGolden(json.loads(str(z["meta"])), z["masks"], z["sizes"], z["supports"])


def has_config_golden(idx: int) -> bool:
    return (GOLD / f"cfg{idx}.npz").exists()
