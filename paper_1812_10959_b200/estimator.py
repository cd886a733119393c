"""Scikit-learn style front end: DicMiner.fit mines on the GPU engine,
DicMiner.transform maps transactions onto the pattern containment matrix
with the dic_containment kernel.

Mirrors /root/reference/pkg/src/dicmine/estimator.py:15-113 (constructor
parameters, fitted attributes, errors) and the input coercion of
_validation.py:14-56 (as_bit_database).  Documented deviation (SURVEY.md
§8(b)): the item universe is not capped at 64 — an incidence array may have
up to MAX_ITEMS columns, and ``itemset_masks_`` is a uint64 array when every
mask fits 64 bits, else an object array of Python ints.
"""

from __future__ import annotations

import os
from typing import Any, Iterable

import numpy as np
from sklearn.base import BaseEstimator, TransformerMixin
from sklearn.exceptions import NotFittedError

from .bitmap import MAX_ITEMS, BitDatabase, database_from_transactions
from .bits import items_of
from .catalog import TransitionAudit
from .config import MiningParams
from .miner import mine_parallel, mine_serial


def resolve_thread_count(threads: int | None) -> int:
    """Turn an optional thread request into a concrete worker count
    (_validation.py:59-65; the GPU engine ignores it, the value is kept for
    MiningParams and get_params parity)."""
    if threads is None:
        return os.cpu_count() or 1
    if threads < 1:
        raise ValueError(f"threads must be >= 1, got {threads}")
    return threads


def as_bit_database(X: Any) -> BitDatabase:
    """Coerce estimator input into a BitDatabase (_validation.py:14-56):
    a BitDatabase as-is, a 2-D 0/1 incidence array (n_transactions, n_items),
    or an iterable of item-id collections (ragged lists are fine)."""
    if isinstance(X, BitDatabase):
        return X
    if isinstance(X, np.ndarray) or (hasattr(X, "__len__") and len(X) and isinstance(X[0], np.ndarray)):
        X = np.asarray(X)
    if isinstance(X, np.ndarray):
        if X.ndim != 2:
            raise ValueError(f"expected a 2D incidence array, got shape {X.shape}")
        n_items = X.shape[1]
        if n_items > MAX_ITEMS:
            raise ValueError(f"incidence array has {n_items} item columns; at most {MAX_ITEMS} supported")
        dense = X.astype(bool)
        if X.dtype != bool and not np.array_equal(X, dense.astype(X.dtype)):
            raise ValueError("incidence array must contain only 0/1 values")
        m = max(n_items, 1)
        W = (m + 63) // 64
        padded = np.zeros((dense.shape[0], W * 64), dtype=bool)
        padded[:, :n_items] = dense
        # bit p of word w <=> column 64w + p (little-endian bit order)
        rows = np.packbits(padded.reshape(-1, W, 64), axis=2, bitorder="little").view("<u8").reshape(-1, W)
        return BitDatabase(rows.astype(np.uint64) if W > 1 else rows[:, 0].astype(np.uint64), m=m)
    if isinstance(X, (str, bytes)):
        raise TypeError("strings are not a transaction collection")
    try:
        rows: Iterable = iter(X)
    except TypeError:
        raise TypeError(f"cannot interpret {type(X).__name__} as transactions") from None
    return database_from_transactions([list(r) for r in rows])


class DicMiner(BaseEstimator, TransformerMixin):
    """Frequent-itemset miner with a fit/transform interface
    (estimator.py:15-56).

    Parameters: ``minsup`` in (0, 1]; ``interval`` (None = half the
    database); ``threads`` (accepted for parity; the GPU engine ignores it);
    ``engine`` "parallel" or "serial" (both run the GPU engine, whose output
    is the reference's by construction); ``prune_bound``.

    Fitted attributes: ``itemset_masks_``, ``supports_``, ``itemsets_``,
    ``n_items_``, ``stats_``, ``result_``.
    """

    def __init__(self, minsup: float = 0.1, interval: int | None = None, threads: int | None = None,
                 engine: str = "parallel", prune_bound: bool = True):
        self.minsup = minsup
        self.interval = interval
        self.threads = threads
        self.engine = engine
        self.prune_bound = prune_bound

    def fit(self, X, y=None, audit: TransitionAudit | None = None):
        """Mine the frequent itemsets of ``X`` (estimator.py:58-82)."""
        if self.engine not in ("parallel", "serial"):
            raise ValueError(f"engine must be 'parallel' or 'serial', got {self.engine!r}")
        db = as_bit_database(X)
        params = MiningParams.create(db.n, self.minsup, interval=self.interval,
                                     threads=resolve_thread_count(self.threads))
        runner = mine_serial if self.engine == "serial" else mine_parallel
        result = runner(db, params, prune_bound=self.prune_bound, audit=audit)
        self.result_ = result
        self.stats_ = result.stats
        self.n_items_ = db.m
        masks = [f.mask for f in result.frequent]
        if all(mk < (1 << 64) for mk in masks):
            self.itemset_masks_ = np.array(masks, dtype=np.uint64)
        else:
            self.itemset_masks_ = np.array(masks, dtype=object)
        self.supports_ = np.array([f.support for f in result.frequent], dtype=np.int64)
        self.itemsets_ = [tuple(items_of(f.mask)) for f in result.frequent]
        self._patterns = None
        return self

    def transform(self, X) -> np.ndarray:
        """Boolean matrix: entry (j, p) says pattern p occurs in transaction j
        (estimator.py:90-99), computed by dic_containment on the GPU."""
        if not hasattr(self, "itemset_masks_"):
            raise NotFittedError("DicMiner must be fitted before calling transform")
        db = as_bit_database(X)
        return self.transform_device(db).cpu().numpy()

    def transform_device(self, db: BitDatabase):
        """The containment matrix as a device bool tensor [n][P] (no host copy)."""
        from . import device as D

        if not hasattr(self, "itemset_masks_"):
            raise NotFittedError("DicMiner must be fitted before calling transform")
        if getattr(self, "_patterns", None) is None:
            self._patterns = D.patterns_to_device(int(mk) for mk in self.itemset_masks_)
        items, offs = self._patterns
        return D.containment(db.device_tids(), db.n, db.m, items, offs)

    def get_feature_names_out(self, input_features=None) -> np.ndarray:
        if not hasattr(self, "itemsets_"):
            raise NotFittedError("DicMiner must be fitted first")
        return np.array(["itemset_" + "_".join(map(str, items)) for items in self.itemsets_], dtype=object)
