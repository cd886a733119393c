"""DicMiner (estimator.py:15-113) and the GPU-encoded text loader, against
golden results of the reference's own DicMiner and load_transactions_with_report
(tests/golden/make_golden_io.py), plus the reference estimator tests'
behaviours (test_estimator.py) and the containment kernel against numpy."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_1812_10959_b200 as dic
from paper_1812_10959_b200 import device as D

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"
EST = json.loads((GOLD / "estimator.json").read_text())
IO = json.loads((GOLD / "io.json").read_text())
TRANSACTIONS = [[0, 1], [0, 1], [0], [0, 1, 2], [2]]


@pytest.mark.parametrize("case", [c for c in EST if "X" in c], ids=lambda c: f"{len(c['X'])}x{c['minsup']}")
def test_fit_transform_match_reference(case):
    miner = dic.DicMiner(minsup=case["minsup"], interval=case["interval"]).fit(case["X"])
    assert [int(v) for v in miner.itemset_masks_] == case["masks"]
    assert [int(s) for s in miner.supports_] == case["supports"]
    assert [list(t) for t in miner.itemsets_] == case["itemsets"]
    assert miner.n_items_ == case["n_items"]
    assert list(miner.get_feature_names_out()) == case["names"]
    out = miner.transform(case["Y"])
    assert out.dtype == bool and out.astype(int).tolist() == case["transform"]


def test_fit_accepts_incidence_matrix():
    case = [c for c in EST if "incidence" in c][0]
    miner = dic.DicMiner(minsup=case["minsup"]).fit(np.array(case["incidence"]))
    assert [int(v) for v in miner.itemset_masks_] == case["masks"] and miner.n_items_ == case["n_items"]
    assert [int(s) for s in miner.supports_] == case["supports"]
    with pytest.raises(ValueError):
        dic.DicMiner().fit(np.array([[0, 2], [1, 0]]))  # non-binary
    with pytest.raises(ValueError):
        dic.DicMiner().fit(np.zeros(4))  # not 2D
    with pytest.raises(TypeError):
        dic.DicMiner().fit("0 1\n2\n")
    with pytest.raises(ValueError):
        dic.DicMiner(engine="gpu").fit(TRANSACTIONS)


def test_sklearn_protocol():
    from sklearn.base import clone
    from sklearn.dummy import DummyClassifier
    from sklearn.exceptions import NotFittedError
    from sklearn.pipeline import Pipeline

    with pytest.raises(NotFittedError):
        dic.DicMiner().transform(TRANSACTIONS)
    with pytest.raises(NotFittedError):
        dic.DicMiner().get_feature_names_out()
    params = {"minsup": 0.3, "interval": 7, "threads": 2, "engine": "serial", "prune_bound": False}
    assert dic.DicMiner(**params).get_params() == params
    assert dic.DicMiner().set_params(**params).get_params() == params
    miner = dic.DicMiner(minsup=0.25, threads=3)
    assert clone(miner).get_params() == miner.get_params()
    out = dic.DicMiner(minsup=0.4).fit_transform(TRANSACTIONS)
    assert out.shape == (5, 4) and out.dtype == bool
    pipe = Pipeline([("patterns", dic.DicMiner(minsup=0.4)), ("clf", DummyClassifier())])
    pipe.fit(TRANSACTIONS, [1, 1, 0, 1, 0])
    assert pipe.predict(TRANSACTIONS).shape == (5,)
    a = dic.DicMiner(minsup=0.4, engine="serial").fit(TRANSACTIONS)
    assert a.stats_.db_passes >= 1.0 and a.result_.frequent


@pytest.mark.parametrize("m,n,P", [(64, 3000, 40), (1000, 20000, 700), (130, 37, 33), (3000, 5000, 64)])
def test_containment_kernel_matches_numpy(m, n, P):
    """dense and packed containment == (row & mask) == mask, incl. empty
    patterns, patterns with items outside the universe, ragged tails."""
    rng = np.random.default_rng(m * 7 + n)
    W = D.words_for(m)
    rows = np.zeros((n, W), dtype=np.uint64)
    bitsm = rng.random((n, m)) < 0.4
    for i in range(m):
        rows[bitsm[:, i], i >> 6] |= np.uint64(1) << np.uint64(i & 63)
    db = dic.BitDatabase(rows, m=m)
    pats = []
    for p in range(P):
        k = int(rng.integers(0, 5))
        its = sorted(set(rng.integers(0, m, size=k).tolist()))
        if p == 3:
            its = [m - 1, m + 5]  # item outside the universe: never contained
        pats.append(sum(1 << i for i in its))
    items, offs = D.patterns_to_device(pats)
    dense = D.containment(db.device_tids(), n, m + 0, items, offs).cpu().numpy()
    packed = D.containment(db.device_tids(), n, m, items, offs, packed=True).cpu().numpy().view(np.uint32)
    for p, mk in enumerate(pats):
        words = dic.bits.to_words(mk, W) if mk < (1 << (64 * W)) else None
        if words is None:
            want = np.zeros(n, dtype=bool)
        else:
            mw = np.array(words, dtype=np.uint64)
            want = np.all((rows & mw) == mw, axis=1)
        assert np.array_equal(dense[:, p], want), p
        bitsp = np.zeros(((n + 31) // 32) * 32, dtype=bool)
        bitsp[:n] = want
        wp = (bitsp.reshape(-1, 32).astype(np.uint64) << np.arange(32, dtype=np.uint64)).sum(axis=1)
        assert np.array_equal(packed[:, p].astype(np.uint64), wp), p


@pytest.mark.parametrize("case", [c for c in IO["text"] if "masks" in c], ids=lambda c: repr(c["text"][:16]))
def test_loader_encodes_on_gpu_like_reference(case, tmp_path):
    p = tmp_path / "t.txt"
    p.write_bytes(case["text"].encode("utf-8"))
    db, rep = dic.load_transactions_with_report(p)
    assert db.m == case["m"] and [int(x) for x in db] == case["masks"]
    assert (rep.transactions, rep.deduplicated) == (case["transactions"], case["deduplicated"])
    q = tmp_path / "c.bin"
    dic.save_bitdb(db, q)
    assert [int(x) for x in dic.load_bitdb(q)] == case["masks"]
