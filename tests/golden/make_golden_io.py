"""Golden fixtures for the input/output and estimator rows,
generated from the REFERENCE itself in a container where /root/reference
exists:

    python tests/golden/make_golden_io.py

  io.json         transaction text files (tricky whitespace, newlines,
                  comments, duplicates, sign/underscore literals) -> the
                  reference loader's masks and LoadReport, or its error
                  (type, line, token/item); binary caches written by the
                  reference's save_bitdb (hex) with their masks
                  and the reference's seeded generator (sha256 of the masks)
  estimator.json  DicMiner fit / transform / feature names on the reference
                  tests' examples and a few seeded random inputs

Item ids stay below 64 (the reference's universe) except in the error cases,
whose ids are out of range for both (negative or >= 65535).
"""

from __future__ import annotations

import json
import random
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

import dicmine  # noqa: E402
from dicmine import datasets as ref_ds  # noqa: E402

TEXT_CASES = [
    "0 1\n0 1\n0\n",
    "0 1\r\n# comment\n\n 2  1_0 +3 -0\r5\x1c6\t7\x0b8\x0c9\n",
    "   # indented comment\n3 3 3 1\n\n\n1 3\n",
    "1 2 3",  # no final newline
    "\r\r4\r\n\r\n5 6 5\n#\n",
    "007 0_0 +0 1_2\n",
    "0 1\nx\n",  # ParseError at line 2
    "0 1\n\n1__0\n",  # ParseError (double underscore)
    "1\n2 -1\n",  # ItemOutOfRange(-1)
    "5\n\n\n# c\n70000\n",  # ItemOutOfRange(70000) at line 5
    "1 + 2\n",  # lone sign
    "3_\n",  # trailing underscore
    "# only comments\n\n",  # EmptyDatabase
    "1 0x10\n",
]


def text_case(text: str) -> dict:
    with tempfile.TemporaryDirectory() as d:
        p = Path(d) / "t.txt"
        p.write_bytes(text.encode("utf-8"))
        try:
            db, rep = ref_ds.load_transactions_with_report(p)
        except dicmine.ParseError as e:
            return {"text": text, "error": "ParseError", "line": e.line, "token": e.token}
        except dicmine.ItemOutOfRange as e:
            return {"text": text, "error": "ItemOutOfRange", "line": e.line, "item": e.item}
        except dicmine.EmptyDatabase:
            return {"text": text, "error": "EmptyDatabase"}
        return {"text": text, "masks": [int(x) for x in db], "m": db.m, "transactions": rep.transactions,
                "deduplicated": rep.deduplicated}


def random_text(rng: random.Random) -> str:
    ws = [" ", "  ", "\t", "\x0b", "\x0c", "\x1c", "\x1f"]
    nl = ["\n", "\r\n", "\r"]
    out = []
    for _ in range(rng.randint(1, 40)):
        r = rng.random()
        if r < 0.1:
            out.append("# " + "".join(rng.choice("abc 12") for _ in range(rng.randint(0, 6))))
        elif r < 0.2:
            out.append(rng.choice(["", " ", "\t"]))
        else:
            toks = [str(rng.randint(0, 63)) for _ in range(rng.randint(1, 8))]
            out.append(rng.choice(["", " "]) + rng.choice(ws).join(toks) + rng.choice(["", " ", "\t"]))
    return "".join(line + rng.choice(nl) for line in out)


def binary_cases() -> list[dict]:
    cases = []
    for masks, m in [([0x3, 0x3, 0x1], None), ([0, 0x8000000000000000, 5], 64), ([1, 2, 4, 8], 10)]:
        db = dicmine.BitDatabase(masks, m=m)
        with tempfile.TemporaryDirectory() as d:
            p = Path(d) / "c.bin"
            ref_ds.save_bitdb(db, p)
            cases.append({"hex": p.read_bytes().hex(), "masks": [int(x) for x in db], "m": db.m})
    return cases


def estimator_cases() -> list[dict]:
    out = []
    tx = [[0, 1], [0, 1], [0], [0, 1, 2], [2]]
    rng = random.Random(0xE57)
    inputs = [(tx, 0.4, None, [[0, 1, 2], [2], []]), (tx, 0.25, 2, tx)]
    for _ in range(4):
        n, m = rng.randint(5, 60), rng.randint(2, 12)
        X = [[i for i in range(m) if rng.random() < 0.35] for _ in range(n)]
        Y = [[i for i in range(m) if rng.random() < 0.5] for _ in range(rng.randint(1, 20))]
        inputs.append((X, rng.choice([0.1, 0.2, 0.3]), rng.choice([None, max(1, n // 3)]), Y))
    for X, minsup, interval, Y in inputs:
        miner = dicmine.DicMiner(minsup=minsup, interval=interval).fit(X)
        out.append({"X": X, "minsup": minsup, "interval": interval, "Y": Y,
                    "masks": [int(v) for v in miner.itemset_masks_], "supports": [int(s) for s in miner.supports_],
                    "itemsets": [list(t) for t in miner.itemsets_], "n_items": miner.n_items_,
                    "names": list(miner.get_feature_names_out()),
                    "transform": miner.transform(Y).astype(int).tolist()})
    inc = np.array([[1, 1, 0], [1, 1, 0], [1, 0, 0], [1, 1, 1], [0, 0, 1]], dtype=np.int64)
    miner = dicmine.DicMiner(minsup=0.4).fit(inc)
    out.append({"incidence": inc.tolist(), "minsup": 0.4, "masks": [int(v) for v in miner.itemset_masks_],
                "supports": [int(s) for s in miner.supports_], "n_items": miner.n_items_})
    return out


SYNTH_SPECS = [(500, 64, 40.0, 42, 0.9), (2000, 20, 5.0, 7, 0.8), (100, 10, 3.5, 1, 0.9), (300, 64, 12.25, 3, 1.0),
               (40000, 64, 12.0, 7, 0.9), (17, 1, 1.0, 5, 0.5)]


def synthetic_cases() -> list[dict]:
    import hashlib

    out = []
    for n, m, avg, seed, skew in SYNTH_SPECS:
        db = ref_ds.generate_synthetic(ref_ds.DatasetSpec(n=n, m=m, avg_len=avg, seed=seed, skew=skew))
        raw = np.asarray(db.masks, dtype="<u8").tobytes()
        out.append({"n": n, "m": m, "avg_len": avg, "seed": seed, "skew": skew, "db_m": db.m,
                    "sha256": hashlib.sha256(raw).hexdigest(), "head": [int(x) for x in db.masks[:5]]})
    return out


def main() -> None:
    rng = random.Random(0x10AD)
    cases = [text_case(t) for t in TEXT_CASES] + [text_case(random_text(rng)) for _ in range(40)]
    (HERE / "io.json").write_text(json.dumps({"text": cases, "binary": binary_cases(),
                                              "synthetic": synthetic_cases()}, indent=0))
    (HERE / "estimator.json").write_text(json.dumps(estimator_cases(), indent=0))
    print("wrote io.json, estimator.json")


if __name__ == "__main__":
    main()
