"""Input/output rows of SURVEY.md §8(f) on the host (no GPU): the C++
transaction-text scanner against the reference loader's golden results and
against the reference's own line loop (restated in datasets._parse_python),
and the binary cache against files written by the reference's save_bitdb."""

from __future__ import annotations

import json
import random
from pathlib import Path

import numpy as np
import pytest

import paper_1812_10959_b200 as dic
from paper_1812_10959_b200 import datasets as ds

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "io.json").read_text())


def masks_of(indptr: np.ndarray, indices: np.ndarray) -> list[int]:
    out = []
    for r in range(indptr.size - 1):
        mk = 0
        for it in indices[indptr[r]: indptr[r + 1]].tolist():
            mk |= 1 << it
        out.append(mk)
    return out


def dedup_of(indptr: np.ndarray, indices: np.ndarray) -> int:
    return sum(int(indptr[r + 1] - indptr[r]) - len(set(indices[indptr[r]: indptr[r + 1]].tolist()))
               for r in range(indptr.size - 1))


@pytest.mark.parametrize("case", GOLD["text"], ids=lambda c: repr(c["text"][:20]))
def test_text_parser_matches_reference_loader(case, tmp_path):
    p = tmp_path / "t.txt"
    p.write_bytes(case["text"].encode("utf-8"))
    err = case.get("error")
    if err in ("ParseError", "ItemOutOfRange"):
        with pytest.raises(getattr(dic, err)) as ei:
            ds.parse_transactions(p)
        assert ei.value.line == case["line"]
        if err == "ParseError":
            assert ei.value.token == case["token"]
        else:
            assert ei.value.item == case["item"]
        return
    indptr, indices = ds.parse_transactions(p)
    if err == "EmptyDatabase":
        assert indptr.size == 1
        return
    assert masks_of(indptr, indices) == case["masks"]
    assert indptr.size - 1 == case["transactions"]
    assert dedup_of(indptr, indices) == case["deduplicated"]


@pytest.mark.parametrize("seed", range(6))
def test_text_parser_threads_equal_reference_loop(seed, tmp_path):
    """A multi-MB file split across threads == the reference's line loop."""
    rng = random.Random(seed)
    nl = ["\n", "\r\n", "\r"]
    lines = []
    for _ in range(60_000):
        r = rng.random()
        if r < 0.05:
            lines.append("# comment " + str(rng.randint(0, 9)))
        elif r < 0.1:
            lines.append(rng.choice(["", " ", "\t "]))
        else:
            lines.append(rng.choice([" ", "\t", "\x1c"]).join(str(rng.randint(0, 999)) for _ in range(rng.randint(1, 30))))
    text = "".join(line + rng.choice(nl) for line in lines)
    if seed % 2:
        text += "17 18"  # no final newline
    p = tmp_path / "big.txt"
    p.write_bytes(text.encode())
    a = ds.parse_transactions(p, threads=8)
    b = ds._parse_python(p)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    # an error deep in the file is reported at the same line by every split
    bad = text.split("\n")
    k = len(bad) * 3 // 4
    bad[k] = bad[k] + " 12x"
    p.write_bytes("\n".join(bad).encode())
    with pytest.raises(dic.ParseError) as e1:
        ds.parse_transactions(p, threads=8)
    with pytest.raises(dic.ParseError) as e2:
        ds._parse_python(p)
    assert (e1.value.line, e1.value.token) == (e2.value.line, e2.value.token)


def test_formatter_round_trip(tmp_path):
    rng = np.random.default_rng(3)
    rows = (rng.random((5000, 5)) < 0.3).astype(np.uint64) * rng.integers(0, 2**63, size=(5000, 5), dtype=np.uint64)
    rows[7] = 0  # an empty transaction -> a blank line, skipped on reload
    db = dic.BitDatabase(rows, m=320)
    p = tmp_path / "out.txt"
    ds.save_transactions(db, p)
    text = p.read_text()
    assert text.count("\n") == 5000
    want = "\n".join(" ".join(str(w * 64 + b) for w in range(5) for b in range(64)
                              if (int(rows[r, w]) >> b) & 1) for r in range(3)) + "\n"
    assert text.startswith(want)
    indptr, indices = ds.parse_transactions(p)
    keep = [r for r in range(5000) if rows[r].any()]
    assert masks_of(indptr, indices) == [dic.bits.from_words(rows[r]) for r in keep]


@pytest.mark.parametrize("case", GOLD["binary"], ids=lambda c: str(c["m"]))
def test_binary_cache_reads_and_writes_reference_files(case, tmp_path):
    p = tmp_path / "c.bin"
    p.write_bytes(bytes.fromhex(case["hex"]))
    db = ds.load_bitdb(p)
    assert db.m == case["m"] and [int(x) for x in db] == case["masks"]
    q = tmp_path / "d.bin"
    ds.save_bitdb(db, q)
    assert q.read_bytes().hex() == case["hex"]
    assert ds.sniff_format(q) == "binary"


def test_binary_cache_wide_and_errors(tmp_path):
    rng = np.random.default_rng(9)
    rows = rng.integers(0, 2**63, size=(100, 5), dtype=np.uint64)
    rows[:, 4] &= np.uint64((1 << 44) - 1)  # m = 300
    db = dic.BitDatabase(rows, m=300)
    p = tmp_path / "w.dat"
    ds.save_bitdb(db, p)
    back = ds.load_bitdb(p)
    assert back.m == 300 and np.array_equal(back.rows, db.rows)
    blob = p.read_bytes()
    for bad, msg in [(blob[:10], "truncated header"), (b"XXXXXXXX" + blob[8:], "bad magic"),
                     (blob[:8] + bytes([7]) + blob[9:], "unsupported version"), (blob[:-8], "expected")]:
        p.write_bytes(bad)
        with pytest.raises(dic.FormatError, match=msg):
            ds.load_bitdb(p)
    p.write_bytes(blob[:9] + (0).to_bytes(8, "little") + blob[17:19])
    with pytest.raises(dic.EmptyDatabase):
        ds.load_bitdb(p)
    v1 = ds._HEADER.pack(ds.MAGIC, 1, 2, 3) + np.array([1, 8], dtype="<u8").tobytes()  # item 3 >= m
    p.write_bytes(v1)
    with pytest.raises(dic.FormatError, match="beyond declared universe"):
        ds.load_bitdb(p)
    assert ds.sniff_format(tmp_path / "x.bin") == "binary" and ds.sniff_format(tmp_path / "x.txt") == "text"


@pytest.mark.parametrize("case", GOLD["synthetic"], ids=lambda c: f"{c['n']}x{c['m']}s{c['seed']}")
def test_synthetic_generator_is_the_reference_stream(case):
    import hashlib

    from paper_1812_10959_b200.synthetic import DatasetSpec, generate_synthetic

    db = generate_synthetic(DatasetSpec(n=case["n"], m=case["m"], avg_len=case["avg_len"], seed=case["seed"],
                                        skew=case["skew"]))
    masks = np.asarray(db.masks, dtype="<u8")
    assert db.m == case["db_m"] and masks[:5].tolist() == case["head"]
    assert hashlib.sha256(masks.tobytes()).hexdigest() == case["sha256"]


def test_synthetic_spec_validation():
    from paper_1812_10959_b200.synthetic import DatasetSpec, generate_synthetic

    for bad in [DatasetSpec(0, 8, 2, 1), DatasetSpec(5, 65, 2, 1), DatasetSpec(5, 8, 0, 1), DatasetSpec(5, 8, 9, 1),
                DatasetSpec(5, 8, 2, 1, skew=0.0)]:
        with pytest.raises(dic.SpecError):
            generate_synthetic(bad)
