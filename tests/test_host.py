"""CPU-only checks: host logic of the drop-in API, the C-ABI library's symbol
table, the sharding arithmetic and the synthetic generators."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import paper_1812_10959_b200 as dic
from paper_1812_10959_b200 import _abi, bits
from paper_1812_10959_b200.workloads import CONFIGS, generate_csr, scaled
from tests.golden_util import csr_digest, has_config_golden, load_config_golden

ROOT = Path(__file__).resolve().parent.parent


def header_functions() -> list[str]:
    text = (ROOT / "include" / "dic_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(dic_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _abi.load()
    names = header_functions()
    assert len(names) >= 25
    for name in names:
        assert hasattr(lib, name), f"{name} declared in include/dic_b200.h but not exported"
        assert name in _abi.SIGNATURES, f"{name} has no ctypes signature"
    assert lib.dic_abi_version() == 1


def test_library_links_no_torch():
    # the boundary is a plain C ABI: no torch / c10 symbols in the library
    out = Path(_abi.lib_path()).read_bytes()
    assert b"c10::" not in out and b"at::Tensor" not in out


def test_argument_errors_surface_before_launch():
    with pytest.raises(_abi.DicError) as ei:
        _abi.call("dic_count_support", None, 10, 64, 5, 3, None, 2, 1, None, None)
    assert ei.value.code == _abi.DIC_EINVAL and "outside database" in ei.value.msg
    with pytest.raises(_abi.DicError):
        _abi.call("dic_count_support", None, 10, 70000, 0, 3, None, 2, 1, None, None)
    with pytest.raises(_abi.DicError):
        _abi.call("dic_engine_create", None, 10, 0, 1, 1, 1, 1, None, ctypes.byref(ctypes.c_void_p()))


def test_params_semantics():
    p = dic.MiningParams.create(10, 0.3)
    assert (p.interval, p.intervals_per_pass, p.min_support_count) == (5, 2, 3)
    assert dic.MiningParams.create(1, 1.0).interval == 1
    assert dic.absolute_support(0.07, 100) == 8  # float ceil, as the reference
    p = dic.MiningParams.create(10, 0.5, interval=3)
    assert [p.chunk_bounds(s) for s in range(1, 5)] == [(0, 2), (3, 5), (6, 8), (9, 9)]
    for bad in [dict(n=0, minsup=0.5), dict(n=3, minsup=0.0), dict(n=3, minsup=1.5),
                dict(n=3, minsup=0.5, interval=4), dict(n=3, minsup=0.5, threads=0)]:
        with pytest.raises(ValueError):
            dic.MiningParams.create(**bad)


def test_bit_helpers():
    assert dic.encode_transaction([63, 0, 0]) == 0x8000000000000001
    assert dic.encode_transaction([200]) == 1 << 200  # no 64-item cap
    with pytest.raises(dic.ItemOutOfRange):
        dic.encode_transaction([-1])
    assert dic.contains(0x5, 0x7) and not dic.contains(0x5, 0x6)
    assert list(dic.immediate_subsets(0x7)) == [0x6, 0x5, 0x3]
    assert list(dic.items_of(0x25)) == [0, 2, 5] and dic.cardinality(1 << 300 | 1) == 2
    # exhaustive 6-item containment == set inclusion
    for a in range(64):
        for b in range(64):
            assert dic.contains(a, b) == ({i for i in range(6) if a >> i & 1} <= {i for i in range(6) if b >> i & 1})
    ints = [0, 1 << 70 | 5, (1 << 128) - 1]
    assert bits.array_to_masks(bits.masks_to_array(ints, 3)) == ints
    assert bits.masks_to_items([0x5, 1 << 65 | 2], 2).tolist() == [[0, 2], [1, 65]]


def test_bitdatabase_host_semantics():
    db = dic.BitDatabase([0x3, 0x3, 0x1])
    assert (db.n, db.m, len(db)) == (3, 2, 3) and db.masks.dtype == np.uint64 and db.masks.ndim == 1
    assert db[0] == 3 and list(db) == [3, 3, 1] and db.union_mask() == 3
    with pytest.raises(ValueError):
        db.masks[0] = 7
    with pytest.raises(dic.EmptyDatabase):
        dic.BitDatabase([])
    with pytest.raises(dic.ItemOutOfRange):
        dic.BitDatabase([0x10], m=4)
    with pytest.raises(ValueError):
        dic.BitDatabase([1], m=0)
    wide = dic.BitDatabase([1 << 100, 3])
    assert wide.m == 101 and wide.masks.shape == (2, 2) and wide.as_int_list() == [1 << 100, 3]
    assert dic.BitDatabase([0, 0]).m == 1  # empty rows allowed, m >= 1
    assert dic.BitDatabase(np.array([5, 1], dtype=np.uint64), m=64) == dic.BitDatabase([5, 1], m=64)


def test_catalog_semantics():
    cat = dic.ItemsetCatalog()
    audit = dic.TransitionAudit()
    r = cat.add_candidate(0x6, audit)
    assert cat.shape_of(0x6) is dic.Shape.DASHED_CIRCLE and r.size == 2
    cat.transition(r, dic.Shape.NIL, audit)
    cat.compact_dashed()
    assert cat.dashed == [] and 0x6 in cat.known  # known keeps every mask ever created
    cat.transition(r, dic.Shape.SOLID_BOX, audit)
    assert audit.illegal() == [(0x6, dic.Shape.NIL, dic.Shape.SOLID_BOX)]


def test_shard_plan_partitions_every_chunk():
    for n, M, G in [(10, 3, 2), (1000, 1000, 8), (977, 50, 8), (7, 1, 4), (3, 2, 8)]:
        p = dic.MiningParams.create(n, 0.5, interval=M)
        plans = [dic.ShardPlan.for_params(p, G, r) for r in range(G)]
        for s in range(1, p.intervals_per_pass + 1):
            first, last = p.chunk_bounds(s)
            covered = []
            for pl in plans:
                b, ln = pl.slice_of(s)
                covered.extend(range(b, b + ln))
                lf, ll = pl.local_chunk(s)
                assert ll - lf + 1 == ln
            assert covered == list(range(first, last + 1))
        assert sum(pl.local_rows() for pl in plans) == n
        for pl in plans:
            chunks = pl.local_chunks()
            assert chunks == [pl.local_chunk(s) for s in range(1, p.intervals_per_pass + 1)]


def test_generators_are_deterministic_and_split_invariant():
    for idx in (1, 2, 3):
        cfg = scaled(CONFIGS[idx], 5000)
        a = generate_csr(cfg, threads=1)
        b = generate_csr(cfg, ranges=[(0, 1234), (1234, 3766)], threads=5)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        # rows are sorted, duplicate-free and inside the universe
        ip, ix = a
        for r in range(0, 5000, 97):
            row = ix[ip[r]:ip[r + 1]]
            assert np.all(np.diff(row) > 0) and (row.size == 0 or (row[0] >= 0 and row[-1] < cfg.m))
    # a shard generated alone equals the same rows of the full set
    cfg = scaled(CONFIGS[4], 20000)
    ip, ix = generate_csr(cfg)
    sip, six = generate_csr(cfg, ranges=[(5000, 100), (15000, 50)])
    want = np.concatenate([ix[ip[5000]:ip[5100]], ix[ip[15000]:ip[15050]]])
    assert np.array_equal(six, want)


@pytest.mark.parametrize("idx", [1, 2, 3])
def test_config_inputs_match_golden_digest(idx):
    if not has_config_golden(idx):
        pytest.skip("golden not generated")
    g = load_config_golden(idx)
    ip, ix = generate_csr(CONFIGS[idx])
    assert csr_digest(ip, ix) == g.meta["csr_sha256"]


def test_config_shapes():
    ip, ix = generate_csr(CONFIGS[1])
    lens = np.diff(ip)
    assert lens.min() >= 1 and lens.max() <= 64 and 9.0 < lens.mean() < 11.0
    ip, ix = generate_csr(scaled(CONFIGS[3], 20000))
    dens = np.diff(ip).mean() / 128
    assert 0.3 < dens < 0.45  # Beta(2,5) mean 0.286 plus planted groups


def test_result_builder_matches_python_construction():
    """csrc/pyresults.c builds MiningResult.frequent: the same FrequentItemset
    tuples (Python ints of any width, LSW-first words) as the reference's
    NamedTuple constructor would, for 1-word and wide masks, in input order."""
    from paper_1812_10959_b200.miner import sorted_frequent
    from paper_1812_10959_b200.phases import FrequentItemset

    rng = np.random.default_rng(3)
    for W in (1, 2, 16, 25):
        F = 500
        masks = rng.integers(0, 2**63, size=(F, W), dtype=np.uint64)
        masks[::7] = 0
        masks[::7, -1] = np.uint64(1) << np.uint64(63)  # the top bit of the top word
        sizes = rng.integers(1, 9, size=F).astype(np.int32)
        sups = rng.integers(0, 2**40, size=F).astype(np.int64)
        got = sorted_frequent(masks, sizes, sups, presorted=True)
        want = tuple(FrequentItemset(int(sum(int(masks[i, w]) << (64 * w) for w in range(W))), int(sizes[i]),
                                     int(sups[i])) for i in range(F))
        assert got == want
        assert all(type(f) is FrequentItemset for f in got) and got[0]._fields == ("mask", "size", "support")
    one = sorted_frequent(np.array([5, 3], dtype=np.uint64), np.array([2, 2], dtype=np.int32),
                          np.array([7, 8], dtype=np.int64), presorted=True)
    assert one == (FrequentItemset(5, 2, 7), FrequentItemset(3, 2, 8))
    assert sorted_frequent(np.zeros((0, 4), dtype=np.uint64), np.zeros(0, np.int32), np.zeros(0, np.int64)) == ()


def header_tids_index(m: int, item: int, g: int) -> int:
    """The tids layout exactly as include/dic_b200.h documents it."""
    TW = 32 if m <= 768 else 16
    t = g // TW
    return t * m * TW + item * TW + (g - t * TW)


@pytest.mark.parametrize("m", [1, 64, 128, 700, 768, 769, 1000, 4096])
def test_tids_layout_matches_header_formula(m):
    """dic_tids_index / dic_tids_words agree with the header's formula (the
    layout an external consumer indexes by)."""
    lib = _abi.load()
    TW = lib.dic_tids_tile_groups(m)
    assert TW == (32 if m <= 768 else 16)
    rng = np.random.default_rng(m)
    for _ in range(200):
        item, g = int(rng.integers(0, m)), int(rng.integers(0, 1 << 22))
        assert _abi.call("dic_tids_index", m, item, g) == header_tids_index(m, item, g)
    for n in (1, 31, 32, 33, TW * 32, TW * 32 + 1, 10_000_000):
        groups = -(-n // 32)
        assert lib.dic_tids_words(n, m) == -(-groups // TW) * m * TW
