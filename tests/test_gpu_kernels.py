"""Kernel-level parity on the GPU: encoder, bit-sliced transform, item support,
the hot support-count kernel and the row-form count, each against a plain
numpy restatement of the reference's `(T & I) == I` count (engine.py:43-58)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_1812_10959_b200 import device as D

pytestmark = pytest.mark.gpu


def np_count(rows: np.ndarray, first: int, last: int, masks: np.ndarray) -> np.ndarray:
    blk = rows[first : last + 1]
    out = np.empty(masks.shape[0], dtype=np.int64)
    for c in range(masks.shape[0]):
        out[c] = int(np.count_nonzero(np.all((blk & masks[c]) == masks[c], axis=1)))
    return out


def random_rows(rng, n, m, density):
    W = D.words_for(m)
    bits = rng.random((n, W * 64)) < density
    bits[:, m:] = False
    rows = np.packbits(bits.reshape(n, W, 64)[:, :, ::-1], axis=2, bitorder="big")
    return np.ascontiguousarray(rows.view(">u8").reshape(n, W).astype(np.uint64))


def items_to_masks(items: np.ndarray, W: int) -> np.ndarray:
    out = np.zeros((items.shape[0], W), dtype=np.uint64)
    for c, row in enumerate(items):
        for it in row:
            out[c, it >> 6] |= np.uint64(1) << np.uint64(it & 63)
    return out


def to_dev(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("m", [1, 7, 64, 65, 128, 300, 1000])
def test_encode_and_transpose(m):
    rng = np.random.default_rng(m)
    n = 2500
    lens = rng.integers(0, min(m, 12) + 1, size=n)
    indptr = np.zeros(n + 1, dtype=np.int64)
    indptr[1:] = np.cumsum(lens)
    indices = rng.integers(0, m, size=int(indptr[-1])).astype(np.int32)  # duplicates on purpose
    rows, status = D.encode_csr(to_dev(indptr), to_dev(indices), n, m)
    W = D.words_for(m)
    want = np.zeros((n, W), dtype=np.uint64)
    dedup = 0
    for r in range(n):
        s = set(indices[indptr[r] : indptr[r + 1]].tolist())
        dedup += lens[r] - len(s)
        for it in s:
            want[r, it >> 6] |= np.uint64(1) << np.uint64(it & 63)
    got = rows.cpu().numpy()
    assert np.array_equal(got, want)
    st = status.cpu().numpy()
    assert st[0] == dedup and st[1] == -1 and st[2] == -1
    tids = D.rows_to_tids(rows, n, m)
    t = tids.cpu().numpy().view(np.uint32)
    assert t.size == D.tids_words(n, m)
    TW = D.tile_groups(m)
    ntiles = t.size // (m * TW)
    tiles = t.reshape(ntiles, m, TW)
    for i in range(m):
        col = (want[:, i >> 6] >> np.uint64(i & 63)) & np.uint64(1)
        padded = np.zeros(ntiles * TW * 32, dtype=np.uint64)
        padded[:n] = col
        words = (padded.reshape(-1, 32) << np.arange(32, dtype=np.uint64)).sum(axis=1).astype(np.uint32)
        assert np.array_equal(tiles[:, i, :TW].reshape(-1), words), f"item {i}"


def test_encode_reports_first_bad_item():
    indptr = np.array([0, 2, 2, 5, 6], dtype=np.int64)
    indices = np.array([1, 3, 0, 70, 99, 64], dtype=np.int32)  # m=64: 70 at pos 3 (row 2) first
    rows, status = D.encode_csr(to_dev(indptr), to_dev(indices), 4, 64)
    st = status.cpu().numpy()
    assert st[1] == 3 and st[2] == 2


@pytest.mark.parametrize("m,n,idx,slabs", [
    (1, 700, "i32", 1), (64, 5000, "u16", 3), (300, 20000, "i32", 4), (1000, 9000, "u16", 2),
    (1000, 513, "i32", 1), (3000, 2100, "u16", 2), (777, 1, "i32", 1)])
def test_encode_straight_to_tiles(m, n, idx, slabs):
    """dic_encode_csr_tids (slab by slab; shared-memory tiles, and the
    global-atomic path at m=3000) == encode_csr + rows_to_tids, same status;
    dic_tids_to_rows inverts it."""
    rng = np.random.default_rng(m + n)
    lens = rng.integers(0, min(m, 25) + 1, size=n)
    indptr = np.zeros(n + 1, dtype=np.int64)
    indptr[1:] = np.cumsum(lens)
    ids = rng.integers(0, m, size=int(indptr[-1]))  # duplicates on purpose
    indices = ids.astype(np.uint16 if idx == "u16" else np.int32)
    rows, st_ref = D.encode_csr(to_dev(indptr), to_dev(ids.astype(np.int32)), n, m)
    want = D.rows_to_tids(rows, n, m).cpu().numpy()
    dip, dix = to_dev(indptr), to_dev(indices)
    tids = torch.full((max(D.tids_words(n, m), 1),), -1, dtype=torch.int32, device="cuda")
    status = torch.empty(4, dtype=torch.int64, device="cuda")
    D.encode_status_init(status)
    rpt = D.tile_groups(m) * 32
    per = -(-n // slabs)
    step = -(-per // rpt) * rpt
    for r0 in range(0, n, step):
        D.encode_csr_tids(dip, dix, n, m, r0, min(n, r0 + step), tids, status)
    D.encode_status_finish(dip, n, status)
    assert np.array_equal(tids.cpu().numpy(), want)
    assert np.array_equal(status.cpu().numpy(), st_ref.cpu().numpy())
    assert np.array_equal(D.tids_to_rows(tids, n, m).cpu().numpy(), rows.cpu().numpy())


def test_encode_tiles_first_bad_item_and_alignment():
    indptr = np.array([0, 2, 2, 5, 6], dtype=np.int64)
    indices = np.array([1, 3, 0, 70, 99, 64], dtype=np.int32)
    tids = torch.empty(D.tids_words(4, 64), dtype=torch.int32, device="cuda")
    status = torch.empty(4, dtype=torch.int64, device="cuda")
    D.encode_status_init(status)
    D.encode_csr_tids(to_dev(indptr), to_dev(indices), 4, 64, 0, 4, tids, status)
    D.encode_status_finish(to_dev(indptr), 4, status)
    st = status.cpu().numpy()
    assert st[1] == 3 and st[2] == 2
    from paper_1812_10959_b200._abi import DicError
    with pytest.raises(DicError):  # slab start not on a tile boundary
        D.encode_csr_tids(to_dev(indptr), to_dev(indices), 4, 64, 1, 4, tids, status)


def test_from_csr_host_slabs_equal_device_path():
    import paper_1812_10959_b200 as dic

    rng = np.random.default_rng(11)
    n, m = 50_000, 1000
    lens = rng.integers(1, 30, size=n)
    indptr = np.zeros(n + 1, dtype=np.int64)
    indptr[1:] = np.cumsum(lens)
    ids = rng.integers(0, m, size=int(indptr[-1])).astype(np.uint16)
    host = dic.BitDatabase.from_csr(torch.from_numpy(indptr).pin_memory(), torch.from_numpy(ids).pin_memory(), m,
                                    slabs=7)
    dev = dic.BitDatabase.from_csr(to_dev(indptr), to_dev(ids.astype(np.int32)), m)
    assert torch.equal(host.device_tids(), dev.device_tids())
    assert np.array_equal(host.rows, dev.rows)
    # int32 offsets (half the PCIe bytes; widened on the device), host and device
    h32 = dic.BitDatabase.from_csr(torch.from_numpy(indptr.astype(np.int32)).pin_memory(),
                                   torch.from_numpy(ids).pin_memory(), m, slabs=5)
    d32 = dic.BitDatabase.from_csr(to_dev(indptr.astype(np.int32)), to_dev(ids), m)
    assert torch.equal(h32.device_tids(), host.device_tids())
    assert torch.equal(d32.device_tids(), host.device_tids())
    with pytest.raises(dic.ItemOutOfRange) as ei:
        bad = ids.copy()
        bad[int(indptr[4321]) + 1] = 1000
        dic.BitDatabase.from_csr(indptr, bad, m, slabs=3)
    assert ei.value.item == 1000 and ei.value.line == 4321


@pytest.mark.parametrize("m,n,first,last", [
    (64, 4000, 0, 3999), (64, 4000, 17, 2049), (130, 3001, 5, 5), (1000, 10000, 999, 8190),
    (512, 70000, 123, 69999), (33, 1, 0, 0)])
def test_item_support(m, n, first, last):
    rng = np.random.default_rng(n + m)
    rows = random_rows(rng, n, m, 0.3)
    tids = D.rows_to_tids(to_dev(rows), n, m)
    got = D.item_support(tids, n, m, first, last).cpu().numpy()
    blk = rows[first : last + 1]
    want = np.array([np.count_nonzero((blk[:, i >> 6] >> np.uint64(i & 63)) & np.uint64(1)) for i in range(m)])
    assert np.array_equal(got, want)


@pytest.mark.parametrize("m,n,k,C,density,first,last", [
    (64, 5000, 2, 700, 0.4, 0, 4999),
    (64, 5000, 3, 300, 0.5, 31, 1031),       # unaligned both ends
    (128, 20000, 1, 128, 0.3, 1, 19998),
    (1000, 30000, 2, 5000, 0.05, 100, 29000),
    (512, 40000, 5, 2000, 0.5, 64, 39999),
    (200, 9000, 8, 500, 0.7, 0, 8999),
    (200, 9000, 11, 300, 0.8, 3, 8000),       # generic-k path
    (70, 100, 4, 50, 0.6, 40, 40),            # single-row chunk
    (1000, 200000, 2, 20000, 0.03, 77, 190000),  # TW=16, several candidate blocks x row splits
    (768, 100000, 3, 9000, 0.2, 0, 99999),      # largest TW=32 universe
    (2000, 5000, 2, 300, 0.1, 10, 4990),        # too wide to stage: global fallback
])
def test_count_support_matches_numpy(m, n, k, C, density, first, last):
    rng = np.random.default_rng(m * 7 + k)
    rows = random_rows(rng, n, m, density)
    items = np.sort(np.stack([rng.choice(m, size=k, replace=False) for _ in range(C)]), axis=1).astype(np.uint16)
    tids = D.rows_to_tids(to_dev(rows), n, m)
    got = D.count_support(tids, n, m, first, last, to_dev(items.view(np.int16))).cpu().numpy()
    want = np_count(rows, first, last, items_to_masks(items, D.words_for(m)))
    assert np.array_equal(got, want)
    # the literal row-form kernel agrees too
    got_rows = D.count_support_rows(to_dev(rows), first, last, to_dev(items_to_masks(items, D.words_for(m)))).cpu().numpy()
    assert np.array_equal(got_rows, want)


def test_count_support_accumulates():
    rng = np.random.default_rng(5)
    m, n = 96, 3000
    rows = random_rows(rng, n, m, 0.5)
    items = np.array([[1, 2], [5, 90], [0, 95]], dtype=np.uint16)
    tids = D.rows_to_tids(to_dev(rows), n, m)
    out = torch.full((3,), 7, dtype=torch.int64, device="cuda")
    D.count_support(tids, n, m, 0, 999, to_dev(items.view(np.int16)), out)
    D.count_support(tids, n, m, 1000, n - 1, to_dev(items.view(np.int16)), out)
    want = np_count(rows, 0, n - 1, items_to_masks(items, 2)) + 7
    assert np.array_equal(out.cpu().numpy(), want)


def test_bad_chunk_rejected():
    rows = to_dev(np.array([[1], [2]], dtype=np.uint64))
    tids = D.rows_to_tids(rows, 2, 2)
    with pytest.raises(D._abi.DicError):
        D.count_support(tids, 2, 2, 1, 0, to_dev(np.array([[0]], dtype=np.int16)))
    with pytest.raises(D._abi.DicError):
        D.count_support(tids, 2, 2, 0, 2, to_dev(np.array([[0]], dtype=np.int16)))


@pytest.mark.parametrize("m,n,density,first,last", [
    (64, 5000, 0.3, 0, 4999), (100, 3000, 0.4, 17, 2900), (700, 40000, 0.05, 123, 39000),
    (1000, 30000, 0.03, 0, 29999), (130, 33, 0.5, 3, 31), (2, 100, 0.5, 0, 99)])
def test_count_pairs_matches_numpy(m, n, density, first, last):
    rng = np.random.default_rng(m + n)
    rows = random_rows(rng, n, m, density)
    tids = D.rows_to_tids(to_dev(rows), n, m)
    tri = D.count_pairs(tids, n, m, first, last).cpu().numpy()
    blk = rows[first:last + 1]
    bitsm = np.stack([(blk[:, i >> 6] >> np.uint64(i & 63)) & np.uint64(1) for i in range(m)], axis=1).astype(np.float64)
    gram = bitsm.T @ bitsm
    iu = np.triu_indices(m, k=1)  # a-major order == tri_index
    assert np.array_equal(tri, gram[iu].astype(np.int64))


def test_tids_select_then_pairs():
    rng = np.random.default_rng(9)
    m, n = 900, 20000
    rows = random_rows(rng, n, m, 0.05)
    tids = D.rows_to_tids(to_dev(rows), n, m)
    items = np.sort(rng.choice(m, size=300, replace=False)).astype(np.int32)
    sub = D.tids_select(tids, n, m, to_dev(items))
    tri = D.count_pairs(sub, n, 300, 5, n - 2).cpu().numpy()
    blk = rows[5:n - 1]
    bitsm = np.stack([(blk[:, i >> 6] >> np.uint64(i & 63)) & np.uint64(1) for i in items], axis=1).astype(np.float64)
    gram = bitsm.T @ bitsm
    assert np.array_equal(tri, gram[np.triu_indices(300, k=1)].astype(np.int64))


@pytest.mark.parametrize("m,n", [(64, 5_000), (700, 3_000), (1000, 2_345), (769, 40)])
def test_encoded_tids_decode_with_header_formula_only(m, n):
    """An external consumer indexing the tids buffer with nothing but the
    header's formula (tests/test_host.py header_tids_index) reads back the
    rows; every word of the buffer is addressed by it and rows past n are zero."""
    from tests.test_host import header_tids_index

    rng = np.random.default_rng(m + n)
    rows = random_rows(rng, n, m, 0.2)
    tids = D.rows_to_tids(to_dev(rows), n, m).cpu().numpy().view(np.uint32)
    TW = 32 if m <= 768 else 16
    G = -(-(-(-n // 32)) // TW) * TW  # groups of the whole tiles
    idx = np.array([[header_tids_index(m, i, g) for i in range(m)] for g in range(G)], dtype=np.int64)
    words = tids[idx]  # [G][m]
    bits_gm = np.unpackbits(words.astype("<u4").view(np.uint8).reshape(G, m, 4), axis=2, bitorder="little")
    rowbits = bits_gm.transpose(0, 2, 1).reshape(G * 32, m)  # row 32g + b, item i
    assert not rowbits[n:].any(), "bits set past the last row"
    back = np.zeros_like(rows)
    for i in range(m):
        back[:, i >> 6] |= rowbits[:n, i].astype(np.uint64) << np.uint64(i & 63)
    assert np.array_equal(back, rows)
    used = np.zeros(tids.size, dtype=bool)
    used[idx.ravel()] = True
    assert used.all(), "the layout has no words outside the formula"
