"""BitDatabase: the transaction bitmap, host view + HBM-resident device copies.

Keeps the reference's constructor and accessors (/root/reference/pkg/src/
dicmine/database.py:13-93): immutable, one mask per row, ``m`` inferred from
the highest set bit or validated.  Generalised to W = ceil(m/64) uint64 words
per row (LSW first); for m <= 64 ``masks`` is the same 1-D uint64 array as
the reference's.

Device residency: ``device_rows()`` is the row bitmap uint64 [n][W] in HBM,
``device_tids()`` the tiled bit-sliced copy the support-count kernel streams
(include/dic_b200.h).  A database built with ``from_csr`` is encoded on the
GPU straight into the tiles (dic_encode_csr_tids); rows and host masks are
derived from them only if asked for.
"""

from __future__ import annotations

from typing import Iterable, Iterator, Sequence

import numpy as np

from . import bits
from .exceptions import EmptyDatabase, ItemOutOfRange

MAX_ITEMS = 65535  # item ids travel as uint16 to the count kernel


def _or_reduce_bits(rows: np.ndarray) -> int:
    """Bit length of the OR of all rows (as one wide int)."""
    acc = np.bitwise_or.reduce(rows, axis=0)
    return bits.from_words(acc).bit_length()


class BitDatabase:
    __slots__ = ("_rows", "_n", "_m", "_ints", "_dev_rows", "_dev_tids")

    def __init__(self, masks: Sequence[int] | np.ndarray, m: int | None = None):
        if isinstance(masks, np.ndarray) and masks.ndim == 2:
            rows = np.array(masks, dtype=np.uint64)
        elif isinstance(masks, np.ndarray):
            if masks.ndim != 1:
                raise ValueError("masks must be a one-dimensional sequence (or [n][W] words)")
            rows = np.array(masks, dtype=np.uint64).reshape(-1, 1)
        else:
            vals = [int(v) for v in masks]
            if any(v < 0 for v in vals):
                raise OverflowError("can't convert negative int to unsigned")
            width = max((v.bit_length() for v in vals), default=0)
            W = bits.words_for(max(width, m or 1))
            rows = bits.masks_to_array(vals, W)
        if rows.shape[0] == 0:
            raise EmptyDatabase("database holds zero transactions")
        used = _or_reduce_bits(rows)
        m = self._check_universe(used, m)
        W = bits.words_for(m)
        if rows.shape[1] < W:
            rows = np.concatenate([rows, np.zeros((rows.shape[0], W - rows.shape[1]), np.uint64)], axis=1)
        elif rows.shape[1] > W:
            rows = np.ascontiguousarray(rows[:, :W])
        rows.setflags(write=False)
        self._rows: np.ndarray | None = rows
        self._n = int(rows.shape[0])
        self._m = m
        self._ints: list[int] | None = None
        self._dev_rows = None
        self._dev_tids = None

    @staticmethod
    def _check_universe(used_bits: int, m: int | None) -> int:
        if m is None:
            m = max(used_bits, 1)
            if m > MAX_ITEMS:
                raise ValueError(f"item universe size must be in [1, {MAX_ITEMS}], got {m}")
            return m
        if not 1 <= m <= MAX_ITEMS:
            raise ValueError(f"item universe size must be in [1, {MAX_ITEMS}], got {m}")
        if used_bits > m:
            raise ItemOutOfRange(used_bits - 1, universe=m)
        return m

    # -- construction on the device --------------------------------------
    @classmethod
    def from_csr(cls, indptr, indices, m: int, *, slabs: int = 8, return_dedup: bool = False):
        """Encode CSR item lists (host or device arrays) on the GPU, straight
        into the bit-sliced tiles the count kernels stream.

        ``indptr`` int64 or int32 [n+1] (int32 halves its PCIe bytes; it is
        widened on the device); ``indices`` uint16 (any universe up to
        MAX_ITEMS fits) or int32 ids.  Host inputs are copied in ``slabs``
        tile-aligned row slabs on a side stream, each slab encoded as soon as
        it lands (pinned host tensors make the copies asynchronous).
        Duplicate ids collapse; an id outside [0, m) raises
        ItemOutOfRange(item, line=row) for the first one in row-major order,
        as encode_transaction would (bitops.py:24-37).  ``return_dedup``:
        also return the number of duplicate ids dropped (LoadReport)."""
        import torch

        from . import device as D

        D.require_cuda()
        if not 1 <= m <= MAX_ITEMS:
            raise ValueError(f"item universe size must be in [1, {MAX_ITEMS}], got {m}")
        ip = indptr if isinstance(indptr, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(indptr))
        ix = indices if isinstance(indices, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(indices))
        if ip.dtype not in (torch.int64, torch.int32):
            ip = ip.to(torch.int64)
        if ix.dtype not in (torch.uint16, torch.int32):
            ix = ix.to(torch.int32)
        n = int(ip.numel()) - 1
        if n < 1:
            raise EmptyDatabase("database holds zero transactions")
        tids = torch.empty(max(D.tids_words(n, m), 1), dtype=torch.int32, device="cuda")
        status = torch.empty(4, dtype=torch.int64, device="cuda")
        D.encode_status_init(status)
        if ix.is_cuda:
            dip = ip.cuda(non_blocking=True).to(torch.int64)
            D.encode_csr_tids(dip, ix, n, m, 0, n, tids, status)
            dix = ix
        else:
            # slab pipeline: H2D of slab i+1 on a copy stream overlaps the
            # encode of slab i on the current stream
            host_ip = ip.numpy() if not ip.is_cuda else ip.cpu().numpy()
            dip = ip.cuda(non_blocking=True).to(torch.int64)  # int32 offsets widen on the device
            dix = torch.empty(max(int(ix.numel()), 1), dtype=ix.dtype, device="cuda")
            rpt = D.tile_groups(m) * 32
            per = -(-n // max(slabs, 1))  # ceil(n / slabs) rows, rounded up to whole tiles
            step = -(-per // rpt) * rpt
            main = torch.cuda.current_stream()
            copy = torch.cuda.Stream()
            copy.wait_stream(main)  # dix / dip allocated on main
            for r0 in range(0, n, step):
                r1 = min(n, r0 + step)
                p0, p1 = int(host_ip[r0]), int(host_ip[r1])
                with torch.cuda.stream(copy):
                    if p1 > p0:
                        dix[p0:p1].copy_(ix[p0:p1], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(copy)
                main.wait_event(ev)
                D.encode_csr_tids(dip, dix, n, m, r0, r1, tids, status)
            dix.record_stream(copy)
        D.encode_status_finish(dip, n, status)
        st = status.cpu().numpy()
        if st[1] >= 0:
            raise ItemOutOfRange(int(dix[int(st[1])].item()), line=int(st[2]), universe=m)
        db = cls.from_device_tids(tids, n, m)
        return (db, int(st[0])) if return_dedup else db

    @classmethod
    def from_device_tids(cls, tids, n: int, m: int) -> "BitDatabase":
        """Wrap HBM-resident bit-sliced tiles (no host copy; rows on demand)."""
        if n < 1:
            raise EmptyDatabase("database holds zero transactions")
        self = object.__new__(cls)
        self._rows = None
        self._n = int(n)
        self._m = int(m)
        self._ints = None
        self._dev_rows = None
        self._dev_tids = tids
        return self

    @classmethod
    def from_device_rows(cls, rows, m: int) -> "BitDatabase":
        """Wrap an HBM-resident row bitmap uint64 [n][W] (no host copy)."""
        self = object.__new__(cls)
        self._rows = None
        self._n = int(rows.shape[0])
        if self._n == 0:
            raise EmptyDatabase("database holds zero transactions")
        self._m = int(m)
        self._ints = None
        self._dev_rows = rows
        self._dev_tids = None
        return self

    # -- host view ---------------------------------------------------------
    def _host_rows(self) -> np.ndarray:
        if self._rows is None:
            rows = self.device_rows().cpu().numpy().view(np.uint64).copy()
            rows.setflags(write=False)
            self._rows = rows
        return self._rows

    @property
    def masks(self) -> np.ndarray:
        rows = self._host_rows()
        return rows[:, 0] if rows.shape[1] == 1 else rows

    @property
    def rows(self) -> np.ndarray:
        """Always the uint64 [n][W] form."""
        return self._host_rows()

    @property
    def n(self) -> int:
        return self._n

    @property
    def m(self) -> int:
        return self._m

    @property
    def words(self) -> int:
        return bits.words_for(self._m)

    def as_int_list(self) -> list[int]:
        if self._ints is None:
            self._ints = bits.array_to_masks(self._host_rows())
        return self._ints

    def union_mask(self) -> int:
        return bits.from_words(np.bitwise_or.reduce(self._host_rows(), axis=0))

    # -- device copies -----------------------------------------------------
    def device_rows(self):
        if self._dev_rows is None:
            import torch

            from . import device as D

            D.require_cuda()
            if self._rows is None and self._dev_tids is not None:
                self._dev_rows = D.tids_to_rows(self._dev_tids, self._n, self._m)
            else:
                self._dev_rows = torch.from_numpy(np.array(self._host_rows(), dtype=np.uint64)).cuda()
        return self._dev_rows

    def device_tids(self):
        if self._dev_tids is None:
            from . import device as D

            self._dev_tids = D.rows_to_tids(self.device_rows(), self._n, self._m)
        return self._dev_tids

    # -- container protocol ------------------------------------------------
    def __len__(self) -> int:
        return self._n

    def __getitem__(self, j: int) -> int:
        return bits.from_words(self._host_rows()[j])

    def __iter__(self) -> Iterator[int]:
        return iter(self.as_int_list())

    def __eq__(self, other: object) -> bool:
        if not isinstance(other, BitDatabase):
            return NotImplemented
        return self._m == other._m and np.array_equal(self._host_rows(), other._host_rows())

    __hash__ = None  # type: ignore[assignment]

    def __repr__(self) -> str:
        return f"BitDatabase(n={self._n}, m={self._m})"


def csr_from_lists(transactions: Iterable[Iterable[int]]) -> tuple[np.ndarray, np.ndarray]:
    """Ragged id lists -> (indptr int64[n+1], indices int32[nnz])."""
    lens, flat = [], []
    for t in transactions:
        row = [int(x) for x in t]
        lens.append(len(row))
        flat.extend(row)
    indptr = np.zeros(len(lens) + 1, dtype=np.int64)
    np.cumsum(lens, out=indptr[1:])
    return indptr, np.asarray(flat, dtype=np.int64)


def database_from_transactions(transactions: Iterable[Iterable[int]]) -> BitDatabase:
    """Ragged id lists -> BitDatabase, encoded on the GPU (duplicates collapse).

    The universe is inferred as max id + 1, as the reference's
    BitDatabase(masks) does from the highest set bit (database.py:34-36);
    a negative id raises ItemOutOfRange like encode_transaction."""
    indptr, flat = csr_from_lists(transactions)
    if flat.size and flat.min() < 0:
        q = int(np.argmax(flat < 0))
        row = int(np.searchsorted(indptr, q, side="right") - 1)
        raise ItemOutOfRange(int(flat[q]), line=row)
    m = max(int(flat.max()) + 1 if flat.size else 1, 1)
    if m > MAX_ITEMS:
        raise ValueError(f"item universe size must be in [1, {MAX_ITEMS}], got {m}")
    return BitDatabase.from_csr(indptr, flat.astype(np.int32), m)
