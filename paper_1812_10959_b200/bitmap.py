"""BitDatabase: the transaction bitmap, host view + HBM-resident device copies.

Keeps the reference's constructor and accessors (/root/reference/pkg/src/
dicmine/database.py:13-93): immutable, one mask per row, ``m`` inferred from
the highest set bit or validated.  Generalised to W = ceil(m/64) uint64 words
per row (LSW first); for m <= 64 ``masks`` is the same 1-D uint64 array as
the reference's.

Device residency: ``device_rows()`` is the row bitmap uint64 [n][W] in HBM,
``device_tids()`` the tiled bit-sliced copy the support-count kernel streams
(include/dic_b200.h).  A database built with ``from_csr`` is encoded on the
GPU (dic_encode_csr) and only copied back to the host if host masks are
asked for.
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
    def from_csr(cls, indptr, indices, m: int) -> "BitDatabase":
        """Encode CSR item lists (host or device arrays) on the GPU.

        Duplicate ids collapse; an id outside [0, m) raises
        ItemOutOfRange(item, line=row) for the first one in row-major order,
        as encode_transaction would (bitops.py:24-37)."""
        import torch

        from . import device as D

        D.require_cuda()
        if not 1 <= m <= MAX_ITEMS:
            raise ValueError(f"item universe size must be in [1, {MAX_ITEMS}], got {m}")
        ip = torch.as_tensor(indptr, dtype=torch.int64).cuda()
        ix = torch.as_tensor(indices, dtype=torch.int32).cuda()
        n = int(ip.numel()) - 1
        if n < 1:
            raise EmptyDatabase("database holds zero transactions")
        rows, status = D.encode_csr(ip, ix, n, m)
        st = status.cpu().numpy()
        if st[1] >= 0:
            raise ItemOutOfRange(int(ix[int(st[1])].item()), line=int(st[2]), universe=m)
        return cls.from_device_rows(rows, m)

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
            rows = self._dev_rows.cpu().numpy().view(np.uint64).copy()
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
            self._dev_rows = torch.from_numpy(np.ascontiguousarray(self._host_rows())).cuda()
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
