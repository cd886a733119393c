"""Dataset ingestion and the binary cache (reference datasets.py:143-268).

The text format — one transaction per line, whitespace-separated integer item
ids, ``#`` comments and blank lines ignored — is parsed by a multithreaded
C++ scanner (csrc/textio.cpp) into CSR and encoded on the GPU straight into
the bit-sliced tiles (BitDatabase.from_csr); duplicate ids are counted by the
encoder.  Files holding non-ASCII bytes take a Python path with the
reference's exact str semantics.  Errors match the reference: ParseError /
ItemOutOfRange with the 1-based line (blank and comment lines counted),
EmptyDatabase, FormatError.

Binary cache: the reference's v1 layout (``<8sBQH`` header: magic, version,
n, m; then n little-endian uint64 masks) is written for m <= 64, so the
reference reads our files; for wider universes the same header carries
version 2 followed by n rows of W = ceil(m/64) little-endian words (LSW
first).  load_bitdb reads both, with the reference's checks and messages.
"""

from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _abi, bits
from .bitmap import MAX_ITEMS, BitDatabase
from .exceptions import EmptyDatabase, FormatError, ItemOutOfRange, ParseError

MAGIC = b"DICBDB01"
FORMAT_VERSION = 1       # the reference's single-word layout (m <= 64)
FORMAT_VERSION_WIDE = 2  # W words per row
_HEADER = struct.Struct(f"<{len(MAGIC)}sBQH")  # magic, version, n, m


@dataclass(frozen=True)
class LoadReport:
    """What the text loader saw: line count kept and duplicate items dropped."""

    transactions: int
    deduplicated: int


def _csr_from_handle(h: C.c_void_p) -> tuple[np.ndarray, np.ndarray]:
    n, nnz = C.c_int64(), C.c_int64()
    _abi.call("dic_csr_info", h, C.byref(n), C.byref(nnz))
    indptr = np.empty(n.value + 1, dtype=np.int64)
    indices = np.empty(max(nnz.value, 1), dtype=np.int32)
    _abi.call("dic_csr_export", h, indptr.ctypes.data, indices.ctypes.data)
    return indptr, indices[: nnz.value]


def _parse_python(path: Path) -> tuple[np.ndarray, np.ndarray]:
    """The reference's line loop (datasets.py:163-185), for Unicode input."""
    lens: list[int] = []
    flat: list[int] = []
    with path.open("r", encoding="utf-8") as fh:
        for lineno, raw in enumerate(fh, start=1):
            line = raw.strip()
            if not line or line.startswith("#"):
                continue
            count = 0
            for token in line.split():
                try:
                    item = int(token)
                except ValueError:
                    raise ParseError(token, lineno, source=str(path)) from None
                if not 0 <= item < MAX_ITEMS:
                    raise ItemOutOfRange(item, line=lineno, source=str(path))
                flat.append(item)
                count += 1
            lens.append(count)
    indptr = np.zeros(len(lens) + 1, dtype=np.int64)
    np.cumsum(lens, out=indptr[1:])
    return indptr, np.asarray(flat, dtype=np.int32)


def parse_transactions(path: str | Path, threads: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """Transaction text file -> CSR (int64 indptr[n+1], int32 ids), raising
    the reference's errors for a bad token."""
    path = Path(path)
    data = path.read_bytes()
    lib = _abi.load()
    h, st = C.c_void_p(), _abi.ParseStatus()
    rc = lib.dic_parse_transactions(data, len(data), MAX_ITEMS, threads, C.byref(h), C.byref(st))
    if rc == _abi.DIC_EDATA:
        if st.kind == 3:
            return _parse_python(path)
        token = data[st.offset: st.offset + st.length].decode("ascii")
        if st.kind == 1:
            raise ParseError(token, st.line, source=str(path))
        raise ItemOutOfRange(int(token), line=st.line, source=str(path))
    if rc != 0:
        raise _abi.DicError("dic_parse_transactions", rc, lib.dic_last_error().decode(errors="replace"))
    try:
        return _csr_from_handle(h)
    finally:
        lib.dic_csr_free(h)


def load_transactions_with_report(path: str | Path) -> tuple[BitDatabase, LoadReport]:
    """Parse a transaction text file, returning the database (encoded on the
    GPU) and a report (datasets.py:156-187)."""
    path = Path(path)
    indptr, indices = parse_transactions(path)
    n = indptr.size - 1
    if n == 0:
        raise EmptyDatabase(f"no transactions in {path}")
    m = max(int(indices.max()) + 1 if indices.size else 1, 1)  # BitDatabase(masks) infers m
    db, dedup = BitDatabase.from_csr(indptr, indices.astype(np.uint16), m, return_dedup=True)
    return db, LoadReport(transactions=n, deduplicated=dedup)


def load_transactions(path: str | Path) -> BitDatabase:
    """Parse a transaction text file into a BitDatabase."""
    db, _ = load_transactions_with_report(path)
    return db


def save_transactions(db: BitDatabase, path: str | Path) -> None:
    """Write the canonical text form: ascending item ids, one line per row
    (an empty transaction gives a blank line, which the loader skips)."""
    rows = np.ascontiguousarray(db.rows, dtype=np.uint64)
    lib = _abi.load()
    buf, ln = C.c_void_p(), C.c_int64()
    _abi.call("dic_format_transactions", rows.ctypes.data, rows.shape[0], rows.shape[1], 0, C.byref(buf),
              C.byref(ln))
    try:
        Path(path).write_bytes(C.string_at(buf, ln.value))
    finally:
        lib.dic_free_buffer(buf)


def save_bitdb(db: BitDatabase, path: str | Path) -> None:
    """Write the binary cache: v1 (the reference's layout) when m <= 64,
    else v2 with W words per row."""
    path = Path(path)
    rows = np.ascontiguousarray(db.rows, dtype="<u8")
    version = FORMAT_VERSION if db.m <= 64 else FORMAT_VERSION_WIDE
    with path.open("wb") as fh:
        fh.write(_HEADER.pack(MAGIC, version, db.n, db.m))
        fh.write((rows[:, 0] if version == FORMAT_VERSION else rows).tobytes())


def load_bitdb(path: str | Path) -> BitDatabase:
    """Read a binary cache written by save_bitdb (or the reference's), bit-exactly."""
    path = Path(path)
    try:
        blob = path.read_bytes()
    except OSError as exc:
        raise FormatError(f"cannot read {path}: {exc}") from exc
    if len(blob) < _HEADER.size:
        raise FormatError(f"{path}: truncated header ({len(blob)} bytes)")
    magic, version, n, m = _HEADER.unpack_from(blob)
    if magic != MAGIC:
        raise FormatError(f"{path}: bad magic {magic!r}")
    if version not in (FORMAT_VERSION, FORMAT_VERSION_WIDE):
        raise FormatError(f"{path}: unsupported version {version}")
    if n == 0:
        raise EmptyDatabase(f"{path}: zero transactions")
    if version == FORMAT_VERSION_WIDE and not 1 <= m <= MAX_ITEMS:
        raise FormatError(f"{path}: item universe {m} out of range")
    W = 1 if version == FORMAT_VERSION else bits.words_for(m)
    expected = _HEADER.size + 8 * n * W
    if len(blob) != expected:
        raise FormatError(f"{path}: expected {expected} bytes, found {len(blob)}")
    rows = np.frombuffer(blob, dtype="<u8", offset=_HEADER.size).astype(np.uint64).reshape(n, W)
    if not 1 <= m <= (64 if version == FORMAT_VERSION else MAX_ITEMS):
        raise FormatError(f"{path}: item universe {m} out of range")
    used = bits.from_words(np.bitwise_or.reduce(rows, axis=0)).bit_length()
    if used > m:
        raise FormatError(f"{path}: mask uses items beyond declared universe {m}")
    return BitDatabase(rows[:, 0] if W == 1 else rows, m=m)


def sniff_format(path: str | Path) -> str:
    """Guess "binary" or "text": magic bytes first, extension second."""
    path = Path(path)
    try:
        with path.open("rb") as fh:
            head = fh.read(len(MAGIC))
    except OSError:
        head = b""
    if head == MAGIC:
        return "binary"
    if path.suffix.lower() in (".bin", ".dicbdb"):
        return "binary"
    return "text"


def item_frequencies(db: BitDatabase) -> np.ndarray:
    """Fraction of transactions containing each item (datasets.py:145-153),
    from the GPU item-support kernel."""
    from . import device as D

    counts = D.item_support(db.device_tids(), db.n, db.m, 0, db.n - 1)
    return counts.cpu().numpy().astype(np.float64) / db.n
