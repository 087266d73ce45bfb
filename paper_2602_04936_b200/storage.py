"""LCPI index snapshots (mirror of lcpsearch.storage, storage.py:12-27,
155-389), produced and consumed by the extension.

``index_snapshot_bytes`` serialises the GPU index's per-depth arena on the
device (lcp_index_snapshot); the bytes are identical to the reference's for
the same dataset.  ``index_from_snapshot_bytes`` validates a snapshot like the
reference loader, recovers the rows, rebuilds the GPU index and checks the
rebuilt snapshot reproduces the input byte for byte.  The LCPD dataset
format (storage.py:52-82) is plain I/O and is restated here for round trips.
"""

from __future__ import annotations

import ctypes
import struct

import numpy as np

from ._native import check, load
from .core import Alphabet, Dataset, InvalidInputError
from .engine import NativeIndex
from .index import TrieIndex

DATASET_MAGIC = b"LCPD"
INDEX_MAGIC = b"LCPI"
FORMAT_VERSION = 1
_DATASET_HEADER = struct.Struct("<4sHBBQII")


def index_snapshot_bytes(index: TrieIndex) -> bytes:
    """Canonical LCPI bytes of a built index (storage.py:155-210)."""
    lib = load()
    h = index.native.handle
    size = ctypes.c_int64(0)
    check(lib.lcp_index_snapshot(h, None, ctypes.byref(size)))
    buf = np.empty(int(size.value), dtype=np.uint8)
    check(lib.lcp_index_snapshot(h, buf.ctypes.data, ctypes.byref(size)))
    return buf.tobytes()


def write_index(path: str, index: TrieIndex) -> int:
    data = index_snapshot_bytes(index)
    with open(path, "wb") as fh:
        fh.write(data)
    return len(data)


def index_from_snapshot_bytes(raw: bytes, name: str = "<bytes>") -> TrieIndex:
    lib = load()
    arr = np.frombuffer(raw, dtype=np.uint8)
    h = ctypes.c_void_p()
    status = lib.lcp_index_from_snapshot(arr.ctypes.data if arr.size else None, arr.size, ctypes.byref(h))
    try:
        check(status)
    except InvalidInputError as e:
        raise InvalidInputError(f"{name}: {e}") from None
    return TrieIndex(NativeIndex.from_handle(h))


def read_index(path: str) -> TrieIndex:
    with open(path, "rb") as fh:
        return index_from_snapshot_bytes(fh.read(), name=path)


def write_dataset(path: str, dataset) -> int:
    """LCPD dataset file (storage.py:52-66)."""
    items = np.ascontiguousarray(dataset.items, dtype="<u2")
    header = _DATASET_HEADER.pack(DATASET_MAGIC, FORMAT_VERSION, 2, 0, items.shape[0],
                                  int(dataset.length), int(dataset.alphabet.size))
    with open(path, "wb") as fh:
        fh.write(header)
        fh.write(items.tobytes())
    return _DATASET_HEADER.size + items.nbytes


def read_dataset(path: str) -> Dataset:
    """LCPD reader (storage.py:69-82)."""
    with open(path, "rb") as fh:
        raw = fh.read()
    if len(raw) < _DATASET_HEADER.size:
        raise InvalidInputError(f"{path}: truncated dataset header")
    magic, version, width, _, n, length, sigma = _DATASET_HEADER.unpack_from(raw, 0)
    if magic != DATASET_MAGIC:
        raise InvalidInputError(f"{path}: not a dataset file (bad magic {magic!r})")
    if version != FORMAT_VERSION or width != 2:
        raise InvalidInputError(f"{path}: unsupported dataset version/width")
    body = raw[_DATASET_HEADER.size:]
    if len(body) != n * length * 2:
        raise InvalidInputError(f"{path}: payload size does not match the header")
    items = np.frombuffer(body, dtype="<u2").reshape(n, length)
    return Dataset.from_rows(items.astype(np.uint16), Alphabet(int(sigma)))
