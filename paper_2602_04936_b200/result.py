"""Result containers with the reference's canonical serialization.

``QueryResult`` mirrors trie.QueryResult (trie.py:51-78): bytes
``b"LCPR" | u8 version=1 | u8 mode | u16 matched_depth | u32 count |
u32[count] ids | u16[count] lcps``, little-endian.  ``FullScanResult``
mirrors oracle.OracleResult (oracle.py:19-35): ``b"ORCL" | u32 count | ids |
lcps``.  ``BatchResult`` is the batched form the GPU produces.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

MODE_CODES = {"strict": 0, "complete": 1, "tal": 2}


@dataclass(frozen=True, eq=False)
class QueryResult:
    indices: np.ndarray = field(repr=False)
    lcps: np.ndarray = field(repr=False)
    matched_depth: int
    mode: str

    @classmethod
    def _new(cls, indices, lcps, matched_depth: int, mode: str) -> "QueryResult":
        """The dataclass constructor without the frozen-field setattr calls
        (a single query's result is built on the latency-critical path)."""
        obj = object.__new__(cls)
        obj.__dict__.update(indices=indices, lcps=lcps, matched_depth=matched_depth, mode=mode)
        return obj

    def pairs(self) -> list[tuple[int, int]]:
        return list(zip(self.indices.tolist(), self.lcps.tolist()))

    def to_bytes(self) -> bytes:
        head = (
            b"LCPR"
            + bytes([1, MODE_CODES[self.mode]])
            + int(self.matched_depth).to_bytes(2, "little")
            + len(self.indices).to_bytes(4, "little")
        )
        return (
            head
            + np.ascontiguousarray(self.indices, dtype="<u4").tobytes()
            + np.ascontiguousarray(self.lcps, dtype="<u2").tobytes()
        )


def empty_result(mode: str, matched_depth: int = 0) -> QueryResult:
    z = np.zeros(0, dtype=np.int64)
    return QueryResult(indices=z, lcps=z.copy(), matched_depth=matched_depth, mode=mode)


@dataclass(frozen=True, eq=False)
class FullScanResult:
    """Exhaustive top-k (same contract and bytes as oracle.OracleResult)."""

    indices: np.ndarray = field(repr=False)
    lcps: np.ndarray = field(repr=False)

    def pairs(self) -> list[tuple[int, int]]:
        return list(zip(self.indices.tolist(), self.lcps.tolist()))

    def to_bytes(self) -> bytes:
        head = b"ORCL" + len(self.indices).to_bytes(4, "little")
        return (
            head
            + np.ascontiguousarray(self.indices, dtype="<u4").tobytes()
            + np.ascontiguousarray(self.lcps, dtype="<u2").tobytes()
        )


@dataclass(eq=False)
class BatchResult:
    """Raw batched output: row q holds ``hits[q]`` (id, lcp) pairs."""

    ids: np.ndarray            # (count, stride) uint32
    lcps: np.ndarray           # (count, stride) uint16
    hits: np.ndarray           # (count,) int32
    matched_depth: np.ndarray | None = None  # (count,) uint16
    aux: np.ndarray | None = None            # (count, 2) uint64
    mode: str = "complete"

    def __len__(self) -> int:
        return int(self.hits.shape[0])

    def pairs(self, q: int) -> list[tuple[int, int]]:
        h = int(self.hits[q])
        return list(zip(self.ids[q, :h].tolist(), self.lcps[q, :h].tolist()))

    def result(self, q: int) -> QueryResult:
        """QueryResult of row q, dtypes as the reference returns them."""
        h = int(self.hits.item(q))
        md = int(self.matched_depth.item(q)) if self.matched_depth is not None else 0
        if h == 0:
            return empty_result(self.mode, md)
        id_dtype = np.int64 if self.mode == "tal" else np.int32
        return QueryResult._new(self.ids[q, :h].astype(id_dtype), self.lcps[q, :h].astype(np.int64), md,
                                self.mode)

    def fullscan_result(self, q: int) -> FullScanResult:
        h = int(self.hits[q])
        return FullScanResult(
            indices=self.ids[q, :h].astype(np.int64), lcps=self.lcps[q, :h].astype(np.int64)
        )
