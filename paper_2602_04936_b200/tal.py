"""TalEngine drop-in (mirror of lcpsearch.tal, pkg/src/lcpsearch/tal.py).

Bucket depth d = min{d : sigma**d >= B} (tal.py:29-36); the GPU build sorts
the rows once and, when 0 < d and sigma**d <= 2**24 (tal.py:26), builds the
dense directory with one binary search per prefix code (== the reference's
``searchsorted(codes, arange(sigma**d + 1))``, tal.py:76-82).  A query scans
only its bucket on the GPU (one CTA per query, warp LCP by XOR/clz, warp
top-k by (lcp desc, id asc)) and reports items_scanned and
sum(min(lcp + 1, L)) exactly like tal.py:173-193.
"""

from __future__ import annotations

import contextlib
import threading

import numpy as np

from .core import InvalidInputError, dataset_parts, validate_query_batch, validate_query_row
from .engine import NativeIndex
from .result import BatchResult, QueryResult
from .work import WorkReport, tal_counters, work_per_symbol

MAX_DIRECTORY_ENTRIES = 1 << 24


def _prefix_depth(sigma: int, bucket_count: int) -> int:
    d, span = 0, 1
    while span < bucket_count:
        span *= sigma
        d += 1
    return d


class InvalidStateNoDirectory(InvalidInputError):
    """Dense directory was not built (bucket count above the cap)."""


class TalEngine:
    """Immutable bucketed scan engine on the GPU."""

    def __init__(self, dataset, bucket_count: int):
        if bucket_count < 1:
            raise InvalidInputError(f"bucket count must be >= 1, got {bucket_count}")
        items, length, sigma = dataset_parts(dataset)
        if bucket_count > sigma**length:
            raise InvalidInputError(
                f"bucket count {bucket_count} needs prefix depth beyond the "
                f"sequence length {length} (alphabet {sigma})"
            )
        depth = _prefix_depth(sigma, bucket_count)
        self._native = NativeIndex(items, length, sigma, tal_depth=depth)
        self.n = int(items.shape[0])
        self.length = length
        self.sigma = sigma
        self.bucket_depth = depth
        self.requested_buckets = bucket_count
        self.bucket_count = sigma**depth
        self.c_sym = work_per_symbol(length)
        self._has_directory = 0 < depth and self.bucket_count <= MAX_DIRECTORY_ENTRIES
        self._directory: np.ndarray | None = None
        self._rows: np.ndarray | None = None
        self._item_index: np.ndarray | None = None

    @property
    def native(self) -> NativeIndex:
        return self._native

    @property
    def directory(self) -> np.ndarray | None:
        if not self._has_directory:
            return None
        if self._directory is None:
            d = self._native.export_directory()
            d.setflags(write=False)
            self._directory = d
        return self._directory

    @property
    def rows(self) -> np.ndarray:
        """Sorted uint16 rows, decoded from the GPU's packed keys."""
        if self._rows is None:
            r = self._native.unpack_sorted_rows() if self.n else np.zeros((0, self.length), np.uint16)
            r.setflags(write=False)
            self._rows = r
        return self._rows

    @property
    def item_index(self) -> np.ndarray:
        if self._item_index is None:
            o = self._native.export_order().astype(np.int64)
            o.setflags(write=False)
            self._item_index = o
        return self._item_index

    @property
    def nbytes(self) -> int:
        return self._native.device_bytes

    def new_work_report(self) -> WorkReport:
        return WorkReport(c_sym=self.c_sym)

    # -- bucket lookup (tal.py:98-152) ---------------------------------------
    def _validate_query(self, q) -> np.ndarray:
        return validate_query_row(q, self.length, self.sigma, tal=True)

    def prefix_code(self, q) -> int:
        code = 0
        for j in range(self.bucket_depth):
            code = code * self.sigma + int(q[j])
        return code

    def bucket_range_directory(self, q) -> tuple[int, int]:
        if self.directory is None:
            raise InvalidStateNoDirectory()
        query = self._validate_query(q)
        code = self.prefix_code(query)
        return int(self.directory[code]), int(self.directory[code + 1])

    def bucket_range_search(self, q) -> tuple[int, int]:
        """GPU binary search on the packed d-prefixes (independent of the directory)."""
        query = self._validate_query(q)
        if self.bucket_depth == 0:
            return 0, self.n
        lo, hi = self._native.bucket_range_search(query.reshape(1, -1))
        return int(lo[0]), int(hi[0])

    def bucket_range(self, q) -> tuple[int, int]:
        if self.directory is not None:
            return self.bucket_range_directory(q)
        return self.bucket_range_search(q)

    def bucket_sizes(self) -> np.ndarray:
        if self.directory is not None:
            return np.diff(self.directory)
        raise InvalidInputError("bucket occupancy enumeration requires the dense directory")

    # -- queries (tal.py:155-194) ---------------------------------------------
    def query(self, q, k: int, work: WorkReport | None = None) -> tuple[QueryResult, WorkReport]:
        if k < 1:
            raise InvalidInputError(f"k must be >= 1, got {k}")
        query = self._validate_query(q)
        tls = getattr(self, "_tls", None)
        srv = getattr(tls, "server", None) if tls is not None else None
        if srv is not None and srv.k == k:
            out = srv.query(query)  # latency mode (low_latency)
        else:
            # the single-query path: pinned staging row and block, so the kernel
            # reads the row and writes the answer over PCIe directly (no copies)
            out = self._native.query_single(query, k, "tal")
        report = self.new_work_report()
        report.queries = 1
        items, sym = tal_counters(out.aux)
        if items:
            report.items_scanned = items
            report.symbols_compared = sym
        if work is not None:
            work.symbols_compared += report.symbols_compared
            work.items_scanned += report.items_scanned
            work.queries += 1
        return out.result(0), report

    @contextlib.contextmanager
    def low_latency(self, k: int):
        """Within the block, this thread's ``query(q, k)`` calls are answered
        by a resident GPU warp (engine.SingleQueryServer, TAL mode); shapes it
        does not cover keep the launch path.  Do not synchronise the whole
        device inside the block (the warp stays resident until 100 ms idle)."""
        from .core import InvalidStateError
        from .engine import SingleQueryServer

        if k < 1:
            raise InvalidInputError(f"k must be >= 1, got {k}")
        srv = None
        if self.n > 0:
            try:
                srv = SingleQueryServer(self._native, k, "tal")
            except InvalidStateError:
                srv = None
        if getattr(self, "_tls", None) is None:
            self._tls = threading.local()
        prev = getattr(self._tls, "server", None)
        self._tls.server = srv
        try:
            yield self
        finally:
            self._tls.server = prev
            if srv is not None:
                srv.close()

    def query_batch(self, queries, k: int, work: WorkReport | None = None,
                    out: BatchResult | None = None) -> BatchResult:
        if k < 1:
            raise InvalidInputError(f"k must be >= 1, got {k}")
        qs = validate_query_batch(queries, self.length, self.sigma)
        res = self._native.query_host(qs, k, "tal", out=out)
        if work is not None:
            items, sym = tal_counters(res.aux)
            work.items_scanned += items
            work.symbols_compared += sym
            work.queries += len(res)
        return res

    def close(self) -> None:
        self._native.close()


def build_tal(dataset, bucket_count: int) -> TalEngine:
    return TalEngine(dataset, bucket_count)


def tal_query(engine: TalEngine, q, k: int) -> tuple[QueryResult, WorkReport]:
    return engine.query(q, k)
