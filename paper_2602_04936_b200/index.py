"""TrieIndex drop-in (mirror of lcpsearch.trie, pkg/src/lcpsearch/trie.py).

``build(dataset)`` (trie.py:397-431) hands the rows to the sm_100a extension,
which packs them into order-preserving u64 keys, sorts them with a stable LSD
radix sort (== core.lexicographic_order, core.py:162-174), computes adjacent
LCPs and the k-ary search levels.  ``TrieIndex.query`` (trie.py:290-342) runs
the batched GPU query (warp lower_bound + bounded range scan + warp top-k);
the reference's per-depth arena (``row_lo``, ``edge_symbol``,
``level_offset``; trie.py:409-419) is produced on the GPU on first access and
backs the structural introspection API (``node``, ``children``,
``check_invariants``), which — like the reference's — is host-side only and
never used by the query path.
"""

from __future__ import annotations

import contextlib
import threading
from dataclasses import dataclass

import numpy as np

from .core import (
    InternalInvariantError,
    InvalidInputError,
    dataset_parts,
    validate_query_batch,
    validate_query_row,
)
from .engine import NativeIndex
from .result import BatchResult, QueryResult
from .work import WorkReport, trie_counters, work_per_symbol

_U16 = np.dtype(np.uint16)  # native-order uint16: the wire format of a query batch


@dataclass(frozen=True)
class TrieNodeView:
    """Read-only handle on one arena node (trie.py:97-126)."""

    index: "TrieIndex"
    node_id: int
    depth: int
    row_lo: int
    row_hi: int

    @property
    def subtree_size(self) -> int:
        return self.row_hi - self.row_lo

    @property
    def edge_symbol(self) -> int | None:
        if self.node_id == 0:
            return None
        return int(self.index.edge_symbol[self.node_id])

    @property
    def posting(self) -> np.ndarray:
        if self.depth != self.index.length:
            return np.zeros(0, dtype=self.index.order.dtype)
        return self.index.order[self.row_lo : self.row_hi]

    def children(self) -> list["TrieNodeView"]:
        return self.index._children(self)


class TrieIndex:
    """Immutable GPU index over a dataset; concurrent readers are safe."""

    def __init__(self, native: NativeIndex):
        self._native = native
        self.n = native.n
        self.length = native.length
        self.sigma = native.sigma
        self.c_sym = work_per_symbol(self.length)
        self._lock = threading.Lock()
        self._tls = threading.local()  # this thread's latency-mode server (low_latency)
        self._order: np.ndarray | None = None
        self._arena: tuple[np.ndarray, np.ndarray, np.ndarray] | None = None

    # -- device-side structure (exported lazily) ---------------------------
    @property
    def native(self) -> NativeIndex:
        return self._native

    @property
    def order(self) -> np.ndarray:
        if self._order is None:
            o = self._native.export_order()
            o.setflags(write=False)
            self._order = o
        return self._order

    def _tables(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        with self._lock:
            if self._arena is None:
                row_lo, edge, off = self._native.export_trie()
                for a in (row_lo, edge, off):
                    a.setflags(write=False)
                self._arena = (row_lo, edge, off)
            return self._arena

    @property
    def row_lo(self) -> np.ndarray:
        return self._tables()[0]

    @property
    def edge_symbol(self) -> np.ndarray:
        return self._tables()[1]

    @property
    def level_offset(self) -> np.ndarray:
        if self._arena is not None:
            return self._arena[2]
        return self._native.level_offsets()

    @property
    def node_count(self) -> int:
        return int(self.level_offset[-1])

    @property
    def nbytes(self) -> int:
        """Device memory held by the GPU index (packed keys, order, search levels)."""
        return self._native.device_bytes

    @property
    def arena_nbytes(self) -> int:
        """Bytes of the reference's arena layout (trie.py:160-168) for this dataset."""
        return int(self.n * 4 + self.node_count * 6 + (self.length + 2) * 8)

    def new_work_report(self) -> WorkReport:
        return WorkReport(c_sym=self.c_sym)

    # -- node views (trie.py:170-211) --------------------------------------
    @property
    def root(self) -> TrieNodeView:
        return TrieNodeView(self, 0, 0, 0, self.n)

    def node(self, node_id: int) -> TrieNodeView:
        if not (0 <= node_id < self.node_count):
            raise InvalidInputError(f"node id {node_id} out of range")
        off = self.level_offset
        depth = int(np.searchsorted(off, node_id, side="right")) - 1
        lo = int(self.row_lo[node_id])
        return TrieNodeView(self, node_id, depth, lo, self._row_hi(node_id, depth))

    def _row_hi(self, node_id: int, depth: int) -> int:
        end = int(self.level_offset[depth + 1])
        return int(self.row_lo[node_id + 1]) if node_id + 1 < end else self.n

    def _children(self, view: TrieNodeView) -> list[TrieNodeView]:
        if view.depth >= self.length or self.n == 0:
            return []
        off = self.level_offset
        base, end = int(off[view.depth + 1]), int(off[view.depth + 2])
        lvl = self.row_lo[base:end]
        c0 = base + int(np.searchsorted(lvl, np.int32(view.row_lo), side="left"))
        c1 = base + int(np.searchsorted(lvl, np.int32(view.row_hi), side="left"))
        return [
            TrieNodeView(self, c, view.depth + 1, int(self.row_lo[c]), self._row_hi(c, view.depth + 1))
            for c in range(c0, c1)
        ]

    def _node_at(self, depth: int, row: int) -> TrieNodeView:
        off = self.level_offset
        base, end = int(off[depth]), int(off[depth + 1])
        j = base + int(np.searchsorted(self.row_lo[base:end], np.int32(row), side="right")) - 1
        return TrieNodeView(self, j, depth, int(self.row_lo[j]), self._row_hi(j, depth))

    # -- queries -----------------------------------------------------------
    def _validate_query(self, q) -> np.ndarray:
        return validate_query_row(q, self.length, self.sigma)

    def descend(self, q) -> tuple[TrieNodeView, int]:
        """Deepest node matching a prefix of q (trie.py:258-263), via the GPU
        strict query: its range is R(d_max)."""
        query = self._validate_query(q)
        if self.n == 0:
            return self.root, 0
        out = self._native.query_host(query.reshape(1, -1), 1, "strict")
        depth = int(out.matched_depth[0])
        rlo = int(out.aux[0, 1] >> np.uint64(32))
        if depth == 0:
            return self.root, 0
        return self._node_at(depth, rlo), depth

    def collect_top_k(self, node: TrieNodeView, k: int) -> np.ndarray:
        """k smallest item ids of a node's subtree (trie.py:265-279); host
        introspection over the exported order, not used by query()."""
        if k < 1:
            raise InvalidInputError(f"k must be >= 1, got {k}")
        rows = self.order[node.row_lo : node.row_hi]
        if k >= rows.size:
            return np.sort(rows)
        return np.sort(np.partition(rows, k - 1)[:k])

    def subtree_items_lexicographic(self, node: TrieNodeView) -> np.ndarray:
        return self.order[node.row_lo : node.row_hi]

    def query(self, q, k: int, mode: str = "strict", work: WorkReport | None = None) -> QueryResult:
        """Top-k by LCP (trie.py:290-342), one query, on the GPU."""
        if mode not in ("strict", "complete"):
            raise InvalidInputError(f"mode must be 'strict' or 'complete', got {mode!r}")
        if k < 1:
            raise InvalidInputError(f"k must be >= 1, got {k}")
        if (type(q) is np.ndarray and q.dtype is _U16 and q.ndim == 1 and q.shape[0] == self.length
                and self.n > 0):
            query = q  # the kernel checks the symbols and raises the same error
        else:
            query = self._validate_query(q)
        tls = getattr(self, "_tls", None)
        srv = getattr(tls, "server", None) if tls is not None else None
        if srv is not None and srv.k == k and srv.mode == mode:
            out = srv.query(query)  # latency mode (low_latency)
        else:
            out = self._native.query_single(query, k, mode)
        if work is not None:
            self._account(out, mode, work)
        return out.result(0)

    @contextlib.contextmanager
    def low_latency(self, k: int, mode: str = "complete"):
        """Within the block, this thread's ``query(q, k, mode)`` calls are
        answered by a resident GPU warp polling page-locked host memory (no
        launch, copy or event per query; engine.SingleQueryServer).  Shapes
        the server does not cover (W > 1, k > 32) keep the launch path.  Do not synchronise the whole device inside the block: the warp
        stays resident until it has been idle for 100 ms."""
        from .core import InvalidStateError
        from .engine import SingleQueryServer

        if mode not in ("strict", "complete"):
            raise InvalidInputError(f"mode must be 'strict' or 'complete', got {mode!r}")
        if k < 1:
            raise InvalidInputError(f"k must be >= 1, got {k}")
        srv = None
        if self.n > 0:
            try:
                srv = SingleQueryServer(self._native, k, mode)
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

    def query_batch(self, queries, k: int, mode: str = "complete", work: WorkReport | None = None,
                    out: BatchResult | None = None) -> BatchResult:
        """Batched query: (count, L) uint16 -> BatchResult (one kernel launch)."""
        if mode not in ("strict", "complete"):
            raise InvalidInputError(f"mode must be 'strict' or 'complete', got {mode!r}")
        if k < 1:
            raise InvalidInputError(f"k must be >= 1, got {k}")
        qs = validate_query_batch(queries, self.length, self.sigma)
        res = self._native.query_host(qs, k, mode, out=out)
        if work is not None:
            self._account(res, mode, work)
        return res

    def query_batch_async(self, queries, k: int, mode: str = "complete", out: BatchResult | None = None):
        """Asynchronous query_batch for pipelined serving: returns a pending
        batch whose result() yields the BatchResult.  ``queries`` and ``out``
        (pinned, from native.alloc_batch) must stay alive until then; up to
        _native.ASYNC_DEPTH batches per thread overlap copies and kernels."""
        if mode not in ("strict", "complete"):
            raise InvalidInputError(f"mode must be 'strict' or 'complete', got {mode!r}")
        if (type(queries) is np.ndarray and queries.dtype is _U16 and queries.ndim == 2
                and queries.shape[1] == self.length and queries.flags.c_contiguous):
            qs = queries  # already in the wire format; symbols are checked on the device
        else:
            qs = validate_query_batch(queries, self.length, self.sigma)
        if out is None:
            out = self._native.alloc_batch(qs.shape[0], k, mode, pinned=True)
        return self._native.query_host_async(qs, k, mode, out)

    def fullscan_batch(self, queries, k: int, out: BatchResult | None = None) -> BatchResult:
        """Brute-force top-k over the same corpus (oracle.py:46-59 semantics)."""
        if k < 1:
            raise InvalidInputError(f"k must be >= 1, got {k}")
        qs = validate_query_batch(queries, self.length, self.sigma)
        return self._native.fullscan_host(qs, k, out=out)

    def _account(self, out: BatchResult, mode: str, work: WorkReport) -> None:
        sym, nodes = trie_counters(out.aux, self.n, self.length, mode == "complete")
        work.symbols_compared += sym
        work.nodes_visited += nodes
        work.queries += len(out)

    def close(self) -> None:
        self._native.close()

    # -- integrity (trie.py:346-394), host-side over the exported arena -----
    def check_invariants(self) -> None:
        n, length = self.n, self.length
        row_lo, edge, off = self._tables()
        if self.node_count > n * length + 1:
            raise InternalInvariantError("node count exceeds n*L + 1")
        if int(off[0]) != 0 or int(off[-1]) != self.node_count:
            raise InternalInvariantError("level offsets do not cover the arena")
        if self.root.subtree_size != n:
            raise InternalInvariantError("root subtree size != n")
        if n == 0:
            if self.node_count != 1:
                raise InternalInvariantError("empty dataset must index to a bare root")
            return
        for d in range(length + 1):
            base, end = int(off[d]), int(off[d + 1])
            if base == end:
                raise InternalInvariantError(f"level {d} is empty")
            lo = row_lo[base:end].astype(np.int64)
            hi = np.append(lo[1:], n)
            sizes = hi - lo
            if int(lo[0]) != 0 or (sizes <= 0).any():
                raise InternalInvariantError(f"level {d} does not partition [0, n)")
            if d < length:
                nb, ne = int(off[d + 1]), int(off[d + 2])
                child_lo = row_lo[nb:ne].astype(np.int64)
                starts = np.searchsorted(child_lo, lo, side="left")
                child_sizes = np.append(child_lo[1:], n) - child_lo
                if not np.array_equal(np.add.reduceat(child_sizes, starts), sizes):
                    raise InternalInvariantError(f"subtree size recurrence fails at depth {d}")
                syms = edge[nb:ne].astype(np.int64)
                parent_of = np.searchsorted(starts, np.arange(ne - nb), side="right") - 1
                if np.any((np.diff(parent_of) == 0) & ~(np.diff(syms) > 0)):
                    raise InternalInvariantError(f"children not symbol-sorted at depth {d}")
        if int(off[length + 1]) - int(off[length]) > n:
            raise InternalInvariantError("more leaves than items")


def build(dataset) -> TrieIndex:
    """Build the GPU index (trie.py:397-431).  An empty dataset is valid."""
    items, length, sigma = dataset_parts(dataset)
    return TrieIndex(NativeIndex(items, length, sigma, tal_depth=-1))


class QueryCache:
    """Memo keyed on (query bytes, k, mode) with atomic get-or-insert
    (trie.py:434-461); values are immutable QueryResults."""

    def __init__(self) -> None:
        self._store: dict = {}
        self._lock = threading.Lock()
        self.hits = 0
        self.misses = 0

    def __len__(self) -> int:
        return len(self._store)

    def lookup(self, key):
        with self._lock:
            res = self._store.get(key)
            if res is None:
                self.misses += 1
            else:
                self.hits += 1
            return res

    def insert(self, key, value):
        with self._lock:
            return self._store.setdefault(key, value)


def memoized_query(index: TrieIndex, q, k: int, mode: str = "strict",
                   cache: QueryCache | None = None, work: WorkReport | None = None) -> QueryResult:
    """TrieIndex.query served from ``cache`` on repeats (trie.py:464-488)."""
    if cache is None:
        raise InvalidInputError("memoized_query requires a cache")
    if (type(q) is np.ndarray and q.dtype is _U16 and q.ndim == 1 and q.shape[0] == index.length
            and q.flags.c_contiguous):
        # a row already in the wire format is its own key: only validated
        # queries are ever inserted, so a hit needs no validation, and a miss
        # is validated below before it is counted (as the reference orders it)
        key = (q.tobytes(), int(k), mode)
        with cache._lock:
            hit = cache._store.get(key)
            if hit is not None:
                cache.hits += 1
        if hit is not None:
            if work is not None:
                work.cache_hits += 1
                work.queries += 1
            return hit
    query = index._validate_query(q)
    key = (query.tobytes(), int(k), mode)
    hit = cache.lookup(key)
    if hit is not None:
        if work is not None:
            work.cache_hits += 1
            work.queries += 1
        return hit
    return cache.insert(key, index.query(query, k, mode, work=work))


def memoized_query_batch(index: TrieIndex, queries, k: int, mode: str = "strict",
                         cache: QueryCache | None = None,
                         work: WorkReport | None = None) -> list[QueryResult]:
    """memoized_query over a batch with one GPU launch for the misses.

    Same results and counters as calling memoized_query on each row in order
    (trie.py:464-488): the first occurrence of a key that is not cached is a
    miss (answered by one query_batch over all misses); later occurrences in
    the batch and cached keys are hits (cache_hits += 1, no scan work)."""
    if cache is None:
        raise InvalidInputError("memoized_query requires a cache")
    if mode not in ("strict", "complete"):
        raise InvalidInputError(f"mode must be 'strict' or 'complete', got {mode!r}")
    if k < 1:
        raise InvalidInputError(f"k must be >= 1, got {k}")
    qs = validate_query_batch(queries, index.length, index.sigma)
    keys = [(row.tobytes(), int(k), mode) for row in qs]
    out: list = [None] * len(keys)
    first: dict = {}
    miss_rows: list[int] = []
    hits = 0
    for i, key in enumerate(keys):
        if key in first:  # repeat inside this batch: served by the first occurrence
            hits += 1
            with cache._lock:
                cache.hits += 1
            continue
        res = cache.lookup(key)
        if res is not None:
            out[i] = res
            hits += 1
        else:
            first[key] = i
            miss_rows.append(i)
    if miss_rows:
        b = index.query_batch(qs[miss_rows], k, mode, work=work)
        for j, i in enumerate(miss_rows):
            out[i] = cache.insert(keys[i], b.result(j))
    for i, key in enumerate(keys):
        if out[i] is None:
            out[i] = out[first[key]]
    if work is not None:
        work.cache_hits += hits
        work.queries += hits
    return out
