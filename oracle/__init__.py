"""TEST INFRASTRUCTURE ONLY — CPU oracle for the LCP top-k path.

ctypes wrapper of ``oracle/liblcp_oracle.so`` (plain-C restatement of the
reference algorithm, see lcp_oracle.c).  Only tests/, __graft_entry__.smoke()
and bench.py's CPU-baseline leg may import this package; the product package
``paper_2602_04936_b200`` never does.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liblcp_oracle.so")

_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64

_SIG = {
    "orc_lexicographic_order": (None, [_P, _I64, _I32, _P]),
    "orc_adjacent_lcp": (None, [_P, _I64, _I32, _P]),
    "orc_trie_build": (_P, [_P, _I64, _I32, _I32]),
    "orc_trie_free": (None, [_P]),
    "orc_trie_node_count": (_I64, [_P]),
    "orc_trie_export": (None, [_P, _P, _P, _P, _P]),
    "orc_trie_query": (_I64, [_P, _P, _I64, _I32, _P, _P, _P, _P, _P]),
    "orc_tal_build": (_P, [_P, _I64, _I32, _I32, _I32]),
    "orc_tal_free": (None, [_P]),
    "orc_tal_has_directory": (ctypes.c_int, [_P]),
    "orc_tal_export": (None, [_P, _P, _P]),
    "orc_tal_bucket_range": (None, [_P, _P, _P, _P]),
    "orc_tal_query": (_I64, [_P, _P, _I64, _P, _P, _P, _P]),
    "orc_oracle_top_k": (_I64, [_P, _I64, _I32, _P, _I64, _P, _P]),
    "orc_trie_query_batch": (None, [_P, _P, _I64, _I64, _I32, _I64, _P, _P, _P, _P, _P, _P, _I32]),
    "orc_tal_query_batch": (None, [_P, _P, _I64, _I64, _I64, _P, _P, _P, _P, _P, _I32]),
    "orc_oracle_top_k_batch": (None, [_P, _I64, _I32, _P, _I64, _I64, _I64, _P, _P, _P, _I32]),
}

_lib = None


def build() -> str:
    """Compile the oracle (gcc, no GPU needed)."""
    src = os.path.join(HERE, "lcp_oracle.c")
    if not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        l = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIG.items():
            fn = getattr(l, name)
            fn.restype = res
            fn.argtypes = args
        _lib = l
    return _lib


def _p(a: np.ndarray) -> int:
    return int(a.ctypes.data)


def _rows(items) -> np.ndarray:
    return np.ascontiguousarray(items, dtype=np.uint16)


def lexicographic_order(rows) -> np.ndarray:
    r = _rows(rows)
    out = np.empty(r.shape[0], dtype=np.int64)
    lib().orc_lexicographic_order(_p(r), r.shape[0], r.shape[1], _p(out))
    return out


def adjacent_lcp(sorted_rows) -> np.ndarray:
    r = _rows(sorted_rows)
    out = np.zeros(max(0, r.shape[0] - 1), dtype=np.int64)
    if r.shape[0] > 1:
        lib().orc_adjacent_lcp(_p(r), r.shape[0], r.shape[1], _p(out))
    return out


def oracle_top_k(items, q, k: int) -> tuple[np.ndarray, np.ndarray]:
    r = _rows(items)
    q = np.ascontiguousarray(q, dtype=np.uint16)
    take = max(0, min(k, r.shape[0]))
    ids = np.empty(max(take, 1), dtype=np.int64)
    lcps = np.empty(max(take, 1), dtype=np.int64)
    h = lib().orc_oracle_top_k(_p(r), r.shape[0], r.shape[1], _p(q), k, _p(ids), _p(lcps))
    return ids[:h], lcps[:h]


def oracle_top_k_batch(items, qs, k: int, nthreads: int = 1):
    r = _rows(items)
    qs = _rows(qs)
    count = qs.shape[0]
    stride = max(1, min(k, r.shape[0]))
    ids = np.zeros((count, stride), dtype=np.int64)
    lcps = np.zeros((count, stride), dtype=np.int64)
    hits = np.zeros(count, dtype=np.int64)
    lib().orc_oracle_top_k_batch(_p(r), r.shape[0], r.shape[1], _p(qs), count, k, stride,
                                 _p(ids), _p(lcps), _p(hits), nthreads)
    return ids, lcps, hits


class OracleTrie:
    """trie.build + TrieIndex.query restated in C (trie.py:229-431)."""

    def __init__(self, items, sigma: int):
        r = _rows(items)
        self.n, self.length, self.sigma = r.shape[0], r.shape[1], sigma
        self._h = lib().orc_trie_build(_p(r), r.shape[0], r.shape[1], sigma)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_trie_free(self._h)
            self._h = None

    @property
    def node_count(self) -> int:
        return int(lib().orc_trie_node_count(self._h))

    def tables(self):
        nc = self.node_count
        order = np.empty(self.n, dtype=np.int32)
        row_lo = np.empty(nc, dtype=np.int32)
        edge = np.empty(nc, dtype=np.uint16)
        off = np.empty(self.length + 2, dtype=np.int64)
        lib().orc_trie_export(self._h, _p(order), _p(row_lo), _p(edge), _p(off))
        return order, row_lo, edge, off

    def query(self, q, k: int, mode: str):
        q = np.ascontiguousarray(q, dtype=np.uint16)
        cap = max(1, min(k, self.n))
        ids = np.empty(cap, dtype=np.int32)
        lcps = np.empty(cap, dtype=np.int64)
        md = np.zeros(1, dtype=np.int32)
        sym = np.zeros(1, dtype=np.int64)
        nodes = np.zeros(1, dtype=np.int64)
        h = lib().orc_trie_query(self._h, _p(q), k, 1 if mode == "complete" else 0, _p(ids),
                                 _p(lcps), _p(md), _p(sym), _p(nodes))
        return ids[:h], lcps[:h], int(md[0]), int(sym[0]), int(nodes[0])

    def query_batch(self, qs, k: int, mode: str, nthreads: int = 1):
        qs = _rows(qs)
        count = qs.shape[0]
        stride = max(1, min(k, self.n))
        ids = np.zeros((count, stride), dtype=np.int32)
        lcps = np.zeros((count, stride), dtype=np.int64)
        hits = np.zeros(count, dtype=np.int64)
        md = np.zeros(count, dtype=np.int32)
        sym = np.zeros(count, dtype=np.int64)
        nodes = np.zeros(count, dtype=np.int64)
        lib().orc_trie_query_batch(self._h, _p(qs), count, k, 1 if mode == "complete" else 0,
                                   stride, _p(ids), _p(lcps), _p(hits), _p(md), _p(sym),
                                   _p(nodes), nthreads)
        return ids, lcps, hits, md, sym, nodes


class OracleTal:
    """TalEngine restated in C (tal.py:29-194)."""

    def __init__(self, items, sigma: int, depth: int):
        r = _rows(items)
        self.n, self.length, self.sigma, self.depth = r.shape[0], r.shape[1], sigma, depth
        self._h = lib().orc_tal_build(_p(r), r.shape[0], r.shape[1], sigma, depth)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_tal_free(self._h)
            self._h = None

    def directory(self):
        if not lib().orc_tal_has_directory(self._h):
            return None
        out = np.empty(self.sigma**self.depth + 1, dtype=np.int64)
        lib().orc_tal_export(self._h, None, _p(out))
        return out

    def item_index(self):
        out = np.empty(self.n, dtype=np.int64)
        lib().orc_tal_export(self._h, _p(out), None)
        return out

    def bucket_range(self, q):
        q = np.ascontiguousarray(q, dtype=np.uint16)
        lo = np.zeros(1, dtype=np.int64)
        hi = np.zeros(1, dtype=np.int64)
        lib().orc_tal_bucket_range(self._h, _p(q), _p(lo), _p(hi))
        return int(lo[0]), int(hi[0])

    def query(self, q, k: int):
        q = np.ascontiguousarray(q, dtype=np.uint16)
        cap = max(1, min(k, self.n))
        ids = np.empty(cap, dtype=np.int64)
        lcps = np.empty(cap, dtype=np.int64)
        items = np.zeros(1, dtype=np.int64)
        sym = np.zeros(1, dtype=np.int64)
        h = lib().orc_tal_query(self._h, _p(q), k, _p(ids), _p(lcps), _p(items), _p(sym))
        return ids[:h], lcps[:h], int(items[0]), int(sym[0])

    def query_batch(self, qs, k: int, nthreads: int = 1):
        qs = _rows(qs)
        count = qs.shape[0]
        stride = max(1, min(k, self.n))
        ids = np.zeros((count, stride), dtype=np.int64)
        lcps = np.zeros((count, stride), dtype=np.int64)
        hits = np.zeros(count, dtype=np.int64)
        items = np.zeros(count, dtype=np.int64)
        sym = np.zeros(count, dtype=np.int64)
        lib().orc_tal_query_batch(self._h, _p(qs), count, k, stride, _p(ids), _p(lcps), _p(hits),
                                  _p(items), _p(sym), nthreads)
        return ids, lcps, hits, items, sym
