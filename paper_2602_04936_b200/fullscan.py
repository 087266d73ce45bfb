"""Brute-force full scan on the GPU (semantics of oracle.oracle_top_k,
pkg/src/lcpsearch/oracle.py:38-59): every item in original row order, top
min(k, n) by (lcp desc, id asc).  This is the contrast path of the paper's
TAL-vs-full-scan comparison, computed by the streaming
kernel k_fullscan + k_merge.  It is *not* the test oracle (see oracle/).
"""

from __future__ import annotations

import threading

import numpy as np

from .core import InvalidInputError, dataset_parts, validate_query_batch
from .engine import NativeIndex
from .result import BatchResult, FullScanResult


class FullScanEngine:
    """Device-resident packed corpus for streaming full scans."""

    def __init__(self, dataset):
        items, length, sigma = dataset_parts(dataset)
        self._native = NativeIndex(items, length, sigma, tal_depth=-1)
        self.n, self.length, self.sigma = self._native.n, length, sigma

    @property
    def native(self) -> NativeIndex:
        return self._native

    def top_k(self, q, k: int) -> FullScanResult:
        if k < 1:
            raise InvalidInputError(f"k must be >= 1, got {k}")
        arr = np.asarray(q)
        if arr.ndim != 1:
            raise InvalidInputError(f"sequence must be 1-D, got shape {arr.shape}")
        if arr.shape[0] != self.length:
            raise InvalidInputError(f"sequence length {arr.shape[0]} != expected {self.length}")
        if arr.size and (int(arr.min()) < 0 or int(arr.max()) >= self.sigma):
            raise InvalidInputError(
                f"symbol {int(arr.max())} out of range for alphabet of size {self.sigma}")
        out = self._native.fullscan_host(np.ascontiguousarray(arr, dtype=np.uint16).reshape(1, -1), k)
        return out.fullscan_result(0)

    def top_k_batch(self, queries, k: int, out: BatchResult | None = None) -> BatchResult:
        if k < 1:
            raise InvalidInputError(f"k must be >= 1, got {k}")
        qs = validate_query_batch(queries, self.length, self.sigma)
        return self._native.fullscan_host(qs, k, out=out)

    def close(self) -> None:
        self._native.close()


_cache_lock = threading.Lock()
_cache: dict[int, tuple[object, FullScanEngine]] = {}


def _engine_for(dataset) -> FullScanEngine:
    key = id(dataset)
    with _cache_lock:
        hit = _cache.get(key)
        if hit is not None and hit[0] is dataset:
            return hit[1]
    eng = FullScanEngine(dataset)
    with _cache_lock:
        if len(_cache) >= 4:
            _cache.pop(next(iter(_cache)))
        _cache[key] = (dataset, eng)
    return eng


def fullscan_top_k(dataset, q, k: int) -> FullScanResult:
    """Exact top-k over the whole dataset on the GPU; always min(k, n) hits."""
    if k < 1:
        raise InvalidInputError(f"k must be >= 1, got {k}")
    return _engine_for(dataset).top_k(q, k)


# Drop-in name of the reference's exhaustive scan (oracle.py:46).
oracle_top_k = fullscan_top_k
