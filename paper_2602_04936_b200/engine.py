"""Owner of one device-resident index built by the sm_100a extension.

``NativeIndex`` wraps an ``lcp_index*`` (include/lcp_b200.h) and exposes the
batched entry points with numpy (host, synchronous) or torch/device-pointer
(asynchronous) buffers.  TrieIndex, TalEngine and the full scan are thin
reference-compatible views over it.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _native
from ._native import IndexInfo, PinnedArray, check, load, ptr, workspace
from .core import InvalidInputError, SYMBOL_DTYPE
from .result import BatchResult

MODES = _native.MODE_CODES


class NativeIndex:
    """Packed, sorted, searchable corpus on the GPU (immutable after build)."""

    def __init__(self, items: np.ndarray, length: int, sigma: int, tal_depth: int = -1):
        lib = load()
        items = np.ascontiguousarray(items, dtype=SYMBOL_DTYPE)
        n = int(items.shape[0])
        h = ctypes.c_void_p()
        check(lib.lcp_index_build(ptr(items) if n else None, n, int(length), int(sigma),
                                  int(tal_depth), ctypes.byref(h)))
        self._h = h
        info = IndexInfo()
        check(lib.lcp_index_get_info(h, ctypes.byref(info)))
        self.info = info
        self.n = int(info.n)
        self.length = int(info.length)
        self.sigma = int(info.sigma)
        self.words = int(info.words)
        self.bits = int(info.bits)

    @classmethod
    def from_handle(cls, h: ctypes.c_void_p):
        """Adopt an lcp_index* built by the library (e.g. from a snapshot)."""
        self = cls.__new__(cls)
        self._h = h
        info = IndexInfo()
        check(load().lcp_index_get_info(h, ctypes.byref(info)))
        self.info = info
        self.n, self.length, self.sigma = int(info.n), int(info.length), int(info.sigma)
        self.words, self.bits = int(info.words), int(info.bits)
        return self

    @classmethod
    def from_device(cls, rows_ptr: int, n: int, length: int, sigma: int, tal_depth: int = -1):
        """Build from a device pointer (e.g. a CUDA uint16 tensor's data_ptr())."""
        self = cls.__new__(cls)
        lib = load()
        h = ctypes.c_void_p()
        check(lib.lcp_index_build(rows_ptr if n else None, int(n), int(length), int(sigma),
                                  int(tal_depth), ctypes.byref(h)))
        self._h = h
        info = IndexInfo()
        check(lib.lcp_index_get_info(h, ctypes.byref(info)))
        self.info = info
        self.n, self.length, self.sigma = int(info.n), int(info.length), int(info.sigma)
        self.words, self.bits = int(info.words), int(info.bits)
        return self

    @property
    def handle(self):
        if not self._h:
            raise RuntimeError("index has been closed")
        return self._h

    def close(self) -> None:
        if getattr(self, "_h", None):
            load().lcp_index_free(self._h)
            self._h = None

    def __del__(self) -> None:  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    @property
    def device_bytes(self) -> int:
        return int(self.info.device_bytes)

    # -- exports (parity / introspection) ------------------------------------
    def export_order(self) -> np.ndarray:
        out = np.empty(self.n, dtype=np.int32)
        if self.n:
            check(load().lcp_index_export_order(self.handle, ptr(out)))
        return out

    def export_sorted_keys(self) -> np.ndarray:
        out = np.empty((self.n, self.words), dtype=np.uint64)
        if self.n:
            check(load().lcp_index_export_sorted_keys(self.handle, ptr(out)))
        return out

    def export_sorted_key_range(self, first: int, count: int) -> np.ndarray:
        out = np.empty((count, self.words), dtype=np.uint64)
        if count:
            check(load().lcp_index_export_sorted_key_range(self.handle, int(first), int(count), ptr(out)))
        return out

    def export_adjacent_lcp(self) -> np.ndarray:
        out = np.empty(max(0, self.n - 1), dtype=np.uint16)
        if self.n > 1:
            check(load().lcp_index_export_adjacent_lcp(self.handle, ptr(out)))
        return out

    def export_directory(self) -> np.ndarray:
        out = np.empty(int(self.info.tal_buckets) + 1, dtype=np.int64)
        check(load().lcp_index_export_directory(self.handle, ptr(out)))
        return out

    def level_offsets(self) -> np.ndarray:
        out = np.empty(self.length + 2, dtype=np.int64)
        check(load().lcp_index_trie_level_offsets(self.handle, ptr(out)))
        return out

    def export_trie(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        off = self.level_offsets()
        nodes = int(off[-1])
        row_lo = np.empty(nodes, dtype=np.int32)
        edge = np.empty(nodes, dtype=np.uint16)
        check(load().lcp_index_export_trie(self.handle, ptr(row_lo), ptr(edge)))
        return row_lo, edge, off

    def bucket_range_search(self, queries: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
        q = np.ascontiguousarray(queries, dtype=np.uint16).reshape(-1, self.length)
        lo = np.empty(q.shape[0], dtype=np.int64)
        hi = np.empty(q.shape[0], dtype=np.int64)
        check(load().lcp_index_bucket_range_search(self.handle, ptr(q), q.shape[0], ptr(lo), ptr(hi)))
        return lo, hi

    def unpack_sorted_rows(self) -> np.ndarray:
        """Sorted uint16 rows decoded from the device's packed keys."""
        keys = self.export_sorted_keys()
        b = self.bits
        spw = 64 // b
        j = np.arange(self.length)
        word = keys[:, j // spw]
        shift = (64 - b * (j % spw + 1)).astype(np.uint64)
        return ((word >> shift) & np.uint64((1 << b) - 1)).astype(np.uint16)

    # -- queries -----------------------------------------------------------
    def stride_for(self, k: int) -> int:
        return max(1, min(int(k), self.n))

    def alloc_batch(self, count: int, k: int, mode: str = "complete", pinned: bool = True,
                    with_work: bool = True, pooled: bool = False) -> BatchResult:
        """Output buffers for ``count`` queries.  Pinned: one page-locked block
        in the lcp_packed_layout_for() layout, so a batch is one D2H copy.
        with_work=False (async path only) leaves matched_depth/aux out of
        the copy (BatchResult.matched_depth/aux are None)."""
        stride = self.stride_for(k)
        if not pinned:
            return BatchResult(
                ids=np.empty((count, stride), dtype=np.uint32),
                lcps=np.empty((count, stride), dtype=np.uint16),
                hits=np.empty(count, dtype=np.int32),
                matched_depth=np.empty(count, dtype=np.uint16),
                aux=np.empty((count, 2), dtype=np.uint64),
                mode=mode,
            )
        lay = _native.PackedLayout()
        check(load().lcp_packed_layout_for(count, stride, ctypes.byref(lay)))
        block = PinnedArray((int(lay.total),), np.uint8, pooled=pooled)
        raw = block.array

        def view(off, dt, shape):
            nbytes = int(np.prod(shape)) * np.dtype(dt).itemsize
            return raw[off:off + nbytes].view(dt).reshape(shape)

        out = BatchResult(
            ids=view(lay.ids, np.uint32, (count, stride)),
            lcps=view(lay.lcps, np.uint16, (count, stride)),
            hits=view(lay.hits, np.int32, (count,)),
            matched_depth=view(lay.matched_depth, np.uint16, (count,)),
            aux=view(lay.aux, np.uint64, (count, 2)),
            mode=mode,
        )
        out._owners = [block]  # the page-locked block lives as long as the result
        out._packed = (block.address, count, stride)
        out._flags = 0 if with_work else 1  # LCP_PACKED_NO_WORK
        if not with_work:
            out.matched_depth = None
            out.aux = None
        return out

    def single_query_buffer(self, k: int, mode: str) -> BatchResult:
        """Per-thread page-locked output block for one query (reused; callers
        copy results out before the next call on the same thread)."""
        cache = getattr(self, "_single", None)
        if cache is None:
            cache = self._single = threading.local()
        key = (self.stride_for(k), mode)
        buf = getattr(cache, "buf", None)
        if buf is None or buf[0] != key:
            buf = (key, self.alloc_batch(1, k, mode, pinned=True))
            cache.buf = buf
        return buf[1]

    def query_single(self, query: np.ndarray, k: int, mode: str) -> BatchResult:
        """One validated (L,) uint16 query, synchronously, with the lowest
        latency: the row is copied into this thread's page-locked staging row
        and submitted through the async packed entry point on the thread's
        workspace, whose graph cache turns H2D + kernel + D2H into a single
        graph launch from the second call on (stable staging / output
        pointers), and — stage and block being lcp_pinned_alloc memory — the
        kernel reads the row and writes the result over PCIe directly (no
        copies); then waits.  Returns the thread's reused one-row block."""
        if mode not in MODES:
            raise InvalidInputError(f"unknown mode {mode!r}")
        if k < 1:
            raise InvalidInputError(f"k must be >= 1, got {k}")
        out = self.single_query_buffer(k, mode)
        cache = self._single
        stage = getattr(cache, "stage", None)
        if stage is None or stage.shape[1] != self.length:
            stage = cache.stage = PinnedArray((1, self.length), np.uint16).array
        stage[0] = query
        out.mode = mode
        ws = workspace()
        packed = out._packed
        fast = _native.host_submit_wait()
        if fast is not None:  # csrc/host_submit.c: submission + wait in one call
            check(fast(self.handle.value, ws.address, stage, self.length, self.stride_for(k), MODES[mode],
                       packed[2], packed[0], 0))
            return out
        check(load().lcp_query_host_packed_async(self._h, ws.handle, ptr(stage), 1, self.stride_for(k),
                                                 MODES[mode], packed[2], packed[0], 0))
        check(load().lcp_workspace_wait(ws.handle))
        return out

    def query_host(self, queries: np.ndarray, k: int, mode: str,
                   out: BatchResult | None = None) -> BatchResult:
        """Synchronous batched query through lcp_query_host (H2D + kernel + D2H)."""
        if mode not in MODES:
            raise InvalidInputError(f"unknown mode {mode!r}")
        if k < 1:
            raise InvalidInputError(f"k must be >= 1, got {k}")
        count = int(queries.shape[0])
        k_eff = self.stride_for(k)
        if out is None:  # a pooled page-locked block: one H2D + one D2H, no per-call pinning
            out = self.alloc_batch(count, k, mode, pinned=True, pooled=True)
        out.mode = mode
        ws = workspace()
        packed = getattr(out, "_packed", None)
        if packed is not None and getattr(out, "_flags", 0):
            raise InvalidInputError("with_work=False blocks are for query_batch_async only")
        if packed is not None and packed[1] == count:
            check(load().lcp_query_host_packed(
                self.handle, ws.handle, ptr(queries), count, k_eff, MODES[mode], packed[2],
                packed[0]))
            return out
        check(load().lcp_query_host(
            self.handle, ws.handle, ptr(queries), count, k_eff, MODES[mode], out.ids.shape[1],
            ptr(out.ids), ptr(out.lcps), ptr(out.hits), ptr(out.matched_depth), ptr(out.aux)))
        return out

    def query_host_async(self, queries: np.ndarray, k: int, mode: str, out: BatchResult) -> "PendingBatch":
        """Enqueue H2D + kernel + D2H for one batch into a pinned packed block
        (from alloc_batch(pinned=True)) and return at once; .result() waits."""
        if mode not in MODES:
            raise InvalidInputError(f"unknown mode {mode!r}")
        if k < 1:
            raise InvalidInputError(f"k must be >= 1, got {k}")
        packed = getattr(out, "_packed", None)
        count = int(queries.shape[0])
        if packed is None or packed[1] != count:
            raise InvalidInputError("async queries need a pinned output block from alloc_batch")
        out.mode = mode
        h = self.handle
        ws = _native.async_workspace()
        fast = _native.host_submit()
        if fast is not None:  # csrc/host_submit.c: the same entry point without ctypes
            check(fast(h.value, ws.address, queries, self.length, self.stride_for(k), MODES[mode],
                       packed[2], packed[0], out._flags))
        else:
            check(load().lcp_query_host_packed_async(
                h, ws.handle, queries.__array_interface__["data"][0], count,
                self.stride_for(k), MODES[mode], packed[2], packed[0], out._flags))
        ws.submitted += 1
        return PendingBatch(ws, ws.submitted, out)

    def query_device(self, queries, k: int, mode: str, ids, lcps, hits, matched_depth=None,
                     aux=None, stream: int | None = None, ws=None) -> None:
        """Asynchronous batched query on device buffers (torch CUDA tensors or
        raw pointers); launches on ``stream`` (default: the workspace stream)."""
        count = int(queries.shape[0])
        ws = ws or workspace()
        st = ws.stream if stream is None else stream
        stride = int(ids.shape[1])
        check(load().lcp_query(
            self.handle, ws.handle, ptr(queries), count, self.stride_for(k), MODES[mode], stride,
            ptr(ids), ptr(lcps), ptr(hits), ptr(matched_depth), ptr(aux), st))

    def fullscan_host(self, queries: np.ndarray, k: int, out: BatchResult | None = None) -> BatchResult:
        if k < 1:
            raise InvalidInputError(f"k must be >= 1, got {k}")
        count = int(queries.shape[0])
        k_eff = self.stride_for(k)
        if out is None:
            out = self.alloc_batch(count, k, "complete", pinned=False)
        ws = workspace()
        check(load().lcp_fullscan_host(
            self.handle, ws.handle, ptr(queries), count, k_eff, out.ids.shape[1],
            ptr(out.ids), ptr(out.lcps), ptr(out.hits)))
        return out

    def fullscan_device(self, queries, k: int, ids, lcps, hits, stream: int | None = None, ws=None) -> None:
        count = int(queries.shape[0])
        ws = ws or workspace()
        st = ws.stream if stream is None else stream
        check(load().lcp_fullscan(
            self.handle, ws.handle, ptr(queries), count, self.stride_for(k), int(ids.shape[1]),
            ptr(ids), ptr(lcps), ptr(hits), st))


class SingleQueryServer:
    """Latency mode for one thread's single queries (lcp_server_*,
    csrc/serve_kernels.cuh): a resident warp answers each query written into
    a page-locked row, straight into a page-locked packed block, with no
    launch, copy or event per query.  Raises InvalidStateError for shapes
    the server does not cover (W > 1, k > 32)."""

    def __init__(self, native: "NativeIndex", k: int, mode: str):
        if mode not in MODES:
            raise InvalidInputError(f"unknown mode {mode!r}")
        self.k, self.mode = int(k), mode
        self._h = None
        self.row = PinnedArray((1, native.length), np.uint16)
        self.out = native.alloc_batch(1, k, mode, pinned=True)
        self.out.mode = mode
        packed = self.out._packed
        h = ctypes.c_void_p()
        check(load().lcp_server_start(native.handle, native.stride_for(k), MODES[mode], packed[2],
                                      self.row.address, packed[0], ctypes.byref(h)))
        self._h = h
        self._native = native  # the index outlives the server

    def query(self, query: np.ndarray) -> BatchResult:
        """``query``: a validated (L,) row (uint16 or any 2-byte integer array)."""
        fast = _native.host_server_query()
        if fast is not None and query.dtype.itemsize == 2 and query.flags.c_contiguous:
            check(fast(self._h.value, query))  # csrc/host_submit.c: the row read in place
            return self.out
        self.row.array[0] = query
        check(load().lcp_server_query(self._h))
        return self.out

    def close(self) -> None:
        if self._h:
            h, self._h = self._h, None
            check(load().lcp_server_stop(h))

    def __del__(self) -> None:  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass


class PendingBatch:
    """An in-flight async batch; result() blocks until its D2H copy landed."""

    __slots__ = ("_ws", "_seq", "_out")

    def __init__(self, ws, seq: int, out: BatchResult):
        self._ws = ws
        self._seq = seq
        self._out = out

    def result(self) -> BatchResult:
        ws = self._ws
        if ws.completed < self._seq:  # still this workspace's in-flight batch
            ws.wait()
        return self._out
