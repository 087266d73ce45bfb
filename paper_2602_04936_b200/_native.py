"""ctypes binding of the C ABI in ``include/lcp_b200.h``.

The shared library ``_lcp_b200.so`` is built in-tree for sm_100a by
:func:`paper_2602_04936_b200._build.build_native`.  There is no CPU fallback:
if the library is missing every entry point raises
:class:`NativeLibraryMissing` instead of computing anything on the host.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .core import InternalInvariantError, InvalidInputError, InvalidStateError

LIB_NAME = "_lcp_b200.so"
# LCP_B200_LIB: A/B hook for tools (a variant build of the same sources)
LIB_PATH = os.environ.get("LCP_B200_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

LCP_OK = 0
LCP_ERR_INVALID_INPUT = 3
LCP_ERR_INTERNAL = 4
LCP_ERR_CUDA = 5
LCP_ERR_STATE = 6

MODE_CODES = {"strict": 0, "complete": 1, "tal": 2}


class NativeLibraryMissing(RuntimeError):
    """The sm_100a extension is not built; there is deliberately no fallback."""


class CudaError(RuntimeError):
    """A CUDA runtime call inside the extension failed."""


class IndexInfo(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64),
        ("length", ctypes.c_int32),
        ("sigma", ctypes.c_int32),
        ("bits", ctypes.c_int32),
        ("syms_per_word", ctypes.c_int32),
        ("words", ctypes.c_int32),
        ("search_levels", ctypes.c_int32),
        ("tal_depth", ctypes.c_int32),
        ("has_directory", ctypes.c_int32),
        ("tal_buckets", ctypes.c_int64),
        ("device_bytes", ctypes.c_int64),
    ]


class PackedLayout(ctypes.Structure):
    _fields_ = [("ids", ctypes.c_int64), ("lcps", ctypes.c_int64), ("hits", ctypes.c_int64),
                ("matched_depth", ctypes.c_int64), ("aux", ctypes.c_int64),
                ("total", ctypes.c_int64), ("err", ctypes.c_int64)]


_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64

# name -> (restype, argtypes); the exported surface of include/lcp_b200.h
SIGNATURES = {
    "lcp_abi_version": (ctypes.c_int, []),
    "lcp_last_error": (ctypes.c_char_p, []),
    "lcp_index_build": (ctypes.c_int, [_P, _I64, _I32, _I32, _I32, ctypes.POINTER(_P)]),
    "lcp_index_free": (ctypes.c_int, [_P]),
    "lcp_index_get_info": (ctypes.c_int, [_P, ctypes.POINTER(IndexInfo)]),
    "lcp_index_export_order": (ctypes.c_int, [_P, _P]),
    "lcp_index_export_sorted_keys": (ctypes.c_int, [_P, _P]),
    "lcp_index_export_adjacent_lcp": (ctypes.c_int, [_P, _P]),
    "lcp_index_export_directory": (ctypes.c_int, [_P, _P]),
    "lcp_index_trie_level_offsets": (ctypes.c_int, [_P, _P]),
    "lcp_index_export_trie": (ctypes.c_int, [_P, _P, _P]),
    "lcp_index_bucket_range_search": (ctypes.c_int, [_P, _P, _I32, _P, _P]),
    "lcp_index_snapshot": (ctypes.c_int, [_P, _P, ctypes.POINTER(_I64)]),
    "lcp_index_from_snapshot": (ctypes.c_int, [_P, _I64, ctypes.POINTER(_P)]),
    "lcp_workspace_create": (ctypes.c_int, [ctypes.POINTER(_P)]),
    "lcp_workspace_free": (ctypes.c_int, [_P]),
    "lcp_workspace_stream": (_P, [_P]),
    "lcp_workspace_check": (ctypes.c_int, [_P, _P]),
    "lcp_packed_layout_for": (ctypes.c_int, [_I32, _I32, ctypes.POINTER(PackedLayout)]),
    "lcp_query_host_packed": (ctypes.c_int, [_P, _P, _P, _I32, _I32, _I32, _I32, _P]),
    "lcp_query_host_packed_async": (ctypes.c_int, [_P, _P, _P, _I32, _I32, _I32, _I32, _P, _I32]),
    "lcp_workspace_wait": (ctypes.c_int, [_P]),
    "lcp_query": (ctypes.c_int, [_P, _P, _P, _I32, _I32, _I32, _I32, _P, _P, _P, _P, _P, _P]),
    "lcp_query_host": (ctypes.c_int, [_P, _P, _P, _I32, _I32, _I32, _I32, _P, _P, _P, _P, _P]),
    "lcp_fullscan": (ctypes.c_int, [_P, _P, _P, _I32, _I32, _I32, _P, _P, _P, _P]),
    "lcp_fullscan_host": (ctypes.c_int, [_P, _P, _P, _I32, _I32, _I32, _P, _P, _P]),
    "lcp_encode_candidates": (ctypes.c_int, [_P, _P, _P, _I32, _I32, _I32, _I32, _I64, _P, _P]),
    "lcp_merge_candidates": (ctypes.c_int, [_P, _I32, _I32, _I32, _I32, _I32, _I32, _P, _P, _P, _P]),
    "lcp_pack_queries": (ctypes.c_int, [_P, _P, _P, _I32, _P, _P]),
    "lcp_route_queries": (ctypes.c_int, [_P, _P, _P, _P, _I32, _P, _I32, _P, _P, _P, _I32, _P, _I32, _P, _P, _P, _P, _I32, _P]),
    "lcp_index_export_sorted_key_range": (ctypes.c_int, [_P, _I64, _I64, _P]),
    "lcp_query_counted": (ctypes.c_int, [_P, _P, _P, _I32, _P, _I32, _I32, _I32, _I32, _P, _P, _P, _P, _P, _P]),
    "lcp_shard_thresholds": (ctypes.c_int, [_P, _P, _P, _P, _P, _I32, _I32, _I32, _I32, _P, _P]),
    "lcp_encode_candidates_sel": (ctypes.c_int, [_P, _P, _P, _P, _P, _I32, _I32, _I32, _I32, _P, _I64, _P, _P]),
    "lcp_signal_peers": (ctypes.c_int, [_P, _I32, _I32, _P, _P]),
    "lcp_merge_candidates_peers": (ctypes.c_int, [_P, _I32, _I32, _I32, _I32, _I32, _I32, _I32, _P, _P, _P, _P, _P, _I32, _P]),
    "lcp_server_start": (ctypes.c_int, [_P, _I32, _I32, _I32, _P, _P, ctypes.POINTER(_P)]),
    "lcp_server_query": (ctypes.c_int, [_P]),
    "lcp_server_query_row": (ctypes.c_int, [_P, _P]),
    "lcp_server_stop": (ctypes.c_int, [_P]),
    "lcp_pinned_alloc": (ctypes.c_int, [_I64, ctypes.POINTER(_P)]),
    "lcp_pinned_free": (ctypes.c_int, [_P]),
    "lcp_stream_sync": (ctypes.c_int, [_P]),
}

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None


def load() -> ctypes.CDLL:
    """Load the extension once; raise NativeLibraryMissing if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryMissing(
                f"{LIB_PATH} is not built; run __graft_entry__.build() "
                "(there is no CPU fallback for the LCP hot path)"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


_host_submit = False  # not yet looked up
_host_submit_wait = None
_host_server_query = None


def _bind_host_module() -> None:
    global _host_submit, _host_submit_wait, _host_server_query
    fn = wait = srvq = None
    if not os.environ.get("LCP_NO_HOST_EXT"):  # A/B switch
        try:
            from . import _lcp_host
        except ImportError:
            _lcp_host = None
        if _lcp_host is not None:
            lib = load()
            _lcp_host.bind(ctypes.cast(lib.lcp_query_host_packed_async, ctypes.c_void_p).value,
                           ctypes.cast(lib.lcp_workspace_wait, ctypes.c_void_p).value,
                           ctypes.cast(lib.lcp_server_query_row, ctypes.c_void_p).value)
            fn, wait, srvq = _lcp_host.submit, _lcp_host.submit_wait, _lcp_host.server_query
    _host_submit, _host_submit_wait, _host_server_query = fn, wait, srvq


def host_submit():
    """submit() of the CPython fast path (csrc/host_submit.c) bound to the
    loaded library's lcp_query_host_packed_async, or None when the module is
    not built (the ctypes call is then used; same entry point, same results)."""
    if _host_submit is False:
        _bind_host_module()
    return _host_submit


def host_server_query():
    """server_query(server, row) of the same module (lcp_server_query_row), or None."""
    if _host_submit is False:
        _bind_host_module()
    return _host_server_query if _host_submit is not None else None


def host_submit_wait():
    """submit_wait() of the same module (submission + lcp_workspace_wait), or None."""
    if _host_submit is False:
        _bind_host_module()
    return _host_submit_wait if _host_submit is not None else None


def last_error() -> str:
    msg = load().lcp_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


def check(status: int) -> None:
    """Map an lcp_status to the reference exception taxonomy (core.py:29-42)."""
    if status == LCP_OK:
        return
    msg = last_error()
    if status == LCP_ERR_INVALID_INPUT:
        raise InvalidInputError(msg)
    if status == LCP_ERR_STATE:
        raise InvalidStateError(msg)
    if status == LCP_ERR_INTERNAL:
        raise InternalInvariantError(msg)
    if status == LCP_ERR_CUDA:
        raise CudaError(msg)
    raise RuntimeError(f"lcp status {status}: {msg}")


def ptr(arr) -> int | None:
    """Raw data pointer of a numpy array or torch tensor (None passes through)."""
    if arr is None:
        return None
    if hasattr(arr, "data_ptr"):
        return int(arr.data_ptr())
    return arr.__array_interface__["data"][0]


class Workspace:
    """One lcp_workspace (own CUDA stream + scratch); not shared across threads."""

    def __init__(self) -> None:
        lib = load()
        h = ctypes.c_void_p()
        check(lib.lcp_workspace_create(ctypes.byref(h)))
        self.handle = h
        self.address = int(h.value)  # for the fast submission path
        self.submitted = 0  # async batches submitted on this workspace
        self.completed = 0  # ... and waited for

    def wait(self) -> None:
        """Complete the in-flight async batch (if any)."""
        if self.completed < self.submitted:
            self.completed = self.submitted
            check(load().lcp_workspace_wait(self.handle))

    @property
    def stream(self) -> int:
        return int(load().lcp_workspace_stream(self.handle) or 0)

    def close(self) -> None:
        if self.handle:
            load().lcp_workspace_free(self.handle)
            self.handle = None

    def __del__(self) -> None:  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass


_tls = threading.local()


def workspace() -> Workspace:
    """Per-thread workspace: concurrent readers never share scratch."""
    ws = getattr(_tls, "ws", None)
    if ws is None:
        ws = Workspace()
        _tls.ws = ws
    return ws


ASYNC_DEPTH = 8  # batches in flight per thread for the async host path (swept 1..16: 8 is best)


def async_workspace() -> Workspace:
    """Next workspace of this thread's async ring; waits for the batch that
    last used it (one batch in flight per workspace)."""
    ring = getattr(_tls, "ring", None)
    if ring is None:
        ring = _tls.ring = [Workspace() for _ in range(ASYNC_DEPTH)]
        _tls.ring_pos = 0
    ws = ring[_tls.ring_pos]
    _tls.ring_pos = (_tls.ring_pos + 1) % len(ring)
    ws.wait()
    return ws


def reset_async_ring() -> None:
    """Complete this thread's in-flight async batches and restart the ring at
    its first workspace (so a caller cycling buffers in lockstep with the ring
    sees the same workspace for the same buffers; its graph cache hits)."""
    ring = getattr(_tls, "ring", None)
    if ring is None:
        return
    for ws in ring:
        ws.wait()
    _tls.ring_pos = 0


class _PinnedMemory:
    """Owner of one page-locked block.  Freed (or returned to the per-size
    pool) only when the last numpy view of it is gone: every view's base chain
    ends here, so results stay valid as long as anything references them."""

    _pool: dict = {}          # nbytes -> [ptr, ...]
    _pool_lock = threading.Lock()
    POOL_PER_SIZE = 8

    def __init__(self, nbytes: int, pooled: bool) -> None:
        self.nbytes = max(int(nbytes), 1)
        self.pooled = pooled
        ptr = None
        if pooled:
            with self._pool_lock:
                free = self._pool.get(self.nbytes)
                if free:
                    ptr = free.pop()
        if ptr is None:
            p = ctypes.c_void_p()
            check(load().lcp_pinned_alloc(self.nbytes, ctypes.byref(p)))
            ptr = int(p.value)
        self.address = ptr

    def release(self) -> None:
        ptr, self.address = self.address, None
        if not ptr:
            return
        if self.pooled:
            with self._pool_lock:
                free = self._pool.setdefault(self.nbytes, [])
                if len(free) < self.POOL_PER_SIZE:
                    free.append(ptr)
                    return
        load().lcp_pinned_free(ctypes.c_void_p(ptr))

    def __del__(self) -> None:  # pragma: no cover - interpreter shutdown order
        try:
            self.release()
        except Exception:
            pass


class _PinnedView:
    """numpy view holder: keeps the _PinnedMemory alive through the array base."""

    def __init__(self, mem: _PinnedMemory, shape, dtype) -> None:
        self.mem = mem
        self.__array_interface__ = {"shape": tuple(shape), "typestr": dtype.str,
                                    "data": (mem.address, False), "version": 3}


class PinnedArray:
    """Page-locked host buffer exposed as a numpy array (for *_host DMA).
    ``pooled``: reuse blocks of the same size (per-call output blocks)."""

    def __init__(self, shape, dtype, pooled: bool = False) -> None:
        import numpy as np

        self.dtype = np.dtype(dtype)
        self.shape = tuple(int(s) for s in (shape if isinstance(shape, (tuple, list)) else (shape,)))
        nbytes = int(np.prod(self.shape, dtype=np.int64)) * self.dtype.itemsize
        self._mem = _PinnedMemory(nbytes, pooled)
        self.address = self._mem.address
        self.array = np.asarray(_PinnedView(self._mem, self.shape, self.dtype))

    def close(self) -> None:
        """Drop this handle; the block is released once no view of it remains."""
        self._mem = None
