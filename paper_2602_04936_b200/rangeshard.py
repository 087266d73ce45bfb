"""Lexicographic range sharding with routed queries.

The reference has no multi-device path.  Row-block sharding
(sharded.py) answers every query on every shard; here each shard owns a
contiguous range of the global sorted order, so a query is answered by the
shard that owns its key range and, only when the answer may spill over a
range boundary, by the neighbouring shards.

Build (collective, once):
  1. every rank samples its rows; the gathered samples are sorted and
     world-1 splitter rows are taken at the quantiles (identical on all ranks);
  2. rows go to the shard owning their range (route = number of splitters
     <= row, lexicographically) with all_to_all, together with their global
     ids; received rows arrive in global-id order (sources in rank order, each
     in row order), so local ids rank exactly like global ids;
  3. each rank indexes its range and publishes its first / last sorted row.

Query step (the batch is broadcast, as in sharded.py):
  1. owner(q) by the same route; a rank answers only the queries it owns;
  2. t = the lcp of the owner's need-th hit (complete) or its d_max
     (strict), -1 when the owner holds fewer than need items.  Another shard s
     can contribute only items with lcp >= t, and the best lcp any item of s
     reaches is max(lcp(q, first_s), lcp(q, last_s)) because q lies outside
     s's range; such shards are "consulted" (flags combined by all_reduce MAX)
     and answer the query locally too;
  3. every rank encodes its answers as (L - lcp) << 32 | global id (UINT64_MAX
     elsewhere), one all_gather, and the merge kernel keeps the top-take —
     exact because (lcp desc, id asc) is a total order and every item that can
     enter the global answer is in an answering shard's local top-k.

Routing and the consult rule are tensor bookkeeping (they run on the device
with NCCL, and on CPU tensors under gloo for the multi-process tests); the
local top-k and the merge are the CUDA kernels.  Local engines are pluggable
so the protocol is testable without a GPU.
"""

from __future__ import annotations

import warnings

import numpy as np

from .core import InvalidInputError

U64_MAX_AS_I64 = -1  # UINT64_MAX bit pattern in an int64 tensor


def torch_empty_like_host(t):
    import torch

    return torch.empty(t.shape, dtype=t.dtype)


def lcp_rows(a, b, length: int):
    """Per-row lcp of broadcastable integer row tensors [..., L]."""
    import torch

    neq = a != b
    first = neq.to(torch.int8).argmax(dim=-1)
    return torch.where(neq.any(dim=-1), first, torch.full_like(first, length))


def route(rows, splitters, length: int, chunk: int = 1 << 16):
    """Owner shard of each row: #splitters <= row (lexicographic)."""
    import torch

    out = torch.empty(rows.shape[0], dtype=torch.int64, device=rows.device)
    if splitters.shape[0] == 0:
        return out.zero_()
    spl = splitters.to(torch.int32)
    for s in range(0, rows.shape[0], chunk):
        r = rows[s:s + chunk].to(torch.int32)
        j = lcp_rows(r[:, None, :], spl[None, :, :], length)          # [m, S]
        jc = j.clamp(max=length - 1)
        rv = torch.gather(r, 1, jc)                                     # r[j] per splitter
        sv = spl[torch.arange(spl.shape[0], device=r.device)[None, :], jc]
        ge = (j == length) | (rv > sv)
        out[s:s + chunk] = ge.sum(dim=1)
    return out


class _Collectives:
    """NCCL collectives on device tensors; any other backend (gloo) through host."""

    def __init__(self, group):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.local = group is None and not dist.is_initialized()  # one process, no group
        self.world = 1 if self.local else dist.get_world_size(group)
        self.rank = 0 if self.local else dist.get_rank(group)
        self.nccl = (not self.local) and dist.get_backend(group) == "nccl"

    def _in(self, t):
        return t if (self.nccl or t.device.type == "cpu") else t.cpu()

    def all_gather(self, t):
        import torch

        if self.local:
            return t.contiguous()[None].clone()
        x = self._in(t.contiguous())
        out = torch.empty((self.world, *x.shape), dtype=x.dtype, device=x.device)
        if self.nccl:
            self.dist.all_gather_into_tensor(out, x, group=self.group)
        else:
            self.dist.all_gather(list(out.unbind(0)), x, group=self.group)
        return out.to(t.device)

    def all_reduce_max(self, t):
        if self.local:
            return t
        x = self._in(t.contiguous())
        self.dist.all_reduce(x, op=self.dist.ReduceOp.MAX, group=self.group)
        return x.to(t.device)

    def all_reduce_sum(self, t):
        if self.local:
            return t
        x = self._in(t.contiguous())
        self.dist.all_reduce(x, group=self.group)
        return x.to(t.device)

    def all_to_all(self, t, send_counts: list[int], recv_counts: list[int], row_elems: int):
        import torch

        if self.local:
            return t.contiguous().reshape(-1).clone()
        x = self._in(t.contiguous())
        out = torch.empty((sum(recv_counts) * row_elems,), dtype=x.dtype, device=x.device)
        self.dist.all_to_all_single(out, x.reshape(-1), [c * row_elems for c in recv_counts],
                                    [c * row_elems for c in send_counts], group=self.group)
        return out.to(t.device)


def pack_keys_host(rows: np.ndarray, length: int, sigma: int) -> np.ndarray:
    """(m, L) symbols -> (m, W) uint64 packed keys in the extension's encoding
    (common.cuh: b = ceil(log2 sigma) rounded up to a power of two, 64/b
    symbols per word, most significant first).  Setup-time helper for the
    few rows routing needs on the device (splitters, shard boundaries)."""
    need = max(1, int(np.ceil(np.log2(sigma))))
    b = 1
    while b < need:
        b <<= 1
    spw = 64 // b
    words = (length + spw - 1) // spw
    rows = np.asarray(rows, dtype=np.uint64).reshape(-1, length)
    out = np.zeros((rows.shape[0], words), dtype=np.uint64)
    for j in range(length):
        out[:, j // spw] |= rows[:, j] << np.uint64(64 - b * (j % spw + 1))
    return out


def unpack_keys_host(keys: np.ndarray, length: int, sigma: int) -> np.ndarray:
    """Inverse of pack_keys_host: (m, W) uint64 -> (m, L) uint16 symbols."""
    need = max(1, int(np.ceil(np.log2(sigma))))
    b = 1
    while b < need:
        b <<= 1
    spw = 64 // b
    j = np.arange(length)
    word = np.asarray(keys, dtype=np.uint64)[:, j // spw]
    shift = (64 - b * (j % spw + 1)).astype(np.uint64)
    return ((word >> shift) & np.uint64((1 << b) - 1)).astype(np.uint16)


class GpuEngine:
    """Local top-k on this rank's range: the CUDA index (NativeIndex; an empty
    range still gets an n = 0 index, which the device routing needs for the
    key encoding)."""

    def __init__(self, rows, length: int, sigma: int):
        """rows: (n, L) uint16 numpy array, or a contiguous CUDA tensor of
        2-byte symbols (int16/uint16 bit patterns), built in place on the GPU."""
        from .engine import NativeIndex

        self.length, self.n = int(length), int(rows.shape[0])
        self.sigma = int(sigma)
        if hasattr(rows, "data_ptr"):
            assert rows.is_cuda and rows.element_size() == 2 and rows.is_contiguous()
            self.native = NativeIndex.from_device(rows.data_ptr() if self.n else 0, self.n, length, sigma)
        else:
            self.native = NativeIndex(rows, length, sigma)
        self.device = "cuda"

    def first_last_rows(self) -> np.ndarray:
        if not self.n:
            return np.zeros((2, self.length), dtype=np.int64)
        keys = np.stack([self.native.export_sorted_key_range(0, 1)[0],
                         self.native.export_sorted_key_range(self.n - 1, 1)[0]])
        return unpack_keys_host(keys, self.length, self.sigma).astype(np.int64)

    def query(self, queries, k: int, mode: str):
        """queries: (m, L) uint16/int16 CUDA tensor -> (ids, lcps, hits, md) int64."""
        import torch

        m = int(queries.shape[0])
        stride = self.native.stride_for(k)
        ids = torch.empty((m, stride), dtype=torch.int32, device=queries.device)
        lcps = torch.empty((m, stride), dtype=torch.int16, device=queries.device)
        hits = torch.empty(m, dtype=torch.int32, device=queries.device)
        md = torch.empty(m, dtype=torch.int16, device=queries.device)
        self.native.query_device(queries.contiguous(), k, mode, ids, lcps, hits, md,
                                 stream=torch.cuda.current_stream().cuda_stream)
        return ids.long(), lcps.long() & 0xFFFF, hits.long(), md.long() & 0xFFFF

    def merge(self, gathered, take: int, strict: bool):
        """gathered: (world, count, k) int64 (u64 bits) CUDA tensor -> merged top-take."""
        import torch

        from . import _native

        world, count, k = (int(s) for s in gathered.shape)
        stride = max(1, take)
        ids = torch.empty((count, stride), dtype=torch.int32, device=gathered.device)
        lcps = torch.empty((count, stride), dtype=torch.int16, device=gathered.device)
        hits = torch.empty(count, dtype=torch.int32, device=gathered.device)
        _native.check(_native.load().lcp_merge_candidates(
            gathered.contiguous().data_ptr(), world, count, k, take, self.length, 1 if strict else 0,
            ids.data_ptr(), lcps.data_ptr(), hits.data_ptr(), torch.cuda.current_stream().cuda_stream))
        return ids.long() & 0xFFFFFFFF, lcps.long() & 0xFFFF, hits.long()


class RangeShardedIndex:
    """One rank's lexicographic range of a corpus split over a process group.

    ``items``: this rank's rows (uint16 (n, L)); their global ids are
    ``id_offset + row``.  Collective: every rank of ``group`` constructs it."""

    SAMPLES = 1024  # rows sampled per rank for the splitters

    def __init__(self, items, length: int, sigma: int, id_offset: int, group=None,
                 engine_factory=GpuEngine, device=None):
        import torch

        self.coll = _Collectives(group)
        self.world, self.rank = self.coll.world, self.coll.rank
        self.length, self.sigma = int(length), int(sigma)
        items = np.ascontiguousarray(items, dtype=np.uint16).reshape(-1, self.length)
        n_local = items.shape[0]
        if device is None:
            device = "cuda" if engine_factory is GpuEngine else "cpu"
        self.device = torch.device(device)
        L = self.length

        # 1. splitters from the gathered samples
        take = min(self.SAMPLES, n_local)
        samp = np.zeros((self.SAMPLES, L), dtype=np.int64)
        if take:
            samp[:take] = items[np.linspace(0, n_local - 1, take).astype(np.int64)]
        valid = np.zeros(self.SAMPLES, dtype=np.int64)
        valid[:take] = 1
        g_samp = self.coll.all_gather(torch.from_numpy(samp).to(self.device)).cpu().numpy()
        g_valid = self.coll.all_gather(torch.from_numpy(valid).to(self.device)).cpu().numpy()
        pool = g_samp.reshape(-1, L)[g_valid.reshape(-1) == 1]
        if pool.shape[0]:
            pool = pool[np.lexsort(pool.T[::-1])]
            cut = [(i + 1) * pool.shape[0] // self.world for i in range(self.world - 1)]
            spl = pool[np.minimum(cut, pool.shape[0] - 1)] if cut else np.zeros((0, L), np.int64)
        else:
            spl = np.zeros((self.world - 1, L), dtype=np.int64)
        self.splitters = torch.from_numpy(np.ascontiguousarray(spl)).to(self.device)

        # 2. rows (+ global ids) to the owner of their range, in global-id order
        if self.world == 1:  # one shard: the rows stay, ids are the row numbers
            self.gids = torch.arange(id_offset, id_offset + n_local, dtype=torch.int64, device=self.device)
            self.engine = engine_factory(items, L, sigma)
            self.n_local = n_local
            self._finish_build()
            return
        # the rows cross PCIe once, as 2-byte symbols, and widen on the device
        # (the host view is only read: torch's read-only-array warning is moot)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", UserWarning)
            host = torch.from_numpy(items.view(np.int16))
        rows_t = host.to(self.device).to(torch.int32) & 0xFFFF
        dest = route(rows_t, self.splitters, L) if n_local else torch.zeros(0, dtype=torch.int64,
                                                                            device=self.device)
        perm = torch.sort(dest, stable=True).indices
        send_counts = torch.bincount(dest, minlength=self.world).to(torch.int64)
        recv_counts = self.coll.all_gather(send_counts)[:, self.rank]
        sc, rc = send_counts.cpu().tolist(), recv_counts.cpu().tolist()
        gids = torch.arange(id_offset, id_offset + n_local, dtype=torch.int64, device=self.device)
        my_rows = self.coll.all_to_all(rows_t[perm], sc, rc, L).reshape(-1, L)
        self.gids = self.coll.all_to_all(gids[perm], sc, rc, 1)
        if engine_factory is GpuEngine and my_rows.is_cuda:
            # the received rows stay on the device: the index is built from them
            # in place (uint16 bit patterns in an int16 tensor)
            local = my_rows.to(torch.int16).contiguous()
        else:
            local = my_rows.cpu().numpy().astype(np.uint16)
        self.engine = engine_factory(local, L, sigma)
        self.n_local = int(local.shape[0])
        self._finish_build()

    def _finish_build(self):
        import torch

        # 3. range boundaries of every shard, corpus size
        fl = torch.from_numpy(self.engine.first_last_rows()).to(self.device)
        g_fl = self.coll.all_gather(fl)
        self.first, self.last = g_fl[:, 0, :].to(torch.int32), g_fl[:, 1, :].to(torch.int32)
        self.nonempty = self.coll.all_gather(torch.tensor([self.n_local], device=self.device))[:, 0] > 0
        self.n_total = int(self.coll.all_reduce_sum(torch.tensor([self.n_local], device=self.device)).item())

    # ---------------------------------------------------------------- queries
    def _encode(self, ids, lcps, hits, k: int):
        """Local answers -> (m, k) int64 u64-bit composites, UINT64_MAX padded."""
        import torch

        m = ids.shape[0]
        cand = torch.full((m, k), U64_MAX_AS_I64, dtype=torch.int64, device=ids.device)
        w = min(k, ids.shape[1])
        gid = self.gids[ids[:, :w].clamp(min=0, max=max(0, self.n_local - 1))]
        comp = ((self.length - lcps[:, :w]) << 32) | gid
        valid = torch.arange(w, device=ids.device)[None, :] < hits[:, None]
        cand[:, :w] = torch.where(valid, comp, torch.full_like(comp, U64_MAX_AS_I64))
        return cand

    def _answer(self, queries, sel, k: int, mode: str, cand):
        if sel.numel() == 0 or self.n_local == 0:
            return None
        ids, lcps, hits, md = self.engine.query(queries.index_select(0, sel), k, mode)
        cand[sel] = self._encode(ids, lcps, hits, k)
        return ids, lcps, hits, md

    def query(self, queries, k: int, mode: str = "complete"):
        """Global top-k for a broadcast (count, L) batch (same on every rank).

        Returns (ids, lcps, hits): int64 tensors (count, max(1, take)), (count,)."""
        import torch

        if mode not in ("complete", "strict"):
            raise InvalidInputError(f"sharded mode must be 'strict' or 'complete', got {mode!r}")
        if k < 1:
            raise InvalidInputError(f"k must be >= 1, got {k}")
        take = max(0, min(int(k), self.n_total))
        if take * self.world > 8192:
            raise InvalidInputError("sharded merge supports world * min(k, n) <= 8192")
        q = queries.to(self.device)
        count, L = int(q.shape[0]), self.length
        kk = max(1, take)
        cand = torch.full((count, kk), U64_MAX_AS_I64, dtype=torch.int64, device=self.device)
        q32 = q.to(torch.int32) & 0xFFFF
        owner = route(q32, self.splitters, L)
        own = (owner == self.rank).nonzero().squeeze(1)
        consult = torch.zeros((count, self.world), dtype=torch.int32, device=self.device)
        if own.numel():
            res = self._answer(q, own, kk, mode, cand)
            if mode == "complete":
                need = min(int(k), self.n_total)
                if res is None or need == 0 or res[1].shape[1] < need:  # owner holds < need items
                    t = torch.full((own.numel(),), -1, dtype=torch.int64, device=self.device)
                else:
                    _, lcps, hits, _ = res
                    t = torch.where(hits >= need, lcps[:, need - 1], torch.full_like(hits, -1))
            else:
                if res is None:
                    t = torch.full((own.numel(),), -1, dtype=torch.int64, device=self.device)
                else:
                    _, _, hits, md = res
                    t = torch.where(hits > 0, md, torch.full_like(hits, -1))
            qo = q32.index_select(0, own)[:, None, :]
            best = torch.maximum(lcp_rows(qo, self.first[None], L), lcp_rows(qo, self.last[None], L))
            c = (best >= t[:, None]) & self.nonempty[None, :]
            c[:, self.rank] = False
            consult[own] = c.to(torch.int32)
        consult = self.coll.all_reduce_max(consult)
        mine = (consult[:, self.rank] > 0).nonzero().squeeze(1)
        self._answer(q, mine, kk, mode, cand)
        gathered = self.coll.all_gather(cand)
        return self.engine.merge(gathered, take, mode == "strict")

    # --------------------------------------------------- device-routed step
    # The same protocol as query(), with no host round trip: routing, the
    # consult rule and the compactions run as kernels (shard_kernels.cuh) and
    # the exchanges as NCCL collectives on the current stream, so the whole
    # step can be captured in a CUDA graph.
    def _device_state(self):
        import torch

        if getattr(self, "_dev", None) is None:
            if not isinstance(self.engine, GpuEngine):
                raise InvalidInputError("query_device needs the CUDA engine (GpuEngine)")
            L, sigma = self.length, self.sigma
            spl = pack_keys_host(self.splitters.cpu().numpy(), L, sigma)
            first = pack_keys_host(self.first.cpu().numpy(), L, sigma)
            last = pack_keys_host(self.last.cpu().numpy(), L, sigma)
            dev = torch.device("cuda", torch.cuda.current_device())
            as_dev = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev)
            self._dev = dict(
                splitters=as_dev(spl), first=as_dev(first), last=as_dev(last),
                nonempty=self.nonempty.to(torch.int32).to(dev),
                gids=self.gids.to(torch.int64).to(dev),
                bufs={})
        return self._dev

    def _step_buffers(self, count: int, kk: int, slot: int = 0):
        import torch

        st = self._device_state()
        key = (count, kk, slot)
        if key not in st["bufs"]:
            dev = st["splitters"].device
            L = self.length
            ls = max(1, min(kk, max(1, self.n_local)))
            mk = lambda *shape, dt: torch.zeros(shape, dtype=dt, device=dev)
            W = self.engine.native.words
            st["bufs"][key] = dict(
                qk=mk(count, W, dt=torch.int64),
                rows=mk(count, L, dt=torch.int16), sel=mk(count, dt=torch.int32),
                cnt=mk(2, dt=torch.int32), ids=mk(count, ls, dt=torch.int32),
                lcps=mk(count, ls, dt=torch.int16), hits=mk(count, dt=torch.int32),
                md=mk(count, dt=torch.int16), tq=mk(count, dt=torch.int32),
                cand=mk(count, kk, dt=torch.int64),
                gathered=mk(self.world, count, kk, dt=torch.int64),
                recv=mk(self.world, max(1, count // self.world), kk, dt=torch.int64),
                ws=None)
        return st["bufs"][key]

    def _peer_buffers(self, b, count: int, kk: int, group=None):
        """Symmetric-memory candidate buffer + signal array for exchange="p2p":
        every rank's allocation mapped into every peer (NVLink), their peer
        pointers as device arrays.  Collective on first use (rendezvous).
        One process without a group: the 'peers' are this rank's own buffers."""
        import torch

        if "peer" in b:
            return b["peer"]
        dev = b["cand"].device
        c = self.coll
        if c.local:
            cand = torch.empty((count, kk), dtype=torch.int64, device=dev)
            sig = torch.zeros(1, dtype=torch.int32, device=dev)
            cand_ptrs, sig_ptrs = [cand.data_ptr()], [sig.data_ptr()]
            keep = (cand, sig)
        else:
            import torch.distributed._symmetric_memory as symm_mem

            grp = (c.group if group is None else group) or c.dist.group.WORLD
            try:
                symm_mem.enable_symm_mem_for_group(grp.group_name)
            except Exception:
                pass
            cand = symm_mem.empty((count, kk), dtype=torch.int64, device=dev)
            sig = symm_mem.empty((self.world,), dtype=torch.int32, device=dev)
            sig.zero_()
            hc = symm_mem.rendezvous(cand, grp)
            hs = symm_mem.rendezvous(sig, grp)
            cand_ptrs, sig_ptrs = list(hc.buffer_ptrs), list(hs.buffer_ptrs)
            keep = (cand, sig, hc, hs)
            c.dist.barrier(group=grp)  # every rank's signal array is zeroed
        b["peer"] = dict(cand=cand, sig=sig, keep=keep,
                         cand_ptrs=torch.tensor(cand_ptrs, dtype=torch.int64, device=dev),
                         sig_ptrs=torch.tensor(sig_ptrs, dtype=torch.int64, device=dev),
                         epoch=torch.zeros(1, dtype=torch.int32, device=dev))
        return b["peer"]

    def query_device(self, queries, k: int, mode: str = "complete", out=None,
                     exchange: str = "all_gather", group=None, slot: int = 0):
        """Global top-k of a broadcast (count, L) uint16 CUDA batch, on the
        current stream, without synchronising the host.  Returns (or fills)
        (ids int32 (m, max(1, take)), lcps int16, hits int32) where m = count
        (exchange "all_gather": every rank gets every answer) or count/world
        (exchange "all_to_all": rank r gets the answers of batch rows
        [r*m, (r+1)*m), the queries its own clients submitted).  ``group``
        overrides the process group of the step's collectives (one NCCL
        communicator per in-flight stream); ``slot`` selects a separate set
        of step buffers (one per in-flight stream)."""
        import torch

        from . import _native
        from ._native import Workspace, check, load

        if mode not in ("complete", "strict"):
            raise InvalidInputError(f"sharded mode must be 'strict' or 'complete', got {mode!r}")
        if k < 1:
            raise InvalidInputError(f"k must be >= 1, got {k}")
        take = max(0, min(int(k), self.n_total))
        if take * self.world > 8192:
            raise InvalidInputError("sharded merge supports world * min(k, n) <= 8192")
        if exchange not in ("all_gather", "all_to_all", "p2p"):
            raise InvalidInputError(f"unknown exchange {exchange!r}")
        st = self._device_state()
        count, L = int(queries.shape[0]), self.length
        if exchange != "all_gather" and count % self.world:
            raise InvalidInputError(f"{exchange} exchange needs count divisible by the world size")
        if exchange == "p2p" and take > 32:
            raise InvalidInputError("p2p exchange supports min(k, n) <= 32")
        kk = max(1, take)
        b = self._step_buffers(count, kk, slot)
        peer = self._peer_buffers(b, count, kk, group) if exchange == "p2p" else None
        cand = peer["cand"] if peer else b["cand"]  # p2p: candidates live in symmetric memory
        if b["ws"] is None:
            b["ws"] = Workspace()
        ws = b["ws"]
        lib = load()
        stream = torch.cuda.current_stream().cuda_stream
        native = self.engine.native
        q = queries.contiguous()
        ls = int(b["ids"].shape[1])
        strict = 1 if mode == "strict" else 0
        need = take if mode == "complete" else kk
        expected = max(1, (count + self.world - 1) // self.world * 5 // 4)
        cnt_own, cnt_con = b["cnt"][0:1], b["cnt"][1:2]

        def answer(cnt, exp):
            check(lib.lcp_query_counted(native.handle, ws.handle, b["rows"].data_ptr(), count,
                                        cnt.data_ptr(), exp, kk, _native.MODE_CODES[mode], ls,
                                        b["ids"].data_ptr(), b["lcps"].data_ptr(),
                                        b["hits"].data_ptr(), b["md"].data_ptr(), None, stream))

        def encode(cnt):
            check(lib.lcp_encode_candidates_sel(
                b["ids"].data_ptr(), b["lcps"].data_ptr(), b["hits"].data_ptr(), b["sel"].data_ptr(),
                cnt.data_ptr(), count, kk, ls, L, st["gids"].data_ptr(), 0, cand.data_ptr(), stream))

        # 0. pack the batch once; routing the own queries also resets the
        #    step's thresholds (-1) and candidates (UINT64_MAX)
        check(lib.lcp_pack_queries(native.handle, ws.handle, q.data_ptr(), count, b["qk"].data_ptr(),
                                   stream))
        # 1. the queries this rank owns: answer, threshold, candidates
        check(lib.lcp_route_queries(native.handle, ws.handle, q.data_ptr(), b["qk"].data_ptr(), count,
                                    st["splitters"].data_ptr(), self.world - 1, None, None, None,
                                    self.rank, b["tq"].data_ptr(), 0, b["rows"].data_ptr(),
                                    b["sel"].data_ptr(), cnt_own.data_ptr(), cand.data_ptr(), kk,
                                    stream))
        answer(cnt_own, expected)
        encode(cnt_own)
        if self.world > 1:  # one shard: nobody else to consult
            check(lib.lcp_shard_thresholds(b["lcps"].data_ptr(), b["hits"].data_ptr(), b["md"].data_ptr(),
                                           b["sel"].data_ptr(), cnt_own.data_ptr(), count, ls, need,
                                           strict, b["tq"].data_ptr(), stream))
            # 2. thresholds of every query from its owner (one int per query)
            self._all_reduce_max_(b["tq"], group)
            # 3. the queries other ranks own whose answer may reach into this range
            check(lib.lcp_route_queries(native.handle, ws.handle, q.data_ptr(), b["qk"].data_ptr(), count,
                                        st["splitters"].data_ptr(), self.world - 1, st["first"].data_ptr(),
                                        st["last"].data_ptr(), st["nonempty"].data_ptr(), self.rank,
                                        b["tq"].data_ptr(), 1, b["rows"].data_ptr(), b["sel"].data_ptr(),
                                        cnt_con.data_ptr(), None, 0, stream))
            answer(cnt_con, max(1, count // 16))
            encode(cnt_con)
        # 4. candidates: every rank's for every query (all_gather), or each
        #    rank's for the queries of rank r's clients to rank r (all_to_all),
        #    or read straight from the peers' symmetric buffers by the merge
        #    kernel after a signal (p2p: the exchange and the merge are one kernel)
        m = count if exchange == "all_gather" else count // self.world
        if exchange == "p2p":
            if out is None:
                out = (torch.empty((m, kk), dtype=torch.int32, device=q.device),
                       torch.empty((m, kk), dtype=torch.int16, device=q.device),
                       torch.empty(m, dtype=torch.int32, device=q.device))
            ids, lcps, hits = out
            check(lib.lcp_signal_peers(peer["sig_ptrs"].data_ptr(), self.world, self.rank,
                                       peer["epoch"].data_ptr(), stream))
            check(lib.lcp_merge_candidates_peers(
                peer["cand_ptrs"].data_ptr(), self.world, self.rank, m, kk, take, L, strict,
                peer["sig"].data_ptr(), peer["epoch"].data_ptr(), ids.data_ptr(), lcps.data_ptr(),
                hits.data_ptr(), int(ids.shape[1]), stream))
            return ids, lcps, hits
        if exchange == "all_gather":
            self._all_gather_into_(b["gathered"], b["cand"], group)
        else:
            self._all_to_all_(b["recv"], b["cand"], group)
        if out is None:
            out = (torch.empty((m, kk), dtype=torch.int32, device=q.device),
                   torch.empty((m, kk), dtype=torch.int16, device=q.device),
                   torch.empty(m, dtype=torch.int32, device=q.device))
        ids, lcps, hits = out
        src = b["gathered"] if exchange == "all_gather" else b["recv"]
        check(lib.lcp_merge_candidates(src.data_ptr(), self.world, m, kk, take, L, strict,
                                       ids.data_ptr(), lcps.data_ptr(), hits.data_ptr(), stream))
        return ids, lcps, hits

    def _all_reduce_max_(self, t, group=None) -> None:
        c = self.coll
        g = c.group if group is None else group
        if c.local:
            return
        if c.nccl:
            c.dist.all_reduce(t, op=c.dist.ReduceOp.MAX, group=g)
        else:  # gloo (multi-process tests on one GPU): host staging, not capturable
            h = t.cpu()
            c.dist.all_reduce(h, op=c.dist.ReduceOp.MAX, group=g)
            t.copy_(h)

    def _all_gather_into_(self, out, t, group=None) -> None:
        c = self.coll
        g = c.group if group is None else group
        if c.local:
            out[0].copy_(t)
        elif c.nccl:
            c.dist.all_gather_into_tensor(out, t, group=g)
        else:
            h = out.cpu()
            c.dist.all_gather(list(h.unbind(0)), t.cpu(), group=g)
            out.copy_(h)

    def _all_to_all_(self, out, t, group=None) -> None:
        """t: (world * m, k) rows, block r to rank r; out: (world, m, k), block s from rank s."""
        c = self.coll
        g = c.group if group is None else group
        if c.local:
            out[0].copy_(t)
            return
        if c.nccl:
            c.dist.all_to_all_single(out, t, group=g)
            return
        h = torch_empty_like_host(out)  # gloo: host staging (tests only)
        c.dist.all_to_all_single(h, t.cpu(), group=g)
        out.copy_(h)
