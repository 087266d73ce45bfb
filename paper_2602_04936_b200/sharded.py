"""Row-block corpus sharding across GPUs with an exact top-k merge.

No reference counterpart: multi-GPU is future work in the paper
(PAPER.md:849).  Rank g holds a contiguous block of item ids
[offset_g, offset_g + n_g) and its own device index.  A query batch is
broadcast (every rank holds the same queries), each rank computes its local
top-min(k, n_g) in complete mode, encodes hits as u64 candidates
``(L - lcp) << 32 | global_id`` padded with UINT64_MAX
(lcp_encode_candidates), the candidates are exchanged with one all-gather
(NCCL over NVLink; the payload carries no arithmetic so the merge stays
deterministic), and lcp_merge_candidates keeps the k smallest per query.
(lcp desc, id asc) is a total order, so the global top-k is contained in the
union of the per-shard top-k's: the merge is exact.

Kernels and the collective run on one CUDA stream (torch's current stream),
so a step is one ordered sequence: query -> encode -> all-gather -> merge.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _native
from .core import InvalidInputError


@dataclass(frozen=True)
class ShardPlan:
    """Row-block partition of n_total items over `world` ranks (sizes differ by <= 1)."""

    n_total: int
    world: int

    def bounds(self, rank: int) -> tuple[int, int]:
        if not (0 <= rank < self.world):
            raise InvalidInputError(f"rank {rank} out of range for world {self.world}")
        base, rem = divmod(self.n_total, self.world)
        lo = rank * base + min(rank, rem)
        return lo, lo + base + (1 if rank < rem else 0)


def local_candidates(index, queries, k: int, id_offset: int, mode: str = "complete",
                     stream: int | None = None, bufs: dict | None = None):
    """One shard's step before the exchange: local top-min(k, n_g) of a CUDA
    (count, L) uint16 batch, encoded as (count, k) int64 candidates
    ``(L - lcp) << 32 | (id + id_offset)`` padded with UINT64_MAX
    (lcp_encode_candidates).  ``index``: NativeIndex or TrieIndex."""
    import torch

    native = getattr(index, "native", index)
    count = int(queries.shape[0])
    dev = queries.device
    st = torch.cuda.current_stream(dev).cuda_stream if stream is None else stream
    if bufs is None:
        ls = native.stride_for(k)
        bufs = dict(ids=torch.empty((count, ls), dtype=torch.int32, device=dev),
                    lcps=torch.empty((count, ls), dtype=torch.int16, device=dev),
                    hits=torch.empty(count, dtype=torch.int32, device=dev),
                    cand=torch.empty((count, k), dtype=torch.int64, device=dev))
    if native.n:
        native.query_device(queries, k, mode, bufs["ids"], bufs["lcps"], bufs["hits"],
                            bufs.get("md"), bufs.get("aux"), stream=st)
    else:
        bufs["hits"].zero_()
    _native.check(_native.load().lcp_encode_candidates(
        bufs["ids"].data_ptr(), bufs["lcps"].data_ptr(), bufs["hits"].data_ptr(), count, k,
        int(bufs["ids"].shape[1]), native.length, int(id_offset), bufs["cand"].data_ptr(), st))
    return bufs["cand"]


def merge_candidates_device(gathered, k: int, length: int, n_total: int, out_ids, out_lcps,
                            out_hits, mode: str = "complete", stream: int | None = None) -> None:
    """The exchange's consumer: (shards, count, k) int64 candidates -> the global
    top-min(k, n_total) per query into (count, max(1, take)) device outputs
    (lcp_merge_candidates; strict keeps only the deepest lcp across shards)."""
    import torch

    shards, count = int(gathered.shape[0]), int(gathered.shape[1])
    take = max(0, min(int(k), int(n_total)))
    st = torch.cuda.current_stream(gathered.device).cuda_stream if stream is None else stream
    _native.check(_native.load().lcp_merge_candidates(
        gathered.data_ptr(), shards, count, k, take, int(length), 1 if mode == "strict" else 0,
        out_ids.data_ptr(), out_lcps.data_ptr(), out_hits.data_ptr(), st))


def merge_candidates(gathered, k: int, length: int, n_total: int, mode: str = "complete"):
    """merge_candidates_device into fresh buffers, returned as a host BatchResult."""
    import numpy as np
    import torch

    from .result import BatchResult

    count, dev = int(gathered.shape[1]), gathered.device
    w = max(1, min(int(k), int(n_total)))
    ids = torch.empty((count, w), dtype=torch.int32, device=dev)
    lcps = torch.empty((count, w), dtype=torch.int16, device=dev)
    hits = torch.empty(count, dtype=torch.int32, device=dev)
    merge_candidates_device(gathered, k, length, n_total, ids, lcps, hits, mode)
    return BatchResult(ids=ids.cpu().numpy().view(np.uint32), lcps=lcps.cpu().numpy().view(np.uint16),
                       hits=hits.cpu().numpy(), mode=mode)


class ShardExchange:
    """The one data-path collective: all-gather of per-shard candidate lists.

    NCCL (CUDA tensors) uses all_gather_into_tensor on the current stream;
    other backends (gloo, for the CPU multi-process tests) gather a list.
    """

    def __init__(self, group=None):
        import torch.distributed as dist

        self._dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def gather(self, cand, out=None):
        """cand: (count, k) int64 tensor -> (world, count, k)."""
        import torch

        dist = self._dist
        if out is None:
            out = torch.empty((self.world, *cand.shape), dtype=cand.dtype, device=cand.device)
        if dist.get_backend(self.group) == "nccl":
            dist.all_gather_into_tensor(out, cand, group=self.group)
        elif cand.is_cuda:  # gloo gathers host tensors only
            host = torch.empty(out.shape, dtype=out.dtype)
            dist.all_gather(list(host.unbind(0)), cand.cpu(), group=self.group)
            out.copy_(host)
        else:
            parts = list(out.unbind(0))
            dist.all_gather(parts, cand, group=self.group)
        return out


class ShardedIndex:
    """One rank's shard of a row-block-partitioned index (torch.distributed)."""

    def __init__(self, items, length: int, sigma: int, id_offset: int, group=None):
        import torch
        import torch.distributed as dist

        from .engine import NativeIndex

        self.exchange = ShardExchange(group)
        self.world, self.rank = self.exchange.world, self.exchange.rank
        self.length, self.sigma = int(length), int(sigma)
        self.id_offset = int(id_offset)
        self.local = NativeIndex(items, length, sigma)
        n = torch.tensor([self.local.n], dtype=torch.int64, device="cuda")
        dist.all_reduce(n, group=group)
        self.n_total = int(n.item())
        self._bufs: dict = {}

    def _buffers(self, count: int, k: int):
        import torch

        key = (count, k)
        if key not in self._bufs:
            ls = self.local.stride_for(k)
            dev = "cuda"
            self._bufs[key] = dict(
                ids=torch.empty((count, ls), dtype=torch.int32, device=dev),
                lcps=torch.empty((count, ls), dtype=torch.int16, device=dev),
                hits=torch.empty(count, dtype=torch.int32, device=dev),
                md=torch.empty(count, dtype=torch.int16, device=dev),
                aux=torch.empty((count, 2), dtype=torch.int64, device=dev),
                cand=torch.empty((count, k), dtype=torch.int64, device=dev),
                gathered=torch.empty((self.world, count, k), dtype=torch.int64, device=dev),
            )
        return self._bufs[key]

    def query_device(self, queries, k: int, out_ids, out_lcps, out_hits, mode: str = "complete") -> None:
        """Global top-k for a broadcast (count, L) uint16 CUDA batch; outputs
        (count, max(1, min(k, n_total))) on the current stream."""
        import torch

        if mode not in ("complete", "strict"):
            raise InvalidInputError(f"sharded mode must be 'strict' or 'complete', got {mode!r}")
        if k < 1:
            raise InvalidInputError(f"k must be >= 1, got {k}")
        take = max(0, min(int(k), self.n_total))
        if take * self.world > 8192:
            raise InvalidInputError("sharded merge supports world * min(k, n) <= 8192")
        count = int(queries.shape[0])
        b = self._buffers(count, k)
        st = torch.cuda.current_stream().cuda_stream
        lib = _native.load()
        if self.local.n:
            self.local.query_device(queries, k, mode, b["ids"], b["lcps"], b["hits"], b["md"],
                                    b["aux"], stream=st)
        else:
            b["hits"].zero_()
        _native.check(lib.lcp_encode_candidates(
            b["ids"].data_ptr(), b["lcps"].data_ptr(), b["hits"].data_ptr(), count, k,
            int(b["ids"].shape[1]), self.length, self.id_offset, b["cand"].data_ptr(), st))
        self.exchange.gather(b["cand"], out=b["gathered"])
        _native.check(lib.lcp_merge_candidates(
            b["gathered"].data_ptr(), self.world, count, k, take, self.length,
            1 if mode == "strict" else 0, out_ids.data_ptr(), out_lcps.data_ptr(),
            out_hits.data_ptr(), st))


class RowBlockShardStep:
    """One rank's row block with a capture-ready query step (no host sync):
    local top-k of the broadcast batch -> encode -> exchange -> merge, all on
    the current stream.  exchange "all_gather": every rank merges every
    query; "all_to_all": rank r merges only rows [r*m, (r+1)*m) of the batch
    (its own clients' queries), receiving each shard's candidates for them.
    ``n_total`` is passed in (no collective at construction)."""

    def __init__(self, items, length: int, sigma: int, id_offset: int, n_total: int, group=None):
        import torch.distributed as dist

        from .engine import NativeIndex

        self.group = group
        self.local = group is None and not dist.is_initialized()
        self.world = 1 if self.local else dist.get_world_size(group)
        self.rank = 0 if self.local else dist.get_rank(group)
        self.length, self.id_offset, self.n_total = int(length), int(id_offset), int(n_total)
        self.native = NativeIndex(items, length, sigma)
        self._bufs: dict = {}

    def query_device(self, queries, k: int, mode: str = "complete", out=None,
                     exchange: str = "all_gather", group=None, slot: int = 0):
        import torch
        import torch.distributed as dist

        if mode not in ("complete", "strict"):
            raise InvalidInputError(f"sharded mode must be 'strict' or 'complete', got {mode!r}")
        take = max(0, min(int(k), self.n_total))
        if take * self.world > 8192:
            raise InvalidInputError("sharded merge supports world * min(k, n) <= 8192")
        count, dev = int(queries.shape[0]), queries.device
        if exchange == "all_to_all" and count % self.world:
            raise InvalidInputError("all_to_all exchange needs count divisible by the world size")
        kk = max(1, take)
        m = count if exchange == "all_gather" else count // self.world
        key = (count, kk, slot)
        if key not in self._bufs:
            ls = self.native.stride_for(kk)
            self._bufs[key] = dict(
                ids=torch.empty((count, ls), dtype=torch.int32, device=dev),
                lcps=torch.empty((count, ls), dtype=torch.int16, device=dev),
                hits=torch.empty(count, dtype=torch.int32, device=dev),
                cand=torch.empty((count, kk), dtype=torch.int64, device=dev),
                recv=torch.empty((self.world, m, kk), dtype=torch.int64, device=dev))
        b = self._bufs[key]
        local_candidates(self.native, queries, kk, self.id_offset, mode, bufs=b)
        g = self.group if group is None else group
        if self.local:
            b["recv"][0].copy_(b["cand"])
        elif dist.get_backend(g) != "nccl":  # gloo (tests on one GPU): host staging, not capturable
            h = torch.empty(b["recv"].shape, dtype=torch.int64)
            if exchange == "all_gather":
                dist.all_gather(list(h.unbind(0)), b["cand"].cpu(), group=g)
            else:
                dist.all_to_all_single(h, b["cand"].cpu(), group=g)
            b["recv"].copy_(h)
        elif exchange == "all_gather":
            dist.all_gather_into_tensor(b["recv"], b["cand"], group=g)
        else:
            dist.all_to_all_single(b["recv"], b["cand"], group=g)
        if out is None:
            out = (torch.empty((m, kk), dtype=torch.int32, device=dev),
                   torch.empty((m, kk), dtype=torch.int16, device=dev),
                   torch.empty(m, dtype=torch.int32, device=dev))
        merge_candidates_device(b["recv"], kk, self.length, self.n_total, *out, mode=mode)
        return out
