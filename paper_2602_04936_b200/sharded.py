"""Row-block corpus sharding across GPUs with an exact top-k merge.

No reference counterpart: multi-GPU is future work in the paper
(PAPER.md:849).  Rank g holds a contiguous block of item ids
[offset_g, offset_g + n_g) and its own device index.  A query batch is
broadcast (every rank holds the same queries), each rank computes its local
top-min(k, n_g) in complete mode, encodes hits as u64 candidates
``(L - lcp) << 32 | global_id`` padded with UINT64_MAX
(lcp_encode_candidates), the candidates are exchanged with one
``all_gather_into_tensor`` (NCCL over NVLink; the payload carries no
arithmetic so the merge stays deterministic), and lcp_merge_candidates keeps
the k smallest per query.  (lcp desc, id asc) is a total order, so the global
top-k is contained in the union of the per-shard top-k's: the merge is exact.

Collective and kernels all run on one CUDA stream (torch's current stream),
so the step is a single ordered sequence: query -> encode -> all-gather ->
merge.  The exchange logic is factored through ``ShardOps`` so the CPU
multi-process tests (gloo, world_size 2) can exercise it without a GPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .core import InvalidInputError


@dataclass
class ShardPlan:
    """Row-block partition of n_total items over `world` ranks."""

    n_total: int
    world: int

    def bounds(self, rank: int) -> tuple[int, int]:
        base, rem = divmod(self.n_total, self.world)
        lo = rank * base + min(rank, rem)
        return lo, lo + base + (1 if rank < rem else 0)


class ShardedIndex:
    """One rank's shard of a row-block-partitioned index (torch.distributed)."""

    def __init__(self, items: np.ndarray, length: int, sigma: int, id_offset: int, group=None):
        import torch
        import torch.distributed as dist

        from .engine import NativeIndex

        self._dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
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
        (count, min(k, n_total)) on the current stream."""
        import torch

        if mode not in ("complete", "strict"):
            raise InvalidInputError(f"sharded mode must be 'strict' or 'complete', got {mode!r}")
        take = max(0, min(int(k), self.n_total))
        if take > 32:
            raise InvalidInputError("sharded merge supports k <= 32")
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
        self._dist.all_gather_into_tensor(b["gathered"], b["cand"], group=self.group)
        _native.check(lib.lcp_merge_candidates(
            b["gathered"].data_ptr(), self.world, count, k, take, self.length,
            1 if mode == "strict" else 0, out_ids.data_ptr(), out_lcps.data_ptr(),
            out_hits.data_ptr(), st))


def encode_candidates_np(ids, lcps, hits, k: int, length: int, id_offset: int) -> np.ndarray:
    """Host statement of k_encode (used by the CPU multi-rank tests)."""
    count = hits.shape[0]
    cand = np.full((count, k), np.iinfo(np.uint64).max, dtype=np.uint64)
    for q in range(count):
        h = int(hits[q])
        cand[q, :h] = ((length - lcps[q, :h].astype(np.uint64)) << np.uint64(32)) | (
            ids[q, :h].astype(np.uint64) + np.uint64(id_offset))
    return cand


def merge_candidates_np(gathered: np.ndarray, take: int, length: int, strict: bool = False):
    """Host statement of k_merge (used by the CPU multi-rank tests)."""
    world, count, k = gathered.shape
    flat = gathered.transpose(1, 0, 2).reshape(count, world * k)
    flat = np.sort(flat, axis=1)
    out = []
    for q in range(count):
        row = flat[q][flat[q] != np.iinfo(np.uint64).max]
        if strict and row.size:
            row = row[(row >> np.uint64(32)) == (row[0] >> np.uint64(32))]
        row = row[:take]
        out.append(list(zip((row & np.uint64(0xFFFFFFFF)).astype(np.int64).tolist(),
                            (length - (row >> np.uint64(32)).astype(np.int64)).tolist())))
    return out
