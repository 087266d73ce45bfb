"""Multi-rank exchange logic of the row-block sharded index, on CPU.

Two processes over the gloo backend run the product's ShardPlan and
ShardExchange (the one data-path collective).  The per-shard top-k comes
from the pinned CPU oracle, and encode/merge are host statements of the
k_encode / k_merge kernels (the GPU versions are checked in
tests/test_gpu_parity.py).  The merged global answer must equal the oracle
on the whole corpus, for complete and strict mode.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_04936_b200.sharded import ShardExchange, ShardPlan

MAXU = np.iinfo(np.uint64).max


def encode(ids, lcps, hits, k, length, id_offset):
    """Host statement of k_encode: (L - lcp) << 32 | (id + offset), UINT64_MAX padded."""
    count = hits.shape[0]
    cand = np.full((count, k), MAXU, dtype=np.uint64)
    for q in range(count):
        h = int(hits[q])
        cand[q, :h] = ((length - lcps[q, :h].astype(np.uint64)) << np.uint64(32)) | (
            ids[q, :h].astype(np.uint64) + np.uint64(id_offset))
    return cand


def merge(gathered, take, length, strict=False):
    """Host statement of k_merge."""
    world, count, k = gathered.shape
    flat = np.sort(gathered.transpose(1, 0, 2).reshape(count, world * k), axis=1)
    out = []
    for q in range(count):
        row = flat[q][flat[q] != MAXU]
        if strict and row.size:
            row = row[(row >> np.uint64(32)) == (row[0] >> np.uint64(32))]
        row = row[:take]
        out.append(list(zip((row & np.uint64(0xFFFFFFFF)).astype(np.int64).tolist(),
                            (length - (row >> np.uint64(32)).astype(np.int64)).tolist())))
    return out


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg):
    import oracle
    from paper_2602_04936_b200 import generate_dataset, generate_queries

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, L, sigma, k = cfg
        ds = generate_dataset(n, L, sigma, seed=11)
        qs = np.vstack([generate_queries(ds, 40, seed=12), generate_queries(ds, 40, seed=13, prefix_len=L // 2)])
        lo, hi = ShardPlan(n, world).bounds(rank)
        local = ds.items[lo:hi]
        ex = ShardExchange()
        assert ex.world == world and ex.rank == rank
        for mode in ("complete", "strict"):
            if hi > lo:
                trie = oracle.OracleTrie(local, sigma)
                ids, lcps, hits, md, _, _ = trie.query_batch(qs, k, mode)
            else:
                ids = np.zeros((len(qs), 1), np.int64)
                lcps = np.zeros((len(qs), 1), np.int64)
                hits = np.zeros(len(qs), np.int64)
            cand = encode(ids, lcps, hits, k, L, lo)
            gathered = ex.gather(torch.from_numpy(cand.view(np.int64)))
            merged = merge(gathered.numpy().view(np.uint64), min(k, n), L, strict=mode == "strict")
            full = oracle.OracleTrie(ds.items, sigma)
            fids, flcps, fhits, _, _, _ = full.query_batch(qs, k, mode)
            for i in range(len(qs)):
                exp = list(zip(fids[i, :fhits[i]].tolist(), flcps[i, :fhits[i]].tolist()))
                assert merged[i] == exp, (rank, mode, i)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [(3000, 12, 4, 10), (500, 8, 2, 5), (7, 4, 3, 10)])
def test_two_rank_exchange_is_exact(oracle_lib, cfg):
    mp.spawn(_worker, args=(2, _free_port(), cfg), nprocs=2, join=True)


def test_shard_plan_partitions_rows():
    for n, world in [(10, 3), (0, 2), (7, 8), (2_000_000, 8)]:
        plan = ShardPlan(n, world)
        spans = [plan.bounds(r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        sizes = [h - l for l, h in spans]
        assert max(sizes) - min(sizes) <= 1
