"""Lexicographic range sharding with routed queries, multi-process on CPU.

world_size 2 and 3 over gloo run the product's RangeShardedIndex protocol
(splitters, row exchange, routing, consult rule, all_gather merge).  The
local top-k per range comes from the pinned C oracle and the merge is a host
statement of k_merge (the GPU engine is covered in test_gpu_parity.py).  The
merged answer must equal the oracle over the whole corpus, for complete and
strict mode, including corpora built to make answers straddle range
boundaries (heavy duplicates, tiny shards, few distinct keys).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_04936_b200.rangeshard import RangeShardedIndex, lcp_rows, route

MAXU = np.iinfo(np.uint64).max


class OracleEngine:
    """Local range engine backed by the C oracle (CPU tensors)."""

    def __init__(self, rows, length, sigma):
        import oracle

        self.rows, self.length, self.n = rows, length, rows.shape[0]
        self.trie = oracle.OracleTrie(rows, sigma) if self.n else None

    def first_last_rows(self):
        if not self.n:
            return np.zeros((2, self.length), dtype=np.int64)
        order = self.trie.tables()[0]
        return np.stack([self.rows[order[0]], self.rows[order[-1]]]).astype(np.int64)

    def query(self, q, k, mode):
        ids, lcps, hits, md, _, _ = self.trie.query_batch(q.cpu().numpy().astype(np.uint16), k, mode)
        return (torch.from_numpy(ids.astype(np.int64)), torch.from_numpy(lcps.astype(np.int64)),
                torch.from_numpy(hits.astype(np.int64)), torch.from_numpy(md.astype(np.int64)))

    def merge(self, gathered, take, strict):
        g = gathered.numpy().view(np.uint64)
        world, count, k = g.shape
        flat = np.sort(g.transpose(1, 0, 2).reshape(count, world * k), axis=1)
        stride = max(1, take)
        ids = np.zeros((count, stride), np.int64)
        lcps = np.zeros((count, stride), np.int64)
        hits = np.zeros(count, np.int64)
        for q in range(count):
            row = flat[q][flat[q] != MAXU]
            if strict and row.size:
                row = row[(row >> np.uint64(32)) == (row[0] >> np.uint64(32))]
            row = row[:take]
            hits[q] = row.size
            ids[q, :row.size] = (row & np.uint64(0xFFFFFFFF)).astype(np.int64)
            lcps[q, :row.size] = self.length - (row >> np.uint64(32)).astype(np.int64)
        return torch.from_numpy(ids), torch.from_numpy(lcps), torch.from_numpy(hits)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _corpus(kind, n, L, sigma, seed):
    from paper_2602_04936_b200 import generate_dataset

    rng = np.random.default_rng(seed)
    if kind == "uniform":
        return generate_dataset(n, L, sigma, seed=seed).items
    if kind == "dups":  # few distinct rows: equal keys straddle every splitter
        base = rng.integers(0, sigma, (5, L)).astype(np.uint16)
        return base[rng.integers(0, 5, n)]
    if kind == "skew":  # one long shared prefix covering most of the corpus
        rows = rng.integers(0, sigma, (n, L)).astype(np.uint16)
        rows[: (3 * n) // 4, : L - 2] = 1
        return rows
    raise ValueError(kind)


def _worker(rank, world, port, cfg):
    import oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        kind, n, L, sigma, ks = cfg
        items = _corpus(kind, n, L, sigma, 11)
        rng = np.random.default_rng(12)
        qs = np.vstack([items[rng.integers(0, max(n, 1), 30)] if n else np.zeros((0, L), np.uint16),
                        rng.integers(0, sigma, (30, L)).astype(np.uint16)])
        if n:  # prefix queries (first half of a row, random tail)
            p = items[rng.integers(0, n, 20)].copy()
            p[:, L // 2:] = rng.integers(0, sigma, (20, L - L // 2))
            qs = np.vstack([qs, p])
        lo, hi = n * rank // world, n * (rank + 1) // world
        sh = RangeShardedIndex(items[lo:hi], L, sigma, id_offset=lo, engine_factory=OracleEngine)
        assert sh.n_total == n
        # every item lives on exactly one shard, in its range
        counts = torch.zeros(world, dtype=torch.int64)
        counts[rank] = sh.n_local
        dist.all_reduce(counts)
        assert int(counts.sum()) == n
        full = oracle.OracleTrie(items, sigma) if n else None
        for k in ks:
            for mode in ("complete", "strict"):
                ids, lcps, hits = sh.query(torch.from_numpy(qs.astype(np.int32)), k, mode)
                if not n:
                    assert int(hits.sum()) == 0
                    continue
                fids, flcps, fhits, _, _, _ = full.query_batch(qs, k, mode)
                for i in range(len(qs)):
                    h = int(hits[i])
                    got = list(zip(ids[i, :h].tolist(), lcps[i, :h].tolist()))
                    exp = list(zip(fids[i, :fhits[i]].tolist(), flcps[i, :fhits[i]].tolist()))
                    assert got == exp, (rank, kind, k, mode, i)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,cfg", [
    (2, ("uniform", 3000, 12, 4, (1, 10, 32, 50))),
    (3, ("uniform", 2000, 8, 2, (5, 17))),
    (3, ("dups", 600, 6, 4, (1, 10, 32))),
    (2, ("skew", 1500, 10, 4, (10, 32))),
    (3, ("uniform", 7, 4, 3, (1, 10))),
    (2, ("uniform", 0, 4, 3, (3,))),
])
def test_range_sharded_is_exact(oracle_lib, world, cfg):
    mp.spawn(_worker, args=(world, _free_port(), cfg), nprocs=world, join=True)


def test_route_and_lcp_rows():
    spl = torch.tensor([[1, 0, 0], [2, 1, 1]])
    rows = torch.tensor([[0, 3, 3], [1, 0, 0], [1, 0, 1], [2, 1, 0], [2, 1, 1], [3, 0, 0]])
    assert route(rows, spl, 3).tolist() == [0, 1, 1, 1, 2, 2]
    assert lcp_rows(rows, torch.tensor([1, 0, 1]), 3).tolist() == [0, 2, 3, 0, 0, 0]
