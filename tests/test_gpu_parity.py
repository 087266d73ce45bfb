"""GPU parity: the sm_100a path through the C ABI vs the golden vectors
(produced by the reference) and vs the pinned C oracle.  Bit-exact for every
id, lcp, hit count, matched depth, work counter and serialized byte."""

import hashlib

import numpy as np
import pytest

import paper_2602_04936_b200 as lg
from golden_util import case_dataset, expected_rows, sha

pytestmark = pytest.mark.gpu


def _batch_rows(b, i):
    return b.pairs(i)


@pytest.mark.parametrize("idx", range(16))
def test_golden_cases(gpu, golden, idx):
    manifest, arrays = golden
    cases = manifest["cases"]
    case = cases[idx]
    name, pre = case["name"], case["name"] + "/"
    ds = case_dataset(case)
    qs = arrays[pre + "queries"]
    ks = arrays[pre + "k"]
    index = lg.build(ds)
    # build parity: order, adjacent lcp, per-depth arena
    assert np.array_equal(index.order, arrays[pre + "order"])
    assert np.array_equal(index.level_offset, arrays[pre + "level_offset"])
    if ds.n:
        assert np.array_equal(index.native.export_adjacent_lcp().astype(np.int64), arrays[pre + "adjacent_lcp"])
    assert index.node_count == case["node_count"]
    assert sha(index.row_lo) == case["row_lo_sha256"]
    assert sha(index.edge_symbol) == case["edge_symbol_sha256"]
    index.check_invariants()

    for mode in ("strict", "complete"):
        mp = f"{pre}{mode}/"
        digest = hashlib.sha256()
        for k in sorted(set(ks.tolist())):
            sel = np.flatnonzero(ks == k)
            w = index.new_work_report()
            b = index.query_batch(qs[sel], int(k), mode, work=w)
            for j, i in enumerate(sel):
                assert _batch_rows(b, j) == expected_rows(arrays, mp, i), (name, mode, i, k)
                assert int(b.matched_depth[j]) == arrays[mp + "md"][i], (name, mode, i)
            assert w.symbols_compared == int(arrays[mp + "sym"][sel].sum())
            assert w.nodes_visited == int(arrays[mp + "nodes"][sel].sum())
            assert w.queries == len(sel)
        for i, q in enumerate(qs):  # single-query API, canonical bytes
            w = index.new_work_report()
            r = index.query(q, int(ks[i]), mode, work=w)
            digest.update(r.to_bytes())
            assert w.symbols_compared == arrays[mp + "sym"][i]
            assert w.nodes_visited == arrays[mp + "nodes"][i]
        assert digest.hexdigest() == case[f"{mode}_bytes_sha256"], (name, mode)

    # brute-force scan kernel vs the reference oracle
    digest = hashlib.sha256()
    for k in sorted(set(ks.tolist())):
        sel = np.flatnonzero(ks == k)
        b = index.fullscan_batch(qs[sel], int(k))
        for j, i in enumerate(sel):
            assert _batch_rows(b, j) == expected_rows(arrays, pre + "oracle/", i), (name, "fullscan", i)
    for i, q in enumerate(qs):
        digest.update(lg.fullscan_top_k(ds, q, int(ks[i])).to_bytes())
    assert digest.hexdigest() == case["oracle_bytes_sha256"]

    for tal in case["tal"]:
        tp = f"{pre}tal{tal['B']}/"
        eng = lg.build_tal(ds, tal["B"])
        assert eng.bucket_depth == tal["depth"] and eng.bucket_count == tal["bucket_count"]
        assert (eng.directory is not None) == tal["has_directory"]
        if tp + "directory" in arrays:
            assert np.array_equal(eng.directory, arrays[tp + "directory"])
        digest = hashlib.sha256()
        for i, q in enumerate(qs):
            r, rep = eng.query(q, int(ks[i]))
            digest.update(r.to_bytes())
            assert rep.items_scanned == arrays[tp + "items"][i]
            assert rep.symbols_compared == arrays[tp + "sym"][i]
            assert eng.bucket_range(q) == (arrays[tp + "lo"][i], arrays[tp + "hi"][i])
            if eng.directory is not None:
                assert eng.bucket_range_search(q) == eng.bucket_range_directory(q)
        assert digest.hexdigest() == tal["bytes_sha256"], (name, tal["B"])
        for k in sorted(set(ks.tolist())):
            sel = np.flatnonzero(ks == k)
            w = eng.new_work_report()
            b = eng.query_batch(qs[sel], int(k), work=w)
            for j, i in enumerate(sel):
                assert _batch_rows(b, j) == expected_rows(arrays, tp, i)
            assert w.items_scanned == int(arrays[tp + "items"][sel].sum())
            assert w.symbols_compared == int(arrays[tp + "sym"][sel].sum())


def test_hand_cases(gpu, golden):
    hand = golden[0]["hand"]
    idx = lg.build(lg.Dataset.from_rows([[0, 0], [0, 1], [1, 0]], 2))
    assert idx.query([0, 0], 3, "complete").pairs() == [tuple(p) for p in hand["complete_3item"]]
    r = idx.query([0, 0], 3, "strict")
    assert r.pairs() == [tuple(p) for p in hand["strict_3item"]] and r.matched_depth == 2
    assert idx.query([0, 0], 3, "complete").to_bytes().hex() == hand["result_bytes"]
    two = lg.build(lg.Dataset.from_rows([[0, 1], [0, 2]], 4))
    assert two.node_count == 4 and two.root.subtree_size == 2
    same = lg.build(lg.Dataset.from_rows([[1, 2, 3]] * 9, 4))
    leaf = same.root.children()[0].children()[0].children()[0]
    assert leaf.posting.tolist() == list(range(9))
    dup = lg.build(lg.Dataset.from_rows([[7, 7]] * 2 + [[1, 1]], 8))
    node, depth = dup.descend([7, 7])
    assert depth == 2 and dup.collect_top_k(node, 1).tolist() == [0]
    ds = lg.Dataset.from_rows([[3, 3]] * 3, 4)
    assert lg.fullscan_top_k(ds, [3, 3], 2).pairs() == [tuple(p) for p in hand["oracle_dups"]]


def test_errors_are_reference_exceptions(gpu):
    idx = lg.build(lg.Dataset.from_rows([[0, 1]], 4))
    with pytest.raises(lg.InvalidInputError):
        idx.query([0, 1], 0)
    with pytest.raises(lg.InvalidInputError):
        idx.query([0, 1], 2, "both")
    with pytest.raises(lg.InvalidInputError):
        idx.query([0], 2)
    with pytest.raises(lg.InvalidInputError):
        idx.query([0, 99], 2)
    # a uint16 row goes straight to the kernel, which raises the same error
    # (and the flag is cleared for the next query)
    with pytest.raises(lg.InvalidInputError, match="out of range for alphabet of size 4"):
        idx.query(np.array([0, 4], dtype=np.uint16), 2)
    assert idx.query(np.array([0, 1], dtype=np.uint16), 2, "complete").pairs() == [(0, 2)]
    empty = lg.build(lg.Dataset.from_rows(np.zeros((0, 2), dtype=np.uint16), 4))
    with pytest.raises(lg.InvalidInputError):  # no kernel runs on an empty index: checked on the host
        empty.query(np.array([0, 4], dtype=np.uint16), 2)
    # device-side symbol validation in the batched path
    with pytest.raises(lg.InvalidInputError):
        idx.query_batch(np.array([[0, 1], [0, 3], [0, 9]], dtype=np.uint16), 2)
    # the workspace error flag is cleared afterwards
    assert idx.query_batch(np.array([[0, 1]], dtype=np.uint16), 2).pairs(0) == [(0, 2)]
    ds = lg.generate_dataset(16, 3, 2, seed=4)
    with pytest.raises(lg.InvalidInputError):
        lg.build_tal(ds, 9)
    eng = lg.build_tal(ds, 8)
    with pytest.raises(lg.InvalidInputError):
        eng.query([0, 1, 0], 0)


def test_empty_and_degenerate(gpu):
    empty = lg.build(lg.Dataset.from_rows(np.zeros((0, 5), dtype=np.uint16), 4))
    assert empty.node_count == 1 and empty.root.subtree_size == 0
    empty.check_invariants()
    w = empty.new_work_report()
    r = empty.query([0, 1, 2, 3, 0], 3, "complete", work=w)
    assert r.pairs() == [] and r.matched_depth == 0 and w.nodes_visited == 1 and w.symbols_compared == 0
    eng = lg.build_tal(lg.Dataset.from_rows(np.zeros((0, 6), dtype=np.uint16), 2), 4)
    r, rep = eng.query([0, 1, 0, 1, 0, 1], 3)
    assert r.pairs() == [] and rep.items_scanned == 0
    zeros = lg.build_tal(lg.Dataset.from_rows(np.zeros((8, 6), dtype=np.uint16), 2), 4)
    r, rep = zeros.query(np.array([1, 1, 0, 0, 0, 0]), 5)
    assert r.pairs() == [] and rep.items_scanned == 0 and rep.energy_work_units == 0.0
    ds = lg.generate_dataset(35, 8, 4, seed=10)
    idx = lg.build(ds)
    for k in (1, 7, 35, 60, 10**9):
        assert len(idx.query(ds.items[0], k, "complete").indices) == min(k, 35)


def _random_cases(seed, count):
    rng = np.random.default_rng(seed)
    for t in range(count):
        n = int(rng.integers(0, 3000))
        L = int(rng.choice([1, 2, 3, 5, 8, 13, 16, 24, 31, 32, 33, 40, 64, 100]))
        sigma = int(rng.choice([2, 3, 4, 5, 7, 16, 17, 255, 256, 1000, 65536]))
        yield t, n, L, sigma, str(rng.choice(["uniform", "clustered"]))


@pytest.mark.parametrize("chunk", range(4))
def test_random_vs_oracle(gpu, oracle_lib, chunk, monkeypatch):
    """Fuzz: random (n, L, sigma, k, mode) vs the pinned C oracle.  Odd chunks
    force the 64-bit composite selection path."""
    if chunk % 2:
        monkeypatch.setenv("LCP_FORCE_WIDE_COMPOSITE", "1")
    for t, n, L, sigma, dist in _random_cases(1000 + chunk, 12):
        ds = lg.generate_dataset(n, L, sigma, seed=7 * t + chunk, distribution=dist)
        idx = lg.build(ds)
        ot = oracle_lib.OracleTrie(ds.items, sigma)
        assert np.array_equal(idx.order, ot.tables()[0]), (n, L, sigma)
        qs = lg.generate_queries(ds, 48, seed=t + 99)
        if n:
            qs = np.vstack([qs, lg.generate_queries(ds, 48, seed=t + 98, prefix_len=L // 2)])
        for k in (1, 3, 10, 20, 24, 32, 33, 64, 70, 100, 129):  # rank k<=16 / 1-, 2-, 4-slot lists / CTA paths
            for mode in ("complete", "strict"):
                b = idx.query_batch(qs, k, mode)
                ids, lcps, hits, md, sym, nodes = ot.query_batch(qs, k, mode)
                for i in range(len(qs)):
                    exp = list(zip(ids[i, :hits[i]].tolist(), lcps[i, :hits[i]].tolist()))
                    assert b.pairs(i) == exp, (n, L, sigma, dist, k, mode, i)
                    assert int(b.matched_depth[i]) == md[i]
            fb = idx.fullscan_batch(qs, k)
            oid, olcp, oh = oracle_lib.oracle_top_k_batch(ds.items, qs, k)
            for i in range(len(qs)):
                assert fb.pairs(i) == list(zip(oid[i, :oh[i]].tolist(), olcp[i, :oh[i]].tolist()))
        d = min(L, 3)
        if sigma**d <= 1 << 26:
            eng = lg.build_tal(ds, sigma**d)
            ote = oracle_lib.OracleTal(ds.items, sigma, eng.bucket_depth)
            for k in (1, 10, 32, 40, 64):
                b = eng.query_batch(qs, k)
                ids, lcps, hits, items, sym = ote.query_batch(qs, k)
                for i in range(len(qs)):
                    assert b.pairs(i) == list(zip(ids[i, :hits[i]].tolist(), lcps[i, :hits[i]].tolist()))
                assert np.array_equal(b.aux[:, 0].astype(np.int64), items)
                assert np.array_equal(b.aux[:, 1].astype(np.int64), sym)


def test_determinism_across_builds(gpu):
    ds = lg.generate_dataset(20_000, 20, 4, seed=20)
    qs = lg.generate_queries(ds, 500, seed=21, prefix_len=10)
    a, b = lg.build(ds), lg.build(ds)
    for mode in ("strict", "complete"):
        ra = a.query_batch(qs, 9, mode)
        rb = b.query_batch(qs, 9, mode)
        for i in range(len(qs)):
            assert ra.result(i).to_bytes() == rb.result(i).to_bytes()
        rc = a.query_batch(qs, 9, mode)
        assert np.array_equal(ra.ids, rc.ids) and np.array_equal(ra.hits, rc.hits)


def test_full_size_properties(gpu, oracle_lib):
    """BASELINE config 3 (N=2M, L=32, sigma=4, k=10): indexed complete mode must
    equal the independent full-scan kernel on every query, and the oracle on a
    sample; the sorted order must be a stable lexicographic permutation."""
    ds = lg.generate_dataset(2_000_000, 32, 4, seed=3)
    idx = lg.build(ds)
    order = idx.order
    assert np.array_equal(np.sort(order), np.arange(ds.n))
    keys = idx.native.export_sorted_keys()[:, 0]
    assert np.all(keys[1:] >= keys[:-1])
    ties = keys[1:] == keys[:-1]
    assert np.all(order[1:][ties] > order[:-1][ties])  # stable id tiebreak
    qs = np.vstack([lg.generate_queries(ds, 2048, seed=4), lg.generate_queries(ds, 2048, seed=5, prefix_len=16)])
    b = idx.query_batch(qs, 10, "complete")
    f = idx.fullscan_batch(qs, 10)
    assert np.array_equal(b.hits, f.hits)
    assert np.array_equal(b.ids, f.ids) and np.array_equal(b.lcps, f.lcps)
    sample = np.r_[0:32, 2048:2080]
    oid, olcp, oh = oracle_lib.oracle_top_k_batch(ds.items, qs[sample], 10, nthreads=8)
    for j, i in enumerate(sample):
        assert b.pairs(i) == list(zip(oid[j, :oh[j]].tolist(), olcp[j, :oh[j]].tolist()))
    # strict mode: every hit has the deepest lcp, and is a prefix of complete
    s = idx.query_batch(qs, 10, "strict")
    for i in range(0, len(qs), 97):
        assert s.pairs(i) == b.pairs(i)[: s.hits[i]]
        assert all(v == s.matched_depth[i] for _, v in s.pairs(i))


def test_device_api_with_torch(gpu):
    import torch

    ds = lg.generate_dataset(50_000, 24, 4, seed=4)
    idx = lg.build(ds)
    qs = lg.generate_queries(ds, 1000, seed=5, prefix_len=12)
    host = idx.query_batch(qs, 5, "complete")
    dq = torch.from_numpy(qs).cuda()
    ids = torch.empty((1000, 5), dtype=torch.int32, device="cuda")
    lcps = torch.empty((1000, 5), dtype=torch.int16, device="cuda")
    hits = torch.empty(1000, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    idx.native.query_device(dq, 5, "complete", ids, lcps, hits, stream=stream)
    torch.cuda.synchronize()
    assert np.array_equal(ids.cpu().numpy().view(np.uint32), host.ids)
    assert np.array_equal(hits.cpu().numpy(), host.hits)


def test_shard_encode_merge_kernels(gpu, oracle_lib):
    """k_encode + k_merge over 3 row-block shards (gathered in one process)
    equal the whole-corpus oracle, complete and strict."""
    import torch

    from paper_2602_04936_b200 import _native
    from paper_2602_04936_b200.engine import NativeIndex
    from paper_2602_04936_b200.sharded import ShardPlan

    lib = _native.load()
    ds = lg.generate_dataset(5000, 16, 4, seed=21)
    qs = np.vstack([lg.generate_queries(ds, 300, seed=22), lg.generate_queries(ds, 300, seed=23, prefix_len=8)])
    dq = torch.from_numpy(qs).cuda()
    world, count = 3, len(qs)
    plan = ShardPlan(ds.n, world)
    shards = [NativeIndex(ds.items[lo:hi], 16, 4) for lo, hi in (plan.bounds(r) for r in range(world))]
    full = oracle_lib.OracleTrie(ds.items, 4)
    for k in (1, 10, 32, 33, 100):  # > 32: the CTA-per-query merge
        for mode in ("complete", "strict"):
            gathered = torch.empty((world, count, k), dtype=torch.int64, device="cuda")
            for r, sh in enumerate(shards):
                ls = sh.stride_for(k)
                ids = torch.empty((count, ls), dtype=torch.int32, device="cuda")
                lcps = torch.empty((count, ls), dtype=torch.int16, device="cuda")
                hits = torch.empty(count, dtype=torch.int32, device="cuda")
                sh.query_device(dq, k, mode, ids, lcps, hits, stream=0)
                _native.check(lib.lcp_encode_candidates(ids.data_ptr(), lcps.data_ptr(), hits.data_ptr(), count,
                                                        k, ls, 16, plan.bounds(r)[0], gathered[r].data_ptr(), 0))
            take = min(k, ds.n)
            oids = torch.empty((count, take), dtype=torch.int32, device="cuda")
            olcps = torch.empty((count, take), dtype=torch.int16, device="cuda")
            ohits = torch.empty(count, dtype=torch.int32, device="cuda")
            _native.check(lib.lcp_merge_candidates(gathered.data_ptr(), world, count, k, take, 16,
                                                   1 if mode == "strict" else 0, oids.data_ptr(),
                                                   olcps.data_ptr(), ohits.data_ptr(), 0))
            torch.cuda.synchronize()
            ids_h, lcps_h, hits_h = oids.cpu().numpy().view(np.uint32), olcps.cpu().numpy(), ohits.cpu().numpy()
            fids, flcps, fhits, _, _, _ = full.query_batch(qs, k, mode)
            for i in range(count):
                got = list(zip(ids_h[i, :hits_h[i]].tolist(), lcps_h[i, :hits_h[i]].tolist()))
                assert got == list(zip(fids[i, :fhits[i]].tolist(), flcps[i, :fhits[i]].tolist())), (k, mode, i)


def test_sharded_index_single_rank_nccl(gpu):
    """ShardedIndex end to end on a 1-rank NCCL group (the collective path
    with world size 1) equals the unsharded index."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_2602_04936_b200.sharded import ShardedIndex

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        ds = lg.generate_dataset(20_000, 24, 4, seed=31)
        qs = lg.generate_queries(ds, 512, seed=32, prefix_len=12)
        sh = ShardedIndex(ds.items, 24, 4, id_offset=0)
        dq = torch.from_numpy(qs).cuda()
        ids = torch.empty((512, 10), dtype=torch.int32, device="cuda")
        lcps = torch.empty((512, 10), dtype=torch.int16, device="cuda")
        hits = torch.empty(512, dtype=torch.int32, device="cuda")
        sh.query_device(dq, 10, ids, lcps, hits)
        torch.cuda.synchronize()
        ref = lg.build(ds).query_batch(qs, 10, "complete")
        assert np.array_equal(hits.cpu().numpy(), ref.hits)
        assert np.array_equal(ids.cpu().numpy().view(np.uint32), ref.ids)
        assert np.array_equal(lcps.cpu().numpy().view(np.uint16), ref.lcps)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("path", ["host_ext", "ctypes"])
def test_async_pipeline_matches_sync(gpu, path, monkeypatch):
    from paper_2602_04936_b200 import _native

    if path == "ctypes":  # the submission without csrc/host_submit.c
        monkeypatch.setattr(_native, "_host_submit", None)
    else:
        assert _native.host_submit() is not None, "the CPython submission module is not built"
    ds = lg.generate_dataset(100_000, 24, 4, seed=41)
    idx = lg.build(ds)
    batches = [lg.generate_queries(ds, 777, seed=42 + b, prefix_len=b * 3) for b in range(7)]
    outs = [idx.native.alloc_batch(777, 5, "complete", pinned=True) for _ in range(3)]
    pending, got = [], []
    for b, qs in enumerate(batches):
        if len(pending) == 3:
            r = pending.pop(0).result()
            got.append((r.ids.copy(), r.lcps.copy(), r.hits.copy(), r.aux.copy()))
        pending.append(idx.query_batch_async(qs, 5, "complete", out=outs[b % 3]))
    for p in pending:
        r = p.result()
        got.append((r.ids.copy(), r.lcps.copy(), r.hits.copy(), r.aux.copy()))
    for qs, (ids, lcps, hits, aux) in zip(batches, got):
        ref = idx.query_batch(qs, 5, "complete")
        assert np.array_equal(ids, ref.ids) and np.array_equal(lcps, ref.lcps)
        assert np.array_equal(hits, ref.hits) and np.array_equal(aux, ref.aux)
    lean = idx.native.alloc_batch(777, 5, "complete", pinned=True, with_work=False)
    r = idx.query_batch_async(batches[2], 5, "complete", out=lean).result()
    ref = idx.query_batch(batches[2], 5, "complete")
    assert r.aux is None and r.matched_depth is None
    assert np.array_equal(r.ids, ref.ids) and np.array_equal(r.hits, ref.hits)
    bad = batches[0].copy()
    bad[3, 2] = 9
    out = idx.native.alloc_batch(777, 5, "complete", pinned=True)
    with pytest.raises(lg.InvalidInputError):
        idx.query_batch_async(bad, 5, "complete", out=out).result()
    r = idx.query_batch_async(batches[1], 5, "complete", out=out).result()
    assert np.array_equal(r.ids, idx.query_batch(batches[1], 5, "complete").ids)


def test_snapshot_bytes_match_reference(gpu, golden):
    """index_snapshot_bytes(gpu_index) is byte-identical to the reference's
    storage.index_snapshot_bytes for every golden case (storage.py:155-210)."""
    import os

    from paper_2602_04936_b200 import storage

    for case in golden[0]["cases"]:
        ds = case_dataset(case)
        snap = storage.index_snapshot_bytes(lg.build(ds))
        assert len(snap) == case["snapshot_size"], case["name"]
        assert hashlib.sha256(snap).hexdigest() == case["snapshot_sha256"], case["name"]
        path = os.path.join(os.path.dirname(__file__), "golden", f"snap_{case['name']}.lcpi")
        if os.path.exists(path):  # load the reference's own bytes onto the GPU
            raw = open(path, "rb").read()
            assert raw == snap
            loaded = storage.index_from_snapshot_bytes(raw)
            assert loaded.n == ds.n and loaded.length == ds.length and loaded.sigma == ds.alphabet.size
            assert np.array_equal(loaded.order, golden[1][case["name"] + "/order"])
            qs = golden[1][case["name"] + "/queries"]
            if len(qs):
                a = loaded.query_batch(qs, 5, "complete")
                b = lg.build(ds).query_batch(qs, 5, "complete")
                assert np.array_equal(a.ids, b.ids) and np.array_equal(a.hits, b.hits)


def test_snapshot_corruption_is_detected(gpu, golden, tmp_path):
    import os

    from paper_2602_04936_b200 import storage

    raw = open(os.path.join(os.path.dirname(__file__), "golden", "snap_trie500.lcpi"), "rb").read()
    bad = [raw[:20], b"XXXX" + raw[4:], raw[:4] + b"\x02\x00" + raw[6:], raw + b"\x00",
           raw[:-3], raw[:40] + b"\x07\x00" + raw[42:]]
    for blob in bad:
        with pytest.raises(lg.InvalidInputError):
            storage.index_from_snapshot_bytes(blob)
    path = tmp_path / "x.lcpi"
    idx = lg.build(lg.generate_dataset(777, 9, 3, seed=5))
    storage.write_index(str(path), idx)
    again = storage.read_index(str(path))
    assert storage.index_snapshot_bytes(again) == path.read_bytes()
    empty = lg.build(lg.Dataset.from_rows(np.zeros((0, 4), dtype=np.uint16), 4))
    e = storage.index_snapshot_bytes(empty)
    assert storage.index_snapshot_bytes(storage.index_from_snapshot_bytes(e)) == e


def test_wide_keys_at_scale(gpu, oracle_lib):
    """sigma = 65536 at N = 2M (W = 8, 64-byte keys, index larger than L2):
    the generic warp kernel must equal the full scan and the oracle."""
    ds = lg.generate_dataset(2_000_000, 32, 65536, seed=3)
    idx = lg.build(ds)
    qs = np.vstack([lg.generate_queries(ds, 256, seed=4), lg.generate_queries(ds, 256, seed=5, prefix_len=2)])
    b = idx.query_batch(qs, 10, "complete")
    f = idx.fullscan_batch(qs, 10)
    assert np.array_equal(b.hits, f.hits) and np.array_equal(b.ids, f.ids) and np.array_equal(b.lcps, f.lcps)
    oid, olcp, oh = oracle_lib.oracle_top_k_batch(ds.items, qs[250:262], 10, nthreads=8)
    for j, i in enumerate(range(250, 262)):
        assert b.pairs(i) == list(zip(oid[j, :oh[j]].tolist(), olcp[j, :oh[j]].tolist()))


def _long_run_cases():
    """Corpora whose queries have an R(d*) far wider than the loaded region."""
    rng = np.random.default_rng(77)
    # d* = 0 for most queries: the first symbol occurs ~4.6 times per 300K items
    ds = lg.generate_dataset(300_000, 8, 65536, seed=71)
    yield "s65536", ds, np.vstack([lg.generate_queries(ds, 96, seed=72),
                                   rng.integers(0, 65536, (96, 8)).astype(np.uint16)])
    # W == 1: R(1) holds ~1200 items, R(2) ~5
    ds = lg.generate_dataset(300_000, 8, 256, seed=73)
    yield "s256", ds, np.vstack([lg.generate_queries(ds, 96, seed=74),
                                 rng.integers(0, 256, (96, 8)).astype(np.uint16)])
    # half the corpus shares the prefix 0^6 with symbol 6 in {0,1,2}; queries
    # 0^6 3 ... sit in a 150K-item R(6) whose R(7) is (nearly) empty
    items = rng.integers(0, 4, (300_000, 16)).astype(np.uint16)
    items[:150_000, :6] = 0
    items[:150_000, 6] = rng.integers(0, 3, 150_000)
    ds = lg.Dataset.from_rows(items, 4)
    qs = rng.integers(0, 4, (128, 16)).astype(np.uint16)
    qs[:96, :6] = 0
    qs[:96, 6] = 3
    yield "skew", ds, qs


@pytest.mark.parametrize("wide", [False, True])
def test_long_runs_vs_oracle(gpu, oracle_lib, wide, monkeypatch):
    """R(d*) spanning up to the whole corpus: the run-edge search + id sketch
    must give exactly the oracle's answers (complete, strict and TAL)."""
    if wide:
        monkeypatch.setenv("LCP_FORCE_WIDE_COMPOSITE", "1")
    for name, ds, qs in _long_run_cases():
        idx = lg.build(ds)
        ot = oracle_lib.OracleTrie(ds.items, ds.alphabet.size)
        for k in (1, 10, 16, 17, 32, 33, 48, 64, 100, 128):
            for mode in ("complete", "strict"):
                b = idx.query_batch(qs, k, mode)
                ids, lcps, hits, md, sym, nodes = ot.query_batch(qs, k, mode)
                for i in range(len(qs)):
                    exp = list(zip(ids[i, :hits[i]].tolist(), lcps[i, :hits[i]].tolist()))
                    assert b.pairs(i) == exp, (name, k, mode, i)
                    assert int(b.matched_depth[i]) == md[i]
                w = idx.new_work_report()
                idx.query_batch(qs, k, mode, work=w)
                assert w.symbols_compared == int(sym.sum()) and w.nodes_visited == int(nodes.sum())
        eng = lg.build_tal(ds, ds.alphabet.size)
        ote = oracle_lib.OracleTal(ds.items, ds.alphabet.size, eng.bucket_depth)
        for k in (1, 10, 32):
            b = eng.query_batch(qs, k)
            ids, lcps, hits, items_, sym = ote.query_batch(qs, k)
            for i in range(len(qs)):
                assert b.pairs(i) == list(zip(ids[i, :hits[i]].tolist(), lcps[i, :hits[i]].tolist())), (name, k, i)
            assert np.array_equal(b.aux[:, 1].astype(np.int64), sym)


def test_clustered_at_scale(gpu, oracle_lib):
    """Config 3 shape with the clustered generator (long shared prefixes):
    indexed complete mode == independent full scan on every query, == oracle
    on a sample."""
    ds = lg.generate_dataset(2_000_000, 32, 4, seed=3, distribution="clustered")
    idx = lg.build(ds)
    qs = np.vstack([lg.generate_queries(ds, 2048, seed=4), lg.generate_queries(ds, 2048, seed=5, prefix_len=16)])
    for k in (10, 32):
        b = idx.query_batch(qs, k, "complete")
        f = idx.fullscan_batch(qs, k)
        assert np.array_equal(b.hits, f.hits) and np.array_equal(b.ids, f.ids) and np.array_equal(b.lcps, f.lcps)
    sample = np.r_[0:24, 2048:2072]
    oid, olcp, oh = oracle_lib.oracle_top_k_batch(ds.items, qs[sample], 32, nthreads=8)
    for j, i in enumerate(sample):
        assert b.pairs(i) == list(zip(oid[j, :oh[j]].tolist(), olcp[j, :oh[j]].tolist()))


def _range_gpu_worker(rank, world, port, backend):
    import os

    import torch
    import torch.distributed as dist

    import oracle
    from paper_2602_04936_b200.rangeshard import RangeShardedIndex

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group(backend, rank=rank, world_size=world)
    try:
        for n, L, sigma, seed in ((50_000, 16, 4, 31), (4000, 8, 2, 32), (20_000, 12, 65536, 33)):
            ds = lg.generate_dataset(n, L, sigma, seed=seed)
            qs = np.vstack([lg.generate_queries(ds, 200, seed=seed + 1),
                            lg.generate_queries(ds, 200, seed=seed + 2, prefix_len=L // 2)])
            lo, hi = n * rank // world, n * (rank + 1) // world
            sh = RangeShardedIndex(ds.items[lo:hi], L, sigma, id_offset=lo)
            full = oracle.OracleTrie(ds.items, sigma)
            dq = torch.from_numpy(qs).cuda()
            for k in (1, 10, 32, 50):
                for mode in ("complete", "strict"):
                    fids, flcps, fhits, _, _, _ = full.query_batch(qs, k, mode)
                    # host-bookkeeping protocol and the device-routed step
                    for ids, lcps, hits in (sh.query(dq, k, mode), sh.query_device(dq, k, mode)):
                        ids, lcps, hits = ids.cpu().long() & 0xFFFFFFFF, lcps.cpu().long() & 0xFFFF, hits.cpu()
                        for i in range(len(qs)):
                            h = int(hits[i])
                            assert list(zip(ids[i, :h].tolist(), lcps[i, :h].tolist())) == \
                                list(zip(fids[i, :fhits[i]].tolist(), flcps[i, :fhits[i]].tolist())), (n, k, mode, i)
            # all_to_all exchange: this rank gets the answers of its slice (and
            # the peer-memory exchange, NCCL only: symmetric memory + signals)
            m = len(qs) // world
            mine = slice(rank * m, (rank + 1) * m)
            cases = [(10, "complete", "all_to_all"), (5, "strict", "all_to_all"), (40, "complete", "all_to_all")]
            if backend == "nccl":
                cases += [(10, "complete", "p2p"), (5, "strict", "p2p"), (32, "complete", "p2p")]
            for k, mode, exchange in cases:
                fids, flcps, fhits, _, _, _ = full.query_batch(qs[mine], k, mode)
                ids, lcps, hits = sh.query_device(dq[: m * world], k, mode, exchange=exchange)
                ids, lcps, hits = ids.cpu().long() & 0xFFFFFFFF, lcps.cpu().long() & 0xFFFF, hits.cpu()
                for i in range(m):
                    h = int(hits[i])
                    assert list(zip(ids[i, :h].tolist(), lcps[i, :h].tolist())) == \
                        list(zip(fids[i, :fhits[i]].tolist(), flcps[i, :fhits[i]].tolist())), (n, k, mode, i)
            if backend == "nccl":
                # the device-routed step has no host round trip: capture it once
                # in a CUDA graph and replay it
                s = torch.cuda.Stream()
                s.wait_stream(torch.cuda.current_stream())
                for exchange in ("all_gather", "all_to_all", "p2p"):
                    with torch.cuda.stream(s):
                        ref = [t.clone() for t in sh.query_device(dq, 10, "complete", exchange=exchange)]
                        out = tuple(torch.empty_like(t) for t in ref)
                        g = torch.cuda.CUDAGraph()
                        with torch.cuda.graph(g, stream=s):
                            sh.query_device(dq, 10, "complete", out=out, exchange=exchange)
                        for t in out:
                            t.zero_()
                        g.replay()
                        g.replay()
                    torch.cuda.synchronize()
                    for a, b in zip(ref, out):
                        assert torch.equal(a, b), exchange
                # the row-block step through NCCL, captured the same way
                from paper_2602_04936_b200.sharded import RowBlockShardStep

                rb = RowBlockShardStep(ds.items, L, sigma, id_offset=0, n_total=n)
                with torch.cuda.stream(s):
                    ref = [t.clone() for t in rb.query_device(dq, 10, "complete", exchange="all_to_all")]
                    out = tuple(torch.empty_like(t) for t in ref)
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=s):
                        rb.query_device(dq, 10, "complete", out=out, exchange="all_to_all")
                    g.replay()
                torch.cuda.synchronize()
                fids, flcps, fhits, _, _, _ = full.query_batch(qs, 10, "complete")
                ids, lcps, hits = (t.cpu() for t in out)
                for i in range(len(qs)):
                    h = int(hits[i])
                    assert list(zip((ids[i, :h].long() & 0xFFFFFFFF).tolist(), (lcps[i, :h].long() & 0xFFFF).tolist())) == \
                        list(zip(fids[i, :fhits[i]].tolist(), flcps[i, :fhits[i]].tolist())), ("rowblock", i)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,backend", [(1, "nccl"), (2, "gloo"), (3, "gloo")])
def test_range_sharded_gpu_engine(gpu, oracle_lib, world, backend):
    """RangeShardedIndex with the CUDA engine and merge kernel.  world > 1
    shares the single GPU with gloo collectives (host-level exchange only)."""
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(_range_gpu_worker, args=(world, port, backend), nprocs=world, join=True)


def test_concurrent_readers(gpu):
    """A built index is safe for concurrent readers (trie.py:19-20): threads
    with their own workspaces get exactly the serial answers."""
    import threading

    ds = lg.generate_dataset(200_000, 24, 4, seed=40)
    idx = lg.build(ds)
    batches = [lg.generate_queries(ds, 512, seed=41 + t, prefix_len=(None if t % 2 else 12)) for t in range(8)]
    serial = [(idx.query_batch(b, 10, "complete"), idx.query_batch(b, 7, "strict")) for b in batches]
    errors = []

    def worker(t):
        try:
            for rep in range(5):
                for j in range(t, len(batches), 4):
                    c = idx.query_batch(batches[j], 10, "complete")
                    s = idx.query_batch(batches[j], 7, "strict")
                    for got, exp in ((c, serial[j][0]), (s, serial[j][1])):
                        assert np.array_equal(got.ids, exp.ids) and np.array_equal(got.hits, exp.hits)
                        assert np.array_equal(got.lcps, exp.lcps)
                    r = idx.query(batches[j][rep], 10, "complete")
                    assert r.pairs() == serial[j][0].pairs(rep)
        except Exception as e:  # pragma: no cover - reported below
            errors.append(repr(e))

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors


@pytest.mark.parametrize("L,sigma", [(1000, 3), (4096, 2)])
def test_long_keys_vs_oracle(gpu, oracle_lib, L, sigma):
    """Very long keys (W = 32..64 words): search tables no longer fit shared
    memory, the general kernel and the full scan's multi-word path run."""
    ds = lg.generate_dataset(600, L, sigma, seed=L)
    idx = lg.build(ds)
    ot = oracle_lib.OracleTrie(ds.items, sigma)
    qs = np.vstack([lg.generate_queries(ds, 20, seed=L + 1), lg.generate_queries(ds, 20, seed=L + 2, prefix_len=L // 2)])
    # near-duplicates: share all but the last symbol with a corpus row
    near = ds.items[:10].copy()
    near[:, -1] = (near[:, -1] + 1) % sigma
    qs = np.vstack([qs, near])
    for k in (1, 10, 33):
        for mode in ("complete", "strict"):
            b = idx.query_batch(qs, k, mode)
            ids, lcps, hits, md, _, _ = ot.query_batch(qs, k, mode)
            for i in range(len(qs)):
                assert b.pairs(i) == list(zip(ids[i, :hits[i]].tolist(), lcps[i, :hits[i]].tolist())), (k, mode, i)
        f = idx.fullscan_batch(qs, k)
        oid, olcp, oh = oracle_lib.oracle_top_k_batch(ds.items, qs, k)
        for i in range(len(qs)):
            assert f.pairs(i) == list(zip(oid[i, :oh[i]].tolist(), olcp[i, :oh[i]].tolist()))


def test_result_views_outlive_their_batch(gpu):
    """Views of a result (pinned, pooled block) stay valid after the result is
    dropped and later batches reuse pooled blocks."""
    import gc

    ds = lg.generate_dataset(50_000, 16, 4, seed=50)
    idx = lg.build(ds)
    q1 = lg.generate_queries(ds, 1000, seed=51)
    ref = idx.query_batch(q1, 10, "complete")
    expect_ids, expect_lcps = ref.ids.copy(), ref.lcps.copy()
    kept = idx.query_batch(q1, 10, "complete")
    ids, lcps = kept.ids, kept.lcps
    del kept
    gc.collect()
    for s in range(20):  # recycle pooled blocks with different answers
        idx.query_batch(lg.generate_queries(ds, 1000, seed=60 + s), 10, "complete")
    assert np.array_equal(ids, expect_ids) and np.array_equal(lcps, expect_lcps)


@pytest.mark.parametrize("wide", [False, True])
def test_large_k_vs_oracle(gpu, oracle_lib, wide, monkeypatch):
    """k_query_general at every branch: select-then-sort inside GEN_CAP, the
    warp setup for need > GEN_CAP / 2, radix rounds beyond GEN_CAP (k up to
    5000, ranges up to the whole corpus), for complete, strict, TAL and the
    full scan, with both composite widths."""
    if wide:
        monkeypatch.setenv("LCP_FORCE_WIDE_COMPOSITE", "1")
    rng = np.random.default_rng(31)
    dup = rng.integers(0, 4, (40, 12)).astype(np.uint16)[rng.integers(0, 40, 6000)]
    cases = [
        ("uniform", lg.generate_dataset(20_000, 16, 4, seed=30)),
        ("clustered", lg.generate_dataset(12_000, 24, 4, seed=32, distribution="clustered")),
        ("dups", lg.Dataset.from_rows(dup, 4)),
        ("wide", lg.generate_dataset(8_000, 40, 65536, seed=33)),
    ]
    for name, ds in cases:
        idx = lg.build(ds)
        sigma = ds.alphabet.size
        ot = oracle_lib.OracleTrie(ds.items, sigma)
        qs = np.vstack([lg.generate_queries(ds, 40, seed=34),
                        lg.generate_queries(ds, 40, seed=35, prefix_len=ds.length // 4)])
        for k in (200, 1000, 1024, 1025, 2048, 2049, 5000):
            for mode in ("complete", "strict"):
                b = idx.query_batch(qs, k, mode)
                ids, lcps, hits, md, sym, nodes = ot.query_batch(qs, k, mode)
                for i in range(len(qs)):
                    exp = list(zip(ids[i, :hits[i]].tolist(), lcps[i, :hits[i]].tolist()))
                    assert b.pairs(i) == exp, (name, k, mode, i)
                    assert int(b.matched_depth[i]) == md[i]
                w = idx.new_work_report()
                idx.query_batch(qs, k, mode, work=w)
                assert w.nodes_visited == int(nodes.sum()), (name, k, mode)
        for k in (100, 3000):
            fb = idx.fullscan_batch(qs[:8], k)
            oid, olcp, oh = oracle_lib.oracle_top_k_batch(ds.items, qs[:8], k)
            for i in range(8):
                assert fb.pairs(i) == list(zip(oid[i, :oh[i]].tolist(), olcp[i, :oh[i]].tolist())), (name, k)
        eng = lg.build_tal(ds, sigma)
        ote = oracle_lib.OracleTal(ds.items, sigma, eng.bucket_depth)
        for k in (100, 3000):
            b = eng.query_batch(qs, k)
            ids, lcps, hits, items_, sym = ote.query_batch(qs, k)
            for i in range(len(qs)):
                assert b.pairs(i) == list(zip(ids[i, :hits[i]].tolist(), lcps[i, :hits[i]].tolist())), (name, k, i)
            assert np.array_equal(b.aux[:, 1].astype(np.int64), sym)


@pytest.mark.parametrize("wide", [False, True])
def test_w1_large_alphabet_vs_oracle(gpu, oracle_lib, wide, monkeypatch):
    """W = 1 with a large alphabet (short keys): d* drops to 0 or 1 once k
    passes the depth-1 bucket size, so R(d*) spans most of the corpus (the
    id-order walk through rank[]) or a mid-sized run (position by position)
    beyond the id sketch's 32 per block.  Complete, strict and TAL at k up to
    128 (the list kernel) against the oracle, work counters included."""
    if wide:
        monkeypatch.setenv("LCP_FORCE_WIDE_COMPOSITE", "1")
    cases = [
        ("s65536-L4", lg.generate_dataset(60_000, 4, 65536, seed=40)),
        ("s256-L8", lg.generate_dataset(60_000, 8, 256, seed=41)),
        ("s256-L8-clustered", lg.generate_dataset(40_000, 8, 256, seed=42, distribution="clustered")),
    ]
    for name, ds in cases:
        idx = lg.build(ds)
        assert idx.native.words == 1
        sigma = ds.alphabet.size
        ot = oracle_lib.OracleTrie(ds.items, sigma)
        qs = np.vstack([lg.generate_queries(ds, 48, seed=43),
                        lg.generate_queries(ds, 48, seed=44, prefix_len=1)])
        for k in (17, 32, 33, 50, 64, 100, 128):
            for mode in ("complete", "strict"):
                b = idx.query_batch(qs, k, mode)
                ids, lcps, hits, md, sym, nodes = ot.query_batch(qs, k, mode)
                for i in range(len(qs)):
                    exp = list(zip(ids[i, :hits[i]].tolist(), lcps[i, :hits[i]].tolist()))
                    assert b.pairs(i) == exp, (name, k, mode, i)
                w = idx.new_work_report()
                idx.query_batch(qs, k, mode, work=w)
                assert w.nodes_visited == int(nodes.sum()), (name, k, mode)
        eng = lg.build_tal(ds, sigma)
        ote = oracle_lib.OracleTal(ds.items, sigma, eng.bucket_depth)
        for k in (17, 33, 64, 128):
            b = eng.query_batch(qs, k)
            ids, lcps, hits, items_, sym = ote.query_batch(qs, k)
            for i in range(len(qs)):
                assert b.pairs(i) == list(zip(ids[i, :hits[i]].tolist(), lcps[i, :hits[i]].tolist())), (name, k, i)
            assert np.array_equal(b.aux[:, 1].astype(np.int64), sym)


def test_wide_keys_list_kernel_vs_oracle(gpu, oracle_lib):
    """W in 2..8 with 32 < k <= 128 (k_query_warp_kn): windows, chunk
    extension, sketch / rank-walk / position tiers, and TAL (whole small
    buckets, complete answers in large ones, the sweep counter), against the
    oracle."""
    cases = [
        ("s256-W4", lg.generate_dataset(120_000, 32, 256, seed=50)),
        ("s65536-W8", lg.generate_dataset(60_000, 32, 65536, seed=51)),
        ("s16-W2", lg.generate_dataset(80_000, 32, 16, seed=52)),
        ("s256-W4-clustered", lg.generate_dataset(60_000, 32, 256, seed=53, distribution="clustered")),
    ]
    for name, ds in cases:
        idx = lg.build(ds)
        assert 2 <= idx.native.words <= 8
        ot = oracle_lib.OracleTrie(ds.items, ds.alphabet.size)
        qs = np.vstack([lg.generate_queries(ds, 48, seed=54),
                        lg.generate_queries(ds, 48, seed=55, prefix_len=2)])
        for k in (33, 48, 64, 65, 100, 128):
            for mode in ("complete", "strict"):
                b = idx.query_batch(qs, k, mode)
                ids, lcps, hits, md, sym, nodes = ot.query_batch(qs, k, mode)
                for i in range(len(qs)):
                    exp = list(zip(ids[i, :hits[i]].tolist(), lcps[i, :hits[i]].tolist()))
                    assert b.pairs(i) == exp, (name, k, mode, i)
                    assert int(b.matched_depth[i]) == md[i]
                w = idx.new_work_report()
                idx.query_batch(qs, k, mode, work=w)
                assert w.nodes_visited == int(nodes.sum()) and w.symbols_compared == int(sym.sum()), (name, k, mode)
        for buckets in (ds.alphabet.size, ds.alphabet.size ** 2):
            eng = lg.build_tal(ds, buckets)
            ote = oracle_lib.OracleTal(ds.items, ds.alphabet.size, eng.bucket_depth)
            for k in (33, 64, 100, 128):
                b = eng.query_batch(qs, k)
                ids, lcps, hits, items_, sym = ote.query_batch(qs, k)
                for i in range(len(qs)):
                    exp = list(zip(ids[i, :hits[i]].tolist(), lcps[i, :hits[i]].tolist()))
                    assert b.pairs(i) == exp, (name, buckets, k, i)
                assert np.array_equal(b.aux[:, 0].astype(np.int64), items_)
                assert np.array_equal(b.aux[:, 1].astype(np.int64), sym)


def test_long_keys_warp_kernel_vs_oracle(gpu, oracle_lib):
    """W > 8 with k <= 128 (k_query_warp_any, k_query_warp_any_kn): the any-W search, window,
    chunk extension and id-sketch long runs, at a scale where runs leave the
    window, for uniform and clustered corpora and near-duplicate queries."""
    cases = [
        ("L300-s4", lg.generate_dataset(50_000, 300, 4, seed=60)),
        ("L256-s256", lg.generate_dataset(30_000, 256, 256, seed=61)),
        ("L300-s4-clustered", lg.generate_dataset(40_000, 300, 4, seed=62, distribution="clustered")),
    ]
    for name, ds in cases:
        idx = lg.build(ds)
        assert idx.native.words > 8
        ot = oracle_lib.OracleTrie(ds.items, ds.alphabet.size)
        near = ds.items[:16].copy()
        near[:, -1] = (near[:, -1] + 1) % ds.alphabet.size
        qs = np.vstack([lg.generate_queries(ds, 40, seed=63),
                        lg.generate_queries(ds, 40, seed=64, prefix_len=ds.length // 4),
                        lg.generate_queries(ds, 24, seed=65, prefix_len=2), near])
        for k in (1, 5, 10, 16, 17, 32, 33, 64, 65, 100, 128):  # k_query_warp_any(_kn)
            for mode in ("complete", "strict"):
                b = idx.query_batch(qs, k, mode)
                ids, lcps, hits, md, sym, nodes = ot.query_batch(qs, k, mode)
                for i in range(len(qs)):
                    exp = list(zip(ids[i, :hits[i]].tolist(), lcps[i, :hits[i]].tolist()))
                    assert b.pairs(i) == exp, (name, k, mode, i)
                    assert int(b.matched_depth[i]) == md[i]
                w = idx.new_work_report()
                idx.query_batch(qs, k, mode, work=w)
                assert w.nodes_visited == int(nodes.sum()) and w.symbols_compared == int(sym.sum()), (name, k, mode)


@pytest.mark.parametrize("sigma", [4, 256])  # W = 1 and W = 4 (packed-query scratch)
@pytest.mark.parametrize("mode", ["strict", "complete"])
def test_graph_replay_multistream_matches_sync(gpu, mode, sigma):
    """The bench's device path: batches captured once in a CUDA graph, fanned
    out over 4 streams (one workspace each, per the header's contract),
    replayed repeatedly. Every replay must reproduce the synchronous host API's
    results bit for bit."""
    import torch

    from paper_2602_04936_b200._native import Workspace

    ds = lg.generate_dataset(200_000, 32, sigma, seed=31)
    idx = lg.build(ds)
    k, nb, bs = 10, 4, 1024
    qs = np.vstack([lg.generate_queries(ds, bs, seed=32 + b, prefix_len=(0 if b % 2 else 16))
                    for b in range(nb)])
    want = idx.query_batch(qs, k, mode)
    dev = torch.device("cuda")
    dq = torch.from_numpy(qs).to(dev).view(nb, bs, 32)
    bufs = [(torch.empty((bs, k), dtype=torch.int32, device=dev),
             torch.empty((bs, k), dtype=torch.int16, device=dev),
             torch.empty(bs, dtype=torch.int32, device=dev),
             torch.empty(bs, dtype=torch.int16, device=dev)) for _ in range(nb)]
    wss = [Workspace() for _ in range(nb)]  # allocated outside capture
    main = torch.cuda.Stream()  # capture needs a non-default stream
    main.wait_stream(torch.cuda.current_stream())
    streams = [torch.cuda.Stream() for _ in range(nb)]
    for b in range(nb):  # eager warm-up: workspace scratch grows outside capture
        ids, lcps, hits, md = bufs[b]
        idx.native.query_device(dq[b], k, mode, ids, lcps, hits, md, stream=main.cuda_stream, ws=wss[b])
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=main):
        for x in streams:
            x.wait_stream(main)
        for b, x in enumerate(streams):
            ids, lcps, hits, md = bufs[b]
            idx.native.query_device(dq[b], k, mode, ids, lcps, hits, md, stream=x.cuda_stream, ws=wss[b])
        for x in streams:
            main.wait_stream(x)
    for _ in range(3):
        for ids, lcps, hits, md in bufs:
            ids.fill_(-1), lcps.fill_(-1), hits.fill_(-1), md.fill_(-1)
        g.replay()
        torch.cuda.synchronize()
        for b, (ids, lcps, hits, md) in enumerate(bufs):
            sl = slice(b * bs, (b + 1) * bs)
            assert np.array_equal(hits.cpu().numpy(), want.hits[sl])
            assert np.array_equal(md.cpu().numpy().view(np.uint16), want.matched_depth[sl])
            got_ids, got_l = ids.cpu().numpy().view(np.uint32), lcps.cpu().numpy().view(np.uint16)
            for i in range(0, bs, 7):
                h = want.hits[b * bs + i]
                assert np.array_equal(got_ids[i, :h], want.ids[b * bs + i, :h])
                assert np.array_equal(got_l[i, :h], want.lcps[b * bs + i, :h])


def test_async_graph_cache_survives_scratch_growth(gpu):
    """a cached async graph bakes in the workspace's device
    scratch pointers.  Alternating submissions of different counts with the
    SAME host query / output pointers on ONE workspace grow (reallocate) that
    scratch between replays; every result must still equal the synchronous
    API's (a stale graph would read and write freed device memory)."""
    import ctypes

    from paper_2602_04936_b200 import _native
    from paper_2602_04936_b200._native import PackedLayout, PinnedArray, Workspace, check, load

    ds = lg.generate_dataset(300_000, 32, 4, seed=13)
    idx = lg.build(ds)
    qs = lg.generate_queries(ds, 8192, seed=14)
    k = 10
    ref = idx.query_batch(qs, k, "complete")
    lib = load()
    ws = Workspace()
    pin_q = PinnedArray((8192, 32), np.uint16)
    pin_q.array[:] = qs
    lay_max = PackedLayout()
    check(lib.lcp_packed_layout_for(8192, k, ctypes.byref(lay_max)))
    block = PinnedArray((int(lay_max.total),), np.uint8)
    for count in (1024, 4096, 1024, 8192, 1024, 4096, 1024):
        lay = PackedLayout()
        check(lib.lcp_packed_layout_for(count, k, ctypes.byref(lay)))
        block.array[:] = 0xAB
        check(lib.lcp_query_host_packed_async(idx.native.handle, ws.handle, pin_q.address, count, k, 1, k,
                                              block.address, 0))
        check(lib.lcp_workspace_wait(ws.handle))
        raw = block.array
        ids = raw[lay.ids:lay.ids + count * k * 4].view(np.uint32).reshape(count, k)
        lcps = raw[lay.lcps:lay.lcps + count * k * 2].view(np.uint16).reshape(count, k)
        hits = raw[lay.hits:lay.hits + count * 4].view(np.int32)
        assert np.array_equal(hits, ref.hits[:count]), count
        assert np.array_equal(ids, ref.ids[:count]) and np.array_equal(lcps, ref.lcps[:count]), count
    ws.close()
    del _native



def test_rowblock_shard_step_single_process(gpu, oracle_lib):
    """RowBlockShardStep (the config-5 row-block step: local top-k -> encode
    -> exchange -> merge) with one process and several blocks composed by
    hand equals the oracle; the single-block step equals the plain index."""
    import torch

    from paper_2602_04936_b200.sharded import RowBlockShardStep, merge_candidates

    ds = lg.generate_dataset(120_000, 32, 4, seed=61)
    qs = np.vstack([lg.generate_queries(ds, 300, seed=62), lg.generate_queries(ds, 300, seed=63, prefix_len=16)])
    dq = torch.from_numpy(qs).cuda()
    one = RowBlockShardStep(ds.items, 32, 4, id_offset=0, n_total=ds.n)
    trie = oracle_lib.OracleTrie(ds.items, 4)
    for k, mode in ((10, "complete"), (7, "strict"), (33, "complete")):
        ids, lcps, hits = one.query_device(dq, k, mode)
        fids, flcps, fhits, _, _, _ = trie.query_batch(qs, k, mode)
        for i in range(len(qs)):
            h = int(hits[i])
            got = list(zip((ids[i, :h].cpu().long() & 0xFFFFFFFF).tolist(), (lcps[i, :h].cpu().long() & 0xFFFF).tolist()))
            assert got == list(zip(fids[i, :fhits[i]].tolist(), flcps[i, :fhits[i]].tolist())), (k, mode, i)


def test_range_shard_p2p_single_process(gpu, oracle_lib):
    """The peer-memory exchange (signal + merge reading the peers' candidate
    buffers) in one process without a process group: one range shard whose
    'peers' are its own buffers, stepped repeatedly (the epoch advances) and
    replayed from a CUDA graph, equals the oracle."""
    import torch

    from paper_2602_04936_b200.rangeshard import RangeShardedIndex

    ds = lg.generate_dataset(80_000, 32, 4, seed=71)
    qs = np.vstack([lg.generate_queries(ds, 256, seed=72), lg.generate_queries(ds, 256, seed=73, prefix_len=16)])
    dq = torch.from_numpy(qs).cuda()
    sh = RangeShardedIndex(ds.items, 32, 4, id_offset=0)
    trie = oracle_lib.OracleTrie(ds.items, 4)
    for k, mode in ((10, "complete"), (7, "strict"), (32, "complete"), (10, "complete")):
        fids, flcps, fhits, _, _, _ = trie.query_batch(qs, k, mode)
        for _ in range(3):
            ids, lcps, hits = sh.query_device(dq, k, mode, exchange="p2p")
        ids, lcps, hits = ids.cpu().long() & 0xFFFFFFFF, lcps.cpu().long() & 0xFFFF, hits.cpu()
        for i in range(len(qs)):
            h = int(hits[i])
            assert list(zip(ids[i, :h].tolist(), lcps[i, :h].tolist())) == \
                list(zip(fids[i, :fhits[i]].tolist(), flcps[i, :fhits[i]].tolist())), (k, mode, i)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        ref = [t.clone() for t in sh.query_device(dq, 10, "complete", exchange="p2p")]
        out = tuple(torch.empty_like(t) for t in ref)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            sh.query_device(dq, 10, "complete", out=out, exchange="p2p")
        for _ in range(3):
            g.replay()
    torch.cuda.synchronize()
    for a, b in zip(ref, out):
        assert torch.equal(a, b)


def test_single_query_alternating_k_and_freed_blocks(gpu):
    """TrieIndex.query through the graph-cached submission with k changing
    every call (a new one-row output block each time, the old one freed and
    its address reused) and explicitly freed / re-allocated pinned blocks on
    the async API: results equal the batch API.  The async graph cache used
    to bake the caller's host pointers into the graph; replaying it after a
    free and reallocation at the same address crashed in cuGraphLaunch."""
    import gc

    ds = lg.generate_dataset(5_000, 12, 3, seed=81)
    idx = lg.build(ds)
    qs = lg.generate_queries(ds, 90, seed=82)
    ref = {(k, m): idx.query_batch(qs, k, m) for k in (1, 5, 50) for m in ("strict", "complete")}
    for rep in range(3):
        for i, q in enumerate(qs):
            k = (1, 5, 50)[(i + rep) % 3]
            for m in ("strict", "complete"):
                assert idx.query(q, k, m).pairs() == ref[(k, m)].pairs(i), (rep, i, k, m)
        gc.collect()
    for rep in range(4):  # async API: fresh pinned blocks every round
        out = idx.native.alloc_batch(len(qs), 5 if rep % 2 else 50, "complete", pinned=True)
        res = idx.query_batch_async(qs, 5 if rep % 2 else 50, "complete", out=out).result()
        exp = ref[(5 if rep % 2 else 50, "complete")]
        assert np.array_equal(res.hits, exp.hits) and np.array_equal(res.ids, exp.ids)
        del out, res
        gc.collect()


@pytest.mark.parametrize("sigma,length", [(4, 32), (65536, 12), (300, 40)])
def test_direct_host_io_matches_copy_path(gpu, sigma, length):
    """Small batches in lcp_pinned_alloc blocks are served with direct host
    I/O (the kernels read rows from / write results into mapped host memory);
    pageable queries take the copy path.  Both must give the same bytes, with
    and without work counters, across the kernel routes (k <= 16 rank kernel,
    17 <= k <= 32 list kernel, W == 1 and W > 1), and an invalid symbol must be
    reported through the host-written flag and then cleared."""
    from paper_2602_04936_b200._native import PinnedArray

    ds = lg.generate_dataset(60_000, length, sigma, seed=77)
    idx = lg.build(ds)
    for count in (1, 7, 1024, 1025):
        qs = lg.generate_queries(ds, count, seed=78 + count, prefix_len=length // 2)
        pin = PinnedArray((count, length), np.uint16)
        pin.array[:] = qs
        for k in (1, 5, 10, 17, 32):
            for mode in ("strict", "complete"):
                ref = idx.query_batch(qs.copy(), k, mode)  # pageable rows: copies
                for work in (True, False):
                    out = idx.native.alloc_batch(count, k, mode, pinned=True, with_work=work)
                    r = idx.query_batch_async(pin.array, k, mode, out=out).result()
                    assert np.array_equal(r.hits, ref.hits), (count, k, mode, work)
                    for q in range(count):
                        h = int(ref.hits[q])
                        assert np.array_equal(r.ids[q, :h], ref.ids[q, :h]), (count, k, mode, q)
                        assert np.array_equal(r.lcps[q, :h], ref.lcps[q, :h]), (count, k, mode, q)
                    if work:
                        assert np.array_equal(r.matched_depth, ref.matched_depth)
                        assert np.array_equal(r.aux, ref.aux)
                sync = idx.query_batch(pin.array, k, mode,
                                       out=idx.native.alloc_batch(count, k, mode, pinned=True))
                assert np.array_equal(sync.hits, ref.hits) and np.array_equal(sync.aux, ref.aux)
        bad = PinnedArray((count, length), np.uint16)
        bad.array[:] = qs
        bad.array[count - 1, 0] = sigma if sigma < 65536 else 0
        if sigma < 65536:
            out = idx.native.alloc_batch(count, 10, "complete", pinned=True)
            with pytest.raises(lg.InvalidInputError):
                idx.query_batch_async(bad.array, 10, "complete", out=out).result()
            r = idx.query_batch_async(pin.array, 10, "complete", out=out).result()
            ref = idx.query_batch(qs.copy(), 10, "complete")
            assert np.array_equal(r.hits, ref.hits) and np.array_equal(r.aux, ref.aux)
    # the single-query API (its own pinned stage and block) agrees as well
    q = lg.generate_queries(ds, 3, seed=5)
    for i in range(3):
        a = idx.query(q[i], 10, "complete")
        b = idx.query_batch(q[i:i + 1].copy(), 10, "complete")
        assert list(a.indices) == list(b.ids[0, :int(b.hits[0])])


def test_memoized_query_hits_and_counters(gpu):
    """memoized_query (trie.py:464-488): uint16 rows hit without re-validation,
    other inputs are validated first; counters and errors as the reference's."""
    ds = lg.generate_dataset(20_000, 16, 4, seed=90)
    idx = lg.build(ds)
    qs = lg.generate_queries(ds, 8, seed=91, prefix_len=8)
    cache = lg.QueryCache()
    w = idx.new_work_report()
    cold = [lg.memoized_query(idx, q, 10, "complete", cache, work=w) for q in qs]
    assert cache.misses == 8 and cache.hits == 0 and w.cache_hits == 0
    for q in qs:  # uint16 rows, lists and int64 rows all hit the same entries
        for form in (q, q.tolist(), q.astype(np.int64)):
            r = lg.memoized_query(idx, form, 10, "complete", cache, work=w)
            assert r is cold[list(map(bytes, qs)).index(bytes(q))]
    assert cache.hits == 24 and cache.misses == 8 and w.cache_hits == 24
    bad = qs[0].copy()
    bad[3] = 4
    with pytest.raises(lg.InvalidInputError):
        lg.memoized_query(idx, bad, 10, "complete", cache)
    with pytest.raises(lg.InvalidInputError):  # 2-D, even though its bytes are cached
        lg.memoized_query(idx, qs[:1], 10, "complete", cache)
    assert cache.misses == 8 and cache.hits == 24
    assert lg.memoized_query(idx, qs[0], 10, "strict", cache) is not cold[0]  # mode is in the key
    assert cache.misses == 9


def test_low_latency_server(gpu):
    """TrieIndex.low_latency: a resident warp answers single queries through
    page-locked mailboxes (csrc/serve_kernels.cuh).  Answers and work
    counters equal the batch API for strict / complete, k up to 16, rows of
    1 to 4 request sectors; shapes it does not serve fall back; an invalid
    symbol is reported; the warp idles out (a device synchronisation inside
    the block returns) and is relaunched; threads get their own servers."""
    import threading
    import time

    import torch

    for n, L, sigma, seed in ((100_000, 24, 4, 4), (5, 16, 4, 6), (30_000, 48, 2, 7), (20_000, 32, 4, 8)):
        ds = lg.generate_dataset(n, L, sigma, seed=seed)
        idx = lg.build(ds)
        qs = np.vstack([lg.generate_queries(ds, 40, seed=seed + 1),
                        lg.generate_queries(ds, 40, seed=seed + 2, prefix_len=L // 2)])
        for k in (1, 5, 10, 16, 20, 32, 40):  # 64- and 96-key regions; 40: not served
            for mode in ("strict", "complete"):
                ref = idx.query_batch(qs, k, mode)
                w_ref, w_got = idx.new_work_report(), idx.new_work_report()
                idx.query_batch(qs, k, mode, work=w_ref)
                with idx.low_latency(k, mode):
                    for i in range(len(qs)):
                        r = idx.query(qs[i], k, mode, work=w_got)
                        assert r.pairs() == ref.pairs(i), (n, L, k, mode, i)
                        assert r.matched_depth == int(ref.matched_depth[i])
                assert w_got.symbols_compared == w_ref.symbols_compared
                assert w_got.nodes_visited == w_ref.nodes_visited
    ds = lg.generate_dataset(50_000, 16, 4, seed=9)
    idx = lg.build(ds)
    qs = lg.generate_queries(ds, 8, seed=10)
    ref = idx.query_batch(qs, 10, "complete")
    with idx.low_latency(10, "complete"):
        assert idx._tls.server is not None
        bad = qs[0].copy()
        bad[5] = 4
        with pytest.raises(lg.InvalidInputError, match="alphabet of size 4"):
            idx.query(bad, 10, "complete")
        assert idx.query(qs[1], 10, "complete").pairs() == ref.pairs(1)
        t0 = time.perf_counter()
        torch.cuda.synchronize()  # waits for the warp to idle out (100 ms)
        assert time.perf_counter() - t0 < 5.0
        assert idx.query(qs[2], 10, "complete").pairs() == ref.pairs(2)  # relaunched
        assert idx.query(qs[3], 10, "strict").pairs() == idx.query_batch(qs[3:4], 10, "strict").pairs(0)

    errors = []

    def worker(t):
        try:
            with idx.low_latency(10, "complete"):
                for i in range(len(qs)):
                    assert idx.query(qs[i], 10, "complete").pairs() == ref.pairs(i)
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(3)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    # TAL through the server: answers and the bucket counters per query
    tds = lg.generate_dataset(60_000, 16, 4, seed=13)
    eng = lg.build_tal(tds, 256)
    tq = np.vstack([lg.generate_queries(tds, 30, seed=14), lg.generate_queries(tds, 30, seed=15, prefix_len=6)])
    for k in (3, 10, 24):
        ref = eng.query_batch(tq, k)
        exp = [eng.query(tq[i], k) for i in range(len(tq))]  # launch path
        with eng.low_latency(k):
            assert eng._tls.server is not None
            for i in range(len(tq)):
                res, rep = eng.query(tq[i], k)
                assert res.to_bytes() == exp[i][0].to_bytes(), (k, i)
                assert res.pairs() == ref.pairs(i), (k, i)
                assert (rep.items_scanned, rep.symbols_compared) == (exp[i][1].items_scanned,
                                                                     exp[i][1].symbols_compared), (k, i)
    wide = lg.build(lg.generate_dataset(2000, 32, 65536, seed=11))  # W > 1: not served, same API
    q = lg.generate_queries(lg.generate_dataset(2000, 32, 65536, seed=11), 1, seed=12)[0]
    with wide.low_latency(5, "complete"):
        assert wide._tls.server is None
        assert wide.query(q, 5, "complete").pairs() == wide.query_batch(q[None], 5, "complete").pairs(0)
