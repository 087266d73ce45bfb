"""Pin the CPU oracle (oracle/lcp_oracle.c) to the reference's own outputs.

The golden vectors in tests/golden were produced by importing the reference
package (tests/golden/make_golden.py).  Every oracle function is checked
against them before any GPU result is judged by the oracle.
"""

import numpy as np
import pytest

from golden_util import case_dataset, expected_rows, sha


def _cases(golden):
    return golden[0]["cases"]


def test_hand_cases(oracle_lib, golden):
    hand = golden[0]["hand"]
    o = oracle_lib
    ids, lcps = o.oracle_top_k(np.array([[0, 0], [0, 1], [1, 1]]), [0, 1], 2)
    assert list(zip(ids.tolist(), lcps.tolist())) == [tuple(p) for p in hand["oracle_hand"]]
    ids, lcps = o.oracle_top_k(np.array([[0, 0], [1, 1], [0, 1]]), [0, 0], 10)
    assert list(zip(ids.tolist(), lcps.tolist())) == [tuple(p) for p in hand["oracle_k_ge_n"]]
    ids, lcps = o.oracle_top_k(np.array([[3, 3]] * 3), [3, 3], 2)
    assert list(zip(ids.tolist(), lcps.tolist())) == [tuple(p) for p in hand["oracle_dups"]]
    assert o.lexicographic_order(np.array([[1, 2], [0, 1], [0, 2], [1, 3]])).tolist() == hand["order_1203"]
    assert o.adjacent_lcp(np.array([[0, 0, 0], [0, 0, 1], [0, 1, 1], [1, 1, 1]])).tolist() == hand["adjacent_210"]
    t = o.OracleTrie(np.array([[0, 0], [0, 1], [1, 0]]), 2)
    ids, lcps, md, _, _ = t.query(np.array([0, 0]), 3, "complete")
    assert list(zip(ids.tolist(), lcps.tolist())) == [tuple(p) for p in hand["complete_3item"]]
    ids, lcps, md, _, _ = t.query(np.array([0, 0]), 3, "strict")
    assert list(zip(ids.tolist(), lcps.tolist())) == [tuple(p) for p in hand["strict_3item"]]
    assert md == 2


@pytest.mark.parametrize("idx", range(16))
def test_oracle_matches_reference_goldens(oracle_lib, golden, idx):
    manifest, arrays = golden
    cases = _cases(golden)
    if idx >= len(cases):
        pytest.skip("no such case")
    case = cases[idx]
    name = case["name"]
    ds = case_dataset(case)
    pre = name + "/"
    qs = arrays[pre + "queries"]
    ks = arrays[pre + "k"]
    trie = oracle_lib.OracleTrie(ds.items, case["sigma"])
    order, row_lo, edge, off = trie.tables()
    assert np.array_equal(order, arrays[pre + "order"])
    assert np.array_equal(off, arrays[pre + "level_offset"])
    assert sha(row_lo) == case["row_lo_sha256"]
    assert sha(edge) == case["edge_symbol_sha256"]
    assert trie.node_count == case["node_count"]
    assert np.array_equal(oracle_lib.lexicographic_order(ds.items), arrays[pre + "order"])
    if ds.n:
        adj = oracle_lib.adjacent_lcp(ds.items[order])
        assert np.array_equal(adj, arrays[pre + "adjacent_lcp"])
    for mode in ("strict", "complete"):
        mp = f"{pre}{mode}/"
        for i, q in enumerate(qs):
            ids, lcps, md, sym, nodes = trie.query(q, int(ks[i]), mode)
            assert list(zip(ids.tolist(), lcps.tolist())) == expected_rows(arrays, mp, i), (name, mode, i)
            assert md == arrays[mp + "md"][i]
            assert sym == arrays[mp + "sym"][i]
            assert nodes == arrays[mp + "nodes"][i]
    for i, q in enumerate(qs):
        ids, lcps = oracle_lib.oracle_top_k(ds.items, q, int(ks[i]))
        assert list(zip(ids.tolist(), lcps.tolist())) == expected_rows(arrays, pre + "oracle/", i)
    for tal in case["tal"]:
        tp = f"{pre}tal{tal['B']}/"
        eng = oracle_lib.OracleTal(ds.items, case["sigma"], tal["depth"])
        if tp + "directory" in arrays:
            assert np.array_equal(eng.directory(), arrays[tp + "directory"])
        for i, q in enumerate(qs):
            ids, lcps, items, sym = eng.query(q, int(ks[i]))
            assert list(zip(ids.tolist(), lcps.tolist())) == expected_rows(arrays, tp, i)
            assert items == arrays[tp + "items"][i] and sym == arrays[tp + "sym"][i]
            assert eng.bucket_range(q) == (arrays[tp + "lo"][i], arrays[tp + "hi"][i])


def test_batch_drivers_match_single(oracle_lib, golden):
    manifest, arrays = golden
    case = next(c for c in manifest["cases"] if c["name"] == "cfg1")
    ds = case_dataset(case)
    qs = arrays["cfg1/queries"][:200]
    trie = oracle_lib.OracleTrie(ds.items, 4)
    ids, lcps, hits, md, sym, nodes = trie.query_batch(qs, 10, "complete", nthreads=3)
    for i in range(len(qs)):
        assert list(zip(ids[i, :hits[i]].tolist(), lcps[i, :hits[i]].tolist())) == expected_rows(
            arrays, "cfg1/complete/", i)
    oid, olcp, oh = oracle_lib.oracle_top_k_batch(ds.items, qs[:50], 10, nthreads=2)
    for i in range(50):
        assert list(zip(oid[i, :oh[i]].tolist(), olcp[i, :oh[i]].tolist())) == expected_rows(
            arrays, "cfg1/oracle/", i)
