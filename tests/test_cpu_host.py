"""CPU-only checks: datagen restatement, C-ABI exports, host-side logic.

No compute call reaches the extension here (there is no GPU); the product
package must import and expose its ABI, and fail loudly when asked to run.
"""

import ast
import os
import re

import numpy as np
import pytest

from golden_util import sha
from paper_2602_04936_b200 import (
    Dataset,
    InvalidInputError,
    QueryResult,
    WorkReport,
    generate_dataset,
    generate_queries,
)
from paper_2602_04936_b200.core import validate_query_batch, validate_query_row
from paper_2602_04936_b200.result import BatchResult
from paper_2602_04936_b200.tal import _prefix_depth
from paper_2602_04936_b200.work import tal_counters, trie_counters

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2602_04936_b200")


# ---------------------------------------------------------------- datagen
def test_datagen_is_byte_identical_to_reference(golden):
    for g in golden[0]["datagen"]:
        args, kw = g["args"], g["kwargs"]
        if args[0] > 200_000:
            continue  # the 2M pin is exercised by the bench/GPU tests
        ds = generate_dataset(*args, **kw)
        assert sha(ds.items) == g["dataset_sha256"], (args, kw)
        assert sha(generate_queries(ds, 257, seed=args[3] + 1)) == g["queries_sha256"]
        assert sha(generate_queries(ds, 129, seed=args[3] + 2, prefix_len=args[1] // 2)) == g["prefix_queries_sha256"]


def test_datagen_errors():
    with pytest.raises(InvalidInputError):
        generate_dataset(-1, 4, 4, seed=1)
    with pytest.raises(InvalidInputError):
        generate_dataset(10, 4, 4, seed=1, distribution="zipf")
    with pytest.raises(InvalidInputError):
        generate_dataset(17, 2, 4, seed=1, distinct=True)
    ds = generate_dataset(0, 4, 4, seed=1)
    with pytest.raises(InvalidInputError):
        generate_queries(ds, 3, seed=1, prefix_len=2)


# ---------------------------------------------------------------- C ABI
def _header_functions():
    text = open(os.path.join(ROOT, "include", "lcp_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(lcp_\w+)\s*\(", text, flags=re.M)))


def test_library_exports_every_header_symbol(native_lib):
    names = _header_functions()
    assert len(names) >= 25
    for name in names:
        assert hasattr(native_lib, name), f"missing export {name}"
    assert native_lib.lcp_abi_version() == 1


def test_ctypes_table_covers_header():
    from paper_2602_04936_b200._native import SIGNATURES

    assert sorted(SIGNATURES) == _header_functions()


def test_host_submit_module_binds_the_abi_entry_point(native_lib):
    """csrc/host_submit.c: built, bound to lcp_query_host_packed_async of the
    loaded library, and it rejects a malformed query batch before any call."""
    from paper_2602_04936_b200 import _native

    submit = _native.host_submit()
    assert submit is not None, "the CPython submission module is not built"
    with pytest.raises(ValueError):  # wrong row length
        submit(0, 0, np.zeros((4, 31), np.uint16), 32, 10, 1, 10, 0, 0)
    with pytest.raises(ValueError):  # 4-byte items
        submit(0, 0, np.zeros((4, 32), np.uint32), 32, 10, 1, 10, 0, 0)
    with pytest.raises((ValueError, BufferError, TypeError)):  # not C-contiguous
        submit(0, 0, np.zeros((32, 4), np.uint16).T, 4, 10, 1, 10, 0, 0)
    with pytest.raises(TypeError):
        submit(0, 0)


def test_library_is_sm100a_only(native_lib):
    from paper_2602_04936_b200._native import LIB_PATH

    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
    assert "sm_90" not in out.stdout and "sm_80" not in out.stdout


def test_product_never_imports_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if not f.endswith(".py"):
                continue
            tree = ast.parse(open(os.path.join(dirpath, f)).read())
            for node in ast.walk(tree):
                if isinstance(node, ast.Import):
                    assert all(not a.name.startswith("oracle") for a in node.names), f
                if isinstance(node, ast.ImportFrom) and node.module:
                    assert not node.module.startswith("oracle"), f
                    assert "lcpsearch" not in node.module, f


def test_missing_library_fails_loudly(monkeypatch):
    from paper_2602_04936_b200 import _native

    monkeypatch.setattr(_native, "_lib", None)
    monkeypatch.setattr(_native, "LIB_PATH", "/nonexistent/_lcp_b200.so")
    with pytest.raises(_native.NativeLibraryMissing):
        _native.load()


# ---------------------------------------------------------------- host logic
def test_query_validation_messages():
    with pytest.raises(InvalidInputError, match="1-D"):
        validate_query_row(np.zeros((2, 2)), 2, 4)
    with pytest.raises(InvalidInputError, match="query length 1 != index length 2"):
        validate_query_row([0], 2, 4)
    with pytest.raises(InvalidInputError, match="out of range"):
        validate_query_row([0, 99], 2, 4)
    with pytest.raises(InvalidInputError, match="must have length 6"):
        validate_query_row([0, 1], 6, 2, tal=True)
    with pytest.raises(InvalidInputError):
        validate_query_batch(np.zeros((3, 5)), 4, 4)
    with pytest.raises(InvalidInputError):
        validate_query_batch(np.full((3, 4), 7), 4, 4)
    assert validate_query_batch(np.zeros(4, dtype=np.int64), 4, 4).shape == (1, 4)


def test_dataset_contract():
    ds = Dataset.from_rows([[0, 1], [1, 1]], 2)
    assert ds.n == 2 and ds.items.dtype == np.uint16 and not ds.items.flags.writeable
    with pytest.raises(InvalidInputError):
        Dataset.from_rows([[0, 2]], 2)
    with pytest.raises(InvalidInputError):
        Dataset.from_rows([0, 1], 2)


def test_result_bytes_match_reference(golden):
    hand = golden[0]["hand"]
    r = QueryResult(indices=np.array([0, 1, 2], dtype=np.int32),
                    lcps=np.array([2, 1, 0], dtype=np.int64), matched_depth=2, mode="complete")
    assert r.to_bytes().hex() == hand["result_bytes"]


def test_prefix_depth():
    assert _prefix_depth(2, 256) == 8
    assert _prefix_depth(4, 5) == 2
    assert _prefix_depth(4, 1) == 0
    assert _prefix_depth(65536, 65536) == 1


def test_work_counter_reconstruction():
    # d_max=3 < L=8, d*=1 complete: symbols 4, nodes 4 + 2;  d_max=L: symbols L
    aux = np.array([[3 | (1 << 32), 0], [8 | (8 << 32), 0]], dtype=np.uint64)
    assert trie_counters(aux, 100, 8, complete=True) == (4 + 8, (4 + 2) + 9)
    assert trie_counters(aux, 100, 8, complete=False) == (12, 4 + 9)
    assert trie_counters(aux, 0, 8, complete=True) == (0, 2)
    assert tal_counters(np.array([[5, 9], [0, 0]], dtype=np.uint64)) == (5, 9)
    w = WorkReport(c_sym=0.125, symbols_compared=8, items_scanned=3)
    assert w.energy_work_units == pytest.approx(4.0)


def test_batch_result_views():
    b = BatchResult(ids=np.array([[4, 2, 0]], dtype=np.uint32), lcps=np.array([[3, 1, 0]], dtype=np.uint16),
                    hits=np.array([2], dtype=np.int32), matched_depth=np.array([3], dtype=np.uint16),
                    aux=np.zeros((1, 2), dtype=np.uint64), mode="tal")
    r = b.result(0)
    assert r.pairs() == [(4, 3), (2, 1)] and r.indices.dtype == np.int64 and r.matched_depth == 3
    b.hits[0] = 0
    assert b.result(0).pairs() == [] and b.result(0).matched_depth == 3


def test_dataset_file_round_trip(tmp_path):
    from paper_2602_04936_b200 import storage

    ds = generate_dataset(321, 7, 5, seed=3)
    path = tmp_path / "d.lcpd"
    storage.write_dataset(str(path), ds)
    back = storage.read_dataset(str(path))
    assert np.array_equal(back.items, ds.items) and back.alphabet.size == 5
    path.write_bytes(b"NOPE" + path.read_bytes()[4:])
    with pytest.raises(InvalidInputError):
        storage.read_dataset(str(path))


def test_row_block_generator_matches_full_dataset():
    """datagen.generate_row_block == slices of generate_dataset (config-5 shards)."""
    from paper_2602_04936_b200.datagen import generate_dataset, generate_row_block

    for n, L, sigma, seed in ((1000, 32, 4, 6), (777, 16, 2, 3), (512, 8, 256, 1), (300, 24, 65536, 9)):
        full = generate_dataset(n, L, sigma, seed=seed).items
        step = 16 // np.gcd(16, L)
        for lo in range(0, n, max(step, n // 7 // step * step)):
            hi = min(n, lo + 123)
            assert np.array_equal(generate_row_block(n, L, sigma, seed, lo, hi), full[lo:hi]), (n, L, lo)


def test_pack_keys_host_matches_encoding_and_roundtrips():
    """rangeshard.pack_keys_host (the splitters / shard boundaries routing reads
    on the device) uses the extension's key encoding: ordering of packed keys
    equals the lexicographic order of the rows, and unpack inverts it."""
    from paper_2602_04936_b200.rangeshard import pack_keys_host, unpack_keys_host

    rng = np.random.default_rng(5)
    for L, sigma in ((32, 4), (24, 4), (16, 2), (20, 65536), (7, 256), (100, 3), (1, 2)):
        rows = rng.integers(0, sigma, size=(300, L)).astype(np.uint16)
        keys = pack_keys_host(rows, L, sigma)
        assert np.array_equal(unpack_keys_host(keys, L, sigma), rows)
        order_rows = np.lexsort(rows.T[::-1])
        order_keys = np.lexsort(keys.T[::-1])
        assert np.array_equal(rows[order_rows], rows[order_keys])


def test_bench_arms_share_one_config():
    """bench.py: the reference arm and the repo arm name the same workload
    (one bench_config function), so the driver's ratio compares like with like."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    assert mod.bench_config(1) == mod.bench_config(1)
    src = open(os.path.join(ROOT, "bench.py")).read()
    assert src.count('"config": bench_config(') == 2
