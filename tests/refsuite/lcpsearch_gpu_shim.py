"""Re-point the reference package's own tests at the GPU package.

Test infrastructure (SURVEY §4 "re-run the reference's own query-level tests
against the GPU index through a thin lcpsearch-compatible shim").  The
UNMODIFIED reference ``lcpsearch`` (installed into baseline/_ref by
tools/install_reference.sh) stays the checker: its ``oracle_top_k``,
``Dataset``, generators, ``lcp`` and storage formats are untouched.  Only the
engines under test are swapped for the sm_100a implementation:

  variant "engines" (default): trie.build / TrieIndex, tal.build_tal /
      TalEngine / tal_query, QueryCache / memoized_query, and the LCPI
      snapshot reader/writer (storage.py:155-389) -> paper_2602_04936_b200.
      oracle_top_k stays the reference's brute force, so every
      "complete == oracle" assertion compares GPU against the reference.
  variant "oracle": oracle.oracle_top_k -> the GPU full-scan kernel, so the
      reference's oracle tests (hand cases, ties, LCP cross-checks against
      the scalar core.lcp) exercise the streaming kernel.

Selected with the environment variable LCPSEARCH_GPU_SHIM; installed at
interpreter start by ``sitecustomize`` in this directory, so subprocesses the
reference tests spawn (determinism_driver.py) see the same swap.
"""

from __future__ import annotations

import os


def install(variant: str | None = None) -> str:
    variant = variant or os.environ.get("LCPSEARCH_GPU_SHIM", "engines")
    import lcpsearch
    import lcpsearch.oracle
    import lcpsearch.storage
    import lcpsearch.tal
    import lcpsearch.trie

    import paper_2602_04936_b200 as gpu
    from paper_2602_04936_b200 import storage as gpu_storage
    from paper_2602_04936_b200._native import load

    load()  # fail loudly (NativeLibraryMissing) rather than test the reference against itself

    if variant == "engines":
        swaps = {
            (lcpsearch, "build"): gpu.build,
            (lcpsearch.trie, "build"): gpu.build,
            (lcpsearch, "TrieIndex"): gpu.TrieIndex,
            (lcpsearch.trie, "TrieIndex"): gpu.TrieIndex,
            (lcpsearch, "build_tal"): gpu.build_tal,
            (lcpsearch.tal, "build_tal"): gpu.build_tal,
            (lcpsearch, "TalEngine"): gpu.TalEngine,
            (lcpsearch.tal, "TalEngine"): gpu.TalEngine,
            (lcpsearch, "tal_query"): gpu.tal_query,
            (lcpsearch.tal, "tal_query"): gpu.tal_query,
            (lcpsearch, "QueryCache"): gpu.QueryCache,
            (lcpsearch.trie, "QueryCache"): gpu.QueryCache,
            (lcpsearch, "memoized_query"): gpu.memoized_query,
            (lcpsearch.trie, "memoized_query"): gpu.memoized_query,
            (lcpsearch.storage, "index_snapshot_bytes"): gpu_storage.index_snapshot_bytes,
            (lcpsearch.storage, "index_from_snapshot_bytes"): gpu_storage.index_from_snapshot_bytes,
            (lcpsearch.storage, "write_index"): gpu_storage.write_index,
            (lcpsearch.storage, "read_index"): gpu_storage.read_index,
        }
    elif variant == "oracle":
        swaps = {
            (lcpsearch, "oracle_top_k"): gpu.oracle_top_k,
            (lcpsearch.oracle, "oracle_top_k"): gpu.oracle_top_k,
        }
    else:
        raise ValueError(f"unknown LCPSEARCH_GPU_SHIM variant {variant!r}")
    for (mod, name), obj in swaps.items():
        if not hasattr(mod, name):
            raise AttributeError(f"reference has no {mod.__name__}.{name} to re-point")
        setattr(mod, name, obj)
    # One exception taxonomy: the GPU package raises its own classes (same
    # names, bases and messages as core.py:29-42); alias the reference's names
    # to them in every lcpsearch module, so `pytest.raises(InvalidInputError)`
    # in a reference test matches whichever side raised.
    import sys

    from paper_2602_04936_b200 import core as gpu_core

    for exc in ("InvalidInputError", "InternalInvariantError", "InvalidStateError", "ConfigError"):
        ours = getattr(gpu_core, exc)
        for modname, mod in list(sys.modules.items()):
            if (modname == "lcpsearch" or modname.startswith("lcpsearch.")) and hasattr(mod, exc):
                setattr(mod, exc, ours)
    lcpsearch.GPU_SHIM_VARIANT = variant
    return variant
