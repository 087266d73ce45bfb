"""Generate the golden vectors from the Python reference itself.

Run in a container that has /root/reference (read-only):

    python tests/golden/make_golden.py

It imports the reference package ``lcpsearch`` from /root/reference/pkg/src,
builds every case below with the reference's own generator, index, TAL
engine and exhaustive oracle, and writes ``golden_v1.npz`` + ``cases.json``.
The GPU box has no /root/reference, so the tests consume only these files.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

# (name, n, L, sigma, seed, distribution, uniform queries, prefix queries, ks, tal buckets)
CASES = [
    # BASELINE config 1 (quickstart.py:12): N=10k, L=16, sigma=4, seed 42, k=10
    ("cfg1", 10_000, 16, 4, 42, "uniform", 500, 500, (10,), (256,)),
    # reference randomized trie test shape (test_trie.py:252-259)
    ("trie500", 500, 12, 3, 0, "uniform", 60, 60, (1, 5, 50), (1, 9)),
    # acceptance C1 grid corners (test_acceptance.py:43-75)
    ("bin64", 2000, 64, 2, 1000, "uniform", 45, 45, (1, 5, 50), (1, 16, 256)),
    ("s4L16", 1000, 16, 4, 1001, "uniform", 60, 60, (1, 5, 50), (4, 256)),
    ("s256L256", 300, 256, 256, 1002, "uniform", 20, 20, (1, 5, 50), (1, 256)),
    ("s16L4n10", 10, 4, 16, 1003, "uniform", 30, 30, (1, 5, 50), (16,)),
    ("empty", 0, 1, 2, 1004, "uniform", 12, 0, (1, 5, 50), (1, 2)),
    ("single", 1, 1, 256, 1005, "uniform", 12, 12, (1, 5, 50), (1, 256)),
    ("s16L256n10", 10, 256, 16, 1006, "uniform", 20, 20, (1, 5, 50), (1,)),
    ("s4L4", 1000, 4, 4, 1007, "uniform", 60, 60, (1, 5, 50), (16, 256)),
    # wide alphabets and skew
    ("s65536", 500, 8, 65536, 11, "uniform", 40, 40, (1, 10, 33), (1, 65536)),
    ("clustered", 3000, 24, 4, 12, "clustered", 60, 60, (1, 10, 32), (64,)),
    ("clusteredL8", 2000, 8, 2, 13, "clustered", 60, 60, (1, 10, 40), (4, 256)),
    ("s5", 800, 10, 5, 14, "uniform", 40, 40, (1, 7, 31), (5, 125)),
    ("dups", 400, 6, 2, 15, "uniform", 40, 40, (3, 17, 64), (2, 32)),
    # GNC shape (config 2) scaled down: L=24, k=5
    ("gnc", 5000, 24, 4, 4, "uniform", 0, 100, (5,), (256,)),
]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main() -> int:
    sys.path.insert(0, REF_SRC)
    import lcpsearch as ref  # noqa: E402
    import lcpsearch.storage  # noqa: E402,F401  (ref.storage)

    arrays: dict[str, np.ndarray] = {}
    manifest = []
    for name, n, L, sigma, seed, dist, nu, npre, ks, buckets in CASES:
        ds = ref.generate_dataset(n, L, sigma, seed=seed, distribution=dist)
        parts = [ref.generate_queries(ds, nu, seed=seed + 7)]
        if npre and n > 0:
            parts.append(ref.generate_queries(ds, npre, seed=seed + 8, prefix_len=L // 2))
        qs = np.vstack(parts) if len(parts) > 1 else parts[0]
        count = qs.shape[0]
        kq = np.array([ks[i % len(ks)] for i in range(count)], dtype=np.int64)
        kmax = max(1, min(int(kq.max()) if count else 1, max(n, 1)))
        pre = f"{name}/"
        arrays[pre + "queries"] = qs
        arrays[pre + "k"] = kq

        index = ref.build(ds)
        arrays[pre + "order"] = index.order.astype(np.int32)
        arrays[pre + "level_offset"] = index.level_offset.astype(np.int64)
        arrays[pre + "adjacent_lcp"] = ref.core.adjacent_lcp(ds.items[index.order]).astype(np.int64)
        entry = {
            "name": name, "n": n, "length": L, "sigma": sigma, "seed": seed,
            "distribution": dist, "queries": count, "ks": list(ks), "tal_buckets": list(buckets),
            "dataset_sha256": sha(ds.items),
            "row_lo_sha256": sha(index.row_lo.astype(np.int32)),
            "edge_symbol_sha256": sha(index.edge_symbol.astype(np.uint16)),
            "node_count": index.node_count,
        }
        snap = ref.storage.index_snapshot_bytes(index)
        entry["snapshot_sha256"] = hashlib.sha256(snap).hexdigest()
        entry["snapshot_size"] = len(snap)
        if len(snap) <= 64 * 1024:  # small reference snapshots for the loader tests
            with open(os.path.join(HERE, f"snap_{name}.lcpi"), "wb") as fh:
                fh.write(snap)
        for mode in ("strict", "complete"):
            ids = np.full((count, kmax), -1, dtype=np.int64)
            lcps = np.full((count, kmax), -1, dtype=np.int64)
            hits = np.zeros(count, dtype=np.int64)
            md = np.zeros(count, dtype=np.int64)
            sym = np.zeros(count, dtype=np.int64)
            nodes = np.zeros(count, dtype=np.int64)
            digest = hashlib.sha256()
            for i, q in enumerate(qs):
                w = index.new_work_report()
                r = index.query(q, int(kq[i]), mode, work=w)
                h = len(r.indices)
                ids[i, :h] = r.indices
                lcps[i, :h] = r.lcps
                hits[i], md[i] = h, r.matched_depth
                sym[i], nodes[i] = w.symbols_compared, w.nodes_visited
                digest.update(r.to_bytes())
            for key, val in (("ids", ids), ("lcps", lcps), ("hits", hits), ("md", md),
                             ("sym", sym), ("nodes", nodes)):
                arrays[f"{pre}{mode}/{key}"] = val
            entry[f"{mode}_bytes_sha256"] = digest.hexdigest()
        # exhaustive oracle
        ids = np.full((count, kmax), -1, dtype=np.int64)
        lcps = np.full((count, kmax), -1, dtype=np.int64)
        hits = np.zeros(count, dtype=np.int64)
        digest = hashlib.sha256()
        for i, q in enumerate(qs):
            r = ref.oracle_top_k(ds, q, int(kq[i]))
            h = len(r.indices)
            ids[i, :h], lcps[i, :h], hits[i] = r.indices, r.lcps, h
            digest.update(r.to_bytes())
        arrays[pre + "oracle/ids"], arrays[pre + "oracle/lcps"], arrays[pre + "oracle/hits"] = ids, lcps, hits
        entry["oracle_bytes_sha256"] = digest.hexdigest()
        # TAL engines
        tal_meta = []
        for B in buckets:
            if B > sigma**L:
                continue
            eng = ref.build_tal(ds, B)
            tp = f"{pre}tal{B}/"
            ids = np.full((count, kmax), -1, dtype=np.int64)
            lcps = np.full((count, kmax), -1, dtype=np.int64)
            hits = np.zeros(count, dtype=np.int64)
            items = np.zeros(count, dtype=np.int64)
            sym = np.zeros(count, dtype=np.int64)
            lo = np.zeros(count, dtype=np.int64)
            hi = np.zeros(count, dtype=np.int64)
            digest = hashlib.sha256()
            for i, q in enumerate(qs):
                r, rep = eng.query(q, int(kq[i]))
                h = len(r.indices)
                ids[i, :h], lcps[i, :h], hits[i] = r.indices, r.lcps, h
                items[i], sym[i] = rep.items_scanned, rep.symbols_compared
                lo[i], hi[i] = eng.bucket_range(q)
                digest.update(r.to_bytes())
            for key, val in (("ids", ids), ("lcps", lcps), ("hits", hits), ("items", items),
                             ("sym", sym), ("lo", lo), ("hi", hi)):
                arrays[tp + key] = val
            if eng.directory is not None and eng.directory.size <= 1 << 17:
                arrays[tp + "directory"] = eng.directory.astype(np.int64)
            tal_meta.append({"B": B, "depth": eng.bucket_depth, "bucket_count": eng.bucket_count,
                             "has_directory": eng.directory is not None,
                             "bytes_sha256": digest.hexdigest()})
        entry["tal"] = tal_meta
        manifest.append(entry)

    # datagen pins: hashes of generated datasets / query batches
    gen = []
    for args, kw in [((1000, 16, 4, 42), {}), ((2000, 24, 4, 4), {}), ((3000, 24, 4, 12), {"distribution": "clustered"}),
                     ((400, 9, 4, 12), {"distinct": True}), ((64, 3, 4, 5), {"distinct": True}),
                     ((300, 40, 2, 8), {"distinct": True}), ((100_000, 24, 4, 4), {}),
                     ((2_000_000, 32, 4, 3), {})]:
        ds = ref.generate_dataset(*args, **kw)
        q1 = ref.generate_queries(ds, 257, seed=args[3] + 1)
        q2 = ref.generate_queries(ds, 129, seed=args[3] + 2, prefix_len=args[1] // 2)
        gen.append({"args": list(args), "kwargs": kw, "dataset_sha256": sha(ds.items),
                    "queries_sha256": sha(q1), "prefix_queries_sha256": sha(q2)})

    hand = {
        # test_trie.py:220-230, test_oracle.py:10-35, test_core.py:127-134
        "complete_3item": ref.build(ref.Dataset.from_rows([[0, 0], [0, 1], [1, 0]], 2)).query([0, 0], 3, "complete").pairs(),
        "strict_3item": ref.build(ref.Dataset.from_rows([[0, 0], [0, 1], [1, 0]], 2)).query([0, 0], 3, "strict").pairs(),
        "oracle_hand": ref.oracle_top_k(ref.Dataset.from_rows([[0, 0], [0, 1], [1, 1]], 2), [0, 1], 2).pairs(),
        "oracle_k_ge_n": ref.oracle_top_k(ref.Dataset.from_rows([[0, 0], [1, 1], [0, 1]], 2), [0, 0], 10).pairs(),
        "oracle_dups": ref.oracle_top_k(ref.Dataset.from_rows([[3, 3], [3, 3], [3, 3]], 4), [3, 3], 2).pairs(),
        "order_1203": ref.core.lexicographic_order(np.array([[1, 2], [0, 1], [0, 2], [1, 3]], dtype=np.uint16)).tolist(),
        "adjacent_210": ref.core.adjacent_lcp(np.array([[0, 0, 0], [0, 0, 1], [0, 1, 1], [1, 1, 1]], dtype=np.uint16)).tolist(),
        "result_bytes": ref.build(ref.Dataset.from_rows([[0, 0], [0, 1], [1, 0]], 2)).query([0, 0], 3, "complete").to_bytes().hex(),
    }
    np.savez_compressed(os.path.join(HERE, "golden_v1.npz"), **arrays)
    with open(os.path.join(HERE, "cases.json"), "w") as f:
        json.dump({"cases": manifest, "datagen": gen, "hand": hand,
                   "generator": "tests/golden/make_golden.py", "reference": REF_SRC}, f, indent=1)
    print(f"wrote {len(manifest)} cases, {len(arrays)} arrays")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
