"""Subprocess driver for the cross-process determinism test (test
infrastructure; modelled on the reference's pkg/tests/determinism_driver.py:21-38).

    determinism_gpu_driver.py N L SIGMA SEED REPS

Builds the GPU index from generate_dataset(N, L, SIGMA, SEED), then REPS
times runs every query path on the same batches (strict / complete at the
warp-rank, warp-list and CTA-per-query k, TAL B=256, the full scan at a
register-list and a CTA k) and prints one SHA-256 per repetition over the
concatenated canonical result bytes (QueryResult.to_bytes / OracleResult
bytes, trie.py:51-87, oracle.py:19-36) and the work counters.
"""

import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2602_04936_b200 as lg  # noqa: E402


def main() -> int:
    n, length, sigma, seed, reps = (int(x) for x in sys.argv[1:6])
    ds = lg.generate_dataset(n, length, sigma, seed=seed)
    qs = np.vstack([lg.generate_queries(ds, 600, seed=seed + 1),
                    lg.generate_queries(ds, 600, seed=seed + 2, prefix_len=length // 2)])
    index = lg.build(ds)
    tal = lg.build_tal(ds, 256)
    for _ in range(reps):
        acc = hashlib.sha256()
        for k in (9, 40, 300):
            for mode in ("strict", "complete"):
                b = index.query_batch(qs, k, mode)
                for i in range(len(qs)):
                    acc.update(b.result(i).to_bytes())
                acc.update(np.ascontiguousarray(b.aux).tobytes())
            t = tal.query_batch(qs, k)
            for i in range(len(qs)):
                acc.update(t.result(i).to_bytes())
            acc.update(np.ascontiguousarray(t.aux).tobytes())
        for k in (10, 200):
            f = index.fullscan_batch(qs, k)
            for i in range(len(qs)):
                acc.update(f.fullscan_result(i).to_bytes())
        print(acc.hexdigest(), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
