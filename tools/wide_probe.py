"""sigma = 65536 (W = 8) at N = 2M: per-query |R(d*)|, d*, and kernel time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2602_04936_b200 as lg

ds = lg.generate_dataset(2_000_000, 32, 65536, seed=3)
idx = lg.build(ds)
for name, qs in [("uniform", lg.generate_queries(ds, 4096, seed=4)),
                 ("prefix2", lg.generate_queries(ds, 4096, seed=4, prefix_len=2))]:
    idx.query_batch(qs[:8], 10, "complete")
    t0 = time.perf_counter()
    b = idx.query_batch(qs, 10, "complete")
    el = time.perf_counter() - t0
    rs = (b.aux[:, 1] & np.uint64(0xFFFFFFFF)).astype(np.int64)
    dmax = (b.aux[:, 0] & np.uint64(0xFFFFFFFF)).astype(np.int64)
    dstar = (b.aux[:, 0] >> np.uint64(32)).astype(np.int64)
    print(f"{name}: {el*1e3:.2f} ms  |R| mean {rs.mean():.1f} max {rs.max()} p99 {np.percentile(rs,99):.0f}  "
          f"dmax mean {dmax.mean():.2f}  d* hist {np.bincount(dstar)[:6]}")
