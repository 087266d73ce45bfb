"""Synchronous query_batch latency: default (fresh pageable outputs) vs a pinned out block."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2602_04936_b200 as lg

ds = lg.generate_dataset(2_000_000, 32, 4, seed=3)
idx = lg.build(ds)
qs = [lg.generate_queries(ds, 4096, seed=s) for s in range(4)]
out = idx.native.alloc_batch(4096, 10, "complete", pinned=True)
for name, kw in (("default (no out)", {}), ("pinned out", {"out": out})):
    for i in range(20):
        idx.query_batch(qs[i % 4], 10, "complete", **kw)
    t = []
    for i in range(300):
        t0 = time.perf_counter()
        idx.query_batch(qs[i % 4], 10, "complete", **kw)
        t.append(time.perf_counter() - t0)
    print(f"{name}: p50 {1e6 * np.median(t):.1f} us per 4096-query batch -> {4096 / np.median(t) / 1e6:.1f} M q/s")
