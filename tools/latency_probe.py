"""One batch in flight: round-trip latency of query_batch_async(...).result()
vs batch size, and the single-query TrieIndex.query loop (config 2), for the
copy path and the direct host-I/O path (LCP_DIRECT_IO_MAX=0 forces copies)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2602_04936_b200 as lg  # noqa: E402
from paper_2602_04936_b200._native import PinnedArray  # noqa: E402

print("LCP_DIRECT_IO_MAX =", os.environ.get("LCP_DIRECT_IO_MAX", "(default)"), flush=True)
ds = lg.generate_dataset(2_000_000, 32, 4, seed=3)
idx = lg.build(ds)
for count in (1, 4, 16, 64, 256, 1024, 4096):
    qs = lg.generate_queries(ds, count * 8, seed=4)
    pin = PinnedArray((8, count, 32), np.uint16)
    pin.array[:] = qs.reshape(8, count, 32)
    row = []
    for work in (False, True):
        out = idx.native.alloc_batch(count, 10, "complete", pinned=True, with_work=work)
        ref = idx.query_batch(qs[:count], 10, "complete")
        r = idx.query_batch_async(pin.array[0], 10, "complete", out=out).result()
        assert np.array_equal(r.ids, ref.ids) and np.array_equal(r.lcps, ref.lcps) and np.array_equal(r.hits, ref.hits)
        if work:
            assert np.array_equal(r.aux, ref.aux) and np.array_equal(r.matched_depth, ref.matched_depth)
        for i in range(100):
            idx.query_batch_async(pin.array[i % 8], 10, "complete", out=out).result()
        ts = []
        for i in range(2000):
            a = time.perf_counter()
            idx.query_batch_async(pin.array[i % 8], 10, "complete", out=out).result()
            ts.append(time.perf_counter() - a)
        row.append(f"{'work' if work else 'lean'} p50 {1e6 * np.median(ts):6.1f} us")
    print(f"count {count:5d}: " + ", ".join(row), flush=True)
# config 2: N=100k, L=24, k=5, prefix_len=12 readings, single-query loop
ds2 = lg.generate_dataset(100_000, 24, 4, seed=7)
idx2 = lg.build(ds2)
qs2 = lg.generate_queries(ds2, 4096, seed=8, prefix_len=12)
for i in range(200):
    idx2.query(qs2[i], 5, "complete")
ts = []
t0 = time.perf_counter()
for i in range(4096):
    a = time.perf_counter()
    idx2.query(qs2[i], 5, "complete")
    ts.append(time.perf_counter() - a)
el = time.perf_counter() - t0
print(f"config 2 TrieIndex.query: {4096 / el / 1e3:.1f} K Hz, p50 {1e6 * np.median(ts):.1f} us, "
      f"p99 {1e6 * np.percentile(ts, 99):.1f} us", flush=True)
