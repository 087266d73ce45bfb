"""Latency mode (TrieIndex.low_latency): config 2 single-query loop through
the resident-warp server vs the launch path, results checked against the
batch API."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2602_04936_b200 as lg  # noqa: E402

ds = lg.generate_dataset(100_000, 24, 4, seed=4)
idx = lg.build(ds)
qs = lg.generate_queries(ds, 1000, seed=5, prefix_len=12)
ref = idx.query_batch(qs, 5, "complete")
for name, ctx in (("launch path", None), ("low_latency", lambda: idx.low_latency(5, "complete"))):
    def loop():
        ts = []
        for rep in range(3):
            for i in range(len(qs)):
                a = time.perf_counter()
                r = idx.query(qs[i], 5, "complete")
                ts.append(time.perf_counter() - a)
                if rep == 0:
                    assert r.pairs() == ref.pairs(i), (name, i)
        return ts
    if ctx is None:
        ts = loop()
    else:
        with ctx():
            ts = loop()
    ts = np.array(ts[200:])
    print(f"{name}: {1 / ts.mean() / 1e3:.1f} K Hz, p50 {1e6 * np.median(ts):.1f} us, p99 {1e6 * np.percentile(ts, 99):.1f} us",
          flush=True)
# an invalid symbol through the server, then a valid query
with idx.low_latency(5, "complete"):
    bad = qs[0].copy()
    bad[3] = 7
    try:
        idx.query(bad, 5, "complete")
        print("ERROR: invalid symbol not reported")
    except lg.InvalidInputError as e:
        print("invalid symbol reported:", e)
    assert idx.query(qs[1], 5, "complete").pairs() == ref.pairs(1)
    time.sleep(0.3)  # the warp idles out; the next query relaunches it
    assert idx.query(qs[2], 5, "complete").pairs() == ref.pairs(2)
print("ok")

# raw round trip: lcp_server_query on an unchanged row (ctypes only)
from paper_2602_04936_b200._native import load  # noqa: E402
from paper_2602_04936_b200.engine import SingleQueryServer  # noqa: E402

srv = SingleQueryServer(idx.native, 5, "complete")
srv.row.array[0] = qs[0]
lib = load()
fn = lib.lcp_server_query
h = srv._h
for _ in range(1000):
    fn(h)
t0 = time.perf_counter()
N = 20000
for _ in range(N):
    fn(h)
el = time.perf_counter() - t0
print(f"raw lcp_server_query: {1e6 * el / N:.2f} us per round trip")
t0 = time.perf_counter()
for i in range(N):
    srv.query(qs[i % len(qs)])
el = time.perf_counter() - t0
print(f"SingleQueryServer.query (row write + call): {1e6 * el / N:.2f} us")
t0 = time.perf_counter()
for i in range(N):
    srv.out.result(0)
el = time.perf_counter() - t0
print(f"BatchResult.result(0): {1e6 * el / N:.2f} us")
srv.close()
