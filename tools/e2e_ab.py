"""A/B of the pipelined e2e loop (bench.py's e2e leg) for a few depths."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2602_04936_b200 as lg
from paper_2602_04936_b200 import _native
from paper_2602_04936_b200._native import PinnedArray

ds = lg.generate_dataset(2_000_000, 32, 4, seed=3)
idx = lg.build(ds)
qs = lg.generate_queries(ds, 4096 * 8, seed=4)
pin = PinnedArray((8, 4096, 32), np.uint16)
pin.array[:] = qs.reshape(8, 4096, 32)
for depth in (2, 3, 4, 6):
    _native.ASYNC_DEPTH = depth
    _native._tls.__dict__.pop("ring", None)
    outs = [idx.native.alloc_batch(4096, 10, "complete", pinned=True) for _ in range(depth)]
    for i in range(50):
        idx.query_batch_async(pin.array[i % 8], 10, "complete", out=outs[i % depth]).result()
    pend = []
    t0 = time.perf_counter()
    steps = 2000
    for i in range(steps):
        if len(pend) == depth:
            pend.pop(0).result()
        pend.append(idx.query_batch_async(pin.array[i % 8], 10, "complete", out=outs[i % depth]))
    for p in pend:
        p.result()
    el = time.perf_counter() - t0
    print(f"{os.environ.get('LCP_NO_GRAPH_CACHE') and 'streams' or 'graphs '} depth {depth}: {1e6 * el / steps:.2f} us/step  {4096 * steps / el / 1e6:.1f} Mq/s")
