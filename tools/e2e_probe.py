"""Where does the end-to-end batch time go?  PCIe copy floor, submission
cost of query_batch_async, and the pipelined loop at several depths."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2602_04936_b200 as lg
from paper_2602_04936_b200 import _native
from paper_2602_04936_b200._native import PinnedArray

B, L, K = 4096, 32, 10
ds = lg.generate_dataset(2_000_000, L, 4, seed=3)
idx = lg.build(ds)
qs = lg.generate_queries(ds, B * 8, seed=4)
pin = PinnedArray((8, B, L), np.uint16)
pin.array[:] = qs.reshape(8, B, L)

# PCIe floor: H2D 256 KB + D2H 270 KB on two streams, pinned
dev = torch.device("cuda")
hq = torch.from_numpy(pin.array.reshape(-1)).view(torch.int16)[: B * L]
hq = torch.empty(B * L, dtype=torch.int16).pin_memory()
ho = torch.empty(B * 66 // 2, dtype=torch.int16).pin_memory()
dq = torch.empty_like(hq, device=dev)
do = torch.empty_like(ho, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, both in (("h2d only", 0), ("d2h only", 1), ("h2d+d2h concurrent", 2)):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = 2000
    for i in range(n):
        if both in (0, 2):
            with torch.cuda.stream(s1):
                dq.copy_(hq, non_blocking=True)
        if both in (1, 2):
            with torch.cuda.stream(s2):
                ho.copy_(do, non_blocking=True)
    torch.cuda.synchronize()
    print(f"{name}: {1e6 * (time.perf_counter() - t0) / n:.2f} us/step")

for depth in (1, 2, 4, 8, 16):
    _native.ASYNC_DEPTH = depth
    _native._tls.__dict__.pop("ring", None)
    outs = [idx.native.alloc_batch(B, K, "complete", pinned=True, with_work=False) for _ in range(depth)]
    for i in range(50):
        idx.query_batch_async(pin.array[i % 8], K, "complete", out=outs[i % depth]).result()
    pending, sub, wait = [], 0.0, 0.0
    steps = 3000
    t0 = time.perf_counter()
    for i in range(steps):
        if len(pending) == depth:
            a = time.perf_counter()
            pending.pop(0).result()
            wait += time.perf_counter() - a
        a = time.perf_counter()
        pending.append(idx.query_batch_async(pin.array[i % 8], K, "complete", out=outs[i % depth]))
        sub += time.perf_counter() - a
    for p in pending:
        p.result()
    el = time.perf_counter() - t0
    print(f"depth {depth}: {1e6 * el / steps:.2f} us/batch  submit {1e6 * sub / steps:.2f}  "
          f"wait {1e6 * wait / steps:.2f}  -> {B * steps / el / 1e6:.1f} M q/s")
