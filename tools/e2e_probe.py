"""Where does an e2e step go: host submit overhead vs PCIe vs kernel."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2602_04936_b200 as lg
from paper_2602_04936_b200._native import PinnedArray

ds = lg.generate_dataset(2_000_000, 32, 4, seed=3)
idx = lg.build(ds)
qs = lg.generate_queries(ds, 4096, seed=4)
pin = PinnedArray((4096, 32), np.uint16)
pin.array[:] = qs
outs = [idx.native.alloc_batch(4096, 10, "complete", pinned=True) for _ in range(3)]
small = [idx.native.alloc_batch(1, 10, "complete", pinned=True) for _ in range(3)]
for i in range(50):
    idx.query_batch_async(pin.array, 10, "complete", out=outs[i % 3]).result()
# host overhead: 1-query batches (device work ~ nothing)
t0 = time.perf_counter()
for i in range(2000):
    idx.query_batch_async(pin.array[:1], 10, "complete", out=small[i % 3]).result()
print(f"submit+wait, 1 query: {1e6 * (time.perf_counter() - t0) / 2000:.2f} us")
pend = []
t0 = time.perf_counter()
for i in range(2000):
    if len(pend) == 3:
        pend.pop(0).result()
    pend.append(idx.query_batch_async(pin.array[:1], 10, "complete", out=small[i % 3]))
for p in pend:
    p.result()
print(f"pipelined 1-query batches: {1e6 * (time.perf_counter() - t0) / 2000:.2f} us/step")
# PCIe alone
dev_in = torch.empty((4096, 32), dtype=torch.int16, device="cuda")
dev_out = torch.empty(outs[0]._owners[0].array.nbytes, dtype=torch.uint8, device="cuda")
host_in = torch.from_numpy(pin.array.view(np.int16))
host_out = torch.from_numpy(outs[0]._owners[0].array)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
for name, fn in [("H2D 256KB", lambda: dev_in.copy_(host_in, non_blocking=True)),
                 ("D2H 336KB", lambda: host_out.copy_(dev_out, non_blocking=True))]:
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(200):
        fn()
    b.record()
    torch.cuda.synchronize()
    print(f"{name}: {1e3 * a.elapsed_time(b) / 200:.2f} us each")
