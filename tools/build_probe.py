"""Index build time at config 3 (N=2M, L=32, sigma=4): first build and steady state."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2602_04936_b200 as lg

ds = lg.generate_dataset(2_000_000, 32, 4, seed=3)
for i in range(10):
    torch.cuda.synchronize()
    t = time.perf_counter()
    idx = lg.build(ds)
    torch.cuda.synchronize()
    print(f"build {i}: {1e3 * (time.perf_counter() - t):.1f} ms (host rows, incl. H2D of {ds.items.nbytes / 1e6:.0f} MB)")
    del idx
dev_rows = torch.from_numpy(ds.items.copy()).cuda()
from paper_2602_04936_b200.engine import NativeIndex

for i in range(10):
    torch.cuda.synchronize()
    t = time.perf_counter()
    ni = NativeIndex.from_device(dev_rows.data_ptr(), ds.n, 32, 4)
    torch.cuda.synchronize()
    print(f"device-rows build {i}: {1e3 * (time.perf_counter() - t):.1f} ms")
    del ni
# replicas kept alive (as bench.py does): pool growth instead of reuse
kept = []
for i in range(8):
    torch.cuda.synchronize()
    t = time.perf_counter()
    kept.append(lg.build(ds))
    torch.cuda.synchronize()
    print(f"kept build {i}: {1e3 * (time.perf_counter() - t):.1f} ms")
