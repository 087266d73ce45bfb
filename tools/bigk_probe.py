"""Config-3 throughput for k beyond the warp path (k > 32 -> k_query_general)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2602_04936_b200 as lg

ds = lg.generate_dataset(2_000_000, 32, 4, seed=3)
idx = lg.build(ds)
B = 4096
dq = torch.from_numpy(lg.generate_queries(ds, B, seed=4)).cuda()
for k in (10, 32, 33, 64, 100, 1000):
    ids = torch.empty((B, k), dtype=torch.int32, device="cuda")
    lcps = torch.empty((B, k), dtype=torch.int16, device="cuda")
    hits = torch.empty(B, dtype=torch.int32, device="cuda")
    for _ in range(3):
        idx.native.query_device(dq, k, "complete", ids, lcps, hits, stream=0)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    a.record()
    for _ in range(n):
        idx.native.query_device(dq, k, "complete", ids, lcps, hits, stream=0)
    b.record()
    torch.cuda.synchronize()
    us = 1e3 * a.elapsed_time(b) / n
    print(f"k={k}: {us:.1f} us/batch -> {B / us:.1f} M q/s")
