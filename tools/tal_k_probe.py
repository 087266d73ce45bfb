"""TAL (B=256) per-batch time across k at config 3 (warp kernel k <= 32, general path beyond)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2602_04936_b200 as lg

ds = lg.generate_dataset(2_000_000, 32, 4, seed=3)
eng = lg.build_tal(ds, 256)
B = 4096
dq = torch.from_numpy(lg.generate_queries(ds, B, seed=4)).cuda()
for k in (10, 16, 17, 24, 32, 33, 64, 100, 1000):
    ids = torch.empty((B, k), dtype=torch.int32, device="cuda")
    lcps = torch.empty((B, k), dtype=torch.int16, device="cuda")
    hits = torch.empty(B, dtype=torch.int32, device="cuda")
    eng.native.query_device(dq, k, "tal", ids, lcps, hits, stream=0)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        eng.native.query_device(dq, k, "tal", ids, lcps, hits, stream=0)
    b.record()
    torch.cuda.synchronize()
    us = 1e3 * a.elapsed_time(b) / 5
    print(f"tal k={k}: {us:.1f} us/batch -> {B / us:.2f} M q/s", flush=True)
