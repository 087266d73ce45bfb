"""One L=256, sigma=256 (W=32) batch at N=1M through k_query_general (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2602_04936_b200 as lg

ds = lg.generate_dataset(1_000_000, 256, 256, seed=3)
idx = lg.build(ds)
B, k = 4096, 10
dq = torch.from_numpy(lg.generate_queries(ds, B, seed=4)).cuda()
ids = torch.empty((B, k), dtype=torch.int32, device="cuda")
lcps = torch.empty((B, k), dtype=torch.int16, device="cuda")
hits = torch.empty(B, dtype=torch.int32, device="cuda")
for _ in range(3):
    idx.native.query_device(dq, k, "complete", ids, lcps, hits, stream=0)
torch.cuda.synchronize()
print("ok")
