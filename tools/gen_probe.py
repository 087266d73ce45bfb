"""One config-3 batch through k_query_general at a given k (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2602_04936_b200 as lg

k = int(sys.argv[1])
mode = sys.argv[2] if len(sys.argv) > 2 else "complete"
ds = lg.generate_dataset(2_000_000, 32, 4, seed=3)
idx = lg.build(ds)
B = 4096
dq = torch.from_numpy(lg.generate_queries(ds, B, seed=4)).cuda()
ids = torch.empty((B, k), dtype=torch.int32, device="cuda")
lcps = torch.empty((B, k), dtype=torch.int16, device="cuda")
hits = torch.empty(B, dtype=torch.int32, device="cuda")
for _ in range(2):
    idx.native.query_device(dq, k, mode, ids, lcps, hits, stream=0)
torch.cuda.synchronize()
print("ok", k, mode)
