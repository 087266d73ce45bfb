"""W = 1 with a large alphabet (sigma 65536, L = 4; sigma 256, L = 8) at N = 2M across k:
d* falls to 0 or 1 once k exceeds the depth-1 bucket size."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2602_04936_b200 as lg

B = 4096
for sigma, L in ((65536, 4), (256, 8)):
    ds = lg.generate_dataset(2_000_000, L, sigma, seed=3)
    idx = lg.build(ds)
    dq = torch.from_numpy(lg.generate_queries(ds, B, seed=4)).cuda()
    for k in (10, 32, 33, 64, 100, 129):
        ids = torch.empty((B, k), dtype=torch.int32, device="cuda")
        lcps = torch.empty((B, k), dtype=torch.int16, device="cuda")
        hits = torch.empty(B, dtype=torch.int32, device="cuda")
        idx.native.query_device(dq, k, "complete", ids, lcps, hits, stream=0)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        idx.native.query_device(dq, k, "complete", ids, lcps, hits, stream=0)
        b.record()
        torch.cuda.synchronize()
        print(f"sigma={sigma} L={L} W={idx.native.words} complete k={k}: {1e3 * a.elapsed_time(b):.1f} us/batch", flush=True)
