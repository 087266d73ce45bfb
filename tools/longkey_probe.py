"""Long keys (W > 8 -> k_query_general even at k = 10): per-batch time at N = 1M."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2602_04936_b200 as lg

B = 4096
for L, sigma in ((256, 4), (512, 4), (1024, 4), (256, 256)):
    ds = lg.generate_dataset(1_000_000, L, sigma, seed=3)
    idx = lg.build(ds)
    dq = torch.from_numpy(lg.generate_queries(ds, B, seed=4)).cuda()
    for k in (10, 64):
        ids = torch.empty((B, k), dtype=torch.int32, device="cuda")
        lcps = torch.empty((B, k), dtype=torch.int16, device="cuda")
        hits = torch.empty(B, dtype=torch.int32, device="cuda")
        idx.native.query_device(dq, k, "complete", ids, lcps, hits, stream=0)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            idx.native.query_device(dq, k, "complete", ids, lcps, hits, stream=0)
        b.record()
        torch.cuda.synchronize()
        print(f"L={L} sigma={sigma} W={idx.native.words} k={k}: {1e3 * a.elapsed_time(b) / 5:.1f} us/batch", flush=True)
    del idx, ds
