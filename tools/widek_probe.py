"""W > 1 paths across k at N=2M (sigma 256: W=4, sigma 65536: W=8): complete and TAL B=256."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2602_04936_b200 as lg

B = 4096
for sigma in (256, 65536):
    ds = lg.generate_dataset(2_000_000, 32, sigma, seed=3)
    eng = lg.build_tal(ds, 256)
    dq = torch.from_numpy(lg.generate_queries(ds, B, seed=4)).cuda()
    for mode in ("complete", "tal"):
        for k in (10, 32, 33, 64, 100):
            ids = torch.empty((B, k), dtype=torch.int32, device="cuda")
            lcps = torch.empty((B, k), dtype=torch.int16, device="cuda")
            hits = torch.empty(B, dtype=torch.int32, device="cuda")
            eng.native.query_device(dq, k, mode, ids, lcps, hits, stream=0)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(5):
                eng.native.query_device(dq, k, mode, ids, lcps, hits, stream=0)
            b.record()
            torch.cuda.synchronize()
            us = 1e3 * a.elapsed_time(b) / 5
            print(f"sigma={sigma} W={eng.native.words} {mode} k={k}: {us:.1f} us/batch", flush=True)
