"""Throughput of the W > 1 paths at 2M: TAL (k_query_tal), full scan (k_fullscan), complete (k_query_warp)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2602_04936_b200 as lg


def timed(fn, n=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return 1e3 * a.elapsed_time(b) / n


B = 4096
for sigma in (256, 65536):
    ds = lg.generate_dataset(2_000_000, 32, sigma, seed=3)
    eng = lg.build_tal(ds, 256)
    dq = torch.from_numpy(lg.generate_queries(ds, B, seed=4)).cuda()
    ids = torch.empty((B, 10), dtype=torch.int32, device="cuda")
    lcps = torch.empty((B, 10), dtype=torch.int16, device="cuda")
    hits = torch.empty(B, dtype=torch.int32, device="cuda")
    nat = eng.native
    t_tal = timed(lambda: nat.query_device(dq, 10, "tal", ids, lcps, hits, stream=0))
    t_cmp = timed(lambda: nat.query_device(dq, 10, "complete", ids, lcps, hits, stream=0))
    t_fs = timed(lambda: nat.fullscan_device(dq, 10, ids, lcps, hits, stream=0), n=3)
    print(f"sigma={sigma} W={nat.words}: TAL B=256 (depth {eng.bucket_depth}) {t_tal:.1f} us, "
          f"complete {t_cmp:.1f} us, full scan {t_fs:.1f} us per 4096 batch")
