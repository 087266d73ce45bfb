"""Config-3 throughput for large k: the warp paths (k <= 128) and k_query_general
(select-then-sort within GEN_CAP, radix rounds beyond), complete and strict."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2602_04936_b200 as lg

ds = lg.generate_dataset(2_000_000, 32, 4, seed=3)
idx = lg.build(ds)
B = 4096
dq = torch.from_numpy(lg.generate_queries(ds, B, seed=4)).cuda()
cases = [(k, "complete") for k in (10, 32, 33, 64, 100, 129, 256, 500, 1000, 2000, 5000)]
cases += [(k, "strict") for k in (256, 1000)]
if os.environ.get("BIGK_KS"):  # e.g. BIGK_KS=1,10,32 (complete and strict)
    ks = [int(x) for x in os.environ["BIGK_KS"].split(",")]
    cases = [(k, m) for m in ("complete", "strict") for k in ks]
for k, mode in cases:
    ids = torch.empty((B, k), dtype=torch.int32, device="cuda")
    lcps = torch.empty((B, k), dtype=torch.int16, device="cuda")
    hits = torch.empty(B, dtype=torch.int32, device="cuda")
    for _ in range(3):
        idx.native.query_device(dq, k, mode, ids, lcps, hits, stream=0)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    a.record()
    for _ in range(n):
        idx.native.query_device(dq, k, mode, ids, lcps, hits, stream=0)
    b.record()
    torch.cuda.synchronize()
    us = 1e3 * a.elapsed_time(b) / n
    print(f"{mode} k={k}: {us:.1f} us/batch -> {B / us:.2f} M q/s", flush=True)
# full scan with k beyond the warp merge (general kernel over the whole corpus)
for nq, k in [] if os.environ.get("BIGK_KS") else ((64, 10), (64, 64), (4096, 10), (4096, 32), (4096, 33), (4096, 64), (4096, 128), (64, 129)):
    fq = dq[:nq]
    ids = torch.empty((nq, k), dtype=torch.int32, device="cuda")
    lcps = torch.empty((nq, k), dtype=torch.int16, device="cuda")
    hits = torch.empty(nq, dtype=torch.int32, device="cuda")
    idx.native.fullscan_device(fq, k, ids, lcps, hits, stream=0)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    idx.native.fullscan_device(fq, k, ids, lcps, hits, stream=0)
    b.record()
    torch.cuda.synchronize()
    print(f"fullscan k={k}, {nq} queries: {1e3 * a.elapsed_time(b):.1f} us", flush=True)
