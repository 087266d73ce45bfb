"""Latency/throughput of the complete-mode query kernel vs batch size
(config 3 index, warm L2, back-to-back launches on one stream)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2602_04936_b200 as lg

ds = lg.generate_dataset(2_000_000, 32, 4, seed=3)
idx = lg.build(ds)
qs = lg.generate_queries(ds, 65536, seed=4)
dq_all = torch.from_numpy(qs).cuda()
st = torch.cuda.current_stream().cuda_stream
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for batch in (1, 32, 148, 512, 1024, 2048, 4096, 8192, 16384, 32768, 65536):
    dq = dq_all[:batch]
    ids = torch.empty((batch, 10), dtype=torch.int32, device="cuda")
    lcps = torch.empty((batch, 10), dtype=torch.int16, device="cuda")
    hits = torch.empty(batch, dtype=torch.int32, device="cuda")
    for _ in range(5):
        idx.native.query_device(dq, 10, "complete", ids, lcps, hits, stream=st)
    torch.cuda.synchronize()
    res = {}
    for mode in ("warm", "cold"):
        ts = []
        for _ in range(30):
            if mode == "cold":
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            idx.native.query_device(dq, 10, "complete", ids, lcps, hits, stream=st)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        res[mode] = float(np.median(ts))
    print(f"batch {batch:6d}: warm {res['warm']:8.2f} us  cold {res['cold']:8.2f} us   "
          f"warm {batch / res['warm']:8.1f} Mq/s  cold {batch / res['cold']:8.1f} Mq/s", flush=True)
