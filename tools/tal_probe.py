"""TAL B=256 at config 3: event-timed device launches (one batch in flight)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2602_04936_b200 as lg

ds = lg.generate_dataset(2_000_000, 32, 4, seed=3)
eng = lg.build_tal(ds, 256)
B = 4096
dq = torch.from_numpy(lg.generate_queries(ds, B * 4, seed=4)).cuda().view(4, B, 32)
ids = torch.empty((B, 10), dtype=torch.int32, device="cuda")
lcps = torch.empty((B, 10), dtype=torch.int16, device="cuda")
hits = torch.empty(B, dtype=torch.int32, device="cuda")
native = eng.native if hasattr(eng, "native") else eng._native
for i in range(5):
    native.query_device(dq[i % 4], 10, "tal", ids, lcps, hits, stream=0)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
n = 50
for i in range(n):
    native.query_device(dq[i % 4], 10, "tal", ids, lcps, hits, stream=0)
b.record()
torch.cuda.synchronize()
us = 1e3 * a.elapsed_time(b) / n
print(f"TAL B=256: {us:.1f} us/batch -> {B / us:.1f} M q/s")
