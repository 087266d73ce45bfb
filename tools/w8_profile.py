"""W > 1 batch query, for ncu and A/B: N=2M, L=32, k=10, 4096 queries,
sigma from argv (default 65536, W = 8; 256: W = 4; 16: W = 2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2602_04936_b200 as lg  # noqa: E402

sigma = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
d8 = lg.generate_dataset(2_000_000, 32, sigma, seed=3)
i8 = lg.build(d8)
q8 = torch.from_numpy(lg.generate_queries(d8, 4096, seed=4, prefix_len=2)).cuda()
ids = torch.empty((4096, 10), dtype=torch.int32, device="cuda")
lcps = torch.empty((4096, 10), dtype=torch.int16, device="cuda")
hits = torch.empty(4096, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for _ in range(4):
    i8.native.query_device(q8, 10, "complete", ids, lcps, hits, stream=st)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50):
    i8.native.query_device(q8, 10, "complete", ids, lcps, hits, stream=st)
b.record()
torch.cuda.synchronize()
print(f"sigma={sigma}: {a.elapsed_time(b) * 1e3 / 50:.2f} us per batch (back-to-back)")
