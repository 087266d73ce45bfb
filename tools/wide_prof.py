import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_04936_b200 as lg
ds = lg.generate_dataset(2_000_000, 32, 65536, seed=3)
idx = lg.build(ds)
dq = torch.from_numpy(lg.generate_queries(ds, 4096, seed=4)).cuda()
ids = torch.empty((4096, 10), dtype=torch.int32, device="cuda")
lcps = torch.empty((4096, 10), dtype=torch.int16, device="cuda")
hits = torch.empty(4096, dtype=torch.int32, device="cuda")
for _ in range(4):
    idx.native.query_device(dq, 10, "complete", ids, lcps, hits, stream=0)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    idx.native.query_device(dq, 10, "complete", ids, lcps, hits, stream=0)
b.record(); torch.cuda.synchronize()
print("us/launch", 1e3 * a.elapsed_time(b) / 20)
