"""BASELINE config 5 on ONE B200: N = 200M sequences, L = 32, sigma = 4, k = 10.

The corpus (12.8 GB of u16 rows, reference generator) is built into one GPU
index; indexed complete-mode batches of 4096 are event-timed (one batch in
flight, graph-free loop), the full scan is timed on one batch, and indexed ==
full scan is checked on that batch.  Prints one JSON object.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2602_04936_b200 as lg

N = int(os.environ.get("CONFIG5_N", 200_000_000))
B, L, K = 4096, 32, 10
t = time.perf_counter()
ds = lg.generate_dataset(N, L, 4, seed=6)
t_gen = time.perf_counter() - t
t = time.perf_counter()
idx = lg.build(ds)
torch.cuda.synchronize()
t_build = time.perf_counter() - t
qs = lg.generate_queries(ds, B * 8, seed=7)
del ds
dq = torch.from_numpy(qs).cuda().view(8, B, L)
ids = torch.empty((B, K), dtype=torch.int32, device="cuda")
lcps = torch.empty((B, K), dtype=torch.int16, device="cuda")
hits = torch.empty(B, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream()
for i in range(20):
    idx.native.query_device(dq[i % 8], K, "complete", ids, lcps, hits, stream=st.cuda_stream)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 400
a.record(st)
for i in range(n):
    idx.native.query_device(dq[i % 8], K, "complete", ids, lcps, hits, stream=st.cuda_stream)
b.record(st)
torch.cuda.synchronize()
us = 1e3 * a.elapsed_time(b) / n
bi = idx.query_batch(qs[:B], K, "complete")
torch.cuda.synchronize()
t = time.perf_counter()
f = idx.fullscan_batch(qs[:B], K)
torch.cuda.synchronize()
t_fs = time.perf_counter() - t
same = bool(np.array_equal(bi.ids, f.ids) and np.array_equal(bi.lcps, f.lcps) and np.array_equal(bi.hits, f.hits))
print(json.dumps({
    "n": N, "generate_s": round(t_gen, 2), "build_s": round(t_build, 3), "device_bytes": idx.nbytes,
    "indexed_us_per_batch": round(us, 2), "indexed_qps": B / (us * 1e-6),
    "fullscan_s_per_batch": round(t_fs, 3), "fullscan_qps": B / t_fs,
    "indexed_equals_fullscan_on_4096": same, "idbits_wide": bool(N > (1 << 26)),
}))
