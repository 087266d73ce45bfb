"""Small-batch full scan (count <= 8) timing: N given (default 2M), L=32,
sigma=4.  Per query count: CUDA-event time per launch over a graph of 20
launches, algorithmic GB/s = (N*K_b + Q*(K_b + 6k)) / time."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2602_04936_b200.datagen import generate_row_block
from paper_2602_04936_b200.engine import NativeIndex

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
k = 10
rows = generate_row_block(n, 32, 4, 6, 0, n)
idx = NativeIndex(rows, 32, 4)
qs = np.random.Generator(np.random.Philox(4)).integers(0, 4, size=(8, 32), dtype=np.uint16)
dq = torch.from_numpy(qs).cuda()
ids = torch.empty((8, k), dtype=torch.int32, device="cuda")
lcps = torch.empty((8, k), dtype=torch.int16, device="cuda")
hits = torch.empty(8, dtype=torch.int32, device="cuda")
peak = 6546.9
for count in (1, 2, 4, 8):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn = lambda: idx.fullscan_device(dq[:count], k, ids[:count], lcps[:count], hits[:count], stream=s.cuda_stream)
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(20):
                fn()
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(5):
            g.replay()
        b.record(s)
        torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / 100
    alg = n * 8 + count * (8 + 6 * k)
    print(f"N={n} count={count}: {us:.2f} us/launch, {alg / us / 1e3:.1f} GB/s algorithmic "
          f"({alg / us / 1e3 / peak:.3f} of {peak} GB/s)", flush=True)
