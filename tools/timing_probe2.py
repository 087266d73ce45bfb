"""Short timed regions with per-stream boundary events: one graph holds W
warm-up steps then K timed steps on 4 streams; each stream records an event
before its first timed step and after its last; time = max(B) - min(A).
Compared with the bench's outer events around a K-step graph."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2602_04936_b200 as lg
from paper_2602_04936_b200._native import Workspace

N, L, S, K, B = 2_000_000, 32, 4, 10, 4096
ds = lg.generate_dataset(N, L, S, seed=3)
qs = lg.generate_queries(ds, B * 8, seed=4)
dev = torch.device("cuda")
dq = torch.from_numpy(qs).to(dev).view(8, B, L)
reps = [lg.build(ds) for _ in range(8)]
main = torch.cuda.Stream()
nst = 4


def make(warm, steps):
    streams = [torch.cuda.Stream() for _ in range(nst)]
    wss = [Workspace() for _ in range(nst)]
    bufs = [(torch.empty((B, K), dtype=torch.int32, device=dev), torch.empty((B, K), dtype=torch.int16, device=dev),
             torch.empty(B, dtype=torch.int32, device=dev), torch.empty(B, dtype=torch.int16, device=dev),
             torch.empty((B, 2), dtype=torch.int64, device=dev)) for _ in range(nst)]
    A = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(nst)]
    Bv = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(nst)]
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=main):
        for x in streams:
            x.wait_stream(main)
        for i in range(warm + steps):
            s = i % nst
            if i == warm + s:
                A[s].record(streams[s])
            ids, lcps, hits, md, aux = bufs[s]
            reps[i % 8].native.query_device(dq[(i // 8) % 8], K, "complete", ids, lcps, hits, md, aux,
                                            stream=streams[s].cuda_stream, ws=wss[s])
        for s in range(nst):
            Bv[s].record(streams[s])
        for x in streams:
            main.wait_stream(x)
    g.keep = (wss, bufs)
    return g, A, Bv


for steps in (20, 64, 640):
    for warm in (8, 32):
        g, A, Bv = make(warm, steps)
        vals = []
        with torch.cuda.stream(main):
            for t in range(6):
                g.replay()
                torch.cuda.synchronize()
                if t:
                    starts = [A[0].elapsed_time(a) for a in A]
                    ends = [A[0].elapsed_time(b) for b in Bv]
                    vals.append(max(ends) - min(starts))
        print(f"steps={steps} warm={warm}: us/step {1e3 * float(np.median(vals)) / steps:.3f}", flush=True)
