"""Timing-method probe for short timed regions (bench.py --steps 20):
the same 4-stream graph of K query steps timed (a) by events on the capture
stream around a replay queued behind a warm replay (bench.py), (b) by
graph-external event nodes at the head and tail of the graph."""
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


def capture(steps, nst, events):
    streams = [torch.cuda.Stream() for _ in range(nst)]
    wss = [Workspace() for _ in range(nst)]
    bufs = [(torch.empty((B, K), dtype=torch.int32, device=dev), torch.empty((B, K), dtype=torch.int16, device=dev),
             torch.empty(B, dtype=torch.int32, device=dev), torch.empty(B, dtype=torch.int16, device=dev),
             torch.empty((B, 2), dtype=torch.int64, device=dev)) for _ in range(nst)]
    ea = torch.cuda.Event(enable_timing=True, external=True)
    eb = torch.cuda.Event(enable_timing=True, external=True)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=main):
        if events:
            ea.record(main)
        for x in streams:
            x.wait_stream(main)
        for i in range(steps):
            x, (ids, lcps, hits, md, aux) = streams[i % nst], bufs[i % nst]
            reps[i % 8].native.query_device(dq[(i // 8) % 8], K, "complete", ids, lcps, hits, md, aux,
                                            stream=x.cuda_stream, ws=wss[i % nst])
        for x in streams:
            main.wait_stream(x)
        if events:
            eb.record(main)
    g.keep = (wss, bufs)
    return g, ea, eb


for steps in (20, 64, 640):
    for nst in (1, 4):
        g, ea, eb = capture(steps, nst, False)
        ge, ea2, eb2 = capture(steps, nst, True)
        res = {}
        for name in ("outer", "inner"):
            vals = []
            for trial in range(5):
                with torch.cuda.stream(main):
                    for _ in range(20):
                        (g if name == "outer" else ge).replay()
                    torch.cuda.synchronize()
                    if name == "outer":
                        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        g.replay()
                        a.record(main)
                        g.replay()
                        b.record(main)
                        torch.cuda.synchronize()
                        vals.append(a.elapsed_time(b))
                    else:
                        ge.replay()
                        ge.replay()
                        torch.cuda.synchronize()
                        vals.append(ea2.elapsed_time(eb2))
            res[name] = 1e3 * float(np.median(vals)) / steps
        print(f"steps={steps} streams={nst}: us/step outer-events {res['outer']:.3f}  in-graph-events {res['inner']:.3f}", flush=True)
