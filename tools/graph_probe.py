"""Host launch cost vs GPU time; CUDA-graph replay of the query step over
R index replicas (R x 24 MB > 126 MB L2, so every step's index misses L2)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2602_04936_b200 as lg

ds = lg.generate_dataset(2_000_000, 32, 4, seed=3)
R = int(os.environ.get("REPLICAS", "8"))
reps = [lg.build(ds) for _ in range(R)]
qs = lg.generate_queries(ds, 4096 * 8, seed=4)
dq = torch.from_numpy(qs).cuda().view(8, 4096, 32)
ids = torch.empty((4096, 10), dtype=torch.int32, device="cuda")
lcps = torch.empty((4096, 10), dtype=torch.int16, device="cuda")
hits = torch.empty(4096, dtype=torch.int32, device="cuda")
md = torch.empty(4096, dtype=torch.int16, device="cuda")
aux = torch.empty((4096, 2), dtype=torch.int64, device="cuda")
s = torch.cuda.Stream()
st = s.cuda_stream
with torch.cuda.stream(s):
    for i in range(20):
        reps[i % R].native.query_device(dq[i % 8], 10, "complete", ids, lcps, hits, md, aux, stream=st)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(2000):
        reps[i % R].native.query_device(dq[i % 8], 10, "complete", ids, lcps, hits, md, aux, stream=st)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"host submit {1e6 * (t1 - t0) / 2000:.2f} us/call; wall incl drain {1e6 * (t2 - t0) / 2000:.2f} us/step")
    g = torch.cuda.CUDAGraph()
    G = 8 * R
    with torch.cuda.graph(g, stream=s):
        for i in range(G):
            reps[i % R].native.query_device(dq[i % 8], 10, "complete", ids, lcps, hits, md, aux, stream=st)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 50
    a.record(s)
    for _ in range(n):
        g.replay()
    b.record(s)
    torch.cuda.synchronize()
    per = a.elapsed_time(b) * 1e3 / (n * G)
    print(f"graph replay over {R} replicas: {per:.2f} us/step  -> {4096 / per:.1f} Mq/s")
    # same index every step (L2-resident)
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2, stream=s):
        for i in range(G):
            reps[0].native.query_device(dq[i % 8], 10, "complete", ids, lcps, hits, md, aux, stream=st)
    g2.replay()
    torch.cuda.synchronize()
    a.record(s)
    for _ in range(n):
        g2.replay()
    b.record(s)
    torch.cuda.synchronize()
    per = a.elapsed_time(b) * 1e3 / (n * G)
    print(f"graph replay, one replica (L2-warm): {per:.2f} us/step -> {4096 / per:.1f} Mq/s")

    # several batches in flight: steps alternate between S streams inside one graph
    for S in (2, 3, 4):
        streams = [torch.cuda.Stream() for _ in range(S)]
        outs = [(torch.empty((4096, 10), dtype=torch.int32, device="cuda"),
                 torch.empty((4096, 10), dtype=torch.int16, device="cuda"),
                 torch.empty(4096, dtype=torch.int32, device="cuda"),
                 torch.empty(4096, dtype=torch.int16, device="cuda"),
                 torch.empty((4096, 2), dtype=torch.int64, device="cuda")) for _ in range(S)]
        g3 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g3, stream=s):
            for x in streams:
                x.wait_stream(s)
            for i in range(G):
                x = streams[i % S]
                o = outs[i % S]
                reps[i % R].native.query_device(dq[i % 8], 10, "complete", *o, stream=x.cuda_stream)
            for x in streams:
                s.wait_stream(x)
        g3.replay()
        torch.cuda.synchronize()
        a.record(s)
        for _ in range(n):
            g3.replay()
        b.record(s)
        torch.cuda.synchronize()
        per = a.elapsed_time(b) * 1e3 / (n * G)
        print(f"graph replay, {S} streams, {R} replicas: {per:.2f} us/step -> {4096 / per:.1f} Mq/s")
