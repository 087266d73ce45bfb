"""Minimal launcher for ncu captures of one kernel family.

    python tools/profile_kernels.py query|fullscan|tal|build|strict [--launches N] [--k K]

Builds the BASELINE config-3 index (N=2M, L=32, sigma=4) and launches the
chosen path a few times on one stream (no L2 flush between launches), so an
``ncu -k regex:<kernel> -s <warm> -c 1`` capture sees a representative launch.
"""

from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["query", "fullscan", "tal", "build", "strict"])
    ap.add_argument("--launches", type=int, default=6)
    ap.add_argument("--batch", type=int, default=4096)
    ap.add_argument("--time", action="store_true")
    ap.add_argument("--k", type=int, default=10)  # 64: k_query_w1_kn, 1000: k_query_general
    args = ap.parse_args()

    import torch

    import paper_2602_04936_b200 as lg

    ds = lg.generate_dataset(2_000_000, 32, 4, seed=3)
    qs = lg.generate_queries(ds, args.batch, seed=4)
    dq = torch.from_numpy(qs).cuda()
    k = args.k
    ids = torch.empty((args.batch, k), dtype=torch.int32, device="cuda")
    lcps = torch.empty((args.batch, k), dtype=torch.int16, device="cuda")
    hits = torch.empty(args.batch, dtype=torch.int32, device="cuda")
    md = torch.empty(args.batch, dtype=torch.int16, device="cuda")
    aux = torch.empty((args.batch, 2), dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    if args.what == "build":
        for _ in range(args.launches):
            lg.build(ds)
        return
    idx = lg.build_tal(ds, 256) if args.what == "tal" else lg.build(ds)
    def launch():
        if args.what == "query":
            idx.native.query_device(dq, k, "complete", ids, lcps, hits, md, aux, stream=st)
        elif args.what == "strict":
            idx.native.query_device(dq, k, "strict", ids, lcps, hits, md, aux, stream=st)
        elif args.what == "tal":
            idx.native.query_device(dq, k, "tal", ids, lcps, hits, md, aux, stream=st)
        else:
            idx.native.fullscan_device(dq, k, ids, lcps, hits, stream=st)

    for _ in range(args.launches):
        launch()
    torch.cuda.synchronize()
    if args.time:
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        reps = 200 if args.what != "fullscan" else 10
        ev[0].record()
        for _ in range(reps):
            launch()
        ev[1].record()
        torch.cuda.synchronize()
        print(f"{args.what}: {1e3 * ev[0].elapsed_time(ev[1]) / reps:.2f} us/launch (back-to-back, warm L2)")
    print("ok", args.what, int(hits.cpu().numpy().sum()))


if __name__ == "__main__":
    main()
