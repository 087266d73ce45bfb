"""config5_leg (bench.py) on one GPU: the range-sharded step at world 1 with
1 and LCP_BENCH_C5_INFLIGHT steps in flight.  Usage: python tools/c5_probe.py [n_items]"""
import json
import os
import sys
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else bench.C5_ITEMS
args = types.SimpleNamespace(steps=256, warmup=8)
res = bench.config5_leg(args, 1, 0, torch.device("cuda"), lambda: None, lambda x: x, "range", n_total=n)
res.pop("query_kernel", None)
print(json.dumps(res, indent=1))
