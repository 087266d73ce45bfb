"""Per-stage latency of the W==1 query kernel from in-kernel clock64 stamps.

Compiles a separate trace build (-DLCP_TRACE) into /tmp and loads it instead
of the shipped library; the shipped .so never contains the trace code.
"""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np

from paper_2602_04936_b200 import _build, _native

out = "/tmp/_lcp_b200_trace.so"
subprocess.run(["nvcc", *_build.NVCC_FLAGS, "-DLCP_TRACE", "-o", out,
                os.path.join(_build.CSRC, "lcp_b200.cu")], check=True)
_native.LIB_PATH = out
lib = _native.load()
lib.lcp_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int64]

import torch

import paper_2602_04936_b200 as lg

ds = lg.generate_dataset(2_000_000, 32, 4, seed=3)
idx = lg.build(ds)
qs = lg.generate_queries(ds, 4096, seed=4)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
names = ["pack", "levels", "region", "dstar", "select", "extend", "write"]
for batch in (1, 4096):
    for cold in (False, True):
        dq = torch.from_numpy(qs[:batch]).cuda()
        ids = torch.empty((batch, 10), dtype=torch.int32, device="cuda")
        lcps = torch.empty((batch, 10), dtype=torch.int16, device="cuda")
        hits = torch.empty(batch, dtype=torch.int32, device="cuda")
        for _ in range(3):
            idx.native.query_device(dq, 10, "complete", ids, lcps, hits, stream=0)
        torch.cuda.synchronize()
        if cold:
            flush.zero_()
        idx.native.query_device(dq, 10, "complete", ids, lcps, hits, stream=0)
        buf = np.zeros(65536 * 8, dtype=np.uint64)
        lib.lcp_debug_trace(buf.ctypes.data, buf.size)
        t = buf.reshape(-1, 8)[:batch].astype(np.int64)
        d = np.diff(t, axis=1)
        print(f"batch {batch} {'cold' if cold else 'warm'}: total cycles median {np.median(t[:, 7] - t[:, 0]):.0f}"
              f" p99 {np.percentile(t[:, 7] - t[:, 0], 99):.0f}")
        for j, nm in enumerate(names):
            print(f"   {nm:7s} median {np.median(d[:, j]):7.0f}  p90 {np.percentile(d[:, j], 90):7.0f}")
