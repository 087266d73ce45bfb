"""Where the e2e loop's time goes: host time inside each async submission vs
time blocked on results, at the bench's 4096-query batches and at tiny
batches (host floor), and per-call driver costs measured in C."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2602_04936_b200 as lg  # noqa: E402
from paper_2602_04936_b200 import _native  # noqa: E402
from paper_2602_04936_b200._native import PinnedArray  # noqa: E402

ds = lg.generate_dataset(2_000_000, 32, 4, seed=3)
idx = lg.build(ds)
for batch in (4096, 1024, 64):
    qs = lg.generate_queries(ds, batch * 8, seed=4)
    pin = PinnedArray((8, batch, 32), np.uint16)
    pin.array[:] = qs.reshape(8, batch, 32)
    depth = _native.ASYNC_DEPTH
    outs = [idx.native.alloc_batch(batch, 10, "complete", pinned=True, with_work=False) for _ in range(depth)]
    _native.reset_async_ring()
    for i in range(16):
        idx.query_batch_async(pin.array[i % 8], 10, "complete", out=outs[i % depth]).result()
    steps = 3000
    pending = []
    t_sub = t_wait = 0.0
    t0 = time.perf_counter()
    for i in range(steps):
        if len(pending) == depth:
            a = time.perf_counter()
            pending.pop(0).result()
            t_wait += time.perf_counter() - a
        a = time.perf_counter()
        pending.append(idx.query_batch_async(pin.array[i % 8], 10, "complete", out=outs[i % depth]))
        t_sub += time.perf_counter() - a
    for p in pending:
        p.result()
    el = time.perf_counter() - t0
    print(f"batch {batch}: {1e6 * el / steps:.2f} us/batch ({batch * steps / el / 1e6:.1f} M q/s); "
          f"submit {1e6 * t_sub / steps:.2f} us, blocked {1e6 * t_wait / steps:.2f} us per batch", flush=True)

# Python + ctypes floor: a no-op ABI call, and a finished workspace's wait
lib = _native.load()
ws = _native.async_workspace()
ws.wait()
for name, fn in (("ctypes lcp_abi_version", lib.lcp_abi_version), ("Workspace.wait (idle)", ws.wait),
                 ("async_workspace()", _native.async_workspace)):
    t0 = time.perf_counter()
    for _ in range(20000):
        fn()
    print(f"{name}: {1e6 * (time.perf_counter() - t0) / 20000:.2f} us per call", flush=True)

# the same submissions as direct ctypes calls (no Python layers above the ABI)
batch = 4096
qs = lg.generate_queries(ds, batch * 8, seed=4)
pin = PinnedArray((8, batch, 32), np.uint16)
pin.array[:] = qs.reshape(8, batch, 32)
depth = _native.ASYNC_DEPTH
outs = [idx.native.alloc_batch(batch, 10, "complete", pinned=True, with_work=False) for _ in range(depth)]
_native.reset_async_ring()
ring = [_native.async_workspace() for _ in range(depth)]
_native.reset_async_ring()
h = idx.native._h
stride = idx.native.stride_for(10)
qptr = [pin.array[i].__array_interface__["data"][0] for i in range(8)]
args = [(h, ring[i % depth].handle, qptr[i % 8], batch, stride, 1, outs[i % depth]._packed[2],
         outs[i % depth]._packed[0], outs[i % depth]._flags) for i in range(depth * 8)]
fn = lib.lcp_query_host_packed_async
wait = lib.lcp_workspace_wait
for rep in range(2):
    t_sub = 0.0
    t0 = time.perf_counter()
    for i in range(3000):
        ws = ring[i % depth]
        wait(ws.handle)
        a = time.perf_counter()
        fn(*args[i % (depth * 8)])
        t_sub += time.perf_counter() - a
    for ws in ring:
        wait(ws.handle)
    el = time.perf_counter() - t0
    print(f"direct ctypes: {1e6 * el / 3000:.2f} us/batch, submit {1e6 * t_sub / 3000:.2f} us", flush=True)

# one batch at a time: the synchronous API vs async submit + immediate wait
out_sync = idx.native.alloc_batch(batch, 10, "complete", pinned=True)
out_lean = idx.native.alloc_batch(batch, 10, "complete", pinned=True, with_work=False)
for name, call in (("query_batch (sync, with work counters)", lambda q: idx.query_batch(q, 10, "complete", out=out_sync)),
                   ("query_batch_async(...).result(), with work counters", lambda q: idx.query_batch_async(q, 10, "complete", out=out_sync).result()),
                   ("query_batch_async(...).result(), lean block", lambda q: idx.query_batch_async(q, 10, "complete", out=out_lean).result())):
    for i in range(50):
        call(pin.array[i % 8])
    ts = []
    for i in range(2000):
        a = time.perf_counter()
        call(pin.array[i % 8])
        ts.append(time.perf_counter() - a)
    print(f"{name}: p50 {1e6 * np.median(ts):.1f} us, mean {1e6 * np.mean(ts):.1f} us", flush=True)
