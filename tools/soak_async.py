"""Soak: thousands of pipelined async batches (graph cache, pooled pinned
blocks, per-thread ring, in-block error flag) checked against precomputed
answers; every 97th batch carries an invalid symbol and must raise."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2602_04936_b200 as lg
from paper_2602_04936_b200 import InvalidInputError, _native
from paper_2602_04936_b200._native import PinnedArray

ds = lg.generate_dataset(500_000, 32, 4, seed=90)
idx = lg.build(ds)
B, K = 4096, 10
pools = [lg.generate_queries(ds, B, seed=91 + i, prefix_len=(None if i % 2 else 16)) for i in range(12)]
expect = [idx.query_batch(p, K, "complete") for p in pools]
exp_ids = [e.ids.copy() for e in expect]
exp_hits = [e.hits.copy() for e in expect]
pin = PinnedArray((12, B, 32), np.uint16)
pin.array[:] = np.stack(pools)
bad = pin.array[3].copy()
bad[17, 5] = 9  # symbol >= sigma
pin_bad = PinnedArray((B, 32), np.uint16)
pin_bad.array[:] = bad
depth = _native.ASYNC_DEPTH
outs = [idx.native.alloc_batch(B, K, "complete", pinned=True, with_work=False) for _ in range(depth)]
pending, checked, errors = [], 0, 0
N = 6000


def finish(p, j, is_bad):
    global checked, errors
    try:
        r = p.result()
    except InvalidInputError:
        assert is_bad, "unexpected invalid-input error"
        errors += 1
        return
    assert not is_bad, "invalid batch did not raise"
    assert np.array_equal(r.hits, exp_hits[j]) and np.array_equal(r.ids, exp_ids[j]), j
    checked += 1


for i in range(N):
    if len(pending) == depth:
        finish(*pending.pop(0))
    j = (i * 7) % 12
    is_bad = i % 97 == 50
    q = pin_bad.array if is_bad else pin.array[j]
    pending.append((idx.query_batch_async(q, K, "complete", out=outs[i % depth]), j, is_bad))
for p in pending:
    finish(*p)
print(f"soak ok: {checked} batches verified, {errors} invalid batches raised")
