"""Whole-build time from device-resident rows (L=32, sigma=4) at 2M and 25M
rows, and the exported order checked against numpy's stable argsort of the
packed keys (LCP_SORT_MSD=0 forces the plain LSD passes; run twice to A/B)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_04936_b200 as lg  # noqa: E402
from paper_2602_04936_b200.engine import NativeIndex  # noqa: E402

print("LCP_SORT_MSD =", os.environ.get("LCP_SORT_MSD", "(default)"), flush=True)
for n, dist in ((2_000_000, "uniform"), (25_000_000, "uniform"), (2_000_000, "clustered")):
    ds = lg.generate_dataset(n, 32, 4, seed=3, distribution=dist)
    rows = np.array(ds.items)
    dev_rows = torch.from_numpy(rows).cuda()
    ts = []
    for _ in range(6):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ni = NativeIndex.from_device(dev_rows.data_ptr(), n, 32, 4)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    order = ni.export_order() if hasattr(ni, "export_order") else None
    ok = "n/a"
    if order is not None and n <= 2_000_000:
        keys = np.zeros(n, np.uint64)
        r = rows.astype(np.uint64)
        for j in range(32):
            keys |= r[:, j] << np.uint64(62 - 2 * j)
        ref = np.argsort(keys, kind="stable")
        ok = bool(np.array_equal(np.asarray(order).astype(np.int64), ref))
    print(f"n={n} {dist}: build {1e3 * np.median(ts[1:]):.2f} ms (min {1e3 * min(ts[1:]):.2f}); order == stable argsort: {ok}",
          flush=True)
    del ni
