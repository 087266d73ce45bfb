"""Event-timed floor of one tiny kernel launch, measured exactly like bench.py
(256 MiB L2 flush queued before each event pair)."""
import numpy as np
import torch

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
x = torch.empty(4096, dtype=torch.int32, device="cuda")
big = torch.empty(1 << 20, dtype=torch.int32, device="cuda")
for name, fn in [("fill 16KB", lambda: x.zero_()), ("fill 4MB", lambda: big.zero_()),
                 ("two fills", lambda: (x.zero_(), x.zero_()))]:
    ts = []
    for i in range(50):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if i >= 5:
            ts.append(a.elapsed_time(b) * 1e3)
    print(f"{name}: median {np.median(ts):.2f} us  min {np.min(ts):.2f} us")
