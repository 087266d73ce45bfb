"""PCIe copy characteristics on the box: pinned H2D / D2H time vs size, and
H2D + D2H pairs on 4 concurrent streams (the e2e pattern)."""
import subprocess

import torch

print(subprocess.run("nvidia-smi topo -m 2>/dev/null | head -5; nvidia-smi -q | grep -i -A3 'PCIe Generation' | head -8; lscpu | grep -i 'numa\\|model name' ", shell=True, capture_output=True, text=True).stdout)
dev = torch.device("cuda")
for size in (64 << 10, 256 << 10, 1 << 20, 4 << 20, 64 << 20):
    h = torch.empty(size, dtype=torch.uint8).pin_memory()
    d = torch.empty(size, dtype=torch.uint8, device=dev)
    for name, fn in (("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 50
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) * 1e3 / reps
        print(f"{name} {size >> 10:6d} KB: {us:8.2f} us  {size / us / 1e3:6.1f} GB/s", flush=True)
# concurrent pairs, 4 streams, 256 KB each way
size = 256 << 10
hs = [torch.empty(size, dtype=torch.uint8).pin_memory() for _ in range(8)]
ho = [torch.empty(size, dtype=torch.uint8).pin_memory() for _ in range(8)]
ds = [torch.empty(size, dtype=torch.uint8, device=dev) for _ in range(8)]
streams = [torch.cuda.Stream() for _ in range(4)]
for rounds in (1, 200):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for s in streams:
        s.wait_stream(torch.cuda.current_stream())
    for r in range(rounds * 4):
        s = streams[r % 4]
        with torch.cuda.stream(s):
            ds[r % 8].copy_(hs[r % 8], non_blocking=True)
            ho[r % 8].copy_(ds[r % 8], non_blocking=True)
    for s in streams:
        torch.cuda.current_stream().wait_stream(s)
    b.record()
    torch.cuda.synchronize()
print(f"pairs of 256 KB H2D + 256 KB D2H on 4 streams: {a.elapsed_time(b) * 1e3 / (200 * 4):.2f} us per pair")
