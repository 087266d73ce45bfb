"""Minimal launcher for ncu captures of the build kernels (k_pack_stream,
k_digit_hist8, k_onesweep): device-resident rows, N given (default 2M),
L=32, sigma=4, a few builds."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2602_04936_b200 as lg
from paper_2602_04936_b200.engine import NativeIndex

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
builds = int(sys.argv[2]) if len(sys.argv) > 2 else 2
ds = lg.generate_dataset(n, 32, 4, seed=3)
dev_rows = torch.from_numpy(np.array(ds.items)).cuda()
for _ in range(builds):
    ni = NativeIndex.from_device(dev_rows.data_ptr(), n, 32, 4)
    torch.cuda.synchronize()
    del ni
