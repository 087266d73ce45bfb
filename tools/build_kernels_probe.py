"""Build-kernel timing from device-resident rows (N=2M and N=25M, L=32,
sigma=4): whole-build CUDA-event time per build, several builds.  Run under
``ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,
dram__throughput.avg.pct_of_peak_sustained_elapsed -k regex:"k_pack|k_onesweep|k_digit"``
for the per-kernel HBM evidence (profiles/build_kernels_r02.csv)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2602_04936_b200 as lg
from paper_2602_04936_b200.engine import NativeIndex

sizes = [int(x) for x in (sys.argv[1:] or ["2000000", "25000000"])]
for n in sizes:
    ds = lg.generate_dataset(n, 32, 4, seed=3)
    dev_rows = torch.from_numpy(ds.items).cuda()
    ms = []
    for i in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        ni = NativeIndex.from_device(dev_rows.data_ptr(), n, 32, 4)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
        del ni
    print(f"N={n}: device-rows build ms {[round(x, 3) for x in ms]}", flush=True)
    del dev_rows, ds
