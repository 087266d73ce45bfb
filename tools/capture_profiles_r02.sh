#!/bin/bash
# Round-2 ncu evidence (run via gpurun from the repo root; one GPU).  Every
# capture runs only after its own command exited 0 without ncu.  Outputs go
# to gpurun_out/ and are copied into profiles/ by hand (summaries only).
set -u
O=gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed
# 1. launch list of the bench's timed step (headline kernel share)
python bench.py --steps 64 --warmup 64 --no-extras --cpu-budget-s 1 > $O/r02_bench_plain.json 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file $O/launches_r02_bench.csv \
    python bench.py --steps 64 --warmup 64 --no-extras --cpu-budget-s 1 > $O/ncu_bench.log 2>&1
# 2. build kernels at 2M and 25M rows (device-resident rows)
python tools/profile_build.py 2000000 1 > /dev/null 2>&1 || exit 1
ncu --metrics $M --clock-control none -k regex:"k_pack|k_digit|k_rs_up|k_scan|k_onesweep" --csv \
    --log-file $O/build_kernels_r02_2m.csv python tools/profile_build.py 2000000 1 > /dev/null 2>&1
ncu --metrics $M --clock-control none -k regex:"k_pack|k_digit|k_rs_up|k_scan|k_onesweep" --csv \
    --log-file $O/build_kernels_r02_25m.csv python tools/profile_build.py 25000000 1 > /dev/null 2>&1
# 3. small-batch full scan at 2M and 200M (Q = 1, 2, 4, 8), and the large-batch scan
python tools/fullscan_smallq_probe.py 2000000 > $O/fsq_r02_2m.txt 2>&1 || exit 1
python tools/fullscan_smallq_probe.py 200000000 > $O/fsq_r02_200m.txt 2>&1 || exit 1
ncu --metrics $M --clock-control none -k regex:"k_fullscan_smallq" -c 4 --csv \
    --log-file $O/fullscan_smallq_r02_2m.csv python tools/fullscan_smallq_probe.py 2000000 > /dev/null 2>&1
ncu --metrics $M --clock-control none -k regex:"k_fullscan_smallq" -c 4 --csv \
    --log-file $O/fullscan_smallq_r02_200m.csv python tools/fullscan_smallq_probe.py 200000000 > /dev/null 2>&1
# 4. full sections for the streaming kernels (details pages; reports stay on the box)
ncu --set full --clock-control none -k regex:"k_fullscan_smallq" -s 1 -c 1 -o /tmp/fsq200 \
    python tools/fullscan_smallq_probe.py 200000000 > /dev/null 2>&1
ncu -i /tmp/fsq200.ncu-rep --page details --csv > $O/ncu_details_fullscan_smallq_r02.csv 2>/dev/null
ncu --set full --clock-control none -k regex:"k_pack_aligned" -c 1 -o /tmp/pack25 \
    python tools/profile_build.py 25000000 1 > /dev/null 2>&1
ncu -i /tmp/pack25.ncu-rep --page details --csv > $O/ncu_details_pack_r02.csv 2>/dev/null
ncu --set full --clock-control none -k regex:"k_onesweep" -c 1 -o /tmp/os2 \
    python tools/profile_build.py 2000000 1 > /dev/null 2>&1
ncu -i /tmp/os2.ncu-rep --page details --csv > $O/ncu_details_onesweep_r02.csv 2>/dev/null
ls -la $O
