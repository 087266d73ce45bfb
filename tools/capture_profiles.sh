#!/bin/bash
# Capture the profiles/ evidence on a GPU box (run via gpurun from the repo root).
# Each capture runs only after its own command exited 0 without ncu.
set -u
R=${1:-r01}
O=gpurun_out
python bench.py --steps 64 --warmup 64 --no-extras --cpu-budget-s 1 > $O/bench_plain.json 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file $O/launches_${R}_bench.csv \
    python bench.py --steps 64 --warmup 64 --no-extras --cpu-budget-s 1 > $O/ncu_bench.log 2>&1
for w in query fullscan tal; do
  case $w in query|tal) k=k_query_w1;; fullscan) k=k_fullscan_w1;; esac
  python tools/profile_kernels.py $w > /dev/null 2>&1 || exit 1
  ncu --set full --import-source on --clock-control none -k regex:$k -s 3 -c 1 \
      -o $O/prof_${w}_${R} python tools/profile_kernels.py $w > $O/ncu_${w}.log 2>&1
  ncu -i $O/prof_${w}_${R}.ncu-rep --page details --csv > $O/ncu_details_${w}_${R}.csv 2>/dev/null
done
ls -la $O
