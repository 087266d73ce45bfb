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
# name:path:k:kernel (kn = the warp top-k list kernel, general = the CTA-per-query kernel)
for spec in query:query:10:k_query_w1 fullscan:fullscan:10:k_fullscan_w1 tal:tal:10:k_query_w1 \
            kn:query:64:k_query_w1_kn general:query:1000:k_query_general; do
  IFS=: read -r w path kk kern <<< "$spec"
  python tools/profile_kernels.py $path --k $kk > /dev/null 2>&1 || exit 1
  ncu --set full --import-source on --clock-control none -k regex:$kern -s 3 -c 1 \
      -o $O/prof_${w}_${R} python tools/profile_kernels.py $path --k $kk > $O/ncu_${w}.log 2>&1
  ncu -i $O/prof_${w}_${R}.ncu-rep --page details --csv > $O/ncu_details_${w}_${R}.csv 2>/dev/null
  ncu -i $O/prof_${w}_${R}.ncu-rep --page raw --csv > $O/ncu_raw_${w}_${R}.csv 2>/dev/null
  # reports are ~35 MB each and gpurun returns at most 64 MiB: keep the headline one
  [ $w = query ] || rm -f $O/prof_${w}_${R}.ncu-rep
done
ls -la $O
