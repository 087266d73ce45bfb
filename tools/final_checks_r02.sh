#!/bin/bash
# End-of-round checks on one B200 (run through gpurun from the repo root):
# the GPU test suite, smoke(), the default bench line, and the ncu launch list
# of the bench's timed step (each ncu pass only after its command exited 0).
set -u
O=gpurun_out
python -m pytest tests -m gpu -q > $O/gpu_tests_final.log 2>&1; tail -3 $O/gpu_tests_final.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_final.log 2>&1; tail -2 $O/smoke_final.log
python bench.py > $O/bench_final.json 2> $O/bench_final.err || { tail -20 $O/bench_final.err; exit 1; }
python bench.py --steps 64 --warmup 64 --no-extras --cpu-budget-s 1 > $O/bench_plain_final.json 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file $O/launches_final_bench.csv \
    python bench.py --steps 64 --warmup 64 --no-extras --cpu-budget-s 1 > $O/ncu_bench_final.log 2>&1
ls -la $O/*final*
