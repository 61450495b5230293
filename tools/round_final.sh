#!/bin/bash
# End-of-round measurement pass (GPU box, repo root): bench line, reference arm, sweep, launch
# list (the ncu captures: tools/profile_round.sh 1 / 2, separate calls: gpurun returns <= 64 MiB).
# Outputs in gpurun_out/final/.
set -u
mkdir -p gpurun_out/final
python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-extras --sweep gpurun_out/final/sweep.json \
    > gpurun_out/final/bench_sweep.json 2> gpurun_out/final/bench_sweep.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv \
    --log-file gpurun_out/final/launches_config4.csv python bench.py --steps 2 --warmup 1 --no-extras --no-e2e \
    --no-cpu-baseline > gpurun_out/final/launches.log 2>&1
