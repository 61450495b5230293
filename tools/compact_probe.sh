#!/bin/bash
# sel_compact durations (ncu, cold) on config 4 and config-5 shapes at s = 1e-4 / 1e-3 / 1e-2
mkdir -p gpurun_out/cp
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:sel_compact -c 2 --csv --log-file gpurun_out/cp/c4.csv \
    python bench.py --steps 2 --warmup 1 --no-extras --no-e2e --no-cpu-baseline > /dev/null 2>&1
for s in 0.0001 0.001 0.01; do
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:sel_compact -c 2 --csv --log-file gpurun_out/cp/s$s.csv \
      python tools/kprof_stream.py $s 600000000 > /dev/null 2>&1
done
for f in gpurun_out/cp/*.csv; do echo "$f $(grep -o '"gpu__time_duration.sum","[a-z]*","[0-9.,]*"' $f | tail -1)"; done
