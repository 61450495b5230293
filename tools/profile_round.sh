#!/bin/bash
# Round profiling captures (run on the GPU box from the repo root); outputs in gpurun_out/prof/.
# Every capture is one launch after warm-up: ncu --set full --clock-control none --import-source on.
set -u
mkdir -p gpurun_out/prof
B="python bench.py --steps 2 --warmup 1 --no-extras --no-e2e --no-cpu-baseline"
N="ncu --set full --clock-control none --import-source on"
PART=${1:-1}   # parts 1, 2, 3: gpurun copies back at most 64 MiB per call
if [ "$PART" = 1 ]; then
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv \
    --log-file gpurun_out/prof/launches_config4.csv $B > gpurun_out/prof/launches.log 2>&1
$N -k regex:esc_scan_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/prof/k1_select_config4 $B > gpurun_out/prof/k1.log 2>&1
$N -k regex:sel_compact --launch-skip 1 --launch-count 1 -o gpurun_out/prof/selcompact_config4 $B > gpurun_out/prof/selc.log 2>&1
$N -k regex:esc_scan_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/prof/k1_count_config5_single \
    python tools/kprof_count.py > gpurun_out/prof/k1c.log 2>&1
$N -k regex:sel_stream --launch-skip 2 --launch-count 1 -o gpurun_out/prof/stream_config5_s0.5 \
    python tools/kprof_stream.py 0.5 200000000 > gpurun_out/prof/stream.log 2>&1
$N -k regex:sel_stream --launch-skip 2 --launch-count 1 -o gpurun_out/prof/stream_config5_s0.1 \
    python tools/kprof_stream.py 0.1 200000000 > gpurun_out/prof/stream01.log 2>&1
elif [ "$PART" = 3 ]; then
# gathered compaction of a sparse selection (config-5 shape, 600M rows, s = 1e-3): warp hit lists
# (the default at this density) vs lane-per-chunk gathers
$N -k regex:sel_compact --launch-skip 2 --launch-count 1 -o gpurun_out/prof/selcompact_hitlist_s1e-3 \
    python tools/kprof_stream.py 0.001 600000000 > gpurun_out/prof/hl.log 2>&1
ESC_HIT_LISTS=0 $N -k regex:sel_compact --launch-skip 2 --launch-count 1 -o gpurun_out/prof/selcompact_lanes_s1e-3 \
    python tools/kprof_stream.py 0.001 600000000 > gpurun_out/prof/hl0.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/prof/launches_f_paths.csv python tools/launches_f.py > gpurun_out/prof/lf.log 2>&1
else
$N -k regex:join_bits --launch-skip 3 --launch-count 1 -o gpurun_out/prof/join_bits_star python tools/diag_join.py \
    > gpurun_out/prof/join.log 2>&1
$N -k regex:csv_ --launch-skip 8 --launch-count 4 -o gpurun_out/prof/csv_ingest python tools/diag_ingest.py \
    > gpurun_out/prof/csv.log 2>&1
$N -k regex:esc_scan_kernel --launch-skip 30 --launch-count 1 -o gpurun_out/prof/k1_config2 python tools/diag_config2.py \
    > gpurun_out/prof/k1c2.log 2>&1
$N -k regex:sel_mid --launch-skip 10 --launch-count 1 -o gpurun_out/prof/mid_config2 python tools/diag_config2.py \
    > gpurun_out/prof/mid2.log 2>&1
$N -k regex:esc_scan_kernel --launch-skip 60 --launch-count 1 -o gpurun_out/prof/onepass_dim python tools/diag_onepass.py \
    > gpurun_out/prof/op.log 2>&1
fi
ls -la gpurun_out/prof
