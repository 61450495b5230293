# compute-sanitizer over the ESC kernels (tools/sanitize.py); summaries -> gpurun_out/san_*.log
CS=/usr/local/cuda/bin/compute-sanitizer
python tools/sanitize.py > gpurun_out/san_plain.log 2>&1; tail -1 gpurun_out/san_plain.log
timeout 1500 $CS --tool memcheck --leak-check no --error-exitcode 9 python tools/sanitize.py > gpurun_out/san_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -3 gpurun_out/san_memcheck.log
timeout 1500 $CS --tool synccheck --error-exitcode 9 python tools/sanitize.py --quick > gpurun_out/san_synccheck.log 2>&1; echo "synccheck rc=$?"; tail -3 gpurun_out/san_synccheck.log
timeout 2400 $CS --tool racecheck --racecheck-report hazard --error-exitcode 9 python tools/sanitize.py --quick > gpurun_out/san_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -3 gpurun_out/san_racecheck.log
