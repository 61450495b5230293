set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_multigpu.py -x -q 2>&1 | tail -30 > gpurun_out/t_mg.log
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/t_all.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-extras > gpurun_out/b1.json 2> gpurun_out/b1.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref1.json 2>&1
tail -3 gpurun_out/t_mg.log gpurun_out/t_all.log; tail -c 3000 gpurun_out/b1.json; tail -5 gpurun_out/b1.err; cat gpurun_out/ref1.json
