mkdir -p gpurun_out/v11
python tools/diag_stream.py 600000000 0.0001,0.001,0.002 > gpurun_out/v11/diag.log 2>&1
ESC_HIT_LISTS=0 python tools/diag_stream.py 600000000 0.0001,0.001 >> gpurun_out/v11/diag.log 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py -x -q > gpurun_out/v11/tests.log 2>&1
