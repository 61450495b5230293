mkdir -p gpurun_out
for c in default 1 2 4; do
  echo "ESC_CHUNKS=$c"
  if [ $c = default ]; then python tools/diag_small.py; else ESC_CHUNKS=$c python tools/diag_small.py; fi
done > gpurun_out/small.log 2>&1
