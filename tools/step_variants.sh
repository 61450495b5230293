for st in 2 3 4; do ESC_STAGES=$st python tools/diag_step_device.py > /tmp/o.txt 2>&1; head -1 /tmp/o.txt | sed "s/^/[stages $st] /"; done
