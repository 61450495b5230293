# config-2 step: per-kernel launch list + one full ncu capture of its kernels
python tools/diag_config2.py > gpurun_out/c2_diag.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/c2_launches.csv python tools/diag_config2.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"esc_scan|sel_|tile_scan|copy_regions" -s 30 -c 8 -o gpurun_out/c2_full -f python tools/diag_config2.py > gpurun_out/c2_ncu.log 2>&1
echo done
