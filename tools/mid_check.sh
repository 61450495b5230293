timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "stream or capture" 2>&1 | tail -3
echo "== mid on"; python tools/diag_config2.py 2>&1 | tail -8
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/c2mid_launches.csv python tools/diag_config2.py > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/c2mid_launches.csv')))
hdr=None; by={}
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); by.setdefault(d['ID'],{})['name']=d['Kernel Name'][:40]; by[d['ID']][d['Metric Name']]=d['Metric Value']
for k,v in list(by.items())[-6:]:
    print(k, v['name'], v.get('gpu__time_duration.sum'), v.get('dram__bytes_read.sum'), v.get('dram__bytes_write.sum'))
PY
