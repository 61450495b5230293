"""Hot source lines of one kernel in an ncu report: `ncu -i R --page source --csv
--print-source cuda,sass` aggregated per CUDA line (instructions executed, stall samples).
Usage: ncu_hotlines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg, fname, cur, hdr = {}, "", None, None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr):
        if r[0]:
            cur = (fname, int(r[0]), r[1].strip()[:90])
            ie = int(r[hdr.index("Instructions Executed")] or 0)
            st = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
            a = agg.setdefault(cur, [0, 0])
            a[0] += ie
            a[1] += st
tot_i = sum(v[0] for v in agg.values()) or 1
tot_s = sum(v[1] for v in agg.values()) or 1
print(f"total warp instructions {tot_i}, stall samples {tot_s}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{v[1] / tot_s * 100:5.1f}% stall {v[0] / tot_i * 100:5.1f}% inst  {k[0]}:{k[1]}  {k[2]}")
