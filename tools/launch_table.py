"""Print an ncu --csv launch list (gpu__time_duration / dram bytes per launch) as a table."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = OrderedDict()
for r in rows[hi + 1:]:
    d.setdefault(r[ii], {"k": r[ki]})[r[mi]] = r[vi]
skip = sys.argv[2] if len(sys.argv) > 2 else "at::"
for i, v in d.items():
    if skip and skip in v["k"]:
        continue
    print(f'{i:>4} {v["k"][:60]:60} {float(v.get("gpu__time_duration.sum", 0)) / 1e3:9.1f} us '
          f'R {float(v.get("dram__bytes_read.sum", 0)) / 1e6:9.1f} MB  W {float(v.get("dram__bytes_write.sum", 0)) / 1e6:8.1f} MB')
