"""Render an ncu launch-list CSV (gpu__time_duration / dram bytes per launch) as a markdown table
(not part of the product).  python tools/launch_table.py <csv> [header-file] > out.md"""
import csv
import sys


def main():
    rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
    h = rows[0]
    iid, ik, im, iv = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    by = {}
    for r in rows[1:]:
        d = by.setdefault(int(r[iid]), {"k": r[ik]})
        d[r[im]] = float(r[iv].replace(",", ""))
    if len(sys.argv) > 2:
        sys.stdout.write(open(sys.argv[2]).read())
    print("| ID | kernel | duration (us) | DRAM read (MB) | DRAM write (MB) |")
    print("|---|---|---|---|---|")
    for i in sorted(by):
        d = by[i]
        name = d["k"].replace("void ", "").split("(")[0][:60]
        print(f"| {i} | `{name}` | {d.get('gpu__time_duration.sum', 0) / 1e3:.1f} | "
              f"{d.get('dram__bytes_read.sum', 0) / 1e6:.1f} | {d.get('dram__bytes_write.sum', 0) / 1e6:.1f} |")


if __name__ == "__main__":
    main()
