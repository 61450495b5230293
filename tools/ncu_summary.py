"""Summarise ncu captures for profiles/ (not part of the product).

python tools/ncu_summary.py <report.ncu-rep> <label> [--traffic-key KEY] [--out FILE]
  -> appends a markdown section to profiles/ncu_r01.md (or FILE) and (with --traffic-key) records the
     launch's DRAM bytes in profiles/traffic.json (read by bench.py for roofline.traffic).
"""

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % (occupancy)"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__sass_inst_executed_op_local_ld.sum", "local loads"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
]


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True, check=True)
    rows = list(csv.reader(io.StringIO(out.stdout)))
    return rows[0], rows[1], rows[2:]


def main():
    report, label = sys.argv[1], sys.argv[2]
    key = sys.argv[sys.argv.index("--traffic-key") + 1] if "--traffic-key" in sys.argv else None
    hdr, units, rows = raw(report)
    lines = [f"\n## {label}\n", f"source: `{os.path.basename(report)}` (ncu --set full --clock-control none)\n"]
    for r in rows:
        name = r[hdr.index("Kernel Name")]
        lines.append(f"\n**{name}**\n\n| metric | value |\n|---|---|")
        for m, title in METRICS:
            if m in hdr:
                lines.append(f"| {title} (`{m}`) | {r[hdr.index(m)]} {units[hdr.index(m)]} |")
        try:  # achieved DRAM bandwidth of this launch (read + write over its duration)
            def _val(m, scale):
                v = float(r[hdr.index(m)])
                u = units[hdr.index(m)].lower()
                return v * scale.get(u, 1.0)
            nbytes = (_val("dram__bytes_read.sum", {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}) +
                      _val("dram__bytes_write.sum", {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}))
            secs = _val("gpu__time_duration.sum", {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6,
                                                    "msecond": 1e-3, "ms": 1e-3, "second": 1.0})
            gbs = nbytes / secs / 1e9
            lines.append(f"| achieved DRAM GB/s (read+write / duration) | {gbs:.0f} GB/s = {gbs / 8000:.2f} of 8 TB/s "
                         f"nominal, {gbs / 6538.3:.2f} of the measured 6538 GB/s copy peak (cold-cache replay) |")
        except (ValueError, KeyError, ZeroDivisionError):
            pass
        stalls = sorted(((float(r[i] or 0), h.replace("smsp__pcsamp_warps_issue_stalled_", ""))
                         for i, h in enumerate(hdr)
                         if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")),
                        reverse=True)[:5]
        lines.append("| top stall reasons (samples) | " + ", ".join(f"{n} {int(v)}" for v, n in stalls) + " |")
        if key:
            def to_bytes(m):
                v = float(r[hdr.index(m)])
                u = units[hdr.index(m)].lower()
                return v * {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "tbyte": 1e12}.get(u, 1)
            path = os.path.join(ROOT, "profiles", "traffic.json")
            data = json.load(open(path)) if os.path.exists(path) else {}
            data[key] = to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum")
            json.dump(data, open(path, "w"), indent=1)
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else os.path.join(ROOT, "profiles", "ncu_r01.md")
    with open(out, "a") as fh:
        fh.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
