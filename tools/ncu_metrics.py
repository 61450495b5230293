"""Print selected metrics of an ncu report (not part of the product): python tools/ncu_metrics.py rep [names...]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
want = sys.argv[2:] or ["Duration", "DRAM Throughput", "Memory Throughput", "Achieved Occupancy",
                        "Registers Per Thread", "Warp Cycles Per Issued Instruction", "Issue Slots Busy",
                        "L1/TEX Hit Rate", "L2 Hit Rate", "Compute (SM) Throughput", "Block Size", "Grid Size",
                        "Dynamic Shared Memory Per Block", "Theoretical Occupancy"]
txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.DictReader(io.StringIO(txt)))
seen = set()
for r in rows:
    k = (r["Kernel Name"][:40], r["Metric Name"])
    if r["Metric Name"] in want and k not in seen:
        seen.add(k)
        print(f'{r["Kernel Name"][:40]:40s} {r["Metric Name"]:40s} {r["Metric Value"]} {r["Metric Unit"]}')
