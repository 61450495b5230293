"""Streamed-compaction speed on the config-5 shape (diagnostics): 600M rows by default, c0/c1
int32 + c4/c5 int64, single range at selectivity s, materialize all four; device time of the
compaction part (sleep-gated) for several s.  Usage: diag_stream.py [rows] [s,s,...]"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1901_01488_b200 import executor, expr as ex
from paper_1901_01488_b200.storage import Column, parse_kind, ColumnTable
n = int(sys.argv[1]) if len(sys.argv) > 1 else 600_000_000
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(5)
cols = [Column(c, parse_kind("INT32"), torch.randint(0, 1_000_000, (n,), generator=g, device=dev, dtype=torch.int32)) for c in ("c0", "c1")]
cols += [Column(c, parse_kind("INT64"), torch.randint(0, 10**12, (n,), generator=g, device=dev, dtype=torch.int64)) for c in ("c4", "c5")]
t = ColumnTable("t", cols)
SS = [float(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else (0.05, 0.1, 0.3, 0.5, 0.9)
for s in SS:
    p = ex.Range(ex.ColumnRef("t", "c0"), 0, int(round(s * 1e6)) - 1)
    for _ in range(2):
        executor.materialize(t, p, ["c0", "c1", "c4", "c5"])
    tt = bench._time_kernels(lambda: executor.materialize(t, p, ["c0", "c1", "c4", "c5"]), 3, dev)
    tc = bench._time_kernels(lambda: executor.count_star(t, p), 3, dev)
    cnt = statistics.median(x for x, k in tc if k == "count")
    sel = statistics.median(x for x, k in tt if k == "select")
    mat = statistics.median(x for x, k in tt if k == "materialize")
    print(f"s={s}: count {cnt:.3f} ms  select {sel:.3f} ms  materialize {mat:.3f} ms  total {sel + mat:.3f} ms")
