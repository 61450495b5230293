"""Scan cost of nullable predicate columns: packed 1-bit NULL staging vs byte masks (diagnostics).
3 int32 columns with 8% NULLs (the reference's custom_nulls fraction), 200M rows, count_star of a
3-atom conjunction; device time with L2 irrelevant (2.4 GB of inputs)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_01488_b200 import compiler, count_star, executor, expr as ex
from paper_1901_01488_b200.storage import KIND_INT32, Column, ColumnTable
import bench
dev = torch.device("cuda", 0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000_000
dt = sys.argv[2] if len(sys.argv) > 2 else "int32"
from paper_1901_01488_b200.storage import parse_kind
kind, tdt, w = {"int32": (KIND_INT32, torch.int32, 4), "int8": (parse_kind("INT8"), torch.int8, 1)}[dt]
g = torch.Generator(device=dev); g.manual_seed(1)
cols = []
for name in ("x", "y", "z"):
    v = torch.randint(0, 100, (n,), generator=g, device=dev, dtype=tdt)
    m = torch.rand(n, generator=g, device=dev) < 0.08
    cols.append(Column(name, kind, v, m))
t = ColumnTable("t", cols)
for packed in (False, True):
    compiler.set_packed_nulls(packed)
    r = lambda c: ex.ColumnRef("t", c)
    p = ex.And((ex.Range(r("x"), 1, 50), ex.Comparison(r("y"), "<", 90), ex.Comparison(r("z"), ">", 3)))
    for _ in range(3): count_star(t, p)
    tt = bench._time_kernels(lambda: count_star(t, p), 7, dev)
    ms = statistics.median(x for x, k in tt if k == "count")
    b = n * (3 * w + (3 / 8 if packed else 3))
    print(f"packed={packed}: count {count_star(t, p)}  {ms:.3f} ms  {b / ms / 1e6:.0f} GB/s of staged bytes  "
          f"({n * 3 * w / ms / 1e6:.0f} GB/s of values)")
