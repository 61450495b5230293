"""Kernels the f1/f3/f4 paths launch (run under ncu for the launch list) and the device sort's
speed against torch.sort (diagnostics): a large hash build, a histogram over a nullable column,
a CSV load with a TEXT column."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1901_01488_b200 import join, sorting
from paper_1901_01488_b200.histogram import build_histogram
from paper_1901_01488_b200.ingest import load_csv
from paper_1901_01488_b200.storage import Column, ColumnTable, parse_kind
dev = torch.device("cuda", 0)
g = np.random.default_rng(1)
mark = lambda s: torch.cuda.nvtx.range_push(s)
t = ColumnTable("b", [Column("k", parse_kind("INT64"), g.integers(-10**9, 10**9, 1_000_000), device=dev),
                      Column("j", parse_kind("INT32"), g.integers(-10**6, 10**6, 1_000_000).astype(np.int32), device=dev)])
join.build_hash(t, "k"); join.build_hash(t, "j")
h = ColumnTable("h", [Column("v", parse_kind("INT32"), g.integers(0, 10**6, 10_000_000).astype(np.int32),
                             g.random(10_000_000) < 0.05, device=dev)])
build_histogram(h, "v", 64)
text = "".join(f'{i},"w{i % 97}",x{i % 13}\n' for i in range(200_000))
load_csv(text, "c", [("i", parse_kind("int64")), ("s", parse_kind("text")), ("u", parse_kind("text"))], device=dev)
torch.cuda.synchronize()
if "--time" in sys.argv:
    for n in (1_000_000, 10_000_000, 100_000_000):
        k = torch.randint(-(1 << 62), 1 << 62, (n,), device=dev)
        v = torch.arange(n, device=dev)
        k32 = torch.randint(0, 1 << 31, (n,), device=dev, dtype=torch.int32)
        for name, fn in (("esc u64 pairs", lambda: sorting.sort_pairs(k, v)), ("torch u64 pairs", lambda: torch.sort(k, stable=True)),
                         ("esc u32 pairs", lambda: sorting.sort_pairs(k32, v)), ("torch i32 pairs", lambda: torch.sort(k32, stable=True))):
            for _ in range(2): fn()
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
            print(f"n={n:>10} {name:16s} {statistics.median(ts):8.3f} ms")
print("ok")
