"""ncu driver for the streamed compaction (not part of the product): config-5-shaped table
(c0, c1 int32; c4, c5 int64), single-range predicate at selectivity s, materialize (c0, c1, c4, c5).
python tools/kprof_stream.py <s> <rows>"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_01488_b200 import ColumnTable, executor, expr as ex
from paper_1901_01488_b200.storage import Column, parse_kind

s, n = float(sys.argv[1]), int(sys.argv[2])
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(5)
cols = []
for c in ("c0", "c1"):
    cols.append(Column(c, parse_kind("INT32"), torch.randint(0, 1_000_000, (n,), generator=g, device=dev, dtype=torch.int32)))
for c in ("c4", "c5"):
    cols.append(Column(c, parse_kind("INT64"), torch.randint(0, 10**12, (n,), generator=g, device=dev, dtype=torch.int64)))
t = ColumnTable("t", cols)
p = ex.Range(ex.ColumnRef("t", "c0"), 0, int(round(s * 1e6)) - 1)
for _ in range(3):
    executor.materialize(t, p, ["c0", "c1", "c4", "c5"])
torch.cuda.synchronize()
print("ok")
