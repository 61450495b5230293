"""Minimal driver for ncu captures of the ESC kernels (not part of the product).
python tools/kprof.py <pred: range1|config4|notnull4> <rows> <mode: count|compact>"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_01488_b200 import ColumnTable, count_star, executor, expr as ex
from paper_1901_01488_b200.storage import Column, parse_kind

name, n, mode = sys.argv[1], int(sys.argv[2]), sys.argv[3]
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(1)
A = torch.randint(1, 1000, (n,), generator=g, device=dev, dtype=torch.int32)
A[torch.rand(n, generator=g, device=dev) < 0.095] = 0
B = torch.randint(-5, 1005, (n,), generator=g, device=dev, dtype=torch.int32)
Cc = torch.randn(n, generator=g, device=dev, dtype=torch.float32)
D = torch.randint(0, 1000, (n,), generator=g, device=dev, dtype=torch.int32)
t = ColumnTable("t", [Column("A", parse_kind("INT32"), A), Column("B", parse_kind("INT32"), B),
                      Column("C", parse_kind("FLOAT32"), Cc), Column("D", parse_kind("INT32"), D)])
r = lambda c: ex.ColumnRef("t", c)
p = {"range1": ex.Range(r("A"), 100, 199),
     "notnull4": ex.And(tuple(ex.FoldedAtom(r(c), True) for c in "ABCD")),
     "config4": ex.And((ex.Equality(r("A"), 0), ex.Range(r("C"), -0.5, 1.0),
                        ex.Or((ex.Equality(r("D"), 17), ex.Comparison(r("D"), ">", 900))),
                        ex.FnCall("b3d", (r("B"), r("D")), ">", 3.0, lambda b, d: (b * 3.0 + d) % 7.0)))}[name]
k = count_star(t, p)
for _ in range(3):
    if mode == "count":
        count_star(t, p)
    else:
        executor.count_and_materialize(t, p, ["A"], k)
torch.cuda.synchronize()
print("ok", k)
