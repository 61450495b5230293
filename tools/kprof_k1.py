"""ncu driver (not part of the product): config-4-shaped table generated on the device; K1
count-only launches, then ESC steps (K1 select + capture + compaction).
python tools/kprof_k1.py [rows]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_01488_b200 import ColumnTable, count_star, expr as ex, optimizer
from paper_1901_01488_b200.catalog import Catalog
from paper_1901_01488_b200.storage import Column, parse_kind

n = int(sys.argv[1]) if len(sys.argv) > 1 else 600_000_000
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
p = ex.And((ex.Equality(r("A"), 0), ex.Range(r("C"), -0.5, 1.0),
            ex.Or((ex.Equality(r("D"), 17), ex.Comparison(r("D"), ">", 900))),
            ex.FnCall("b3d", (r("B"), r("D")), ">", 3.0, lambda b, d: (b * 3.0 + d) % 7.0)))
cat = Catalog(); cat.register(t)
for _ in range(3): count_star(t, p)                     # K1 count launches 0..2
for _ in range(3):                                      # ESC steps: K1 select launches 3..5
    optimizer.esc_subquery(cat, "t", p, ["A", "C", "D"], optimizer.EscConfig()); cat.temps.sweep()
torch.cuda.synchronize()
print("ok")
