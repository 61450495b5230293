"""K1 select time vs the number of captured columns (not part of the product): config-4-shaped
table on the device, ESC steps projecting 3 / 2 / 1 / 0 predicate columns."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
from paper_1901_01488_b200 import ColumnTable, expr as ex, optimizer
from paper_1901_01488_b200.catalog import Catalog
from paper_1901_01488_b200.storage import Column, parse_kind
n = 600_000_000
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(1)
A = torch.randint(1, 1000, (n,), generator=g, device=dev, dtype=torch.int32); A[torch.rand(n, generator=g, device=dev) < 0.095] = 0
B = torch.randint(-5, 1005, (n,), generator=g, device=dev, dtype=torch.int32)
Cc = torch.randn(n, generator=g, device=dev, dtype=torch.float32)
D = torch.randint(0, 1000, (n,), generator=g, device=dev, dtype=torch.int32)
E = torch.randint(0, 1000, (n,), generator=g, device=dev, dtype=torch.int32)  # a non-predicate column
t = ColumnTable("t", [Column("A", parse_kind("INT32"), A), Column("B", parse_kind("INT32"), B),
                      Column("C", parse_kind("FLOAT32"), Cc), Column("D", parse_kind("INT32"), D), Column("E", parse_kind("INT32"), E)])
r = lambda c: ex.ColumnRef("t", c)
p = ex.And((ex.Equality(r("A"), 0), ex.Range(r("C"), -0.5, 1.0), ex.Or((ex.Equality(r("D"), 17), ex.Comparison(r("D"), ">", 900))),
            ex.FnCall("b3d", (r("B"), r("D")), ">", 3.0, lambda b, d: (b * 3.0 + d) % 7.0)))
cat = Catalog(); cat.register(t)
cfg = optimizer.EscConfig()
for proj in (["A", "C", "D"], ["A", "C"], ["A"], ["E"]):
    step = lambda: (optimizer.esc_subquery(cat, "t", p, proj, cfg), cat.temps.sweep())
    for _ in range(3): step()
    tt = bench._time_kernels(step, 8, dev)
    sel = statistics.median(x for x, k in tt if k == "select")
    mat = statistics.median(x for x, k in tt if k == "materialize")
    print(proj, f"select {sel:.4f} ms  materialize {mat:.4f} ms", flush=True)
