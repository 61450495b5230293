"""Host-side overhead of the ESC step (not part of the product): cProfile of repeated
optimizer.esc_subquery calls on a config-4-shaped device table."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_01488_b200 import ColumnTable, expr as ex, optimizer
from paper_1901_01488_b200.catalog import Catalog
from paper_1901_01488_b200.storage import Column, parse_kind

n = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000_000
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
cfg = optimizer.EscConfig()
def step():
    d = optimizer.esc_subquery(cat, "t", p, ["A", "C", "D"], cfg)
    cat.temps.sweep()
    return d
for _ in range(5): step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
N = 50
w0 = time.perf_counter(); e0.record()
for _ in range(N): step()
e1.record(); torch.cuda.synchronize()
print(f"wall {((time.perf_counter()-w0)/N)*1e3:.3f} ms/step, device {e0.elapsed_time(e1)/N:.3f} ms/step")
pr = cProfile.Profile(); pr.enable()
for _ in range(N): step()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
