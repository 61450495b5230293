"""Host timeline of the queued ESC step as the bench runs it (not part of the product)."""
import os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_01488_b200 import ColumnTable, expr as ex, optimizer, executor as E
from paper_1901_01488_b200.catalog import Catalog
from paper_1901_01488_b200.storage import Column, parse_kind

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
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
marks = {}
def timed(name, fn):
    def w(*a, **k):
        t0 = time.perf_counter(); out = fn(*a, **k); marks.setdefault(name, []).append((time.perf_counter() - t0) * 1e6)
        return out
    return w
E.launch_step = timed("launch_step", E.launch_step)
E.finish_step = timed("finish_step", E.finish_step)
E._trim = timed("trim", E._trim)
E._step_plan = timed("plan", E._step_plan)
E.compile_predicate = timed("compile", E.compile_predicate)
cat.materialize_temp = timed("temp", cat.materialize_temp)
def step():
    d = optimizer.esc_subquery(cat, "t", p, ["A", "C", "D"], cfg)
    t0 = time.perf_counter(); cat.temps.sweep(); marks.setdefault("sweep", []).append((time.perf_counter() - t0) * 1e6)
for _ in range(5): step()
marks.clear()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
E.KERNEL_EVENTS = None
w0 = time.perf_counter(); e0.record()
for _ in range(30):
    t0 = time.perf_counter(); step(); marks.setdefault("step", []).append((time.perf_counter() - t0) * 1e6)
e1.record(); torch.cuda.synchronize()
E.KERNEL_EVENTS = []
for _ in range(10): step()
torch.cuda.synchronize()
ev = E.KERNEL_EVENTS; E.KERNEL_EVENTS = None
sel = statistics.median(a.elapsed_time(b) for a, b, k in ev if k == "select")
mat = statistics.median(a.elapsed_time(b) for a, b, k in ev if k == "materialize")
print(f"device {e0.elapsed_time(e1)/30:.3f} ms/step; select {sel:.3f} mat {mat:.3f} (sum {sel+mat:.3f})")
for k, v in marks.items(): print(f"{k:12s} {statistics.median(v):8.1f} us")
