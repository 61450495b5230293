"""Host time per ESC step on a config-4-shaped table (not part of the product): wall vs device,
and how the host time splits over the step's Python phases (monkeypatched timers)."""
import functools, os, statistics, sys, time
from collections import defaultdict
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_01488_b200 import ColumnTable, expr as ex, optimizer, executor, catalog as catmod
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
acc = defaultdict(float)
def timed(mod, name, label):
    f = getattr(mod, name)
    @functools.wraps(f)
    def w(*a, **k):
        t0 = time.perf_counter()
        try:
            return f(*a, **k)
        finally:
            acc[label] += time.perf_counter() - t0
    setattr(mod, name, w)
timed(executor, "launch_step", "launch_step")
timed(executor, "finish_step", "finish_step")
timed(executor, "_trim", "  _trim")
timed(executor, "compile_predicate", "  compile_predicate")
timed(executor, "_step_plan", "  _step_plan")
timed(executor, "raise_udf_errors", "  raise_udf_errors")
timed(torch.cuda.Stream, "synchronize", "stream sync (wait)")
timed(Catalog, "materialize_temp", "materialize_temp")
def step():
    d = optimizer.esc_subquery(cat, "t", p, ["A", "C", "D"], cfg)
    cat.temps.sweep()
    return d
for _ in range(10): step()
torch.cuda.synchronize()
acc.clear()
N = 100
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
w0 = time.perf_counter(); e0.record()
for _ in range(N): step()
e1.record(); torch.cuda.synchronize()
wall = (time.perf_counter() - w0) / N * 1e6
print(f"n={n}: wall {wall:.1f} us/step, device span {e0.elapsed_time(e1)/N*1e3:.1f} us/step")
for k, v in acc.items(): print(f"  {k:24s} {v/N*1e6:8.1f} us")
executor.KERNEL_EVENTS = []
for _ in range(20): step()
torch.cuda.synchronize()
by = defaultdict(list)
for a, b, k in executor.KERNEL_EVENTS: by[k].append(a.elapsed_time(b) * 1e3)
executor.KERNEL_EVENTS = None
print("  kernels:", {k: round(statistics.median(v), 1) for k, v in by.items()})
