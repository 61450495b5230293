"""Host timeline of one ESC step (not part of the product): where the GPU waits for Python."""
import os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_01488_b200 import ColumnTable, expr as ex, optimizer, executor as E, _native as N
from paper_1901_01488_b200.catalog import Catalog
from paper_1901_01488_b200.compiler import compile_predicate
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
needed = ["A", "C", "D"]
cap = n // 5
marks = {k: [] for k in ("compile", "select_launch", "mat_launch", "sync", "trim", "temp")}
def step():
    t0 = time.perf_counter()
    cp = compile_predicate(t, p)
    t1 = time.perf_counter()
    ws = N.workspace(dev, torch.cuda.current_stream())
    _, _, sel = E.launch_select(cp, t, None, n, capture=needed, sync=False, d_count=ws.dcount)
    t2 = time.perf_counter()
    proj = [t.column(c) for c in needed]
    vals, nulls, _ = E.launch_materialize_selection(sel, proj, cap, want_row_ids=False, skip_over_capacity=True)
    t3 = time.perf_counter()
    count, fails = E.finish_select(sel, cp)
    t4 = time.perf_counter()
    cols = [v[:count].clone() for v in vals]
    t5 = time.perf_counter()
    h = cat.materialize_temp([Column(c.name, c.kind, v) for c, v in zip(proj, cols)])
    cat.temps.sweep()
    t6 = time.perf_counter()
    for k, a, b in (("compile", t0, t1), ("select_launch", t1, t2), ("mat_launch", t2, t3), ("sync", t3, t4),
                    ("trim", t4, t5), ("temp", t5, t6)):
        marks[k].append((b - a) * 1e6)
for _ in range(5): step()
for k in marks: marks[k].clear()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(30): step()
e1.record(); torch.cuda.synchronize()
print(f"device {e0.elapsed_time(e1)/30:.3f} ms/step")
for k, v in marks.items(): print(f"{k:14s} median {statistics.median(v):8.1f} us")
t0 = time.perf_counter()
for _ in range(30): optimizer.esc_subquery(cat, "t", p, needed, cfg); cat.temps.sweep()
torch.cuda.synchronize()
print(f"esc_subquery wall {(time.perf_counter()-t0)/30*1e3:.3f} ms/step")
