"""Config-3 ESC overhead breakdown (not part of the product): plan() wall time, the ESC batch's
kernels (events) and a cProfile of the host side."""
import cProfile, os, pstats, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1901_01488_b200 import Engine, datagen, executor, optimizer, ra, serde, expr as ex
from paper_1901_01488_b200.storage import Column, ColumnTable, Dictionary, parse_kind

dev = torch.device("cuda", 0)
cfg = optimizer.EscConfig()
g = datagen.config3(fact_rows=int(sys.argv[1]) if len(sys.argv) > 1 else 6_000_000)
eng = Engine(cfg)
names = {"date": "dates"}
for name, cols in g.items():
    eng.catalog.register(ColumnTable(names.get(name, name), [
        Column(k, parse_kind(v[0]), v[1], None, Dictionary(v[2]) if len(v) > 2 else None, device=dev)
        for k, v in cols.items()]))
conj = [ex.ColumnCompare(ex.ColumnRef("fact", a), "=", ex.ColumnRef(names.get(dim, dim), b))
        for _, a, dim, b in datagen.CONFIG3_EDGES]
conj += [serde.from_json(j, names.get(dim, dim)) for dim, j in datagen.CONFIG3_WHERE.items()]
q = ra.query(eng.catalog, ["fact", "dates", "customer", "supplier", "part"], ex.And(tuple(conj)))
import functools
from collections import defaultdict
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
from paper_1901_01488_b200.catalog import Catalog
timed(executor, "launch_step", "launch_step")
timed(executor, "_onepass_plan", "  _onepass_plan")
timed(executor, "compile_predicate", "  compile_predicate")
timed(executor, "finish_step", "finish_step")
timed(executor, "_take_outputs", "  _take_outputs")
timed(optimizer, "_esc_batch", "_esc_batch")
timed(optimizer, "build_join_graph", "build_join_graph")
timed(optimizer, "order_builds", "order_builds")
timed(Catalog, "materialize_temp", "materialize_temp")
timed(torch.cuda.Stream, "synchronize", "stream sync (wait)")
def once():
    p = optimizer.plan(q, eng.catalog, cfg)
    eng.catalog.temps.sweep()
    return p
for _ in range(10): once()
acc.clear()
walls, ovs = [], []
for _ in range(50):
    torch.cuda.synchronize(); t0 = time.perf_counter(); p = once(); walls.append((time.perf_counter() - t0) * 1e6)
    ovs.append(optimizer.esc_overhead_ms(p) * 1e3)
print(f"plan wall median {statistics.median(walls):.1f} us, esc overhead median {statistics.median(ovs):.1f} us")
for k, v in acc.items(): print(f"  {k:24s} {v/50*1e6:8.1f} us per plan")
executor.KERNEL_EVENTS = []
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); once(); e1.record(); torch.cuda.synchronize()
print(f"device span of one plan(): {e0.elapsed_time(e1)*1e3:.1f} us")
for a, b, k in executor.KERNEL_EVENTS: print(f"   {k:12s} {a.elapsed_time(b)*1e3:7.1f} us  (start +{e0.elapsed_time(a)*1e3:6.1f})")
executor.KERNEL_EVENTS = None
pr = cProfile.Profile(); pr.enable()
for _ in range(100): once()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(35)
