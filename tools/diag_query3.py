"""Config-3 query breakdown (not part of the product): Engine.run wall time split into planning
(ESC), hash builds, factor arrays and the COUNT probe (monkeypatched host timers)."""
import functools, os, statistics, sys, time
from collections import defaultdict
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_01488_b200 import Engine, datagen, join, optimizer, ra, serde, expr as ex
from paper_1901_01488_b200.storage import Column, ColumnTable, Dictionary, parse_kind

dev = torch.device("cuda", 0)
cfg = optimizer.EscConfig()
g = datagen.config3(fact_rows=60_000_000)
eng = Engine(cfg)
names = {"date": "dates"}
for name, cols in g.items():
    eng.catalog.register(ColumnTable(names.get(name, name), [
        Column(k, parse_kind(v[0]), v[1], None, Dictionary(v[2]) if len(v) > 2 else None, device=dev)
        for k, v in cols.items()]))
del g
conj = [ex.ColumnCompare(ex.ColumnRef("fact", a), "=", ex.ColumnRef(names.get(dim, dim), b))
        for _, a, dim, b in datagen.CONFIG3_EDGES]
conj += [serde.from_json(j, names.get(dim, dim)) for dim, j in datagen.CONFIG3_WHERE.items()]
q = ra.query(eng.catalog, ["fact", "dates", "customer", "supplier", "part"], ex.And(tuple(conj)))
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
import paper_1901_01488_b200.engine as E
timed(optimizer, "plan", "plan (ESC + ordering)")
timed(join, "execute_plan", "execute_plan")
timed(join, "build_hash", "  build_hash")
timed(join, "_factor_array", "  _factor_array")
timed(join, "_stage_weights", "  _stage_weights")
timed(join, "_count_pipeline", "  _count_pipeline")
for _ in range(5): eng.run(q)
torch.cuda.synchronize(); acc.clear()
N = 20
walls = []
for _ in range(N):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = eng.run(q); torch.cuda.synchronize()
    walls.append((time.perf_counter() - t0) * 1e3)
print(f"Engine.run median {statistics.median(walls):.3f} ms, count {r.count}")
for k, v in acc.items(): print(f"  {k:28s} {v / N * 1e3:8.3f} ms")

# cProfile of the execution half and the device span of one run
import cProfile, pstats
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); w0 = time.perf_counter(); e0.record(); eng.run(q); e1.record(); torch.cuda.synchronize()
print(f"one run: wall {(time.perf_counter() - w0) * 1e3:.3f} ms, device span {e0.elapsed_time(e1):.3f} ms")
pr = cProfile.Profile(); pr.enable()
for _ in range(50): eng.run(q)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(30)

# build phase split
import paper_1901_01488_b200.join as J
acc.clear()
timed(J, "HashTableIndex", "  HashTableIndex (ctor)")
timed(J.HashTableIndex, "_finish", "  _finish")
from paper_1901_01488_b200 import executor
timed(executor, "eval_predicate", "  eval_predicate")
timed(J, "build_indexes", "build_indexes")
for _ in range(20): eng.run(q)
for k, v in acc.items(): print(f"  {k:28s} {v / 20 * 1e3:8.3f} ms")
