"""Host profile of optimizer.plan on the config-3 star (not part of the product)."""
import cProfile, os, pstats, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_01488_b200 import Catalog, datagen, expr as ex, optimizer, ra, serde
from paper_1901_01488_b200.storage import Column, ColumnTable, Dictionary, parse_kind

dev = torch.device("cuda", 0)
g = datagen.config3(fact_rows=1)
cat = Catalog()
names = {"date": "dates"}
for tname, cols in g.items():
    if tname == "fact":
        continue
    cat.register(ColumnTable(names.get(tname, tname), [
        Column(c, parse_kind(s[0]), s[1], None, Dictionary(s[2]) if len(s) > 2 else None, device=dev)
        for c, s in cols.items()]))
fact = torch.ones(60_000_000, dtype=torch.int32, device=dev)
cat.register(ColumnTable("fact", [Column(c, parse_kind("INT32"), fact) for c in
                                  ("f_datekey", "f_custkey", "f_suppkey", "f_partkey")]))
r = ex.ColumnRef
conj = [ex.ColumnCompare(r("fact", a), "=", r(names.get(d, d), b)) for _, a, d, b in datagen.CONFIG3_EDGES]
conj += [serde.from_json(j, names.get(d, d)) for d, j in datagen.CONFIG3_WHERE.items()]
q = ra.query(cat, ["fact", "dates", "customer", "supplier", "part"], ex.And(tuple(conj)))
cfg = optimizer.EscConfig()
for _ in range(5):
    optimizer.plan(q, cat, cfg); cat.temps.sweep()
ov, wall = [], []
for _ in range(30):
    t0 = time.perf_counter()
    p = optimizer.plan(q, cat, cfg)
    wall.append((time.perf_counter() - t0) * 1e3)
    ov.append(optimizer.esc_overhead_ms(p))
    cat.temps.sweep()
print(f"overhead median {statistics.median(ov):.3f} ms, plan wall {statistics.median(wall):.3f} ms")
for d in p.decisions:
    print(d.table, d.exact_count, round(d.subquery_ms, 3), round(d.materialize_ms, 3))
pr = cProfile.Profile(); pr.enable()
for _ in range(30):
    optimizer.plan(q, cat, cfg); cat.temps.sweep()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
