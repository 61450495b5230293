"""ncu driver for one config-3 query (not part of the product): warm-up runs, then ONE Engine.run
inside a cudaProfilerStart/Stop window (ncu --profile-from-start off) for its launch list."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_01488_b200 import Engine, datagen, optimizer, ra, serde, expr as ex
from paper_1901_01488_b200.storage import Column, ColumnTable, Dictionary, parse_kind

dev = torch.device("cuda", 0)
g = datagen.config3(fact_rows=60_000_000)
eng = Engine(optimizer.EscConfig())
names = {"date": "dates"}
for name, cols in g.items():
    eng.catalog.register(ColumnTable(names.get(name, name), [
        Column(k, parse_kind(v[0]), v[1], None, Dictionary(v[2]) if len(v) > 2 else None, device=dev)
        for k, v in cols.items()]))
conj = [ex.ColumnCompare(ex.ColumnRef("fact", a), "=", ex.ColumnRef(names.get(dim, dim), b))
        for _, a, dim, b in datagen.CONFIG3_EDGES]
conj += [serde.from_json(j, names.get(dim, dim)) for dim, j in datagen.CONFIG3_WHERE.items()]
q = ra.query(eng.catalog, ["fact", "dates", "customer", "supplier", "part"], ex.And(tuple(conj)))
for _ in range(5):
    eng.run(q)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
r = eng.run(q)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("count", r.count)
