"""Per-kernel timing of the selection compaction routes (not part of the product).
Usage: python tools/diag_compact.py [rows]"""
import json, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_01488_b200 import ColumnTable, executor, expr as ex, _native as N
from paper_1901_01488_b200.storage import Column, parse_kind

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(5)
c0 = torch.randint(0, 1_000_000, (n,), generator=g, device=dev, dtype=torch.int32)
c1 = torch.randint(0, 1_000_000, (n,), generator=g, device=dev, dtype=torch.int32)
c4 = torch.randint(0, 10**12, (n,), generator=g, device=dev, dtype=torch.int64)
t = ColumnTable("t", [Column("c0", parse_kind("INT32"), c0), Column("c1", parse_kind("INT32"), c1),
                      Column("c4", parse_kind("INT64"), c4)])
out = {}
for div in [int(x) for x in os.environ.get("DIVS", "32,0").split(",")]:
    N.set_stream_div(div)
    for s in (0.002, 0.05, 0.1, 0.5, 0.9):
        p = ex.Range(ex.ColumnRef("t", "c0"), 0, int(s * 1e6) - 1)
        for _ in range(2):
            executor.count_and_materialize(t, p, ["c0", "c1", "c4"], n)
        torch.cuda.synchronize()
        executor.KERNEL_EVENTS = []
        w0 = time.perf_counter()
        for _ in range(3):
            executor.count_and_materialize(t, p, ["c0", "c1", "c4"], n)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - w0) / 3 * 1e3
        ev = executor.KERNEL_EVENTS
        executor.KERNEL_EVENTS = None
        sel = statistics.median(a.elapsed_time(b) for a, b, k in ev if k == "select")
        mat = statistics.median(a.elapsed_time(b) for a, b, k in ev if k == "materialize")
        out[f"div{div}_s{s}"] = {"select_ms": round(sel, 3), "materialize_ms": round(mat, 3), "wall_ms": round(wall, 3)}
        print(f"div={div} s={s}: select {sel:.3f} ms, materialize {mat:.3f} ms, wall {wall:.3f} ms", flush=True)
print(json.dumps({"rows": n, "res": out}))
