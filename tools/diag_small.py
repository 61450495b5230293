"""K1 count time vs table size (not part of the product): finds the fixed cost of a scan."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1901_01488_b200 import ColumnTable, count_star, expr as ex, executor
from paper_1901_01488_b200.storage import Column, parse_kind

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(3)
for n in (1_000_000, 3_000_000, 6_000_000, 12_000_000, 24_000_000, 48_000_000, 96_000_000):
    cols = [Column(c, parse_kind("INT32"), torch.randint(0, 100, (n,), generator=g, device=dev, dtype=torch.int32))
            for c in ("x", "y", "z")]
    t = ColumnTable("t", cols)
    r = lambda c: ex.ColumnRef("t", c)
    p = ex.And((ex.Range(r("x"), 10, 50), ex.Range(r("y"), 5, 7), ex.Comparison(r("z"), "<", 24)))
    for _ in range(3): count_star(t, p)
    res = []
    for flush in (False, True):
        tt = bench._time_kernels(lambda: count_star(t, p), 20, dev, flush=flush)
        res.append(statistics.median(x for x, k in tt) * 1e3)
    print(f"n={n:>10d} warm {res[0]:7.1f} us  flushed {res[1]:7.1f} us  -> {n*12/res[1]/1e3:7.1f} GB/s", flush=True)
