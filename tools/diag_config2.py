"""Config-2 step breakdown (not part of the product): device time of the ESC sub-query on the
exact 6M-row recipe, with and without an L2 flush, and its kernels."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1901_01488_b200 import datagen, executor, optimizer, serde, count_star, _native as N
from paper_1901_01488_b200.catalog import Catalog
from paper_1901_01488_b200.storage import Column, ColumnTable, Dictionary, parse_kind

dev = torch.device("cuda", 0)
w2 = datagen.config2()
t2 = ColumnTable("lineitem", [Column(k, parse_kind(v[0]), v[1], None, Dictionary(v[2]) if len(v) > 2 else None,
                                     device=dev) for k, v in w2.columns.items()])
c2 = Catalog(); c2.register(t2)
p2 = serde.from_json(w2.pred, "lineitem")
cfg = optimizer.EscConfig()
step = lambda: (optimizer.esc_subquery(c2, "lineitem", p2, w2.project, cfg), c2.temps.sweep())
for _ in range(5): step()
for flush in (False, True):
    tt = bench._time_kernels(step, 20, dev, flush=flush)
    by = {}
    for x, k in tt: by.setdefault(k, []).append(x)
    print("flush" if flush else "warm ", {k: round(statistics.median(v) * 1e3, 1) for k, v in by.items()}, "us")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    xs = []
    for _ in range(20):
        if flush: bench._flush_l2(dev)
        torch.cuda.synchronize(); e0.record(); step(); e1.record(); torch.cuda.synchronize()
        xs.append(e0.elapsed_time(e1) * 1e3)
    print("   whole step (events, incl host gaps)", round(statistics.median(xs), 1), "us")
for _ in range(3): count_star(t2, p2)
tt = bench._time_kernels(lambda: count_star(t2, p2), 20, dev, flush=True)
print("count_star flush", round(statistics.median(x for x, k in tt) * 1e3, 1), "us")
print("launches/step", end=" ")
a = N.load_library().esc_launch_count(); step(); torch.cuda.synchronize(); print(N.load_library().esc_launch_count() - a)
print("onepass max rows", executor.ONEPASS_MAX_ROWS, "rows", t2.row_count)
