import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1901_01488_b200 import Catalog, ColumnTable, expr as ex, optimizer, executor, count_star
from paper_1901_01488_b200.storage import KIND_INT32, KIND_INT64, Column
dev = torch.device("cuda", 0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_003
g = np.random.default_rng(8 + n)
x = g.integers(0, 100_000, n).astype(np.int32)
y = g.integers(-(1 << 40), 1 << 40, n).astype(np.int64)
yn = g.random(n) < 0.05
print("zeros at", np.flatnonzero(x == 0)[:5], "ONEPASS", executor.ONEPASS_MAX_ROWS)
full = ColumnTable("t", [Column("x", KIND_INT32, x, device=dev), Column("y", KIND_INT64, y, yn, device=dev)])
cat = Catalog(); cat.register(full)
cfg = optimizer.EscConfig()
bad = ex.FnCall("inv", (ex.ColumnRef("t", "x"),), ">", 0.5, lambda v: 1.0 / v)
for what, fn in (("count", lambda: count_star(full, bad)), ("esc", lambda: optimizer.esc_subquery(cat, "t", bad, ["x"], cfg))):
    try:
        r = fn(); print(what, "no error", getattr(r, "exact_count", r))
    except Exception as e:
        print(what, type(e).__name__, e)
for hi_x in (99, 9_999, 29_999):
    p = ex.Range(ex.ColumnRef("t", "x"), 0, hi_x)
    ref = optimizer.esc_subquery(cat, "t", p, ["y", "x"], cfg); cat.temps.sweep()
    print("range", hi_x, ref.exact_count)
for what, fn in (("count", lambda: count_star(full, bad)), ("esc", lambda: optimizer.esc_subquery(cat, "t", bad, ["x"], cfg))):
    try:
        r = fn(); print(what, "no error", getattr(r, "exact_count", r))
    except Exception as e:
        print(what, type(e).__name__, e)
