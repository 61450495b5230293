"""Count-only K1 time vs ring stages for a few row widths (not part of the product).
ESC_STAGES caps the stage count; run once per setting."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_01488_b200 import ColumnTable, count_star, executor, expr as ex
from paper_1901_01488_b200.storage import Column, parse_kind
n = 400_000_000
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(3)
i32 = lambda: torch.randint(0, 1_000_000, (n,), generator=g, device=dev, dtype=torch.int32)
cases = {}
a, b = i32(), i32()
t1 = ColumnTable("t", [Column("a", parse_kind("INT32"), a)])
cases["i32x1"] = (t1, ex.Range(ex.ColumnRef("t", "a"), 0, 9999), 4)
t2 = ColumnTable("t", [Column("a", parse_kind("INT32"), a), Column("b", parse_kind("INT32"), b)])
cases["i32x2"] = (t2, ex.And((ex.Range(ex.ColumnRef("t", "a"), 0, 99999), ex.Range(ex.ColumnRef("t", "b"), 0, 99999))), 8)
del b
c8 = torch.randint(0, 100, (n,), generator=g, device=dev, dtype=torch.int8)
t3 = ColumnTable("t", [Column("c", parse_kind("INT8"), c8)])
cases["i8x1"] = (t3, ex.Range(ex.ColumnRef("t", "c"), 0, 9), 1)
out = {}
for name, (t, p, w) in cases.items():
    for _ in range(2): count_star(t, p)
    executor.KERNEL_EVENTS = []
    for _ in range(7): count_star(t, p)
    torch.cuda.synchronize()
    ms = statistics.median(x.elapsed_time(y) for x, y, _ in executor.KERNEL_EVENTS)
    executor.KERNEL_EVENTS = None
    out[name] = (round(ms, 4), round(n * w / ms / 1e6))
print(json.dumps({"stages": os.environ.get("ESC_STAGES", "default"), "res": out}))
