"""One K1 count at a given size (for ncu; not part of the product)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_01488_b200 import ColumnTable, count_star, expr as ex
from paper_1901_01488_b200.storage import Column, parse_kind
dev = torch.device("cuda", 0)
n = int(sys.argv[1])
g = torch.Generator(device=dev); g.manual_seed(3)
cols = [Column(c, parse_kind("INT32"), torch.randint(0, 100, (n,), generator=g, device=dev, dtype=torch.int32))
        for c in ("x", "y", "z")]
t = ColumnTable("t", cols)
r = lambda c: ex.ColumnRef("t", c)
p = ex.And((ex.Range(r("x"), 10, 50), ex.Range(r("y"), 5, 7), ex.Comparison(r("z"), "<", 24)))
for _ in range(4): count_star(t, p)
torch.cuda.synchronize()
