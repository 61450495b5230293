"""ncu driver: K1 count-only over the config-5 single-range shape (600M int32 c0), not part of the product."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_01488_b200 import ColumnTable, count_star, expr as ex
from paper_1901_01488_b200.storage import Column, parse_kind
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(5)
c0 = torch.randint(0, 1_000_000, (600_000_000,), generator=g, device=dev, dtype=torch.int32)
t = ColumnTable("t", [Column("c0", parse_kind("INT32"), c0)])
p = ex.Range(ex.ColumnRef("t", "c0"), 0, 99_999)
for _ in range(4):
    count_star(t, p)
torch.cuda.synchronize()
print("ok")
