"""ncu driver (not part of the product): K1 on the config-4 recipe (150M rows), count-only then
select (the ESC step's scan), each after warm-ups — compare the two modes' launches."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_01488_b200 import count_star, datagen, executor, serde
from paper_1901_01488_b200.storage import Column, ColumnTable, parse_kind
n = 150_000_000
dev = torch.device("cuda", 0)
w = datagen.config4_blocked(n, 0, n)
t = ColumnTable("t", [Column(k, parse_kind(w.columns[k][0]), w.columns[k][1], device=dev) for k in "ABCD"])
pred = serde.from_json(w.pred, "t", w.udfs)
cap = n // 5
for _ in range(3):
    count_star(t, pred)
    ps = executor.launch_step(t, pred, w.project, cap); torch.cuda.synchronize(); executor.finish_step(ps)
torch.cuda.synchronize()
count_star(t, pred)                       # launch 7 of esc_scan_kernel: count
ps = executor.launch_step(t, pred, w.project, cap); torch.cuda.synchronize(); executor.finish_step(ps)  # 8: select
print("ok")
