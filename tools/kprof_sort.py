"""ncu driver for the device radix sort (not part of the product): 100M u64 keys + u64 values
(python tools/kprof_sort.py [n] [u32])."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_01488_b200 import sorting
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
dev = torch.device("cuda", 0)
if len(sys.argv) > 2 and sys.argv[2] == "u32":
    k = torch.randint(0, 1 << 31, (n,), device=dev, dtype=torch.int32)
else:
    k = torch.randint(-(1 << 62), 1 << 62, (n,), device=dev)
v = torch.arange(n, device=dev)
for _ in range(2):
    sorting.sort_pairs(k, v)
torch.cuda.synchronize()
print("ok")
