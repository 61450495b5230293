"""Cold-L2 floors for a mid-size scan (diagnostics): device time of torch reads/copies of the
config-2 predicate bytes (72 MB) after an L2 flush, next to the ESC kernels."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
dev = torch.device("cuda", 0)
for mb in (24, 72, 288):
    n = mb * 2**20 // 4
    x = torch.randint(0, 100, (n,), dtype=torch.int32, device=dev)
    y = torch.empty_like(x)
    for name, fn in (("sum", lambda: x.sum()), ("copy", lambda: y.copy_(x)), ("count(x<50)", lambda: (x < 50).sum())):
        ts = []
        for _ in range(10):
            bench._flush_l2(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        print(f"{mb} MB {name:12s} {statistics.median(ts):7.1f} us  ({mb * 2**20 / statistics.median(ts) / 1e6:.2f} TB/s read)")
