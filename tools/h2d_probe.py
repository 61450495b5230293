"""H2D bandwidth of pinned host columns (not part of the product): one stream vs several."""
import time, torch
dev = torch.device("cuda", 0)
cols = [torch.empty(600_000_000, dtype=torch.int32).pin_memory() for _ in range(4)]
for c in cols: c.fill_(1)
def run(nstreams):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    torch.cuda.synchronize(); t0 = time.perf_counter()
    outs = []
    for i, c in enumerate(cols):
        s = streams[i % nstreams]
        with torch.cuda.stream(s):
            outs.append(c.to(dev, non_blocking=True))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    return sum(c.numel() * 4 for c in cols) / dt / 1e9
for ns in (1, 2, 4, 1, 2, 4):
    print(ns, f"{run(ns):.1f} GB/s", flush=True)
