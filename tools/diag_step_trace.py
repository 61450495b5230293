"""One config-2 ESC step (K1 select + sel_mid_kernel) with per-CTA %globaltimer stamps of both
kernels on one time axis (esc_debug_trace; L2 flushed before; diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_1901_01488_b200 import datagen, executor, serde, _native as N
from paper_1901_01488_b200.storage import Column, ColumnTable, Dictionary, parse_kind
dev = torch.device("cuda", 0)
lib = N.load_library()
buf = torch.zeros(8 * 8192, dtype=torch.int64, device=dev)
lib.esc_debug_trace(buf.data_ptr())  # before the plan is prepared (plans capture it)
w2 = datagen.config2()
t2 = ColumnTable("lineitem", [Column(k, parse_kind(v[0]), v[1], None, Dictionary(v[2]) if len(v) > 2 else None,
                                     device=dev) for k, v in w2.columns.items()])
p2 = serde.from_json(w2.pred, "lineitem")
cap = int(0.2 * t2.row_count)
for _ in range(3):
    ps = executor.launch_step(t2, p2, w2.project, cap); torch.cuda.synchronize(); executor.finish_step(ps)
buf.zero_()
bench._flush_l2(dev)
torch.cuda._sleep(2_000_000)
ps = executor.launch_step(t2, p2, w2.project, cap)
torch.cuda.synchronize(); executor.finish_step(ps)
lib.esc_debug_trace(None)
st = buf.view(-1, 8).cpu().numpy().astype(np.int64)
k1 = st[:148]; k1 = k1[k1[:, 0] > 0]
mid = st[1024:]; mid = mid[mid[:, 1] > 0]
t0 = k1[:, 0].min()
def show(name, a, names):
    rel = (a - t0) / 1e3
    print(name, len(a))
    for k, nm in enumerate(names):
        v = rel[:, k][a[:, k] > 0]
        if len(v): print(f"  {nm:15s} min {v.min():7.1f}  med {np.median(v):7.1f}  max {v.max():7.1f} us")
show("K1", k1, ["start", "first tile", "consumers done", "producer done", "cta finished", "last: final begin", "last: final end"])
show("mid", mid, ["start", "ticket", "published", "offsets", "expanded", "base read", "end"])
# the slowest mid blocks (block id = ticket order) with their phase stamps
rel = (mid - t0) / 1e3
order = np.argsort(-rel[:, 6])[:6]
blocks = (np.nonzero(st[1024:, 1] > 0)[0])[order]
v = rel[:, 7][mid[:, 7] > 0]
if len(v): print(f"  first word     min {v.min():7.1f}  med {np.median(v):7.1f}  max {v.max():7.1f} us")
print("slowest mid blocks (ticket, start, ticket, published, offsets, expanded, base read, end):")
for b, r in zip(blocks, rel[order]):
    print(f"  {b:5d} " + " ".join(f"{x:6.1f}" for x in r[:7]))
