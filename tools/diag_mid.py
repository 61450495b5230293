"""Per-block timeline of one sel_mid_kernel launch on config 2 (esc_debug_trace; diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_1901_01488_b200 import datagen, executor, serde, _native as N
from paper_1901_01488_b200.storage import Column, ColumnTable, Dictionary, parse_kind
dev = torch.device("cuda", 0)
lib = N.load_library()
w2 = datagen.config2()
t2 = ColumnTable("lineitem", [Column(k, parse_kind(v[0]), v[1], None, Dictionary(v[2]) if len(v) > 2 else None,
                                     device=dev) for k, v in w2.columns.items()])
p2 = serde.from_json(w2.pred, "lineitem")
proj = [t2.column(c) for c in w2.project]
for _ in range(3):
    sel = executor.select(t2, p2, capture=w2.project)
    executor.launch_materialize_selection(sel, proj, sel.count, False)
torch.cuda.synchronize()
buf = torch.zeros(8 * 8192, dtype=torch.int64, device=dev)
bench._flush_l2(dev)
sel = executor.select(t2, p2, capture=w2.project)  # L2 flushed before the scan, as in the bench step
lib.esc_debug_trace(buf.data_ptr())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record(); executor.launch_materialize_selection(sel, proj, sel.count, False); e1.record()
torch.cuda.synchronize()
lib.esc_debug_trace(None)
st = buf.view(-1, 8).cpu().numpy().astype(np.int64)[1024:]
st = st[st[:, 1] > 0]
t0 = st[:, 0].min()
rel = (st - t0) / 1e3
print(f"mid kernel: events {e0.elapsed_time(e1)*1e3:.1f} us, blocks {len(st)}, hits {sel.count}")
for k, name in enumerate(["start", "ticket", "published", "offsets", "expanded", "base read", "end"]):
    v = rel[:, k][st[:, k] > 0]
    if len(v): print(f"  {name:12s} min {v.min():7.1f}  med {np.median(v):7.1f}  max {v.max():7.1f} us")
