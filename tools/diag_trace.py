"""Per-CTA timeline of one K1 launch (esc_debug_trace; not part of the product)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1901_01488_b200 import ColumnTable, count_star, expr as ex, _native as N
from paper_1901_01488_b200.storage import Column, parse_kind
dev = torch.device("cuda", 0)
lib = N.load_library()
for n in [int(a) for a in sys.argv[1:]] or [1_000_000, 6_000_000, 96_000_000]:
    g = torch.Generator(device=dev); g.manual_seed(3)
    cols = [Column(c, parse_kind("INT32"), torch.randint(0, 100, (n,), generator=g, device=dev, dtype=torch.int32))
            for c in ("x", "y", "z")]
    t = ColumnTable("t", cols)
    r = lambda c: ex.ColumnRef("t", c)
    p = ex.And((ex.Range(r("x"), 10, 50), ex.Range(r("y"), 5, 7), ex.Comparison(r("z"), "<", 24)))
    for _ in range(3): count_star(t, p)
    buf = torch.zeros(8 * 1024, dtype=torch.int64, device=dev)
    lib.esc_debug_trace(C_ptr := buf.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(); count_star(t, p); e1.record(); torch.cuda.synchronize()
    lib.esc_debug_trace(None)
    st = buf.view(-1, 8).cpu().numpy().astype(np.int64)
    st = st[st[:, 0] > 0]
    t0 = st[:, 0].min()
    rel = (st - t0) / 1e3
    print(f"n={n} events {e0.elapsed_time(e1)*1e3:.1f} us, ctas {len(st)}")
    for k, name in enumerate(["start", "first tile", "consumers done", "producer done", "cta finished",
                              "last: final begin", "last: final end"]):
        v = rel[:, k][st[:, k] > 0]
        if not len(v): continue
        print(f"  {name:15s} min {v.min():7.1f}  med {np.median(v):7.1f}  max {v.max():7.1f} us")
    late = np.argsort(-rel[:, 2])[:5]
    print("  slowest CTAs:", [(int(i), [round(x, 1) for x in rel[i]]) for i in late])
