"""One-pass ESC step on small tables (not part of the product): event time of the launch and
the per-CTA timeline (esc_debug_trace)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_1901_01488_b200 import ColumnTable, expr as ex, executor, _native as N
from paper_1901_01488_b200.storage import Column, parse_kind
dev = torch.device("cuda", 0)
lib = N.load_library()
for n in (2556, 30000, 200000, 2000000):
    g = torch.Generator(device=dev); g.manual_seed(3)
    t = ColumnTable("t", [Column("k", parse_kind("INT32"), torch.arange(n, dtype=torch.int32, device=dev)),
                          Column("r", parse_kind("INT32"), torch.randint(0, 25, (n,), generator=g, device=dev, dtype=torch.int32))])
    p = ex.Range(ex.ColumnRef("t", "r"), 3, 4)
    step = lambda: executor.count_and_materialize(t, p, ["k"], n)
    for _ in range(5): step()
    tt = bench._time_kernels(step, 20, dev)
    ms = [x for x, k in tt]
    buf = torch.zeros(8 * 1024, dtype=torch.int64, device=dev)
    lib.esc_debug_trace(buf.data_ptr()); step(); torch.cuda.synchronize(); lib.esc_debug_trace(None)
    st = buf.view(-1, 8).cpu().numpy().astype(np.int64)
    st = st[st[:, 0] > 0]
    rel = (st - st[:, 0].min()) / 1e3
    desc = []
    for k, name in enumerate(["start", "first", "writers done", "prod done", "finished", "final0", "final1"]):
        v = rel[:, k][st[:, k] > 0]
        if len(v): desc.append(f"{name} {np.median(v):.1f}/{v.max():.1f}")
    print(f"n={n:>8d} launch-bracket {statistics.median(ms)*1e3:6.1f} us | ctas {len(st)} | " + ", ".join(desc), flush=True)

# host cost of re-issuing a prepared one-pass launch, and the device time per launch back to back
import ctypes as C, time
n = 2556
t = ColumnTable("t", [Column("k", parse_kind("INT32"), torch.arange(n, dtype=torch.int32, device=dev)),
                      Column("r", parse_kind("INT32"), torch.randint(0, 25, (n,), device=dev, dtype=torch.int32))])
p = ex.Range(ex.ColumnRef("t", "r"), 3, 4)
executor.count_and_materialize(t, p, ["k"], n)
ps = executor.launch_step(t, p, ["k"], n, slot=1)
torch.cuda.synchronize()
from paper_1901_01488_b200.compiler import compile_predicate
cp = compile_predicate(t, p)
h = list(cp.c_plans.values())[0]
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(100): lib.esc_step_plan_launch(C.c_void_p(h.ptr), 3, sp)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
w0 = time.perf_counter(); e0.record()
for _ in range(1000): lib.esc_step_plan_launch(C.c_void_p(h.ptr), 3, sp)
w1 = time.perf_counter(); e1.record(); torch.cuda.synchronize()
print(f"one-pass re-issue: host {(w1-w0)*1e3:.2f} us/launch, device {e0.elapsed_time(e1):.2f} us/launch back to back")
# K1 count on the same tiny table, host issue cost through the public path
from paper_1901_01488_b200 import count_star
for _ in range(10): count_star(t, p)
w0 = time.perf_counter()
for _ in range(200): count_star(t, p)
print(f"count_star tiny: {(time.perf_counter()-w0)/200*1e6:.1f} us wall per call (incl. sync)")
