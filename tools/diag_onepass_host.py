"""Line-level host cost of the one-pass ESC launch (not part of the product): the statements of
executor.launch_step's one-pass branch timed one by one on a 30K-row table."""
import ctypes as C, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_01488_b200 import ColumnTable, executor as E, expr as ex, _native as N
from paper_1901_01488_b200.compiler import compile_predicate
from paper_1901_01488_b200.storage import Column, parse_kind
dev = torch.device("cuda", 0)
n = 30000
t = ColumnTable("t", [Column("k", parse_kind("INT32"), torch.arange(n, dtype=torch.int32, device=dev)),
                      Column("r", parse_kind("INT32"), torch.randint(0, 25, (n,), device=dev, dtype=torch.int32))])
p = ex.Range(ex.ColumnRef("t", "r"), 3, 4)
for _ in range(20): E.count_and_materialize(t, p, ["k"], n // 5)
torch.cuda.synchronize()
marks = {}
def mark(k, t0):
    t1 = time.perf_counter(); marks.setdefault(k, []).append((t1 - t0) * 1e6); return t1
for _ in range(300):
    t0 = time.perf_counter()
    cp = compile_predicate(t, p); t0 = mark("compile", t0)
    lib = N.load_library(); stream = E._stream(t.device); t0 = mark("lib+stream", t0)
    ws = N.workspace(t.device, stream); ws_ptr, ws_bytes = ws.ensure(n, stream.cuda_stream); t0 = mark("workspace", t0)
    res = C.c_void_p(ws.result_ptr(1)); sp = C.c_void_p(stream.cuda_stream); t0 = mark("ptrs", t0)
    proj = [t.column("k")]; cap = n // 5; t0 = mark("proj", t0)
    plan = E._onepass_plan(cp, t, proj, cap, ws); t0 = mark("_onepass_plan", t0)
    ckey = (plan.key[3:], n, 1, ws_ptr, N.TUNING[0]); handle = cp.c_plans.get(ckey); t0 = mark("ckey", t0)
    N.check(lib.esc_step_plan_rebind(C.c_void_p(handle.ptr), C.byref(plan.outs)), "rebind"); t0 = mark("rebind", t0)
    N.check(lib.esc_step_plan_launch(C.c_void_p(handle.ptr), 3, sp), "launch"); t0 = mark("launch", t0)
    ps = E.PendingStep(t, cp, proj, cap, "onepass", 1, plan); t0 = mark("PendingStep", t0)
    stream.synchronize(); t0 = mark("sync", t0)
    out = E.finish_step(ps); t0 = mark("finish_step", t0)
for k, v in marks.items(): print(f"{k:14s} {statistics.median(v):7.2f} us")
