"""Host timeline of one small-table ESC step (config-3 customer dimension; not part of the product)."""
import ctypes as C, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_01488_b200 import datagen, serde, executor as E, _native as N
from paper_1901_01488_b200.compiler import compile_predicate
from paper_1901_01488_b200.storage import Column, ColumnTable, Dictionary, parse_kind

dev = torch.device("cuda", 0)
g = datagen.config3(fact_rows=1)
cols = g["customer"]
t = ColumnTable("customer", [Column(c, parse_kind(s[0]), s[1], None, Dictionary(s[2]) if len(s) > 2 else None,
                                    device=dev) for c, s in cols.items()])
pred = serde.from_json(datagen.CONFIG3_WHERE["customer"], "customer")
needed = ["c_custkey"]
cap = 6000
lib = N.load_library()
marks = {k: [] for k in ("compile", "ensure", "plan", "launch", "sync", "read", "trim", "total")}
for it in range(60):
    t0 = time.perf_counter()
    cp = compile_predicate(t, pred)
    t1 = time.perf_counter()
    stream = E._stream(dev)
    ws = N.workspace(dev, stream)
    ws_ptr, ws_bytes = ws.ensure(t.row_count, stream.cuda_stream)
    t2 = time.perf_counter()
    proj = [t.column(n) for n in needed]
    plan = E._onepass_plan(cp, t, proj, cap, ws)
    t3 = time.perf_counter()
    N.check(lib.esc_compact_onepass(C.byref(cp.program), plan.mat_cols, plan.mat_ncols, t.row_count, None,
                                    C.byref(plan.outs), C.c_void_p(ws.result.data_ptr()), C.c_void_p(ws_ptr),
                                    C.c_size_t(ws_bytes), C.c_void_p(stream.cuda_stream)), "x")
    t4 = time.perf_counter()
    stream.synchronize()
    t5 = time.perf_counter()
    count, fails = ws.read_result(cp.n_udfs)
    t6 = time.perf_counter()
    out = E._trim(proj, plan.out_values, plan.out_nulls, min(count, cap), stream)
    t7 = time.perf_counter()
    if it >= 10:
        for k, a, b in (("compile", t0, t1), ("ensure", t1, t2), ("plan", t2, t3), ("launch", t3, t4),
                        ("sync", t4, t5), ("read", t5, t6), ("trim", t6, t7), ("total", t0, t7)):
            marks[k].append((b - a) * 1e6)
for k, v in marks.items():
    print(f"{k:8s} {statistics.median(v):8.1f} us")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    lib.esc_compact_onepass(C.byref(cp.program), plan.mat_cols, plan.mat_ncols, t.row_count, None, C.byref(plan.outs),
                            C.c_void_p(ws.result.data_ptr()), C.c_void_p(ws_ptr), C.c_size_t(ws_bytes),
                            C.c_void_p(stream.cuda_stream))
e1.record(); torch.cuda.synchronize()
print(f"kernel back-to-back {e0.elapsed_time(e1)/50*1e3:.1f} us per launch")
