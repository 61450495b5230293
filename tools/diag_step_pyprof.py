"""Python profile of the single-GPU ESC step's host path (config-4 recipe, default 75M rows):
cProfile over 200 steps, top functions by own time, plus the step's event time and host wall.
Usage: diag_step_pyprof.py [rows] [sharded]"""
import cProfile
import os
import pstats
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1901_01488_b200 import datagen, optimizer, serde
from paper_1901_01488_b200.catalog import Catalog
from paper_1901_01488_b200.storage import Column, ColumnTable, parse_kind

n = int(sys.argv[1]) if len(sys.argv) > 1 else 75_000_000
dev = torch.device("cuda", 0)
w = datagen.config4_blocked(n, 0, n)
t = ColumnTable("t", [Column(k, parse_kind(w.columns[k][0]), w.columns[k][1], device=dev) for k in "ABCD"])
pred = serde.from_json(w.pred, "t", w.udfs)
cfg = optimizer.EscConfig()
cat = Catalog()
cat.register(t)


def step():
    optimizer.esc_subquery(cat, "t", pred, w.project, cfg)
    cat.temps.sweep()


for _ in range(10):
    step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
walls = []
e0.record()
for _ in range(50):
    a = time.perf_counter()
    step()
    walls.append((time.perf_counter() - a) * 1e6)
e1.record()
torch.cuda.synchronize()
print(f"step {e0.elapsed_time(e1) / 50 * 1e3:.1f} us (events), host wall per step {statistics.median(walls):.1f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    step()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(30)
st.sort_stats("cumulative").print_stats(25)

# sections of the step without the profiler (medians over 100 steps, us)
from paper_1901_01488_b200 import executor

secs = {"launch": [], "wait": [], "finish": [], "register": [], "sweep": []}
prepared = ("t", t, pred, list(w.project), n, True, (1 * n) // 5)
for i in range(120):
    a = time.perf_counter()
    ps = executor.launch_step(t, pred, list(w.project), (1 * n) // 5, materialize=True, slot=1)
    b = time.perf_counter()
    executor._stream(dev).synchronize()
    c = time.perf_counter()
    count, cols = executor.finish_step(ps)
    d = time.perf_counter()
    cat.materialize_temp(cols)
    e = time.perf_counter()
    cat.temps.sweep()
    f = time.perf_counter()
    if i >= 20:
        for k, v in zip(secs, (b - a, c - b, d - c, e - d, f - e)):
            secs[k].append(v * 1e6)
print("sections (us):", {k: round(statistics.median(v), 1) for k, v in secs.items()})

# the host functions of one step, each timed by a wrapper (medians over 100 steps, us)
import functools

from paper_1901_01488_b200 import _native as N, compiler
from paper_1901_01488_b200 import storage

parts = {}


def timed(mod, name):
    f = getattr(mod, name)

    @functools.wraps(f)
    def g(*a, **k):
        t0 = time.perf_counter()
        r = f(*a, **k)
        parts.setdefault(f"{getattr(mod, '__name__', type(mod).__name__).rsplit('.', 1)[-1]}.{name}", []).append((time.perf_counter() - t0) * 1e6)
        return r

    setattr(mod, name, g)


for mod, name in ((executor, "compile_predicate"), (N, "workspace"), (executor, "_step_plan"),
                  (executor, "_take_outputs"), (executor, "raise_udf_errors"), (executor, "_plan_lend")):
    timed(mod, name)
timed(cat, "materialize_temp")
for i in range(120):
    step()
print("functions (us):", {k: round(statistics.median(v[20:]), 2) for k, v in parts.items()})
