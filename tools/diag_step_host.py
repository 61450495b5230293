"""Host-side anatomy of one ESC step at the 8-GPU shard size (75M rows of config 4): the
single-GPU step vs the sharded step in a one-rank NCCL group.  Prints where host time goes
(launch / wait / finish) and the device time of the step's kernels.  Diagnostics."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
from paper_1901_01488_b200 import datagen, executor, multigpu, optimizer, serde
from paper_1901_01488_b200.catalog import Catalog
from paper_1901_01488_b200.storage import Column, ColumnTable, parse_kind
import bench
n = int(sys.argv[1]) if len(sys.argv) > 1 else 75_000_000
dev = torch.device("cuda", 0); torch.cuda.set_device(0)
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(bench._free_port()))
dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
w = datagen.config4_blocked(n, 0, n)
t = ColumnTable("t", [Column(k, parse_kind(w.columns[k][0]), w.columns[k][1], device=dev) for k in "ABCD"])
pred = serde.from_json(w.pred, "t", w.udfs)
cfg = optimizer.EscConfig()
cat = Catalog(); cat.register(t)
st = multigpu.ShardedTable("t", t, n, 0, 0, 1)
def single():
    d = optimizer.esc_subquery(cat, "t", pred, w.project, cfg); cat.temps.sweep(); return d
def sharded():
    return multigpu.sharded_esc_subquery(st, pred, w.project, cfg)
for name, fn in (("single", single), ("sharded", sharded)):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    walls = []
    e0.record()
    for _ in range(20):
        t0 = time.perf_counter(); fn(); walls.append((time.perf_counter() - t0) * 1e6)
    e1.record(); torch.cuda.synchronize()
    print(f"{name:8s} step {e0.elapsed_time(e1) / 20 * 1e3:7.1f} us (events), host wall per call {statistics.median(walls):7.1f} us")
# where the sharded step's host time goes (sections of multigpu.esc_batch, no profiler)
from fractions import Fraction
tt = st.table()
gcap = (1 * n) // 5
secs = {"prep": [], "launch": [], "wait": [], "finish": [], "register": []}
scratch = Catalog()
for i in range(40):
    torch.cuda.synchronize()
    a = time.perf_counter()
    it = multigpu._Launched("t", tt, pred, list(w.project), n, True, gcap, min(gcap, tt.row_count))
    b = time.perf_counter()
    multigpu._launch(it, 1)
    c = time.perf_counter()
    executor._stream(dev).synchronize()
    d = time.perf_counter()
    local, counts, cols = multigpu._finish(it)
    e = time.perf_counter()
    scratch.materialize_temp(cols); scratch.temps.sweep()
    f = time.perf_counter()
    if i >= 10:
        for k, v in zip(secs, (b - a, c - b, d - c, e - d, f - e)):
            secs[k].append(v * 1e6)
print("sharded sections (us):", {k: round(statistics.median(v), 1) for k, v in secs.items()})
# inside _finish: the pieces it calls (timed by wrapping them)
import functools
parts = {}
def timed(mod, name):
    f = getattr(mod, name)
    @functools.wraps(f)
    def g(*a, **k):
        t = time.perf_counter(); r = f(*a, **k); parts.setdefault(name, []).append((time.perf_counter() - t) * 1e6); return r
    setattr(mod, name, g)
timed(multigpu, "_global_replay"); timed(executor, "_take_outputs"); timed(multigpu, "allreduce_min")
for i in range(30):
    it = multigpu._Launched("t", tt, pred, list(w.project), n, True, gcap, min(gcap, tt.row_count))
    multigpu._launch(it, 1); executor._stream(dev).synchronize()
    local, counts, cols = multigpu._finish(it)
    scratch.materialize_temp(cols); scratch.temps.sweep()
print("finish parts (us):", {k: round(statistics.median(v[10:]), 1) for k, v in parts.items()},
      "may_fail", it.ps.cp.may_fail, "unbound", it.ps.cp.unbound)
dist.destroy_process_group()
