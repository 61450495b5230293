"""Host time around the device work of one ESC step (diagnostics): from the step's start to the
scan's launch call (the device idles unless a previous step still runs), and from the host wait's
return to the step's end (the device idles). Single-GPU step (default) or the sharded step in a
one-rank NCCL group (--sharded); 75M rows of config 4 = the 8-GPU shard."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from paper_1901_01488_b200 import datagen, executor, multigpu, optimizer, serde, _native as N
from paper_1901_01488_b200.catalog import Catalog
from paper_1901_01488_b200.storage import Column, ColumnTable, parse_kind
import bench
n = 75_000_000
sharded = "--sharded" in sys.argv
dev = torch.device("cuda", 0); torch.cuda.set_device(0)
if sharded:
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(bench._free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
w = datagen.config4_blocked(n, 0, n)
t = ColumnTable("t", [Column(k, parse_kind(w.columns[k][0]), w.columns[k][1], device=dev) for k in "ABCD"])
pred = serde.from_json(w.pred, "t", w.udfs)
cfg = optimizer.EscConfig()
cat = Catalog(); cat.register(t)
st = multigpu.ShardedTable("t", t, n, 0, 0, 1)
lib = N.load_library()
marks = {}
orig_launch = lib.esc_step_plan_launch
def launch(*a):
    marks.setdefault("launch", time.perf_counter())
    return orig_launch(*a)
lib.esc_step_plan_launch = launch
orig_sync = torch.cuda.Stream.synchronize
def sync(self):
    r = orig_sync(self); marks["synced"] = time.perf_counter(); return r
torch.cuda.Stream.synchronize = sync
def step():
    if sharded:
        return multigpu.sharded_esc_subquery(st, pred, w.project, cfg)
    d = optimizer.esc_subquery(cat, "t", pred, w.project, cfg); cat.temps.sweep(); return d
for _ in range(5): step()
pre, post, total = [], [], []
for _ in range(30):
    torch.cuda.synchronize(); marks.clear()
    t0 = time.perf_counter(); step(); t1 = time.perf_counter()
    pre.append((marks["launch"] - t0) * 1e6); post.append((t1 - marks["synced"]) * 1e6); total.append((t1 - t0) * 1e6)
print(f"{'sharded' if sharded else 'single'}: to first launch {statistics.median(pre):6.1f} us, after the wait "
      f"{statistics.median(post):6.1f} us, step wall {statistics.median(total):6.1f} us")
# where the time after the wait goes (single path): the pieces it calls, timed by wrapping them
if not sharded:
    import functools
    from paper_1901_01488_b200 import catalog as catmod, storage
    parts = {}
    def timed(obj, name, label):
        f = getattr(obj, name)
        @functools.wraps(f)
        def g(*a, **k):
            t = time.perf_counter(); r = f(*a, **k); parts.setdefault(label, []).append((time.perf_counter() - t) * 1e6); return r
        setattr(obj, name, g)
    timed(executor, "finish_step", "finish_step")
    timed(executor, "_take_outputs", "  _take_outputs")
    timed(catmod.Catalog, "materialize_temp", "materialize_temp")
    timed(storage.TempTableStore, "sweep", "sweep")
    timed(optimizer, "decide_pushdown", "decide_pushdown")
    timed(executor, "compile_predicate", "compile_predicate")
    timed(executor, "_step_plan", "_step_plan")
    for _ in range(30): step()
    for k, v in parts.items(): print(f"  {k:22s} {statistics.median(v[5:]):6.1f} us")
