"""Config-4 ESC step (600M rows) on the device alone (diagnostics): the queued step (K1 select +
compaction chain, one graph) behind a sleep kernel so the events see device work only, vs the
count-only scan and vs the bench's host-inclusive step."""
import os, sys, statistics, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_01488_b200 import count_star, datagen, executor, optimizer, serde
from paper_1901_01488_b200.catalog import Catalog
from paper_1901_01488_b200.storage import Column, ColumnTable, parse_kind
n = int(sys.argv[1]) if len(sys.argv) > 1 else 600_000_000
dev = torch.device("cuda", 0)
w = datagen.config4_blocked(n, 0, n)
t = ColumnTable("t", [Column(k, parse_kind(w.columns[k][0]), w.columns[k][1], device=dev) for k in "ABCD"])
pred = serde.from_json(w.pred, "t", w.udfs)
cap = n // 5
def dev_time(fn, reps=20):
    for _ in range(3): fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.cuda._sleep(20_000_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); r = fn(); e1.record(); torch.cuda.synchronize()
        if isinstance(r, executor.PendingStep): executor.finish_step(r)
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)
step = lambda: executor.launch_step(t, pred, w.project, cap)
scan = lambda: executor.launch_step(t, pred, w.project, cap, materialize=False)
print(f"device: queued step {dev_time(step):.4f} ms, count-only scan {dev_time(scan):.4f} ms")
cat = Catalog(); cat.register(t); cfg = optimizer.EscConfig()
def host_step():
    d = optimizer.esc_subquery(cat, "t", pred, w.project, cfg); cat.temps.sweep()
for _ in range(3): host_step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): host_step()
e1.record(); torch.cuda.synchronize()
print(f"host-inclusive step (bench loop) {e0.elapsed_time(e1) / 20:.4f} ms")
# K1 select alone (profiling split: part 1 with events around it), with and without the scan-time
# capture of the hit rows' values
import bench
for capture in (True, False):
    prev = executor.set_capture(capture)
    executor.release_step_plans(dev)
    tt = bench._time_kernels(lambda: executor.finish_step(step()) if False else (lambda ps: (torch.cuda.synchronize(), executor.finish_step(ps)))(step()), 10, dev)
    sel = statistics.median(x for x, k in tt if k == "select")
    mat = statistics.median(x for x, k in tt if k == "materialize")
    print(f"capture={capture}: K1 select {sel:.4f} ms, compaction {mat:.4f} ms")
    executor.set_capture(prev)
# the one-pass kernel (K2: scan + decoupled look-back + compaction in one launch) on the same table
if "--onepass" in sys.argv:
    def one():
        return executor.materialize_onepass(t, pred, w.project, cap)
    for _ in range(3): one()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): one()
    e1.record(); torch.cuda.synchronize()
    print(f"one-pass K2 materialize (host-inclusive) {e0.elapsed_time(e1) / 10:.4f} ms")
