"""Device time of a queued ESC step (scan + compaction, no host gaps): a sleep kernel holds the
stream while the step is enqueued, so the events around it see only device work.  Config 2
(6M rows) by default; L2 flushed before each rep.  Diagnostics, not product."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1901_01488_b200 import datagen, executor, optimizer, serde, _native as N
from paper_1901_01488_b200.catalog import Catalog
from paper_1901_01488_b200.storage import Column, ColumnTable, Dictionary, parse_kind

dev = torch.device("cuda", 0)
w2 = datagen.config2()
t2 = ColumnTable("lineitem", [Column(k, parse_kind(v[0]), v[1], None, Dictionary(v[2]) if len(v) > 2 else None,
                                     device=dev) for k, v in w2.columns.items()])
p2 = serde.from_json(w2.pred, "lineitem")
cap = int(0.2 * t2.row_count)


REPS = int(os.environ.get("REPS", "15"))


def measure(label, parts=None, reps=None, clean=False):
    reps = reps or REPS
    for _ in range(3):
        ps = executor.launch_step(t2, p2, w2.project, cap)
        torch.cuda.synchronize(); executor.finish_step(ps)
    ts = []
    for _ in range(reps):
        bench._flush_l2(dev, clean)
        torch.cuda._sleep(2_000_000)  # ~1 ms: the host enqueues the step meanwhile
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ps = executor.launch_step(t2, p2, w2.project, cap)
        e1.record()
        torch.cuda.synchronize()
        executor.finish_step(ps)
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"{label:28s} device step {statistics.median(ts):6.1f} us  (min {min(ts):6.1f}, mean {statistics.mean(ts):6.2f})")


measure("default")
measure("default, clean L2", clean=True)
N.set_mid_max_rows(0); measure("mid off"); measure("mid off, clean L2", clean=True); N.set_mid_max_rows(32 << 20)
for k, v in list(os.environ.items()):
    pass
