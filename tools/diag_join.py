"""Star-join COUNT micro-benchmark (not part of the product): config-3-shaped fact with device
generated keys, four dimension builds, timing of esc_join_count."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_01488_b200 import ColumnTable, executor, expr as ex, join
from paper_1901_01488_b200.storage import Column, parse_kind

n = int(sys.argv[1]) if len(sys.argv) > 1 else 60_000_000
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(7)
sizes = {"d0": 2000, "d1": 2556, "d2": 30000, "d3": 200000}
steps, fcols = [], []
for i, (a, nd) in enumerate(sizes.items()):
    keys = torch.arange(1, nd + 1, device=dev, dtype=torch.int64)
    attr = torch.randint(0, 25, (nd,), generator=g, device=dev)
    t = ColumnTable(a, [Column("k", parse_kind("INT64"), keys), Column("a", parse_kind("INT64"), attr)])
    idx = join.build_hash(t, "k", ex.Comparison(ex.ColumnRef(a, "a"), "<", 6))
    steps.append(join.BuildStep(a, idx, ex.ColumnRef("f", f"k{i}")))
    fcols.append(Column(f"k{i}", parse_kind("INT32"), torch.randint(1, nd + 1, (n,), generator=g, device=dev,
                                                                     dtype=torch.int32)))
fact = ColumnTable("f", fcols)
for _ in range(3):
    join.probe_joins(fact, "f", None, steps, None)
executor.KERNEL_EVENTS = []
for _ in range(10):
    _, st = join.probe_joins(fact, "f", None, steps, None)
torch.cuda.synchronize()
ms = statistics.median(a.elapsed_time(b) for a, b, k in executor.KERNEL_EVENTS if k == "join")
executor.KERNEL_EVENTS = None
print(f"rows={n} join_kernel_ms={ms:.3f} GBps={n * 16 / ms / 1e6:.0f} probe_out={st.probe_out}")
