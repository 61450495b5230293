"""Streamed vs warp compaction on a mid-size table (not part of the product): 6M rows, the
config-5 column shapes, selectivity 0.02 / 0.1 / 0.5, L2 flushed; ESC_STREAM_DIV from the env."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
from paper_1901_01488_b200 import ColumnTable, executor, expr as ex
from paper_1901_01488_b200.storage import Column, parse_kind
dev = torch.device("cuda", 0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 6_000_000
g = torch.Generator(device=dev); g.manual_seed(5)
cols = [Column(c, parse_kind("INT32"), torch.randint(0, 1_000_000, (n,), generator=g, device=dev, dtype=torch.int32)) for c in ("c0", "c1")]
cols += [Column(c, parse_kind("INT64"), torch.randint(0, 10**12, (n,), generator=g, device=dev, dtype=torch.int64)) for c in ("c4", "c5")]
t = ColumnTable("t", cols)
for s in (0.02, 0.1, 0.5):
    p = ex.Range(ex.ColumnRef("t", "c0"), 0, int(round(s * 1e6)) - 1)
    step = lambda: executor.count_and_materialize(t, p, ["c0", "c1", "c4", "c5"], n)
    for _ in range(3): step()
    tt = bench._time_kernels(step, 10, dev, flush=True)
    print(os.environ.get("ESC_STREAM_DIV", "default"), n, s, round(sum(x for x, k in tt) / 10 * 1e3, 1), "us", flush=True)
