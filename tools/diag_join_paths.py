"""Star-join COUNT probe timing per kernel path (not part of the product): bits (PK bitmaps),
dense (duplicate keys -> u8 factors), hash (sparse key ranges)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_01488_b200 import ColumnTable, executor, expr as ex, join
from paper_1901_01488_b200.storage import Column, parse_kind
n = 60_000_000
dev = torch.device("cuda", 0)
for mode in ("bits", "dense", "hash"):
    g = torch.Generator(device=dev); g.manual_seed(7)
    mult = 1_000_003 if mode == "hash" else 1
    steps, fcols = [], []
    for i, nd in enumerate((2000, 2556, 30000, 200000)):
        keys = torch.arange(1, nd + 1, device=dev, dtype=torch.int64) * mult
        if mode == "dense" and i == 2:
            keys = torch.cat([keys, keys[::3]])
        attr = torch.randint(0, 25, (keys.numel(),), generator=g, device=dev)
        t = ColumnTable(f"d{i}", [Column("k", parse_kind("INT64"), keys), Column("a", parse_kind("INT64"), attr)])
        idx = join.build_hash(t, "k", ex.Comparison(ex.ColumnRef(f"d{i}", "a"), "<", 6))
        steps.append(join.BuildStep(f"d{i}", idx, ex.ColumnRef("f", f"k{i}")))
        v = torch.randint(1, nd + 1, (n,), generator=g, device=dev, dtype=torch.int64) * mult
        fcols.append(Column(f"k{i}", parse_kind("INT32" if mode != "hash" else "INT64"),
                            v.to(torch.int32) if mode != "hash" else v))
    fact = ColumnTable("f", fcols)
    for _ in range(3): join.probe_joins(fact, "f", None, steps, None)
    executor.KERNEL_EVENTS = []
    for _ in range(5): _, st = join.probe_joins(fact, "f", None, steps, None)
    torch.cuda.synchronize()
    ms = statistics.median(a.elapsed_time(b) for a, b, k in executor.KERNEL_EVENTS if k == "join")
    executor.KERNEL_EVENTS = None
    w = 16 if mode != "hash" else 32
    print(f"{mode}: join_kernel_ms={ms:.3f} GBps={n * w / ms / 1e6:.0f} probe_out={st.probe_out}")
    del fact, fcols, steps
    torch.cuda.empty_cache()
