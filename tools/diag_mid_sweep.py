"""Mid-size compaction (one kernel) vs the scan chain: device time of the queued step over a
4-column int32/int64 table at several sizes and selectivities (sleep-gated events, L2 flushed).
Sets ESC_MID_MAX_ROWS by measurement; diagnostics."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_1901_01488_b200 import executor, expr as ex, _native as N
from paper_1901_01488_b200.storage import KIND_INT32, KIND_INT64, Column, ColumnTable
dev = torch.device("cuda", 0)
for n in (4_000_000, 12_000_000, 24_000_000, 48_000_000):
    g = torch.Generator(device=dev); g.manual_seed(5)
    t = ColumnTable("t", [Column("c0", KIND_INT32, torch.randint(0, 1_000_000, (n,), generator=g, device=dev, dtype=torch.int32)),
                          Column("c1", KIND_INT32, torch.randint(0, 1_000_000, (n,), generator=g, device=dev, dtype=torch.int32)),
                          Column("c4", KIND_INT64, torch.randint(0, 1 << 40, (n,), generator=g, device=dev, dtype=torch.int64)),
                          Column("c5", KIND_INT64, torch.randint(0, 1 << 40, (n,), generator=g, device=dev, dtype=torch.int64))])
    for s in (0.001, 0.02, 0.1, 0.5):
        p = ex.Range(ex.ColumnRef("t", "c0"), 0, int(s * 1_000_000) - 1)
        row = []
        for mid in (1 << 40, 0):
            N.set_mid_max_rows(mid)
            ms = bench._device_step_ms(lambda: executor.launch_step(t, p, ["c0", "c1", "c4", "c5"], n // 4), executor.finish_step, 7, dev)
            row.append(ms * 1e3)
        print(f"n={n:>10} s={s:<6} mid {row[0]:8.1f} us   chain {row[1]:8.1f} us   {'MID' if row[0] < row[1] else 'chain'}")
    del t
    torch.cuda.empty_cache()
