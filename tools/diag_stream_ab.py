"""A/B of sel_stream_kernel ring settings inside ONE process (diagnostics): the config-5 shape
(c0/c1 int32 + c4/c5 int64, single range at selectivity s, materialize all four), each setting
given as env overrides (ESC_STREAM_SPT / ESC_STREAM_STAGES / ESC_STREAM_WARPS, read when the
compaction is planned), settings interleaved over several rounds so box drift hits all alike.
python tools/diag_stream_ab.py [rows] [settings...]   (setting: "SPT=4,ST=3" or "default")"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1901_01488_b200 import executor, expr as ex
from paper_1901_01488_b200.storage import Column, parse_kind, ColumnTable

n = int(sys.argv[1]) if len(sys.argv) > 1 else 600_000_000
settings = sys.argv[2:] or ["default", "SPT=2", "SPT=4"]
KEYS = {"SPT": "ESC_STREAM_SPT", "ST": "ESC_STREAM_STAGES", "WARPS": "ESC_STREAM_WARPS"}
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(5)
cols = [Column(c, parse_kind("INT32"), torch.randint(0, 1_000_000, (n,), generator=g, device=dev, dtype=torch.int32)) for c in ("c0", "c1")]
cols += [Column(c, parse_kind("INT64"), torch.randint(0, 10**12, (n,), generator=g, device=dev, dtype=torch.int64)) for c in ("c4", "c5")]
t = ColumnTable("t", cols)


def apply(setting):
    for v in KEYS.values():
        os.environ.pop(v, None)
    if setting != "default":
        for kv in setting.split(","):
            k, v = kv.split("=")
            os.environ[KEYS[k]] = v


res = {}
for s in (0.05, 0.1, 0.3, 0.5, 0.9):
    p = ex.Range(ex.ColumnRef("t", "c0"), 0, int(round(s * 1e6)) - 1)
    for rnd in range(3):
        for st in settings:
            apply(st)
            executor.materialize(t, p, ["c0", "c1", "c4", "c5"])
            tt = bench._time_kernels(lambda: executor.materialize(t, p, ["c0", "c1", "c4", "c5"]), 3, dev)
            res.setdefault((s, st), []).append(statistics.median(x for x, k in tt if k == "materialize"))
apply("default")
print("materialize ms (median of rounds)   " + "  ".join(f"{st:>10}" for st in settings))
for s in (0.05, 0.1, 0.3, 0.5, 0.9):
    print(f"s={s:<5}" + " " * 28 + "  ".join(f"{statistics.median(res[(s, st)]):>10.3f}" for st in settings))
