"""K1 geometry sweep on the current kernels (not part of the product): config-4-shaped select
(ESC step) and count, and a 1-column count, per (ESC_CHUNKS, ESC_STAGES) in child processes.
python tools/stage_sweep2.py [rows]"""
import itertools, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, statistics
sys.path.insert(0, %r)
import torch, bench
from paper_1901_01488_b200 import ColumnTable, count_star, expr as ex, optimizer, executor
from paper_1901_01488_b200.catalog import Catalog
from paper_1901_01488_b200.storage import Column, parse_kind
n = %d
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(1)
A = torch.randint(1, 1000, (n,), generator=g, device=dev, dtype=torch.int32); A[torch.rand(n, generator=g, device=dev) < 0.095] = 0
B = torch.randint(-5, 1005, (n,), generator=g, device=dev, dtype=torch.int32)
Cc = torch.randn(n, generator=g, device=dev, dtype=torch.float32)
D = torch.randint(0, 1000, (n,), generator=g, device=dev, dtype=torch.int32)
t = ColumnTable("t", [Column("A", parse_kind("INT32"), A), Column("B", parse_kind("INT32"), B),
                      Column("C", parse_kind("FLOAT32"), Cc), Column("D", parse_kind("INT32"), D)])
r = lambda c: ex.ColumnRef("t", c)
p = ex.And((ex.Equality(r("A"), 0), ex.Range(r("C"), -0.5, 1.0), ex.Or((ex.Equality(r("D"), 17), ex.Comparison(r("D"), ">", 900))),
            ex.FnCall("b3d", (r("B"), r("D")), ">", 3.0, lambda b, d: (b * 3.0 + d) %% 7.0)))
p1 = ex.Range(r("D"), 0, 9)
cat = Catalog(); cat.register(t)
cfg = optimizer.EscConfig()
step = lambda: (optimizer.esc_subquery(cat, "t", p, ["A", "C", "D"], cfg), cat.temps.sweep())
out = {}
for name, fn, kind in (("select", step, "select"), ("count4", lambda: count_star(t, p), "count"), ("count1", lambda: count_star(t, p1), "count")):
    for _ in range(3): fn()
    tt = bench._time_kernels(fn, 8, dev)
    out[name] = statistics.median(x for x, k in tt if k == kind)
print("RESULT", out)
'''
rows = int(sys.argv[1]) if len(sys.argv) > 1 else 600_000_000
res = []
combos = [(None, None), ("4", "2"), ("4", "3"), ("2", "3"), ("2", "4"), ("2", "6"), ("1", "6"), ("1", "8"), ("1", "12"),
          ("8", "3"), ("8", "4"), ("8", "6")]
if len(sys.argv) > 2:  # a quick run: the default geometry only
    combos = combos[:1]
for c, s in combos:
    env = dict(os.environ)
    if c: env["ESC_CHUNKS"] = c
    if s: env["ESC_STAGES"] = s
    o = subprocess.run([sys.executable, "-c", CHILD % (ROOT, rows)], env=env, capture_output=True, text=True, timeout=600)
    line = [l for l in o.stdout.splitlines() if l.startswith("RESULT")]
    r = eval(line[0][7:]) if line else {"error": o.stderr[-300:]}
    print(c, s, r, flush=True)
    res.append({"chunks": c, "stages": s, **r})
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "stage_sweep2.json"), "w"), indent=1)
