"""Profile ingest.load_csv (not part of the product)."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1901_01488_b200.engine import parse_schema_spec
from paper_1901_01488_b200.ingest import load_csv
rows = 1_000_000
g = np.random.default_rng(2026)
ints = g.integers(-10**12, 10**12, rows); cents = g.integers(0, 10**8, rows)
words = np.array(["alpha", "beta", '"gamma, delta"', "epsilon", '"say ""hi"""', "zeta"])
w = words[g.integers(0, len(words), rows)]
text = "\n".join(f"{a},{c // 100}.{c % 100:02d},2020-01-{1 + (a % 28):02d},{s}" for a, c, s in zip(ints.tolist(), cents.tolist(), w.tolist()))
data = (text + "\n").encode()
schema = parse_schema_spec("i:int64,d:decimal(12,2),t:date,s:text")
dev = torch.device("cuda", 0)
load_csv(data, "t", schema, device=dev); torch.cuda.synchronize()
t0 = time.perf_counter(); load_csv(data, "t", schema, device=dev); torch.cuda.synchronize()
print("wall ms", (time.perf_counter() - t0) * 1e3)
pr = cProfile.Profile(); pr.enable()
load_csv(data, "t", schema, device=dev); torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
