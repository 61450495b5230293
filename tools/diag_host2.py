"""Host-side overhead of the config-2 ESC step (not part of the product): wall vs device time and
a cProfile of repeated optimizer.esc_subquery calls on the exact 6M-row recipe."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_01488_b200 import datagen, optimizer, serde
from paper_1901_01488_b200.catalog import Catalog
from paper_1901_01488_b200.storage import Column, ColumnTable, Dictionary, parse_kind

dev = torch.device("cuda", 0)
w2 = datagen.config2()
t2 = ColumnTable("lineitem", [Column(k, parse_kind(v[0]), v[1], None, Dictionary(v[2]) if len(v) > 2 else None,
                                     device=dev) for k, v in w2.columns.items()])
cat = Catalog(); cat.register(t2)
p2 = serde.from_json(w2.pred, "lineitem")
cfg = optimizer.EscConfig()
def step():
    d = optimizer.esc_subquery(cat, "lineitem", p2, w2.project, cfg)
    cat.temps.sweep()
    return d
for _ in range(10): step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
N = 200
w0 = time.perf_counter(); e0.record()
for _ in range(N): step()
e1.record(); torch.cuda.synchronize()
print(f"wall {((time.perf_counter()-w0)/N)*1e6:.1f} us/step, device span {e0.elapsed_time(e1)/N*1e3:.1f} us/step")
pr = cProfile.Profile(); pr.enable()
for _ in range(N): step()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
