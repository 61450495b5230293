"""cProfile of the single-GPU and sharded ESC steps at the 8-GPU shard size (75M rows of config 4):
where the host's per-step Python time goes (diagnostics)."""
import cProfile, os, pstats, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
import bench
from paper_1901_01488_b200 import datagen, multigpu, optimizer, serde
from paper_1901_01488_b200.catalog import Catalog
from paper_1901_01488_b200.storage import Column, ColumnTable, parse_kind
n = 75_000_000
dev = torch.device("cuda", 0); torch.cuda.set_device(0)
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(bench._free_port()))
dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
w = datagen.config4_blocked(n, 0, n)
t = ColumnTable("t", [Column(k, parse_kind(w.columns[k][0]), w.columns[k][1], device=dev) for k in "ABCD"])
pred = serde.from_json(w.pred, "t", w.udfs)
cfg = optimizer.EscConfig()
cat = Catalog(); cat.register(t)
st = multigpu.ShardedTable("t", t, n, 0, 0, 1)
def single():
    optimizer.esc_subquery(cat, "t", pred, w.project, cfg); cat.temps.sweep()
def sharded():
    multigpu.sharded_esc_subquery(st, pred, w.project, cfg)
for name, fn in (("single", single), ("sharded", sharded)):
    for _ in range(10): fn()
    torch.cuda.synchronize()
    pr = cProfile.Profile(); pr.enable()
    for _ in range(200): fn()
    pr.disable()
    print("=====", name)
    pstats.Stats(pr).sort_stats("tottime").print_stats(22)
dist.destroy_process_group()
