"""Debug: dense-tile list size after one materialisation (not part of the product)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_01488_b200 import ColumnTable, executor, expr as ex, _native as N
from paper_1901_01488_b200.storage import Column, parse_kind
n = 20_000_000
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(5)
c0 = torch.randint(0, 1_000_000, (n,), generator=g, device=dev, dtype=torch.int32)
c4 = torch.randint(0, 10**12, (n,), generator=g, device=dev, dtype=torch.int64)
t = ColumnTable("t", [Column("c0", parse_kind("INT32"), c0), Column("c4", parse_kind("INT64"), c4)])
lib = N.load_library()
for s in (0.002, 0.05, 0.5):
    p = ex.Range(ex.ColumnRef("t", "c0"), 0, int(s * 1e6) - 1)
    sel = executor.select(t, p, capture=["c0"])
    executor.materialize_selection(sel, ["c0", "c4"])
    torch.cuda.synchronize()
    ws = N.workspace(dev, torch.cuda.current_stream())
    total = lib.esc_workspace_bytes(n)
    segs = C.c_int64()
    lib.esc_selection_sizes(n, None, C.byref(segs), None)
    up = lambda x: (x + 255) & ~255
    dense_off = total - up(256 + 4 * segs.value)
    nd = int(ws.buf[dense_off:dense_off + 4].view(torch.int32).item())
    counts = sel.buffers[1][: (n + 4095) // 4096 * 8].cpu().numpy() & 0x7FFFFFFF
    tiles = counts[: (len(counts) // 8) * 8].reshape(-1, 8).sum(1)
    print(f"s={s} count={sel.count} n_dense={nd} expected={(tiles >= 128).sum()} of {len(tiles)} "
          f"seg_rows={sel.desc.seg_rows}", flush=True)
