"""Host cost of a kernel launch on this box (not part of the product): a tiny esc_gather and a torch
fill_, 2000 each, timed on the host."""
import ctypes as C, sys, time, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch
from paper_1901_01488_b200 import _native as N
lib = N.load_library()
dev = torch.device("cuda", 0)
src = torch.arange(1024, dtype=torch.int32, device=dev); idx = torch.zeros(1, dtype=torch.int64, device=dev)
out = torch.empty(1, dtype=torch.int32, device=dev)
desc = N.EscColumn(); desc.data = src.data_ptr(); desc.nulls = None; desc.dtype = N.dtype_code(src)
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
args = (C.byref(desc), C.c_void_p(idx.data_ptr()), 1, C.c_void_p(out.data_ptr()), None, sp)
for _ in range(100): lib.esc_gather(*args)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(2000): lib.esc_gather(*args)
t1 = time.perf_counter(); torch.cuda.synchronize()
print(f"esc_gather (<<<>>>, small params): {(t1-t0)/2000*1e6:.2f} us/launch host")
f = torch.empty(1, dtype=torch.int32, device=dev)
t0 = time.perf_counter()
for _ in range(2000): f.fill_(1)
t1 = time.perf_counter(); torch.cuda.synchronize()
print(f"torch fill_: {(t1-t0)/2000*1e6:.2f} us/launch host")
