"""Cold-L2 read floor of a plain streaming kernel (tools/probe/readprobe.cu) at mid sizes, vs K1
(diagnostics): is the ESC scan's ~20 us for 72 MB its design or the DRAM ramp?"""
import ctypes as C, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
dev = torch.device("cuda", 0)
lib = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "probe", "_readprobe.so"))
out = torch.zeros(1, dtype=torch.int64, device=dev)
for mb in (24, 72, 288, 1152):
    x = torch.randint(0, 1 << 30, (mb * 2**20 // 4,), dtype=torch.int32, device=dev)
    best = None
    for blocks, threads, unroll in ((148, 1024, 8), (148 * 2, 1024, 8), (148 * 4, 512, 8), (148 * 8, 256, 8),
                                    (148 * 16, 256, 4), (148 * 32, 256, 1)):
        ts = []
        for _ in range(7):
            bench._flush_l2(dev, True)
            torch.cuda._sleep(1_000_000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            lib.read_probe(C.c_void_p(x.data_ptr()), C.c_int64(x.numel() * 4), C.c_void_p(out.data_ptr()), blocks,
                           threads, unroll, C.c_void_p(torch.cuda.current_stream().cuda_stream))
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        m = statistics.median(ts)
        print(f"{mb:5d} MB  grid {blocks:5d} x {threads:4d} U{unroll}: {m:8.1f} us  {mb * 2**20 / m / 1e6:5.2f} TB/s")
