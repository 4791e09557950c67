"""Zero-copy probe: the gather kernels reading the AoS straight from pinned
host memory (UVA pointer) over PCIe, vs a whole-record H2D copy."""
import ctypes as C
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "benchmarks"))
import torch
import workloads as W
from paper_2512_05516_b200 import api, _lib as L

n = 1 << 24
P, v, src = W.random_default_aos(n)
host = torch.empty(v.nbytes + 16, dtype=torch.uint8, pin_memory=True)
host[: v.nbytes].copy_(src.data[: v.nbytes].cpu())
dev_copy = torch.empty_like(src.data)

def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record(); b.synchronize()
    return a.elapsed_time(b) / reps

ms = t(lambda: dev_copy[: v.nbytes].copy_(host[: v.nbytes], non_blocking=True))
print("H2D whole records: %.2f ms = %.1f GB/s, %.0f M rec/s" % (ms, v.nbytes / ms / 1e6, n / ms / 1e3), flush=True)
for kern, prec in (("density", 16), ("kick", 16), ("drift", 16), (None, 16)):
    dst = api.View(P, n, "soa", kern, prec)
    out = api.PackedBuffer.empty(dst)
    def go():
        if kern in ("kick", "drift"):
            st = L.lib().sf_b200_gather_kernel(v.handle, C.c_void_p(host.data_ptr()), dst.handle,
                                               C.c_void_p(out.data.data_ptr()), kern.encode(), C.c_double(1e-3), 0,
                                               C.c_void_p(torch.cuda.current_stream().cuda_stream))
        else:
            st = L.lib().sf_b200_gather(v.handle, C.c_void_p(host.data_ptr()), dst.handle,
                                        C.c_void_p(out.data.data_ptr()),
                                        C.c_void_p(torch.cuda.current_stream().cuda_stream))
        L.check(st)
    try:
        ms = t(go)
        print("zero-copy gather %-8s: %.2f ms, %.0f M rec/s (whole-record equiv %.1f GB/s)" % (
            kern or "full", ms, n / ms / 1e3, v.nbytes / ms / 1e6), flush=True)
    except Exception as e:
        print("zero-copy gather %s failed: %s" % (kern, e), flush=True)
