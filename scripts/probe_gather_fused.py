"""Fused AoS -> SoA gathers (kick / drift) at 16M records: device time per launch."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "benchmarks"))
import torch
import workloads as W
from paper_2512_05516_b200 import api

n = 1 << 24
P, v, src = W.random_default_aos(n)
for kern, prec in (("kick", 16), ("kick", 32), ("kick", api.SF_PREC_BF16), ("drift", 16), ("drift", 32)):
    dst = api.View(P, n, "soa", kern, prec)
    out = api.PackedBuffer.empty(dst)
    for _ in range(3):
        api.gather_kernel(src, dst, kern, 1e-3, out=out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        api.gather_kernel(src, dst, kern, 1e-3, out=out)
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / 20
    print("%-6s prec %-4d %.3f ms  %.1f G rec/s  whole-record bytes %.2f TB/s" % (
        kern, prec, ms, n / ms / 1e6, (v.nbytes + dst.nbytes) / ms / 1e9), flush=True)
