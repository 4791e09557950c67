"""Full-record AoS (default 88-B schema) -> SoA at T16 / T32 / bf16, 16M records: device time per launch."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_05516_b200 import api

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "benchmarks"))
import workloads as W

n = 1 << 24
P, v, src = W.random_default_aos(n)
for name, prec, access in (("T16 all fields", 16, None), ("bf16 all fields", api.SF_PREC_BF16, None),
                           ("T32 all fields", 32, None), ("T16 kick set", 16, "kick"), ("T16 drift set", 16, "drift"),
                           ("T16 density set", 16, "density")):
    dst = api.View(P, n, "soa", access, prec)
    out = api.PackedBuffer.empty(dst)
    for _ in range(3):
        api.gather(src, dst, out=out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        api.gather(src, dst, out=out)
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / 20
    nbytes = v.nbytes + dst.nbytes
    print("%-18s %.3f ms  %.1f G rec/s  whole-record bytes %.2f TB/s" % (name, ms, n / ms / 1e6, nbytes / ms / 1e9),
          flush=True)
