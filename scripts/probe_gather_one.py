"""One full-record AoS -> SoA T16 gather launch (for ncu)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "benchmarks"))
import torch
import workloads as W
from paper_2512_05516_b200 import api

n = 1 << 24
access = sys.argv[1] if len(sys.argv) > 1 and sys.argv[1] != "all" else None
P, v, src = W.random_default_aos(n)
dst = api.View(P, n, "soa", access, 16)
out = api.PackedBuffer.empty(dst)
for _ in range(4):
    api.gather(src, dst, out=out)
torch.cuda.synchronize()
