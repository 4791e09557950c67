"""C4 in-place orchestration: chunk-size sweep (64M host-resident records)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "benchmarks"))
import torch
import workloads as W
from paper_2512_05516_b200 import api

n = 1 << 26
P, v, src = W.random_default_aos(n)
pinned = api.HostBuffer(v.nbytes, 0)
hp = pinned.numpy()
step = 1 << 22
for b in range(0, v.nbytes, step * 88):
    e = min(v.nbytes, b + step * 88)
    hp[b:e] = src.data[b:e].cpu().numpy()
del src
torch.cuda.empty_cache()
dst = api.View(P, n, "soa", "drift", 16)
for chunk in (1 << 19, 1 << 20, 1 << 21, 1 << 22, 1 << 23):
    api.run_host(v, pinned, dst, "drift", 1e-3, chunk=chunk, mode=2)
    secs = [api.run_host(v, pinned, dst, "drift", 1e-3, chunk=chunk, mode=2)["seconds"] for _ in range(3)]
    s = sum(secs) / len(secs)
    print("chunk %8d: %.1f ms  %.0f M rec/s  %.1f GB/s both ways" % (chunk, s * 1e3, n / s / 1e6, 2 * v.nbytes / s / 1e9),
          flush=True)
pinned.free()
