"""C4 managed-memory orchestrations (64M host-resident records): migrate-per-chunk vs mapped in place."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "benchmarks"))
import torch
import workloads as W
from paper_2512_05516_b200 import api

n = 1 << 26
P, v, src = W.random_default_aos(n)
managed = api.HostBuffer(v.nbytes, 1)
pinned = api.HostBuffer(v.nbytes, 0)
hm, hp = managed.numpy(), pinned.numpy()
step = 1 << 22
for b in range(0, v.nbytes, step * 88):
    e = min(v.nbytes, b + step * 88)
    blk = src.data[b:e].cpu().numpy()
    hm[b:e] = blk
    hp[b:e] = blk
del src
torch.cuda.empty_cache()
dst = api.View(P, n, "soa", "drift", 16)
for mode, name, hb in ((1, "managed (prefetch)", managed), (3, "managed mapped", managed), (2, "pinned in-place", pinned)):
    api.run_host(v, hb, dst, "drift", 1e-3, mode=mode)
    secs = [api.run_host(v, hb, dst, "drift", 1e-3, mode=mode)["seconds"] for _ in range(3)]
    s = sum(secs) / len(secs)
    print("%-20s %.1f ms  %.0f M rec/s" % (name, s * 1e3, n / s / 1e6), flush=True)
managed.free()
pinned.free()
