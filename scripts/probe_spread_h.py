"""C3-sized density / force timing with uniform h and with h spread over [0.9, 1.0] h0 (the general pair term)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "benchmarks"))
from paper_2512_05516_b200 import api  # noqa: E402
from paper_2512_05516_b200.sharded import grid_for  # noqa: E402
from workloads import timed_each  # noqa: E402

n = 1 << 22
h, nc, cell = grid_for(n)
g = torch.Generator(device="cuda").manual_seed(3)
x = torch.rand(n, 3, generator=g, device="cuda")
m = torch.full((n,), 1.0 / n, device="cuda")
fine, dims = cell / 2, (nc * 2,) * 3
cs, perm = api.bin_particles(x, (0, 0, 0), fine, dims)
out = {}
for name, hh in (("uniform", torch.full((n,), h, device="cuda")),
                 ("spread", h * (0.9 + 0.1 * torch.rand(n, generator=g, device="cuda")))):
    rho = torch.empty(n, device="cuda")
    fd = lambda: api.density_cells(x, m, hh, cs, perm, (0, 0, 0), fine, dims, reach=2, rho=rho)  # noqa: E731
    for _ in range(3):
        fd()
    td = timed_each(fd, 10)
    v = torch.rand(n, 3, generator=g, device="cuda") * 2 - 1
    P = rho * (2.0 / 3.0)
    a, du = torch.empty(n, 3, device="cuda"), torch.empty(n, device="cuda")
    ff = lambda: api.force_cells(x, v, m, hh, rho, P, cs, perm, (0, 0, 0), fine, dims, reach=2, a=a, du=du)  # noqa: E731
    for _ in range(3):
        ff()
    tf = timed_each(ff, 10)
    out[name] = {"density_ms": sum(td) / len(td), "force_ms": sum(tf) / len(tf)}
print(json.dumps(out))
