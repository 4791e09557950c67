"""Debug: C3 sampled parity mismatch (GPU rho vs subset oracle vs brute force)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import numpy as np, torch
import oracle as O
from paper_2512_05516_b200 import api
from paper_2512_05516_b200.sharded import grid_for
from test_gpu_config_sizes import _subbox_homes

n = 1 << 22
hh, nc, cell = grid_for(n)
print("h", hh, "nc", nc, "cell", cell)
refine = 2
g = torch.Generator(device="cuda").manual_seed(3)
x0 = torch.rand(n, 3, generator=g, device="cuda")
for dt, prec in ((torch.float16, 16), (torch.bfloat16, 100)):
  x = x0.to(dt)
  m = torch.full((n,), 1.0 / n, device="cuda").to(dt)
  h = torch.full((n,), hh, device="cuda").to(dt)
  for reach_refine in (1, 2):
    dd = (nc * reach_refine,) * 3
    cs, perm = api.bin_particles(x.float().contiguous(), (0, 0, 0), cell / reach_refine, dd)
    rho = api.density_cells(x, m, h, cs, perm, (0, 0, 0), cell / reach_refine, dd, reach=reach_refine, prec=prec)
    for lo in ((0.41, 0.37, 0.52), (0.0, 0.0, 0.0), (0.93, 0.0, 0.6)):
        side = 0.07
        idx, homes = _subbox_homes(x.float(), lo, side, 2 * float(h.float().max()) * 1.001)
        xd = x[idx].double().cpu().numpy(); md = m[idx].double().cpu().numpy(); hd = h[idx].double().cpu().numpy()
        hn = homes.cpu().numpy().astype(np.uint64)
        c = float(2 * hd.max()) * 1.0001
        want = O.density_cells_at(xd.reshape(-1), md, hd, float(min(lo)), float(max(lo)) + side, c, hn)
        got = rho[idx[homes]].double().cpu().numpy()
        bad = np.nonzero(np.abs(got - want) > 1e-5 * np.abs(want))[0]
        print(dt, "refine", reach_refine, "box", lo, "homes", len(hn), "bad", len(bad))
        for b in bad[:4]:
            i = int(idx[homes[b]])
            d = torch.sqrt(((x.double() - x[i].double()) ** 2).sum(1))
            sel = (d < 2 * float(h[0])).nonzero().squeeze(1)
            bf = sum(float(m[j]) * O.w(float(d[j]), float(h[0])) for j in sel.tolist())
            ins = sum(1 for j in sel.tolist() if j in set(idx.tolist()))
            print("  i", i, "x", x[i].tolist(), "gpu", got[b], "oracle", want[b], "brute", bf, "nbrs", len(sel), "in box", ins)
