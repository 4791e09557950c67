"""Per-call timing of the C5 full step's force phase (diagnostic)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_05516_b200 import api
from paper_2512_05516_b200.sharded import ShardedState, Slab, grid_for, gpu_force_backend, force_with_ghosts

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 27
h, nc, cell = grid_for(n)
st = ShardedState(n, Slab(nc, cell, 0, 1), prec=32, h=h)
st.sort_by_cell()
for it in range(3):
    st.density()
    torch.cuda.synchronize()
    names = ["x", "v", "m", "h", "rho", "P"]
    own = [st.stream(k) for k in names]
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    t0 = time.perf_counter()
    ev[0].record()
    a = torch.zeros((n, 3), device="cuda"); du = torch.zeros(n, device="cuda")
    ev[1].record()
    b = st._binning
    api.force_cells(*[o.contiguous() for o in own], b["cs"], b["perm"], (0, 0, 0), cell / 2, (nc * 2,) * 3,
                    n_home=n, reach=2, a=a, du=du)
    ev[2].record()
    st.stream("a").copy_(a); st.stream("du").copy_(du)
    ev[3].record()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print("iter", it, "zeros %.2f ms, force_cells %.2f ms, copy %.2f ms, wall %.2f ms" % (
        ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3]), 1e3 * (t1 - t0)), flush=True)
    t0 = time.perf_counter()
    st.force()
    torch.cuda.synchronize()
    print("   st.force wall %.2f ms" % (1e3 * (time.perf_counter() - t0)), flush=True)
