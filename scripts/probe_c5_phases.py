"""CUDA-event timing of the pieces of one C5 density call (PeerBlocks), 128M."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_05516_b200 import api
from paper_2512_05516_b200.sharded import ShardedState, Slab, grid_for

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 27
h, nc, cell = grid_for(n)
st = ShardedState(n, Slab(nc, cell, 0, 1), prec=32, h=h)
st.sort_by_cell()
pb = st._peer
x, m, hh = st.stream("x"), st.stream("m"), st.stream("h")
for it in range(4):
    st.kick_drift()
    pb(x, m, hh)  # sizes buffers
    torch.cuda.synchronize()
    posb, massb, hmaxb, _, _, _ = pb.layout(pb.ncell, pb.cap)
    cs = pb.buf.tensor(0, (pb.ncell + 1,), torch.int32)
    pos = pb.buf.tensor(posb, (pb.cap, 4), torch.float32)[:n]
    mass = pb.buf.tensor(massb, (pb.cap,), torch.float32)[:n]
    hmax = pb.buf.tensor(hmaxb, (4,), torch.int32)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record()
    api.bin_particles(x.float().contiguous(), (pb.x_origin, 0.0, 0.0), pb.cell, (pb.nx, pb.ny, pb.nz), cell_start=cs,
                      perm=pb.perm[:n])
    ev[1].record()
    api.cells_pack(x, m, hh, pb.perm, pos, mass, hmax, pb.prec)
    ev[2].record()
    blocks = [api.cell_block(pos, mass, cs, hmax, pb.x0, pb.nx, pb.x_origin)]
    api.density_cells_blocks(blocks, n, pb.perm, (0.0, 0.0), pb.cell, pb.NX, pb.ny, pb.nz, reach=2)
    ev[3].record()
    torch.cuda.synchronize()
    print("iter %d bin %.2f pack %.2f pairs %.2f ms" % (it, ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]),
                                                      ev[2].elapsed_time(ev[3])), flush=True)
