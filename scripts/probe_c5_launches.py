"""One C5 step (128M particles, one rank; `full` = the reference timestep
order) after warm-up, inside cudaProfilerStart/Stop, for an ncu launch list:
`ncu --profile-from-start off --metrics gpu__time_duration.sum --csv python scripts/probe_c5_launches.py [n] [full]`."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_05516_b200.sharded import ShardedState, Slab, grid_for  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 27
full = len(sys.argv) > 2 and sys.argv[2] == "full"
h, nc, cell = grid_for(n)
st = ShardedState(n, Slab(nc, cell, 0, 1), prec=32, h=h)
st.sort_by_cell()
for _ in range(2):
    st.full_step() if full else st.step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
st.full_step() if full else st.step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("grid", nc, "cell", cell, "h", h)
