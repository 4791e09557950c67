"""One launch of each C1 in-place kernel (kick, drift, kick,drift) on a 1M-record
default AoS, for ncu: `ncu --set full -k regex:k_update_rec python scripts/probe_c1_kernels.py`."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from benchmarks.workloads import random_default_aos  # noqa: E402
from paper_2512_05516_b200 import api  # noqa: E402

n = 1 << 20
P, _, src = random_default_aos(n)
nat = api.convert(src, api.View(P, n, "aos", None, api.SF_PREC_NATIVE))
for k in sys.argv[1:] or ["kick", "drift", "kick,drift"]:
    api.run_kernel(nat, k, 1e-3, buffer_size=64)
torch.cuda.synchronize()
