"""Compare the handle's launch counter for one geninv_d call with the kernels ncu sees (run under
   ncu --profile-from-start off --metrics gpu__time_duration.sum --csv).
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0804_4809_b200 import inputs as I
from paper_0804_4809_b200.binding import Handle
name = sys.argv[1]
G = I.make_single(I.CONFIGS["C3"], 1, device="cuda").T.contiguous() if name == "C3T" else I.make_single(I.CONFIGS[name], I.QSEED[name], device="cuda")
h = Handle(0)
Gp, info = h.geninv_d(G)
torch.cuda.synchronize()
l0 = h.launch_count
torch.cuda.profiler.start()
h.geninv_d(G, Gp)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("claimed", h.launch_count - l0)
