"""One emulated-a7 geninv_d call on C4 under the CUDA profiler range (ncu --profile-from-start off)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_0804_4809_b200 import inputs as I  # noqa: E402
from paper_0804_4809_b200.binding import Handle  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
G = I.make_single(I.CONFIGS[name], I.QSEED[name], device="cuda")
h = Handle(0)
h.set_emulation(1)
Gp, info = h.geninv_d(G)
torch.cuda.synchronize()
torch.cuda.profiler.start()
h.geninv_d(G, Gp)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
