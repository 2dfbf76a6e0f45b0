"""One geninv_batched_d launch on `nb` matrices of C5 (measurement target for ncu)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0804_4809_b200 import inputs as I          # noqa: E402
from paper_0804_4809_b200.binding import Handle       # noqa: E402

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
h = Handle(0)
G = I.make_batch(I.CONFIGS["C5"], 1, 0, nb, device="cuda")
for _ in range(2):
    Gp, rk = h.geninv_batched_d(G)
torch.cuda.synchronize()
print("ok")
