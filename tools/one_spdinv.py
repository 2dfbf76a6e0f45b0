"""One geninv_spd_inverse_d of an r x r SPD matrix (measurement target for ncu launch lists)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0804_4809_b200 import inputs as I          # noqa: E402
from paper_0804_4809_b200.binding import Handle       # noqa: E402

r = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
h = Handle(0)
G = I.dense_normal(1, 4 * r, r, device="cuda")
B = (G.T @ G).contiguous()
for _ in range(3):
    h.geninv_spd_inverse_d(B)
torch.cuda.synchronize()
print("ok")
