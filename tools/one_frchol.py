"""One full-rank Cholesky (geninv_frchol_d) of a C2-sized Gram on the device: a target for ncu captures
of the panel kernel (measurement tool).   python tools/one_frchol.py [s]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0804_4809_b200 import inputs as I          # noqa: E402
from paper_0804_4809_b200.binding import Handle       # noqa: E402

s = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
h = Handle(0)
G = I.dense_normal(1, 4 * s, s, device="cuda")
A = torch.zeros(s, s, dtype=torch.float64, device="cuda")
h.geninv_gram_d(G, 0, A)
for _ in range(2):
    h.geninv_frchol_d(A)
torch.cuda.synchronize()
print("ok")
