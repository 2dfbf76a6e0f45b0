"""frchol (a2 + a3) and the SPD inverse (a5) at several sizes, median of reps (CUDA events): for
choosing the lookahead depth by s (run once per GENINV_LOOKAHEAD setting).

    GENINV_LOOKAHEAD=1 python tools/frchol_sizes.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0804_4809_b200 import inputs as I  # noqa: E402
from paper_0804_4809_b200.binding import Handle  # noqa: E402


def med(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


h = Handle(0)
for s in (512, 768, 1024, 1536, 2048, 3072, 4096):
    r = s * 3 // 4
    G = I.low_rank(3, 4 * s, s, r, device="cuda")
    A = torch.zeros(s, s, dtype=torch.float64, device="cuda")
    h.geninv_gram_d(G, 0, A)
    Bf = torch.eye(s, dtype=torch.float64, device="cuda") * s + A / A.diagonal().max()
    print(f"s={s}: frchol {med(lambda: h.geninv_frchol_d(A)):.3f} ms, spd_inverse {med(lambda: h.geninv_spd_inverse_d(Bf)):.3f} ms",
          flush=True)
