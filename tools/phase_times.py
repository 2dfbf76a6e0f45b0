"""Per-step device times of one geninv through the split entry points (gram_d, from_gram_d, apply_d)
and of the whole-call geninv_d, median of reps, CUDA events on the handle's (current) stream.

    python tools/phase_times.py C3T [reps]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_0804_4809_b200 import inputs as I  # noqa: E402
from paper_0804_4809_b200.binding import Handle  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3T"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
if name == "C3T":
    G = I.make_single(I.CONFIGS["C3"], I.QSEED["C3"], device="cuda").T.contiguous()
else:
    G = I.make_single(I.CONFIGS[name], I.QSEED[name], device="cuda")
m, n = G.shape
trans = int(m < n)
s = min(m, n)
h = Handle(0)
A = torch.zeros(s, (s + 1) // 2 * 2, dtype=torch.float64, device="cuda")
Gp = torch.empty(n, m, dtype=torch.float64, device="cuda")


def timed(fn):
    ts = []
    for i in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if i:
            ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


t_gram = timed(lambda: h.geninv_gram_d(G, trans, A))
t_chain = timed(lambda: h.geninv_from_gram_d(A))
t_apply = timed(lambda: h.geninv_apply_d(G, trans, Gp))
t_all = timed(lambda: h.geninv_d(G, Gp))
print(f"{name} {m}x{n}: gram {t_gram:.3f} ms, factorisation chain (a2-a6) {t_chain:.3f} ms, "
      f"output {t_apply:.3f} ms; sum {t_gram + t_chain + t_apply:.3f} ms; whole geninv_d {t_all:.3f} ms")

# the chain's two factorisations through their step entry points
Ah = A.clone()
L, piv, info = h.geninv_frchol_d(Ah)
t_fr = timed(lambda: h.geninv_frchol_d(Ah))
Lc = L.contiguous()
B = (Lc.T @ Lc).contiguous()
Bp = torch.zeros(B.shape[0], (B.shape[0] + 1) // 2 * 2, dtype=torch.float64, device="cuda")
Bp[:, :B.shape[0]] = B
t_spd = timed(lambda: h.geninv_spd_inverse_d(Bp[:, :B.shape[0]]))
print(f"  frchol (a2+a3, s={s}) {t_fr:.3f} ms; spd inverse (a5, r={info.rank}) {t_spd:.3f} ms")
if "--profile-spd" in sys.argv:   # ncu --profile-from-start off ... python tools/phase_times.py C3T 1 --profile-spd
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    h.geninv_spd_inverse_d(Bp[:, :B.shape[0]])
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
