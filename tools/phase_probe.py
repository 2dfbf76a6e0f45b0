"""Time the factorisation steps separately (frchol a2+a3, spd inverse a5) at C3/C4 sizes."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_0804_4809_b200 import inputs as I  # noqa: E402
from paper_0804_4809_b200.binding import Handle  # noqa: E402


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


h = Handle(0)
cases = [(16384, 4096, 3072), (8192, 1024, 1024), (65536, 4096, 3584)]
if len(sys.argv) > 1:
    cases = cases[:int(sys.argv[1])]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
for (m, n, r) in cases:
    G = I.low_rank(1, m, n, r, device="cuda")
    A = torch.zeros(n, n, dtype=torch.float64, device="cuda")
    h.geninv_gram_d(G, 0, A)
    t_fr = timeit(lambda: h.geninv_frchol_d(A), reps)
    L, piv, info = h.geninv_frchol_d(A)
    B = (L.T @ L).contiguous()
    t_inv = timeit(lambda: h.geninv_spd_inverse_d(B), reps)
    t_fg = timeit(lambda: h.geninv_from_gram_d(A), reps)
    print(f"s={n} r={info.rank}: frchol {t_fr:.2f} ms  spd_inverse {t_inv:.2f} ms  from_gram {t_fg:.2f} ms", flush=True)
