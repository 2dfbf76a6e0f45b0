"""Time the pieces of the factorisation chain for one shape through the step entry points (CUDA events,
median of 10): a2-a3 geninv_frchol_d, a5 geninv_spd_inverse_d (POTRF + TRTRI + LAUUM) on B = L'L, and the
whole a2-a6 geninv_from_gram_d -- the rest of from_gram is the chain GEMMs (L'L, K = L M, X = K K').

    python tools/chain_breakdown.py [m n r]      (default C2: 4096 1024 1024)
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0804_4809_b200 import inputs as I          # noqa: E402
from paper_0804_4809_b200.binding import Handle       # noqa: E402

m, n, r = [int(x) for x in sys.argv[1:4]] if len(sys.argv) > 3 else (4096, 1024, 1024)
h = Handle(0)
G = I.dense_normal(1, m, n, device="cuda") if r >= min(m, n) else I.low_rank(1, m, n, r, device="cuda")
s = min(m, n)
A = torch.zeros(s, s, dtype=torch.float64, device="cuda")
h.geninv_gram_d(G, int(m < n), A)
st = torch.cuda.current_stream()


def timed(fn, reps=10):
    fn()
    fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


L, piv, info = h.geninv_frchol_d(A)
rk = info.rank
B = (L[:, :rk].T @ L[:, :rk]).contiguous()
out = {"shape": [m, n, r], "rank": rk,
       "frchol_ms": timed(lambda: h.geninv_frchol_d(A)),
       "spd_inverse_ms": timed(lambda: h.geninv_spd_inverse_d(B)),
       "from_gram_ms": timed(lambda: h.geninv_from_gram_d(A)),
       "gram_ms": timed(lambda: h.geninv_gram_d(G, int(m < n), A))}
Gp = torch.empty(n, m, dtype=torch.float64, device="cuda")
h.geninv_from_gram_d(A)
out["apply_ms"] = timed(lambda: h.geninv_apply_d(G, int(m < n), Gp))
out["geninv_d_ms"] = timed(lambda: h.geninv_d(G, Gp))
out["chain_gemms_ms"] = out["from_gram_ms"] - out["frchol_ms"] - out["spd_inverse_ms"]
print(json.dumps(out))
