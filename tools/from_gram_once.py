"""One geninv_from_gram_d (steps a2-a6) on the Gram of a tall exact-rank matrix, between
cudaProfilerStart/Stop, for an ncu launch list of the replicated factorisation chain.

    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv python tools/from_gram_once.py [m n r]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_0804_4809_b200 import inputs as I  # noqa: E402
from paper_0804_4809_b200.binding import Handle  # noqa: E402

m, n, r = [int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (65536, 4096, 3584))]
h = Handle(0)
G = I.low_rank(5, m, n, r, device="cuda")
A = torch.zeros(n, n, dtype=torch.float64, device="cuda")
h.geninv_gram_d(G, 0, A)
h.geninv_from_gram_d(A)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
h.geninv_from_gram_d(A)
e1.record()
torch.cuda.synchronize()
print(f"from_gram {n} r={r}: {e0.elapsed_time(e1):.2f} ms")
torch.cuda.profiler.start()
h.geninv_from_gram_d(A)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
