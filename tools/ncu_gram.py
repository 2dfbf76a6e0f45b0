"""One a1 Gram launch (A = G'G, lower tiles, split-K) of a C4 row block between cudaProfilerStart/Stop.

    ncu --profile-from-start off --set full python tools/ncu_gram.py [rows]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_0804_4809_b200 import inputs as I  # noqa: E402
from paper_0804_4809_b200.binding import Handle  # noqa: E402

cfg = I.CONFIGS["C4"]
rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
h = Handle(0)
G = I.make_single(cfg, I.QSEED["C4"], device="cuda", rows=rows)
A = torch.zeros(cfg.n, cfg.n, dtype=torch.float64, device="cuda")
h.geninv_gram_d(G, 0, A)
torch.cuda.synchronize()
torch.cuda.profiler.start()
h.geninv_gram_d(G, 0, A)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("gram rows", rows)
