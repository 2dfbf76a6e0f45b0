"""Time the a7 output product of C4 (geninv_apply_d, CUDA events, median of 3) for the raster-band knob in
the environment (GENINV_BAND_MB) -- measurement tool.   python tools/time_apply.py"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0804_4809_b200 import inputs as I          # noqa: E402
from paper_0804_4809_b200.binding import Handle       # noqa: E402

cfg = I.CONFIGS["C4"]
h = Handle(0)
G = I.make_single(cfg, I.QSEED["C4"], device="cuda")
A = torch.zeros(cfg.n, cfg.n, dtype=torch.float64, device="cuda")
Gp = torch.empty(cfg.n, cfg.m, dtype=torch.float64, device="cuda")
h.geninv_gram_d(G, 0, A)
h.geninv_from_gram_d(A)
ts = []
for _ in range(4):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    h.geninv_apply_d(G, 0, Gp)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(json.dumps({"band_mb": os.environ.get("GENINV_BAND_MB", "48"), "apply_ms": float(np.median(ts[1:]))}))
