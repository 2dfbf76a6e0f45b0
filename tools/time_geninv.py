"""Time geninv_d (the whole call) on a config: median of reps, CUDA events, input resident.

    python tools/time_geninv.py C3T [reps]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_0804_4809_b200 import inputs as I  # noqa: E402
from paper_0804_4809_b200.binding import Handle  # noqa: E402

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
if name == "C3T":
    G = I.make_single(I.CONFIGS["C3"], I.QSEED["C3"], device="cuda").T.contiguous()
else:
    G = I.make_single(I.CONFIGS[name], I.QSEED[name], device="cuda")
h = Handle(0)
Gp, info = h.geninv_d(G)
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h.geninv_d(G, Gp)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"{name} geninv_d: median {np.median(ts):.3f} ms  min {np.min(ts):.3f} ms  rank {info.rank}  "
      f"graphs {'off' if os.environ.get('GENINV_NO_GRAPH') else 'on'}")
