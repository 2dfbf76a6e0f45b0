"""Per-panel phase times of frchol from the GI_PANEL_TIMING build (libgeninv_timing.so)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
os.environ["GENINV_LIB"] = os.path.abspath("paper_0804_4809_b200/libgeninv_timing.so")
from paper_0804_4809_b200 import inputs as I  # noqa: E402
from paper_0804_4809_b200 import binding  # noqa: E402

h = binding.Handle(0)
lib = binding.load()
m, n, r = [int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (16384, 4096, 3072))]
G = I.low_rank(1, m, n, r, device="cuda")
A = torch.zeros(n, n, dtype=torch.float64, device="cuda")
h.geninv_gram_d(G, 0, A)
for _ in range(3):
    h.geninv_frchol_d(A)
torch.cuda.synchronize()
np_ = (n + 31) // 32
buf = (ctypes.c_ulonglong * (np_ * 8))()
lib.geninv_debug_panel_times(buf, np_)
t = np.array(buf, dtype=np.float64).reshape(np_, 8)
ph = np.diff(t[:, [0, 1, 2, 3, 4]], axis=1) / 1e3
tot = (t[:, 6] - t[:, 0]) / 1e3
gap = (t[1:, 0] - t[:-1, 6]) / 1e3
print(f"panels {np_}: kernel total {tot.sum():.1f} us, gaps (update GEMM + launch) {gap.sum():.1f} us")
print("mean us per phase [load, diag factor, T/publish, trsm]:", ph.mean(axis=0).round(2), " write-back+tail:",
      ((t[:, 6] - t[:, 4]) / 1e3).mean().round(2))
for p in (0, 1, 10, 60, 100, np_ - 1):
    print(p, ph[p].round(2), round(tot[p], 2), round(gap[p - 1], 2) if p else "")
