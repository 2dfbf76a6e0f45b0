"""Per-panel phase times of frchol from the GI_PANEL_TIMING build (libgeninv_timing.so).

    python -m paper_0804_4809_b200.build --timing
    python tools/panel_timing.py [m n r]

Stamps (CTA 0, %globaltimer ns; thread 0 = the diagonal warp, thread 32 = the first row warp):
0 start, 5 loads done, 1 diagonal-block correction done, 2 diagonal factor done and published
(thread 0), 7 row correction of warp 1 done, 4 rows of warp 1 solved, 6 written back (thread 32).
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["GENINV_LIB"] = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "paper_0804_4809_b200",
                                                        "libgeninv_timing.so"))
from paper_0804_4809_b200 import binding  # noqa: E402
from paper_0804_4809_b200 import inputs as I  # noqa: E402

h = binding.Handle(0)
lib = binding.load()
m, n, r = [int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (4096, 1024, 1024))]
G = I.low_rank(1, m, n, r, device="cuda") if r < n else I.dense_normal(1, m, n, device="cuda")
A = torch.zeros(n, n, dtype=torch.float64, device="cuda")
h.geninv_gram_d(G, 0, A)
for _ in range(3):
    h.geninv_frchol_d(A)
torch.cuda.synchronize()
np_ = (n + 31) // 32
buf = (ctypes.c_ulonglong * (np_ * 8))()
lib.geninv_debug_panel_times(buf, np_)
t = np.array(buf, dtype=np.float64).reshape(np_, 8)
d = np.stack([t[:, 5] - t[:, 0], t[:, 1] - t[:, 5], t[:, 2] - t[:, 1], t[:, 7] - t[:, 1], t[:, 4] - t[:, 1],
              t[:, 6] - t[:, 4], np.maximum(t[:, 2], t[:, 6]) - t[:, 0]], axis=1) / 1e3
end = np.maximum(t[:, 2], t[:, 6])
gap = (t[1:, 0] - end[:-1]) / 1e3
names = ["loads", "correction", "diag factor", "row correction done", "rows solved (from correction)",
         "write-back", "kernel"]
med = np.median(d[2:-1], axis=0)
print(f"s={n}: {np_} panels; median us per phase (panels >= 2): " +
      ", ".join(f"{a} {b:.2f}" for a, b in zip(names, med)) + f"; gap to next {np.median(gap):.2f}")
print(f"  span of the whole factorisation: {(end[-1] - t[0, 0]) / 1e3:.0f} us")
kern = d[:, 6]
print(f"  sum of kernel times {kern.sum():.0f} us, sum of gaps {gap.sum():.0f} us; gap percentiles 50/90/99: "
      + " / ".join(f"{np.percentile(gap, q):.2f}" for q in (50, 90, 99))
      + "; largest gaps (panel: us): " + ", ".join(f"{i + 1}: {gap[i]:.1f}" for i in np.argsort(gap)[::-1][:8]))
