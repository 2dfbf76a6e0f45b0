"""Per-phase cycle counts of the batched kernel (debug build with GI_BATCHED_TIMING).

    python -m paper_0804_4809_b200.build --timing      # -> libgeninv_timing.so
    GENINV_LIB=paper_0804_4809_b200/libgeninv_timing.so python tools/batched_phases.py [batch]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_0804_4809_b200 import binding as B  # noqa: E402
from paper_0804_4809_b200 import inputs as I  # noqa: E402

NAMES = ["load G", "Gram+store", "tol", "frchol", "L'L", "M = inv(L'L) (sweep)", "K", "X", "output"]


def main():
    nb = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    cfg = I.CONFIGS["C5"]
    h = B.Handle(0)
    G = I.make_batch(cfg, 1, 0, nb, device="cuda")
    Gp, rk = h.geninv_batched_d(G)
    Gp, rk = h.geninv_batched_d(G, Gp, rk)
    torch.cuda.synchronize()
    lib = B.load()
    buf = np.zeros((4096, 16), dtype=np.int64)
    lib.geninv_debug_batched_times.argtypes = [ctypes.c_void_p, ctypes.c_int]
    lib.geninv_debug_batched_times(buf.ctypes.data, 4096)
    t = buf[:min(nb, 4096)]
    seq = [0, 1, 2, 3, 4, 5, 6, 8, 9, 10]
    d = np.diff(t[:, seq], axis=1)
    tot = t[:, 10] - t[:, 0]
    print(f"cycles per matrix (median over {len(t)} CTAs): total {np.median(tot):.0f}")
    for name, col in zip(NAMES, d.T):
        print(f"  {name:12s} {np.median(col):8.0f}  ({np.median(col) / np.median(tot) * 100:4.1f} %)")
    # one sweep step (k0 = 8): chain (V rows), barrier 1, update + K entries + publish, barrier 2
    if t[:, 12].any():
        st = np.diff(t[:, [12, 7, 13, 11]], axis=1)
        print("  sweep step k0 = 8: chain %.0f, barrier %.0f, update/fix/publish %.0f cycles" % tuple(np.median(st, axis=0)))
    if t[:, 14].any():
        print("  output: start -> chunk 0 ready %.0f, chunk 0 products %.0f cycles" % (
            np.median(t[:, 14] - t[:, 9]), np.median(t[:, 15] - t[:, 14])))


if __name__ == "__main__":
    main()
