"""Time the batched kernel (C5: 65,536 x 96 x 64, rank 40) through geninv_batched_d.

    python tools/time_batched.py [reps]

Prints ms per batch, us per matrix and GFLOP/s (F_alg of bench.py with the detected ranks).
Set GENINV_BATCHED_MINB=2 to time the 2-CTA/SM build of the kernel.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_0804_4809_b200 import inputs as I  # noqa: E402
from paper_0804_4809_b200.binding import Handle  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    cfg = I.CONFIGS["C5"]
    if len(sys.argv) > 2:                            # smaller batch (profiling)
        cfg = I.Config("C5", cfg.m, cfg.n, cfg.rank, batch=int(sys.argv[2]))
    h = Handle(0)
    G = I.make_batch(cfg, 1, 0, cfg.batch, device="cuda")
    Gp = torch.empty(cfg.batch, cfg.n, cfg.m, dtype=torch.float64, device="cuda")
    rk = torch.empty(cfg.batch, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream()
    h.use_stream(st)
    for _ in range(3):
        h.geninv_batched_d(G, Gp, rk)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        h.geninv_batched_d(G, Gp, rk)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    r = rk.cpu().numpy().astype(np.int64)
    s, ell = cfg.s, cfg.ell
    # F_alg per matrix with rank r and the r leading columns accepted (bench.py's batched model)
    fl = 0.0
    for rv, cnt in zip(*np.unique(r, return_counts=True)):
        k = np.arange(s)
        rk_ = np.minimum(k, rv)
        chol = float(np.sum(2.0 * (s - k) * rk_ + (s - k)))
        fl += cnt * (ell * s * (s + 1) + chol + s * rv * (rv + 1) + rv ** 3 + 2.0 * s * rv * rv
                     + s * (s + 1) * rv + 2.0 * s * s * ell)
    print(f"minb={os.environ.get('GENINV_BATCHED_MINB', '3')} ms {ms:.3f}  us/matrix {ms * 1e3 / cfg.batch:.4f}  "
          f"GFLOP/s {fl / ms / 1e6:.0f}  ranks {np.unique(r, return_counts=True)}")


if __name__ == "__main__":
    main()
