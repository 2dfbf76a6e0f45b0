"""One a7 output-product launch (G+ = X G') of the C4 workload, bracketed by cudaProfilerStart/Stop
so that `ncu --profile-from-start off` captures exactly that kernel.

    ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        python tools/ncu_apply.py [rows] [seed]

rows defaults to the full 2^21 of C4 (the launch bench.py times); a smaller row count gives a
smaller launch of the same kernel for `--set full` captures (replay has to save its 64 GiB output).
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_0804_4809_b200 import inputs as I  # noqa: E402
from paper_0804_4809_b200.binding import Handle  # noqa: E402


def main():
    cfg = I.CONFIGS["C4"]
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else cfg.m
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else I.QSEED["C4"]
    h = Handle(0)
    G = I.make_single(cfg, seed, device="cuda", rows=rows)
    A = torch.zeros(cfg.n, cfg.n, dtype=torch.float64, device="cuda")
    Gp = torch.empty(cfg.n, rows, dtype=torch.float64, device="cuda")
    h.geninv_gram_d(G, 0, A)
    h.geninv_from_gram_d(A)
    h.geninv_apply_d(G, 0, Gp)                       # warm (tensor maps, L2)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    h.geninv_apply_d(G, 0, Gp)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print(f"apply launch: {cfg.n} x {rows} x {cfg.n}, flops {2.0 * cfg.n * cfg.n * rows:.4g}")


if __name__ == "__main__":
    main()
