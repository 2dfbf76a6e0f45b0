"""The paper's own workload on B200: a Table-1-style column for geninv.

    python tools/table1.py [max_log2_n] [reps]  > profiles/r01_table1.json

PAPER.md P:84 (section 3): m = 2n, n = 2^k, rank r = 7n/8, coefficients uniform in [-1, 1]
(construction: reading R16, inputs.paper_family).  For each n: the wall time of one geninv_d call
(median of `reps`, CUDA events, input resident in HBM), its GFLOP/s (F_alg of bench.py), the detected
rank, and the largest absolute coefficient of the four Penrose error matrices (the paper's 2e-10
criterion, P:84 / Table 1 caption), computed with cuBLAS (test-only checker).  For n <= 64 the
batched kernel's time per matrix over a batch of 65,536 copies of the family is added.
The paper's own times (Matlab 6.5.1, 2005 PC, Table 1) are quoted as context only.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_0804_4809_b200 import inputs as I  # noqa: E402
from paper_0804_4809_b200.binding import Handle  # noqa: E402

PAPER_S = {32: 0.007, 64: 0.022, 128: 0.105, 256: 0.768, 512: 6.445, 1024: 54.137}  # Table 1, geninv column


def f_alg(s, ell, r):
    k = np.arange(s)
    rk = np.minimum(k, r)
    chol = float(np.sum(2.0 * (s - k) * rk + (s - k)))
    return ell * s * (s + 1) + chol + s * r * (r + 1) + r ** 3 + 2.0 * s * r * r + s * (s + 1) * r + 2.0 * s * s * ell


def main():
    kmax = int(sys.argv[1]) if len(sys.argv) > 1 else 13
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    h = Handle(0)
    st = torch.cuda.current_stream()
    rows = []
    for k in range(5, kmax + 1):
        n = 1 << k
        m = 2 * n
        G = I.paper_family(n, I.PAPER_QSEED.get(n, 1), device="cuda")
        Gp = torch.empty(n, m, dtype=torch.float64, device="cuda")
        _, info = h.geninv_d(G, Gp)
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            h.geninv_d(G, Gp)
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        GX, XG = G @ Gp, Gp @ G
        err = max(float((GX @ G - G).abs().max()), float((XG @ Gp - Gp).abs().max()),
                  float((GX.T - GX).abs().max()), float((XG.T - XG).abs().max()))
        row = {"n": n, "m": m, "seed": I.PAPER_QSEED.get(n, 1), "rank": info.rank, "rank_constructed": 7 * n // 8, "ms": ms,
               "gflops": f_alg(n, m, info.rank) / (ms * 1e-3) / 1e9, "penrose_abs_max": err,
               "paper_matlab_s": PAPER_S.get(n)}
        if n <= 64:
            nb = 65536
            Gb = G.unsqueeze(0).expand(nb, m, n).contiguous()
            Gpb, rk = h.geninv_batched_d(Gb)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(5):
                h.geninv_batched_d(Gb, Gpb, rk)
            e1.record(st)
            torch.cuda.synchronize()
            row["batched_us_per_matrix"] = e0.elapsed_time(e1) / 5 / nb * 1e3
            del Gb, Gpb
        rows.append(row)
        print(json.dumps(row), file=sys.stderr, flush=True)
    print(json.dumps({"what": "Table-1 analogue: geninv_d on the paper's family (P:84) on one B200",
                      "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
