"""Time the minimum-norm least-squares solve W = G+ F (geninv_solve_d) against forming G+
(geninv_d) on a BASELINE config, k right-hand sides, inputs resident in HBM, CUDA events, median.

    python tools/time_solve.py [C4|C3T|C2] [k] [reps]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_0804_4809_b200 import inputs as I  # noqa: E402
from paper_0804_4809_b200.binding import Handle  # noqa: E402


def timed(fn, reps):
    fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C4"
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    if name == "C3T":
        G = I.make_single(I.CONFIGS["C3"], I.QSEED["C3"], device="cuda").T.contiguous()
    else:
        G = I.make_single(I.CONFIGS[name], I.QSEED[name], device="cuda")
    m, n = G.shape
    F = I.normal_matrix(I.stream_key(7, 99), m, k, device="cuda")
    h = Handle(0)
    W, info = h.geninv_solve_d(G, F)
    t_solve = timed(lambda: h.geninv_solve_d(G, F, W), reps)
    res = {"config": name, "m": m, "n": n, "k": k, "rank": info.rank, "solve_ms": t_solve}
    if m * n * 8 * 2 < 150e9:   # room for G+ next to G (C4: 64 + 64 GiB)
        Gp = torch.empty(n, m, dtype=torch.float64, device="cuda")
        t_gp = timed(lambda: h.geninv_d(G, Gp), reps)
        res["geninv_ms"] = t_gp
        res["geninv_then_gemm_ms"] = t_gp + timed(lambda: Gp @ F, reps)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
