"""geninv_d with the a7 product on the FP64 tensor cores (mode 0) and emulated on the INT8 tensor
cores (mode 1): time of each (median, CUDA events, input resident) and the relative difference of the
two G+ (Frobenius; C4 on a column sample).

    python tools/time_emulated.py C2 C3T C4
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
    torch.cuda.synchronize()
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
    for name in sys.argv[1:] or ["C2", "C3T"]:
        if name == "C3T":
            G = I.make_single(I.CONFIGS["C3"], I.QSEED["C3"], device="cuda").T.contiguous()
        else:
            G = I.make_single(I.CONFIGS[name], I.QSEED[name], device="cuda")
        m, n = G.shape
        h = Handle(0)
        reps = 2 if name == "C4" else 10
        res = {"config": name}
        out = {}
        for mode in (0, 1):
            h.set_emulation(mode)
            Gp = torch.empty(n, m, dtype=torch.float64, device="cuda")
            res[f"ms_mode{mode}"] = timed(lambda: h.geninv_d(G, Gp), reps)
            # keep a sample of columns (C4: 64 GiB per G+)
            cols = torch.arange(0, m, max(1, m // 4096), device="cuda")
            out[mode] = Gp[:, cols].clone()
            del Gp
            torch.cuda.empty_cache()
        res["rel_diff_sampled"] = float(torch.linalg.norm(out[1] - out[0]) / torch.linalg.norm(out[0]))
        print(json.dumps(res), flush=True)
        del G
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
