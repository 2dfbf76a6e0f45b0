"""Full-size C4 (2^21 x 4096, rank 3584): Gram time and the four Penrose residuals of the device's G+
(tests/gpu_checks.py checker), for the Gram-accumulation knob in the environment
(GENINV_GRAM_CHUNK_ROWS) -- measurement tool, one JSON line per run.

    python tools/c4_rho.py [seed]
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0804_4809_b200 import inputs as I           # noqa: E402
from paper_0804_4809_b200.binding import Handle        # noqa: E402
from tests.gpu_checks import penrose_streamed          # noqa: E402


def main():
    seed = int(sys.argv[1]) if len(sys.argv) > 1 else I.QSEED["C4"]
    cfg = I.CONFIGS["C4"]
    m, n = cfg.m, cfg.n
    h = Handle(0)
    G = I.make_single(cfg, seed, device="cuda")
    A = torch.zeros(n, n, dtype=torch.float64, device="cuda")
    Gp = torch.empty(n, m, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream()
    ts = []
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        A.zero_()
        torch.cuda.synchronize()
        e0.record(st)
        h.geninv_gram_d(G, 0, A)
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    info = h.geninv_from_gram_d(A)
    h.geninv_apply_d(G, 0, Gp)
    torch.cuda.synchronize()
    t0 = time.time()
    rho = penrose_streamed(G, Gp)
    out = {"seed": seed, "chunk_rows": os.environ.get("GENINV_GRAM_CHUNK_ROWS", "default"), "rank": info.rank,
           "mu_acc": info.mu_acc, "mu_drop": info.mu_drop, "gram_ms": ts, "rho": rho, "check_s": time.time() - t0}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
