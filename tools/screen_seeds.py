"""Pre-screen seeds of the large configs by the device's own decision margins.

    python tools/screen_seeds.py C4 1 12

For each seed: build G on the GPU (same generator as tests/bench), run the
split C ABI (gram -> from_gram) and print the device's mu_acc = min accepted
pivot / tol and mu_drop = max |dropped pivot| / tol.  This is a screen only:
the chosen seed (inputs.QSEED) is confirmed against the ORACLE's margins in
tests/test_gpu_c4_full.py / test_gpu_parity.py, which assert predicate Q.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_0804_4809_b200 import inputs as I  # noqa: E402
from paper_0804_4809_b200.binding import Handle  # noqa: E402


def main():
    name = sys.argv[1]
    s0, s1 = int(sys.argv[2]), int(sys.argv[3])
    cfg = I.CONFIGS[name]
    h = Handle(0)
    tr = int(cfg.m < cfg.n)
    s = cfg.s
    A = torch.zeros(s, s, dtype=torch.float64, device="cuda")
    G = torch.empty(cfg.m, cfg.n, dtype=torch.float64, device="cuda")
    for seed in range(s0, s1 + 1):
        I.make_single(cfg, seed, device="cuda", out=G) if cfg.ncopy == 0 else G.copy_(I.make_single(cfg, seed, device="cuda"))
        A.zero_()
        h.geninv_gram_d(G, tr, A)
        info = h.geninv_from_gram_d(A)
        print(json.dumps({"config": name, "seed": seed, "rank": info.rank, "mu_acc": info.mu_acc,
                          "mu_drop": info.mu_drop, "Q": info.mu_acc >= 1e4 and info.mu_drop <= 1e-2,
                          "Qstar": info.mu_acc >= 1e6 and info.mu_drop <= 1e-3}), flush=True)


if __name__ == "__main__":
    main()
