"""One geninv_d call of a config between cudaProfilerStart/Stop (for ncu --profile-from-start off).

    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv python tools/one_call.py C2
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_0804_4809_b200 import inputs as I  # noqa: E402
from paper_0804_4809_b200.binding import Handle  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    if name == "C3T":
        G = I.make_single(I.CONFIGS["C3"], I.QSEED["C3"], device="cuda").T.contiguous()
    else:
        cfg = I.CONFIGS[name]
        G = I.make_single(cfg, I.QSEED[name], device="cuda")
    h = Handle(0)
    Gp, info = h.geninv_d(G)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    h.geninv_d(G, Gp)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print(name, "rank", info.rank)


if __name__ == "__main__":
    main()
