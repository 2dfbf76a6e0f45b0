import os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
from paper_0804_4809_b200 import inputs as I
from paper_0804_4809_b200.binding import Handle
G = I.make_single(I.CONFIGS["C3"], I.QSEED["C3"], device="cuda").T.contiguous()
h = Handle(0); h.set_emulation(1)
Gp, info = h.geninv_d(G); torch.cuda.synchronize()
torch.cuda.profiler.start(); h.geninv_d(G, Gp); torch.cuda.synchronize(); torch.cuda.profiler.stop()
