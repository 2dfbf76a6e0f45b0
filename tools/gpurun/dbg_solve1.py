import sys, os, torch, numpy as np
sys.path.insert(0, os.getcwd())
from paper_0804_4809_b200 import inputs as I
from paper_0804_4809_b200.binding import Handle
H = Handle(0)
m, n = 1000, 333
G = I.low_rank(31334, m, n, 260).numpy()
F = I.dense_normal(3, m, 5).numpy()
mode = sys.argv[1]
Gd = torch.as_tensor(G).cuda()                          # ld 333: staged
Fp = torch.zeros(m, 6, dtype=torch.float64, device="cuda"); Fp[:, :5] = torch.as_tensor(F)
print("G", hex(Gd.data_ptr()), "F", hex(Fp.data_ptr()), flush=True)
if mode == "d":
    Gp, info = H.geninv_d(Gd); torch.cuda.synchronize(); print("geninv_d ok", flush=True)
try:
    W, info = H.geninv_solve_d(Gd, Fp[:, :5])
    torch.cuda.synchronize()
    print(mode, "ok", info.rank, flush=True)
except Exception as e:
    print(mode, "FAIL", e, flush=True)
