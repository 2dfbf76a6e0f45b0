import sys, os, torch, numpy as np
sys.path.insert(0, os.getcwd())
from paper_0804_4809_b200 import inputs as I
from paper_0804_4809_b200.binding import Handle
H = Handle(0)
m, n, k = 1000, 333, 5
G = I.low_rank(31334, m, n, 260).numpy()
F = I.dense_normal(3, m, k).numpy()
padval = float(sys.argv[1])
tG = torch.full((m, 334), padval, dtype=torch.float64, device="cuda"); tG[:, :n] = torch.as_tensor(G)
tF = torch.zeros(m, 6, dtype=torch.float64, device="cuda"); tF[:, :k] = torch.as_tensor(F)
try:
    W, info = H.geninv_solve_d(tG[:, :n], tF[:, :k]); torch.cuda.synchronize(); print(padval, "ok", flush=True)
except Exception as e:
    print(padval, "FAIL", e, flush=True)
