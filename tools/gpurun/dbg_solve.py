import sys, os, subprocess, torch, numpy as np
sys.path.insert(0, os.getcwd())
from paper_0804_4809_b200 import inputs as I
from paper_0804_4809_b200.binding import Handle
H = Handle(0)
case = sys.argv[1:]
m, n, r, k = map(int, case)
G = torch.as_tensor(I.low_rank(31334, m, n, r).numpy()).cuda()
if n % 2:
    Gq = torch.zeros(m, n + 1, dtype=torch.float64, device="cuda"); Gq[:, :n] = G; G = Gq[:, :n]
F = torch.zeros(m, (k + 1) // 2 * 2, dtype=torch.float64, device="cuda"); F[:, :k] = torch.as_tensor(I.dense_normal(3, m, k).numpy())
try:
    W, info = H.geninv_solve_d(G, F[:, :k])
    torch.cuda.synchronize()
    print(case, "ok", info.rank, flush=True)
except Exception as e:
    print(case, "FAIL", e, flush=True)
