import sys, os, torch
sys.path.insert(0, "/root/repo")
from paper_0804_4809_b200 import inputs as I
from paper_0804_4809_b200.binding import Handle
cfg = I.CONFIGS["C4"]
rows = 1 << 20
h = Handle(0)
G = I.make_single(cfg, I.QSEED["C4"], device="cuda", rows=rows)
A = torch.zeros(cfg.n, cfg.n, dtype=torch.float64, device="cuda")
Gp = torch.empty(cfg.n, rows, dtype=torch.float64, device="cuda")
h.geninv_gram_d(G, 0, A); h.geninv_from_gram_d(A)
def t(f, n=3):
    ts=[]
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record(); f(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return sorted(ts)[n//2]
tg = t(lambda: h.geninv_gram_d(G, 0, A))
ta = t(lambda: h.geninv_apply_d(G, 0, Gp))
print(f"{os.path.basename(os.environ.get('GENINV_LIB','libgeninv.so'))}: gram {tg:.2f} ms  apply {ta:.2f} ms")
