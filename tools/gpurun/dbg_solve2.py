import sys, os, ctypes, torch, numpy as np
sys.path.insert(0, os.getcwd())
from cuda.bindings import runtime as cudart
from paper_0804_4809_b200 import inputs as I
from paper_0804_4809_b200.binding import Handle, _Info, _opts
H = Handle(0)
m, n, k = 1000, 333, 5
G = I.low_rank(31334, m, n, 260).numpy()
F = I.dense_normal(3, m, k).numpy()
which = sys.argv[1]
def exact(arr, ld):
    rows, cols = arr.shape
    buf = np.zeros((rows, ld)); buf[:, :cols] = arr
    err, p = cudart.cudaMalloc(buf.nbytes)
    cudart.cudaMemcpy(p, buf.ctypes.data, buf.nbytes, cudart.cudaMemcpyKind.cudaMemcpyHostToDevice)
    return p
pG = exact(G, 334) if which in ("G", "both") else None
pF = exact(F, 6) if which in ("F", "both") else None
tG = torch.zeros(m, 334, dtype=torch.float64, device="cuda"); tG[:, :n] = torch.as_tensor(G)
tF = torch.zeros(m, 6, dtype=torch.float64, device="cuda"); tF[:, :k] = torch.as_tensor(F)
W = torch.empty(n, k, dtype=torch.float64, device="cuda")
rank, info, o = ctypes.c_int64(), _Info(), _opts()
st = H._lib.geninv_solve_d(H._h, pG if pG else tG.data_ptr(), m, n, 334, pF if pF else tF.data_ptr(), k, 6,
                           W.data_ptr(), k, ctypes.byref(rank), ctypes.byref(o), ctypes.byref(info))
print(which, "status", st, rank.value, flush=True)
