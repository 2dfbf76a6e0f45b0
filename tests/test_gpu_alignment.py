"""Any leading dimension >= n and any 8-byte-aligned base pointer through the C ABI (`-m gpu`).

The tensor-core path needs 16-byte-aligned bases and even leading dimensions for its TMA views;
the library stages such operands into an aligned copy (include/geninv.h "Alignment").  The paper's
problem is any real m x n G, so odd shapes stored contiguously (odd ld) and views
starting at an odd element must give the oracle's result.
"""
import ctypes

import numpy as np
import pytest
import torch

from oracle import checks as C
from oracle import geninv_oracle as O
from paper_0804_4809_b200 import inputs as I

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def H():
    from paper_0804_4809_b200.binding import Handle
    return Handle(0)


def offset_view(G, off):
    """G (m x n) stored contiguously (ld = n) starting `off` doubles into a fresh device buffer."""
    m, n = G.shape
    buf = torch.zeros(m * n + off + 1, dtype=torch.float64, device="cuda")
    v = buf[off:off + m * n].view(m, n)
    v.copy_(torch.as_tensor(G))
    return v


CASES = [  # (m, n, rank, seed, full_rank): seeds in Q (tools/screen_q_cpu.py; full rank: dense N(0,1))
    (1000, 333, 260, 31334, False),
    (333, 1000, 260, 31334, False),
    (4097, 1023, 1023, 7, True),
]


def make(m, n, r, seed, full):
    return I.dense_normal(seed, m, n).numpy() if full else I.low_rank(seed, m, n, r).numpy()


@pytest.mark.parametrize("off", [0, 1])
@pytest.mark.parametrize("m,n,r,seed,full", CASES)
def test_geninv_d_any_ld_and_offset(H, m, n, r, seed, full, off):
    G = make(m, n, r, seed, full)
    R = O.geninv(G)
    assert R.in_Q() and R.rank == r
    Gd = offset_view(G, off)
    # odd n (contiguous: odd ld) or off = 1 (base 8 mod 16): operands the TMA path cannot read in place
    Gp, info = H.geninv_d(Gd)
    assert info.rank == R.rank
    assert C.rel_fro(Gp.cpu().numpy(), R.Gp) <= 1e-9
    # the input is never written
    assert np.array_equal(Gd.cpu().numpy(), G)
    # async variant: same G+
    Ga, rk = H.geninv_d_async(Gd)
    torch.cuda.synchronize()
    assert int(rk[0]) == R.rank
    assert C.rel_fro(Ga.cpu().numpy(), R.Gp) <= 1e-9


@pytest.mark.parametrize("m,n,r,seed,full", CASES[:1])
def test_split_api_and_solve_unaligned(H, m, n, r, seed, full):
    G = make(m, n, r, seed, full)
    R = O.geninv(G)
    Gd = offset_view(G, 1)
    A = torch.zeros(n, n + 2, dtype=torch.float64, device="cuda")[:, :n]   # odd lda (335) as well
    H.geninv_gram_d(Gd, 0, A)
    info = H.geninv_from_gram_d(A)
    assert info.rank == R.rank
    Gp = torch.empty(n, m, dtype=torch.float64, device="cuda")
    H.geninv_apply_d(Gd, 0, Gp)
    torch.cuda.synchronize()
    assert C.rel_fro(Gp.cpu().numpy(), R.Gp) <= 1e-9
    # least squares with an odd-width, offset right-hand side F
    F = I.dense_normal(3, m, 5).numpy()
    Fd = offset_view(F, 1)
    W, winfo = H.geninv_solve_d(Gd, Fd)
    Wo, ro = O.solve(G, F)
    assert winfo.rank == ro
    assert C.rel_fro(W.cpu().numpy(), Wo) <= 1e-9


def test_frchol_odd_ldl(H):
    # the step entry point with an odd leading dimension of L (its TMA operand is then the handle's L)
    from paper_0804_4809_b200.binding import _Info, _opts, _check
    G = make(1000, 333, 260, 31334, False)
    A, _ = O.gram(G)
    ch = O.full_rank_cholesky(A, O.tolerance(A))
    s = 333
    Ad = torch.as_tensor(A).cuda()
    L = torch.full((s, s), 5.0, dtype=torch.float64, device="cuda")   # ld = 333 (odd)
    piv = torch.empty(s, dtype=torch.int32, device="cuda")
    rank, info, o = ctypes.c_int64(), _Info(), _opts()
    _check(H._lib.geninv_frchol_d(H._h, Ad.data_ptr(), s, s, L.data_ptr(), s, piv.data_ptr(), ctypes.byref(rank),
                                  ctypes.byref(o), ctypes.byref(info)))
    r = rank.value
    assert r == ch.rank
    assert np.array_equal(piv[:r].cpu().numpy(), ch.piv)
    assert bool((L[:, r:] == 0).all())
    # the same kernels as the aligned call: identical bits
    La, pa, ia = H.geninv_frchol_d(Ad)
    assert ia.rank == r and torch.equal(pa, piv[:r])
    assert torch.equal(La, L[:, :r])
