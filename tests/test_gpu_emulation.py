"""a7 emulated on the INT8 tensor cores (geninv_set_emulation(1)) against the oracle
(`-m gpu`): the same gates as the native path (rank exact, G+ within 1e-9 of the oracle, Penrose
residuals <= 1e-10 on inputs in Q) on ragged shapes -- M, N, K off the 128 / 256 / 128-byte tile
grid, K not a multiple of 16 (padded slices), several G chunks -- and agreement with the native
FP64 tensor-core path within the summation-order noise of the chain (1e-10, as the schedule variants
of tests/test_gpu_variants.py; the emulated products' own error bound is below an FP64 GEMM's).
The Gram is emulated from s >= 3072 (test_emulated_gram_c3t), a7 on every shape of both branches."""
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
    h = Handle(0)
    yield h
    h.set_emulation(0)


def dev(X):
    m, n = X.shape
    t = torch.zeros(m, (n + 1) // 2 * 2, dtype=torch.float64, device="cuda")
    t[:, :n] = torch.as_tensor(X)
    return t[:, :n]


def penrose(G, X):
    G = torch.as_tensor(G).cuda()
    X = torch.as_tensor(X).cuda()
    GX, XG = G @ X, X @ G
    E = [GX @ G - G, XG @ X - X, GX.T - GX, XG.T - XG]
    D = [G, X, GX, XG]
    return [float(torch.linalg.norm(e) / torch.linalg.norm(d)) for e, d in zip(E, D)]


@pytest.mark.parametrize("m,n,r", [(300, 140, 100), (1000, 333, 260), (2050, 530, 400), (700, 200, 200),
                                   (4100, 129, 120), (1500, 1024, 1024),
                                   (140, 300, 100), (333, 1000, 260), (530, 2050, 400), (129, 4100, 120)])
def test_emulated_matches_oracle(H, m, n, r):
    G = I.low_rank(m * 7 + n, m, n, r).numpy() if r < n else I.dense_normal(m * 7 + n, m, n).numpy()
    R = O.geninv(G)
    assert R.in_Q()
    H.set_emulation(1)
    Gp, info = H.geninv_d(dev(G))
    H.set_emulation(0)
    Gn, _ = H.geninv_d(dev(G))
    assert info.rank == R.rank
    gp = Gp.cpu().numpy()
    assert C.rel_fro(gp, R.Gp) <= 1e-9
    assert max(penrose(G, gp)) <= 1e-10
    assert C.rel_fro(gp, Gn.cpu().numpy()) <= 1e-10   # summation-order noise, as test_gpu_variants


def test_emulated_c2(H):
    G = I.make_single(I.CONFIGS["C2"], I.QSEED["C2"], device="cuda")
    H.set_emulation(1)
    Gp, info = H.geninv_d(G)
    H.set_emulation(0)
    R = O.geninv(G.cpu().numpy())
    assert info.rank == R.rank == 1024
    assert C.rel_fro(Gp.cpu().numpy(), R.Gp) <= 1e-9
    assert max(penrose(G.cpu().numpy(), Gp.cpu().numpy())) <= 1e-10


def test_emulated_deterministic(H):
    G = I.low_rank(5, 3000, 700, 600, device="cuda")
    H.set_emulation(1)
    a, _ = H.geninv_d(G)
    b, _ = H.geninv_d(G)
    H.set_emulation(0)
    assert torch.equal(a, b)


def test_emulated_gram_c3t(H):
    """C3T (s = 4096): the Gram (K-chunks of 16384 rows, column digit planes) and a7 both emulated."""
    G = I.make_single(I.CONFIGS["C3"], I.QSEED["C3"], device="cuda").T.contiguous()
    H.set_emulation(1)
    Gp, info = H.geninv_d(G)
    H.set_emulation(0)
    Gh = G.cpu().numpy()
    R = O.geninv(Gh)
    assert R.in_Q()
    assert info.rank == R.rank == 3072
    assert C.rel_fro(Gp.cpu().numpy(), R.Gp) <= 1e-9
    assert max(penrose(Gh, Gp.cpu().numpy())) <= 1e-10


def test_emulated_c3_t_branch(H):
    """C3 (4096 x 16384, T branch): the Gram from row digit planes, a7 = G' X from column digit planes."""
    G = I.make_single(I.CONFIGS["C3"], I.QSEED["C3"], device="cuda")
    H.set_emulation(1)
    Gp, info = H.geninv_d(G)
    H.set_emulation(0)
    Gh = G.cpu().numpy()
    R = O.geninv(Gh)
    assert R.in_Q() and info.transposed
    assert info.rank == R.rank == 3072
    assert C.rel_fro(Gp.cpu().numpy(), R.Gp) <= 1e-9
    assert max(penrose(Gh, Gp.cpu().numpy())) <= 1e-10


@pytest.mark.parametrize("scale", [1e-150, 1e150])
def test_emulated_extreme_scales(H, scale):
    G0 = I.low_rank(31, 300, 140, 100).numpy()
    R = O.geninv(G0)
    H.set_emulation(1)
    Gp, info = H.geninv_d(dev(G0 * scale))
    H.set_emulation(0)
    assert info.rank == R.rank
    assert C.rel_fro(Gp.cpu().numpy() * scale, R.Gp) <= 1e-9


def test_emulated_nonfinite_and_zero(H):
    from paper_0804_4809_b200.binding import GENINV_ENONFINITE, GeninvError
    G = I.dense_normal(3, 4000, 3100).numpy()        # s >= 3072: the emulated Gram path
    G[17, 5] = np.nan
    H.set_emulation(1)
    try:
        with pytest.raises(GeninvError) as exc:
            H.geninv_d(dev(G))
        assert exc.value.status == GENINV_ENONFINITE
        Z = torch.zeros(400, 130, dtype=torch.float64, device="cuda")
        Gp, info = H.geninv_d(Z)
        assert info.rank == 0 and not Gp.any()
    finally:
        H.set_emulation(0)


@pytest.mark.parametrize("m,n,seed", [(6200, 4500, 10700), (4500, 6200, 10701)])   # seeds in Q (oracle)
def test_emulated_two_k_passes(H, m, n, seed):
    """s = 4500 > 4096: a7 over two exact int32 K passes with their own exponents, the Gram in
    K-chunks (both branches)."""
    G = I.low_rank(seed, m, n, 4300, device="cuda")
    H.set_emulation(1)
    Gp, info = H.geninv_d(G)
    H.set_emulation(0)
    Gh = G.cpu().numpy()
    R = O.geninv(Gh)
    assert R.in_Q()
    assert info.rank == R.rank == 4300
    assert C.rel_fro(Gp.cpu().numpy(), R.Gp) <= 1e-9
    assert max(penrose(Gh, Gp.cpu().numpy())) <= 1e-10
