"""Degenerate and boundary inputs through the C ABI (`-m gpu`): vectors, rank 0 and 1, the
small / general path boundary, padded and odd leading dimensions, strided batches, invalid
arguments.  Expected values come from the oracle (or exact closed forms)."""
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


def dev(X, pad=0):
    m, n = X.shape
    t = torch.zeros(m, n + pad, dtype=torch.float64, device="cuda")
    t[:, :n] = torch.as_tensor(X)
    return t[:, :n]


@pytest.mark.parametrize("m,n", [(1, 1), (1, 7), (9, 1), (1, 300), (500, 1), (2, 2)])
def test_vectors_and_tiny(H, m, n):
    G = I.dense_normal(m * 100 + n, m, n).numpy()
    Gp, info = H.geninv_d(dev(G, pad=(n & 1)))
    R = O.geninv(G)
    assert info.rank == R.rank == min(m, n)
    assert C.rel_fro(Gp.cpu().numpy(), R.Gp) <= 1e-12


def test_rank_one_closed_form(H):
    # G = u v': G+ = v u' / (|u|^2 |v|^2)
    u = I.dense_normal(1, 200, 1).numpy()
    v = I.dense_normal(2, 90, 1).numpy()
    G = u @ v.T
    Gp, info = H.geninv_d(dev(G))
    assert info.rank == 1
    want = (v @ u.T) / (float((u.T @ u)[0, 0]) * float((v.T @ v)[0, 0]))
    assert C.rel_fro(Gp.cpu().numpy(), want) <= 1e-12


@pytest.mark.parametrize("m,n", [(64, 64), (128, 64), (64, 128), (129, 64), (64, 65), (65, 64)])
def test_small_path_boundary(H, m, n):
    # min(m, n) <= 64 and max(m, n) <= 128 run the one-CTA kernel, the rest the general path
    r = min(m, n) - 3
    # seed: first >= m * 7 + n with oracle margins in Q (tools/screen_q_cpu.py)
    seed = {(64, 64): 512, (128, 64): 960, (64, 128): 576, (129, 64): 967, (64, 65): 513, (65, 64): 519}[(m, n)]
    G = I.low_rank(seed, m, n, r).numpy()
    R = O.geninv(G)
    assert R.in_Q()
    Gp, info = H.geninv_d(dev(G, pad=1))   # odd leading dimension on both paths (staged copy on the general path)
    assert info.rank == R.rank == r
    assert C.rel_fro(Gp.cpu().numpy(), R.Gp) <= 1e-9


def test_zero_matrix_both_paths(H):
    for (m, n) in ((50, 30), (600, 300), (300, 600)):
        Gp = torch.full((n, m), 3.0, dtype=torch.float64, device="cuda")
        _, info = H.geninv_d(torch.zeros(m, n, dtype=torch.float64, device="cuda"), Gp)
        assert info.rank == 0 and bool((Gp == 0).all())


def test_batched_strided_and_odd_ld(H):
    # a batch stored with padding between matrices and an odd leading dimension (8-byte copies)
    cfg = I.CONFIGS["C1"]
    base = torch.zeros(5, 64 + 3, 49, dtype=torch.float64, device="cuda")
    for i in range(5):
        base[i, :64, :48] = I.make_single(cfg, i + 1).cuda()
    G = base[:, :64, :48]                          # ld 49 (odd), stride 67 * 49
    Gp, rk = H.geninv_batched_d(G)
    torch.cuda.synchronize()
    for i in range(5):
        R = O.geninv(G[i].cpu().numpy())
        assert int(rk[i]) == R.rank
        assert C.rel_fro(Gp[i].cpu().numpy(), R.Gp) <= 1e-9


def test_batched_rank_zero_and_mixed(H):
    cfg = I.CONFIGS["C1"]
    Gs = torch.stack([I.make_single(cfg, 1), torch.zeros(64, 48, dtype=torch.float64),
                      I.low_rank(3, 64, 48, 1)]).cuda()
    Gp, rk = H.geninv_batched_d(Gs)
    torch.cuda.synchronize()
    assert rk.tolist() == [32, 0, 1]
    assert bool((Gp[1] == 0).all())
    for i in (0, 2):
        assert C.rel_fro(Gp[i].cpu().numpy(), O.geninv(Gs[i].cpu().numpy()).Gp) <= 1e-9


def test_invalid_arguments(H):
    from paper_0804_4809_b200.binding import GeninvError
    lib = H._lib
    G = torch.zeros(10, 4, dtype=torch.float64, device="cuda")
    Gp = torch.zeros(4, 10, dtype=torch.float64, device="cuda")
    # ld < n, ldp < m, m = 0, too large batched shapes -> GENINV_EINVAL (1)
    assert lib.geninv_d(H._h, G.data_ptr(), 10, 4, 3, Gp.data_ptr(), 10, None, None, None) == 1
    assert lib.geninv_d(H._h, G.data_ptr(), 10, 4, 4, Gp.data_ptr(), 9, None, None, None) == 1
    assert lib.geninv_d(H._h, G.data_ptr(), 0, 4, 4, Gp.data_ptr(), 10, None, None, None) == 1
    big = torch.zeros(2, 65, 65, dtype=torch.float64, device="cuda")
    with pytest.raises(GeninvError):
        H.geninv_batched_d(big)
    # split API: apply before any factorisation of that size -> GENINV_ESTATE (7)
    from paper_0804_4809_b200.binding import Handle
    h2 = Handle(0)
    assert h2._lib.geninv_apply_d(h2._h, G.data_ptr(), 10, 4, 4, 0, Gp.data_ptr(), 10) == 7


@pytest.mark.parametrize("m,n,r,seed", [(2000, 500, 350, 4500), (500, 2000, 350, 10500), (700, 300, 300, 2200),
                                        (400, 200, 0, 0)])
def test_async_matches_sync(H, m, n, r, seed):
    # geninv_d_async: no host synchronisation, rank on the device; the inverse runs at full size with
    # an identity block past the rank, which gives the same G+ as the rank-sized inverse of geninv_d.
    # seed: first >= m + 5n with oracle margins in Q (tools/screen_q_cpu.py)
    G = I.low_rank(seed, m, n, r).numpy() if r > 0 else np.zeros((m, n))
    Gs, info = H.geninv_d(dev(G))
    Ga, rk = H.geninv_d_async(dev(G))
    torch.cuda.synchronize()
    assert int(rk[0]) == info.rank == r
    R = O.geninv(G)
    if r == 0:
        assert bool((Ga == 0).all())
    else:
        assert C.rel_fro(Ga.cpu().numpy(), Gs.cpu().numpy()) <= 1e-9
        assert R.in_Q()
        assert C.rel_fro(Ga.cpu().numpy(), R.Gp) <= 1e-9


@pytest.mark.parametrize("scale", [1e-150, 1e-100, 1e100, 1e150])
@pytest.mark.parametrize("m,n,r", [(300, 140, 100), (90, 60, 40)])
def test_extreme_scales(H, scale, m, n, r):
    """G scaled by 1e+-150 (the Gram's entries near 1e+-300, still normal numbers): the relative
    tolerance makes the decisions scale-free, so rank and G+ * scale match the unscaled oracle's
    (the panel kernel's branch-free sqrt / reciprocal assumes normal pivots; the batched path
    covers the small shape)."""
    G0 = I.low_rank(31, m, n, r).numpy()
    R = O.geninv(G0)
    assert R.in_Q()
    G = G0 * scale
    Gp, info = H.geninv_d(dev(G))
    assert info.rank == R.rank
    assert C.rel_fro(Gp.cpu().numpy() * scale, R.Gp) <= 1e-9


@pytest.mark.parametrize("m,n", [(300, 140), (90, 60)])
def test_tiny_scale_fails_loudly(H, m, n):
    """Pivots below 2^-1022 are outside the branch-free sqrt / reciprocal's range: the call reports
    GENINV_ERANGE (general path) / rank -9 with NaN G+ (batched), never a silent wrong G+."""
    from paper_0804_4809_b200.binding import GENINV_ERANGE, GeninvError
    G = I.low_rank(32, m, n, 40).numpy() * 1e-158   # Gram ~1e-313: subnormal pivots
    with pytest.raises(GeninvError) as exc:
        H.geninv_d(dev(G))
    assert exc.value.status == GENINV_ERANGE
    if max(m, n) > 128:
        return
    Gb = torch.as_tensor(G[None]).cuda()
    Gp, rk = H.geninv_batched_d(Gb)
    torch.cuda.synchronize()
    assert int(rk[0]) == -GENINV_ERANGE
    assert torch.isnan(Gp).all()


# seeds: first seed >= m * 13 + n with oracle margins in Q (tools/screen_q_cpu.py test_batched_shape_sweep)
BATCHED_SWEEP_SEED = {(1, 1, 1): 14, (7, 3, 3): 94, (3, 7, 2): 46, (64, 64, 64): 896, (128, 64, 64): 1728,
                      (64, 128, 64): 960, (100, 63, 41): 1363, (63, 100, 41): 919, (128, 17, 17): 1681,
                      (17, 128, 9): 349, (96, 64, 40): 1312, (64, 96, 40): 928, (127, 57, 33): 1708,
                      (57, 127, 56): 868, (120, 8, 5): 1568, (9, 121, 9): 238,
                      (80, 50, 30): 1090, (50, 80, 27): 730}


@pytest.mark.parametrize("m,n,r", list(BATCHED_SWEEP_SEED))
def test_batched_shape_sweep(H, m, n, r):
    # ragged s / ell, both orientations, full rank; every tile count r8 / 8 = 1..8 of the templated block
    # sweep (M = inv(L'L), reading R28), and ranks that end the Cholesky early (rank-exhausted exit)
    G = I.low_rank(BATCHED_SWEEP_SEED[(m, n, r)], m, n, r)
    R = O.geninv(G.numpy())
    assert R.in_Q() and R.rank == r
    Gs = torch.stack([G, torch.zeros(m, n, dtype=torch.float64), 2.0 * G]).cuda()
    Gp, rk = H.geninv_batched_d(Gs)
    torch.cuda.synchronize()
    assert rk.tolist() == [r, 0, r]
    assert C.rel_fro(Gp[0].cpu().numpy(), R.Gp) <= 1e-9
    assert bool((Gp[1] == 0).all())
    assert C.rel_fro(2.0 * Gp[2].cpu().numpy(), R.Gp) <= 1e-9
