"""Minimum-norm least-squares solve W = G+ F through the C ABI (geninv_solve_d)
against the oracle's W = Y F (P:32-34 read as W = G+ F, reading R10).

Gates as for G+ (north star): rank exact, ||W_gpu - W_oracle||_F / ||W_oracle||_F <= 1e-9 on inputs
whose decision margins are in Q; plus the normal equations and the minimum-norm property.
"""
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


def dev(X):
    m, n = X.shape
    t = torch.zeros(m, (n + 1) // 2 * 2, dtype=torch.float64, device="cuda")
    t[:, :n] = torch.as_tensor(X)
    return t[:, :n]


# seeds: the first seed >= m * 7 + n whose oracle margins are in Q (tools/screen_q_cpu.py)
SOLVE_SEED = {(300, 130, 70): 2230, (130, 300, 70): 1211, (2050, 530, 400): 14880, (257, 255, 200): 2054,
              (96, 64, 40): 736, (64, 64, 64): 512}


@pytest.mark.parametrize("m,n,r,k", [(300, 130, 70, 1), (130, 300, 70, 7), (2050, 530, 400, 64), (257, 255, 200, 3),
                                     (96, 64, 40, 10), (64, 64, 64, 5)])
def test_solve_parity(H, m, n, r, k):
    G = I.low_rank(SOLVE_SEED[(m, n, r)], m, n, r).numpy()
    F = I.dense_normal(m + k, m, k).numpy()
    Wo, ro = O.solve(G, F)
    R = O.geninv(G)
    assert R.in_Q()
    W, info = H.geninv_solve_d(dev(G), torch.as_tensor(F).cuda())
    assert info.rank == ro == r
    assert C.rel_fro(W.cpu().numpy(), Wo) <= 1e-9


def test_solve_tall_split_k(H):
    # K = m = 2^18 rows: the G'F product runs split-K with a fixed-order reduction
    m, n, r, k = 1 << 18, 96, 80, 4
    G = I.low_rank(31, m, n, r, device="cuda")
    F = I.dense_normal(32, m, k, device="cuda")
    W, info = H.geninv_solve_d(G, F)
    Gh, Fh = G.cpu().numpy(), F.cpu().numpy()
    Wo, ro = O.solve(Gh, Fh)
    assert info.rank == ro == r
    assert C.rel_fro(W.cpu().numpy(), Wo) <= 1e-9
    # normal equations G'G W = G'F (checked with cuBLAS, test-only)
    lhs = G.T @ (G @ W)
    rhs = G.T @ F
    assert float((lhs - rhs).abs().max() / rhs.abs().max()) <= 1e-8


def test_solve_matches_geninv_times_f(H):
    G = I.low_rank(41, 700, 300, 250).numpy()
    F = I.dense_normal(42, 700, 9).numpy()
    Gp, _ = H.geninv_d(dev(G))
    W, _ = H.geninv_solve_d(dev(G), torch.as_tensor(F).cuda())
    assert C.rel_fro(W.cpu().numpy(), Gp.cpu().numpy() @ F) <= 1e-10
