"""Step-level parity of the sm_100a kernels against the oracle (`-m gpu`).

Integer constructions make every partial sum exact, so the GPU must be
BIT-EXACT there whatever its summation order:
  P1  integer G -> Gram (both layouts, split-K, ragged tiles)
  P2  integer L_true -> full-rank Cholesky L, piv, r (drops interleaved)
  P3  unimodular B = U U' -> M = inv(B)
Random inputs are graded at the floating-point level.
"""
import json
import os

import numpy as np
import pytest
import torch

from oracle import checks as C
from oracle import geninv_oracle as O
from paper_0804_4809_b200 import inputs as I

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


@pytest.fixture(scope="module")
def H():
    from paper_0804_4809_b200.binding import Handle
    return Handle(0)


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64).cuda()


def padded(a, cols):
    """Device copy of `a` with an even leading dimension >= cols."""
    ld = (max(cols, a.shape[1]) + 1) // 2 * 2
    t = torch.zeros(a.shape[0], ld, dtype=torch.float64, device="cuda")
    t[:, :a.shape[1]] = torch.as_tensor(a)
    return t


@pytest.mark.parametrize("shape", [(37, 12), (12, 38), (300, 130), (130, 300), (4096, 200), (200, 4096),
                                   (1000, 1000), (9000, 260)])
def test_gram_integer_bit_exact(H, shape):
    rng = np.random.default_rng(shape[0] * 7 + shape[1])
    G = rng.integers(-3, 4, size=shape).astype(float)
    m, n = shape
    tr = int(m < n)
    s = min(m, n)
    A = torch.full((s, (s + 1) // 2 * 2), np.nan, dtype=torch.float64, device="cuda")
    H.geninv_gram_d(padded(G, n), tr, A)
    torch.cuda.synchronize()
    Ao, _ = O.gram(G)
    got = A[:, :s].cpu().numpy()
    low = np.tril_indices(s)
    assert np.array_equal(got[low], Ao[low])


@pytest.mark.parametrize("shape", [(1 << 18, 200), (200, 1 << 18), (300000, 130)])
def test_gram_two_level_integer_bit_exact(H, shape):
    # long sums: each CTA's k-range exceeds the 8192-row register chunk, so the CHUNK instance of the
    # Gram runs (chunk sums added into the tile in memory, then the pairwise split-K reduction); with
    # integer entries every partial sum is exact, so the result must be the exact Gram bit for bit (P1)
    rng = np.random.default_rng(shape[0] + shape[1])
    G = rng.integers(-3, 4, size=shape).astype(float)
    m, n = shape
    tr = int(m < n)
    s = min(m, n)
    A = torch.full((s, (s + 1) // 2 * 2), np.nan, dtype=torch.float64, device="cuda")
    H.geninv_gram_d(padded(G, n), tr, A)
    torch.cuda.synchronize()
    # the exact Gram: integer entries, |every partial sum| <= 9 * 300000 < 2^53, so any FP64 summation order
    # (here the host BLAS) is exact
    Ao = (G @ G.T) if tr else (G.T @ G)
    low = np.tril_indices(s)
    assert np.array_equal(A[:, :s].cpu().numpy()[low], Ao[low])


@pytest.mark.parametrize("shape", [(3000, 257), (257, 3000)])
def test_gram_random(H, shape):
    G = I.dense_normal(3, *shape).numpy()
    m, n = shape
    s = min(m, n)
    A = torch.zeros(s, (s + 1) // 2 * 2, dtype=torch.float64, device="cuda")
    H.geninv_gram_d(padded(G, n), int(m < n), A)
    Ao, _ = O.gram(G)
    low = np.tril_indices(s)
    got = A[:, :s].cpu().numpy()
    assert np.abs(got[low] - Ao[low]).max() <= 1e-14 * np.abs(Ao).max() * 10


def integer_ltrue(s, r, seed):
    rng = np.random.default_rng(seed)
    piv = np.sort(rng.choice(s, size=r, replace=False))
    L = np.zeros((s, r))
    for j, p in enumerate(piv):
        L[p, j] = rng.integers(1, 4)
        L[p + 1:, j] = rng.integers(-3, 4, size=s - p - 1)
    return L, piv


@pytest.mark.parametrize("s,r,seed", [(64, 40, 0), (33, 33, 1), (50, 7, 2), (96, 64, 3), (300, 170, 4),
                                      (129, 1, 5)])
def test_frchol_integer_bit_exact(H, s, r, seed):
    Lt, piv = integer_ltrue(s, r, seed)
    Li = Lt.astype(np.int64)
    A = C.int_matmul(Li, Li.T).astype(float)
    assert np.abs(A).max() < 2 ** 52
    ch = O.full_rank_cholesky(A, O.tolerance(A))
    assert np.array_equal(ch.L, Lt)                     # oracle pinned first
    L, pv, info = H.geninv_frchol_d(padded(A, s))
    assert info.rank == r
    assert np.array_equal(pv.cpu().numpy(), piv)
    assert np.array_equal(L.cpu().numpy(), Lt)


def test_frchol_strict_tolerance(H):
    # R3: a pivot equal to tol is dropped; one ulp below tol it would be kept
    A = np.diag([4.0, 1.0, 9.0, 1.0])
    L, pv, info = H.geninv_frchol_d(padded(A, 4), tol_abs=1.0)
    assert info.rank == 2 and pv.cpu().tolist() == [0, 2]
    L, pv, info = H.geninv_frchol_d(padded(A, 4), tol_abs=float(np.nextafter(1.0, 0.0)))
    assert info.rank == 4


@pytest.mark.parametrize("k", [0, 1])
def test_frchol_margins_golden(H, k):
    # the hand-worked margins (tests/golden "margins", negative dropped pivots): the device reports the same
    # decisions and min accepted / max |dropped| / min pivot, exactly (every value is a small dyadic rational)
    ex = GOLD["margins"][k]
    A = np.array(ex["A"], dtype=float)
    kw = {"tol_abs": ex["tol"]} if ex["tol"] is not None else {}
    L, pv, info = H.geninv_frchol_d(padded(A, 4), **kw)
    assert info.rank == ex["rank"] and pv.cpu().tolist()[:ex["rank"]] == ex["piv"]
    assert np.array_equal(L.cpu().numpy()[:, :ex["rank"]], np.array(ex["L"], dtype=float))
    assert info.min_acc == min(ex["accepted"])
    assert info.max_drop == max(abs(v) for v in ex["dropped"])
    assert info.min_pivot == ex["min_pivot"]
    if ex["tol"] is None:
        assert info.tol == ex["tol_expected"]
    # this A is not PSD: the pivot -7 is far below -s * tol with the paper's tol (reported, not an error);
    # with tol = 1 the worst dropped pivot -1/2 is within -s * tol
    assert info.not_psd_hint == (1 if ex["tol"] is None else 0)


@pytest.mark.parametrize("r,seed", [(8, 0), (32, 1), (33, 2), (64, 3), (100, 4)])
def test_spd_inverse_unimodular_bit_exact(H, r, seed):
    rng = np.random.default_rng(seed)
    # bidiagonal-ish unimodular U keeps |M| small enough to stay exact
    U = np.eye(r, dtype=np.int64)
    for i in range(1, r):
        U[i, i - 1] = rng.integers(-1, 2)
        if i >= 2 and rng.random() < 0.3:
            U[i, i - 2] = rng.integers(-1, 2)
    B = C.int_matmul(U, U.T)
    Ui = np.eye(r, dtype=object)
    Uo = U.astype(object)
    for i in range(r):
        for j in range(i):
            Ui[i, j] = -sum(Uo[i, k] * Ui[k, j] for k in range(j, i))
    Mx = C.int_matmul(Ui.T, Ui)
    if max(abs(int(v)) for v in Mx.flat) >= 2 ** 40:
        pytest.skip("|M| too large for exact FP64 partial sums")
    M = H.geninv_spd_inverse_d(padded(B.astype(float), r))
    assert np.array_equal(M.cpu().numpy(), Mx.astype(float))


def test_spd_inverse_random(H):
    G = I.dense_normal(4, 700, 300).numpy()
    B = G.T @ G
    M = H.geninv_spd_inverse_d(padded(B, 300)).cpu().numpy()
    assert C.rel_fro(M, O.inverse(B)) <= 1e-12
    assert np.array_equal(M, M.T)


def test_spd_inverse_rejects_indefinite(H):
    from paper_0804_4809_b200.binding import GeninvError, GENINV_ENOTSPD
    B = np.array([[1.0, 2.0], [2.0, 1.0]])
    with pytest.raises(GeninvError) as e:
        H.geninv_spd_inverse_d(padded(B, 2))
    assert e.value.status == GENINV_ENOTSPD
