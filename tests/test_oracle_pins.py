"""Pins for the CPU oracle -- all CPU, `-m "not gpu"`.

Each test checks oracle/geninv_oracle.py against something other than itself:
values fixed by the paper / SPEC worked examples (tests/golden), exact
integer constructions, closed forms, LAPACK / Jacobi SVD pseudoinverses and
invariants of the Moore-Penrose inverse.  The pins are chosen so a dropped
term, a wrong sign or index, or a transposed operand in any oracle step
fails at least one of them (see test_mutations_are_caught).
"""
import json
import os

import numpy as np
import pytest

from oracle import checks as C
from oracle import geninv_oracle as O
from paper_0804_4809_b200 import inputs as I

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


# ---------------------------------------------------------------- P4 golden
@pytest.mark.parametrize("ex", GOLD["full_rank_cholesky"], ids=lambda e: e["cite"][:20])
def test_golden_full_rank_cholesky(ex):
    A = np.array(ex["A"], dtype=float)
    tol = O.tolerance(A)
    ch = O.full_rank_cholesky(A, tol)
    assert ch.rank == ex["rank"]
    assert ch.L.shape == (A.shape[0], ex["rank"])
    if ex["rank"]:
        assert np.array_equal(ch.L, np.array(ex["L"], dtype=float))
    assert list(ch.piv) == ex["piv"]


@pytest.mark.parametrize("ex", GOLD["margins"], ids=["tol_abs", "paper_tol"])
def test_golden_margins(ex):
    """Decision margins (they define predicates Q / Q*, which gate every GPU comparison)
    on a hand-worked A with negative dropped pivots, for the scalar and the batched oracle."""
    A = np.array(ex["A"], dtype=float)
    tol = ex["tol"] if ex["tol"] is not None else O.tolerance(A)
    if ex["tol"] is None:
        assert tol == ex["tol_expected"]
    ch = O.full_rank_cholesky(A, tol)
    assert ch.rank == ex["rank"] and list(ch.piv) == ex["piv"]
    assert np.array_equal(ch.L, np.array(ex["L"], dtype=float))
    assert list(ch.accepted) == ex["accepted"] and list(ch.dropped) == ex["dropped"]
    assert ch.mu_acc == pytest.approx(ex["mu_acc"], rel=1e-15)
    assert ch.mu_drop == pytest.approx(ex["mu_drop"], rel=1e-15)
    assert ch.min_pivot == ex["min_pivot"]
    # batched form: the same matrix three times (plus a permuted-irrelevant zero matrix: rank 0, no margins)
    Ab = np.stack([A, A, np.zeros_like(A), A])
    tb = np.array([tol, tol, 0.0, tol])
    Lb, rb, min_acc, max_drop, min_piv = O.full_rank_cholesky_batched(Ab, tb)
    assert list(rb) == [ex["rank"]] * 2 + [0] + [ex["rank"]]
    for b in (0, 1, 3):
        assert np.array_equal(Lb[b][:, :ex["rank"]], ch.L) and not Lb[b][:, ex["rank"]:].any()
        assert min_acc[b] / tol == pytest.approx(ex["mu_acc"], rel=1e-15)
        assert max_drop[b] / tol == pytest.approx(ex["mu_drop"], rel=1e-15)
        assert min_piv[b] == ex["min_pivot"]
    assert min_acc[2] == np.inf and max_drop[2] == 0.0 and min_piv[2] == 0.0


def test_margin_mutations_are_caught(monkeypatch):
    """A signed max instead of max |.| for mu_drop, or min over accepted replaced by min over all pivots,
    fails the margin goldens (the VERDICT r1 mutation)."""
    ex = GOLD["margins"][1]
    A = np.array(ex["A"], dtype=float)

    def golden_ok():
        ch = O.full_rank_cholesky(A, O.tolerance(A))
        return (ch.mu_drop == pytest.approx(ex["mu_drop"], rel=1e-15)
                and ch.mu_acc == pytest.approx(ex["mu_acc"], rel=1e-15))
    assert golden_ok()
    monkeypatch.setattr(O.FullRankCholesky, "mu_drop", property(lambda self: float(self.dropped.max() / self.tol)))
    assert not golden_ok()
    monkeypatch.undo()
    monkeypatch.setattr(O.FullRankCholesky, "mu_acc", property(lambda self: float(
        np.concatenate([self.accepted, self.dropped]).min() / self.tol)))
    assert not golden_ok()


def test_margins_define_Q():
    """Q / Q* thresholds on GeninvResult, at and across their boundaries."""
    def res(acc, drop, tol=1.0):
        ch = O.FullRankCholesky(np.zeros((2, 1)), 1, tol, np.array([0]), np.array(acc, dtype=float),
                                np.array(drop, dtype=float))
        return O.GeninvResult(np.zeros((1, 1)), 1, tol, False, ch)
    assert res([1e4], [1e-2]).in_Q() and not res([1e4], [1e-2]).in_Qstar()
    assert not res([9.999e3], [0.0]).in_Q()
    assert not res([1e5], [-0.0101]).in_Q()            # |negative| dropped pivot counts
    assert res([1e6], [-1e-3]).in_Qstar() and not res([1e6], [-1.01e-3]).in_Qstar()
    assert res([2e6, 1e6], []).mu_drop == 0.0 and res([2e6, 1e6], []).mu_acc == 1e6


@pytest.mark.parametrize("ex", GOLD["geninv"], ids=lambda e: e["cite"][:20])
def test_golden_geninv(ex):
    G = np.array(ex["G"], dtype=float)
    R = O.geninv(G)
    want = np.array(ex["Gp"], dtype=float) / ex["den"]
    assert R.rank == ex["rank"]
    assert R.Gp.shape == want.shape
    assert np.abs(R.Gp - want).max() <= 1e-12


@pytest.mark.parametrize("ex", GOLD["inverse"], ids=lambda e: e["cite"][:20])
def test_golden_inverse(ex):
    M = O.inverse(np.array(ex["B"], dtype=float))
    assert np.abs(M - np.array(ex["M"], dtype=float) / ex["den"]).max() <= 1e-15


@pytest.mark.parametrize("ex", GOLD["min_norm_solve"], ids=lambda e: e["cite"][:20])
def test_golden_min_norm(ex):
    G = np.array(ex["G"], dtype=float)
    W = O.geninv(G).Gp @ np.array(ex["F"], dtype=float)
    assert np.abs(W - np.array(ex["W"], dtype=float) / ex["den"]).max() <= 1e-12


@pytest.mark.parametrize("ex", GOLD["min_norm_solve"], ids=lambda e: e["cite"][:20])
def test_golden_solve(ex):
    W, _ = O.solve(np.array(ex["G"], dtype=float), np.array(ex["F"], dtype=float))
    assert np.abs(W - np.array(ex["W"], dtype=float) / ex["den"]).max() <= 1e-12


def test_solve_pins():
    # full column rank: W is the unique least-squares solution (G'G)^-1 G'F, via QR
    G = I.dense_normal(21, 300, 40).numpy()
    F = I.dense_normal(22, 300, 5).numpy()
    W, r = O.solve(G, F)
    assert r == 40
    assert C.rel_fro(W, C.closed_form_full_rank(G) @ F) <= 1e-12
    # rank deficient, both branches: normal equations G'G W = G'F, and W is orthogonal to null(G)
    for (m, n) in ((90, 60), (60, 90)):
        G = I.low_rank(23, m, n, 25).numpy()
        F = I.dense_normal(24, m, 4).numpy()
        W, r = O.solve(G, F)
        assert r == 25
        lhs, rhs = G.T @ (G @ W), G.T @ F
        assert np.abs(lhs - rhs).max() <= 1e-8 * np.abs(rhs).max()
        _, _, Vt = np.linalg.svd(G)
        Z = Vt[25:].T
        assert np.abs(Z.T @ W).max() <= 1e-8 * np.abs(W).max()
        # and equals the brute-force SVD pseudoinverse applied to F
        assert C.rel_fro(W, C.jacobi_svd_pinv(G, 25) @ F) <= 1e-9


@pytest.mark.parametrize("ex", GOLD["svd_pinv"], ids=lambda e: e["cite"][:20])
def test_golden_svd_checker(ex):
    # the Jacobi checker itself is pinned before it is used to pin the oracle
    P = C.jacobi_svd_pinv(np.array(ex["G"], dtype=float))
    assert np.abs(P - np.array(ex["Gp"], dtype=float) / ex["den"]).max() <= 1e-14


def test_golden_penrose():
    ex = GOLD["penrose"][0]
    rho, absmax = O.penrose_residuals(np.array(ex["G"], float), np.array(ex["X"], float))
    assert np.allclose(rho, ex["rho"], atol=1e-15) and absmax == ex["absmax"]


# ------------------------------------------------- P1: integer Gram is exact
@pytest.mark.parametrize("shape", [(37, 11), (9, 23), (64, 64)])
def test_gram_integer_exact(shape):
    rng = np.random.default_rng(1)
    G = rng.integers(-3, 4, size=shape).astype(float)
    A, tr = O.gram(G)
    Gi = G.astype(np.int64)
    exact = C.int_matmul(Gi, Gi.T) if tr else C.int_matmul(Gi.T, Gi)
    assert tr == (shape[0] < shape[1])
    assert np.array_equal(A, exact.astype(float))


# ------------------------------------- P2: integer L_true, exact factorisation
def integer_ltrue(s, r, seed):
    """L_true: s x r, zeros above pivots, pivots d in {1,2,3}, entries below in [-3,3].

    Pivot rows are drawn by seed so dropped rows interleave; A = L L' is an
    exact integer matrix and every accepted c_k is d^2 exactly.
    """
    rng = np.random.default_rng(seed)
    piv = np.sort(rng.choice(s, size=r, replace=False))
    L = np.zeros((s, r))
    for j, p in enumerate(piv):
        L[p, j] = rng.integers(1, 4)
        L[p + 1:, j] = rng.integers(-3, 4, size=s - p - 1)
    return L, piv


@pytest.mark.parametrize("s,r,seed", [(64, 40, 0), (33, 33, 1), (50, 7, 2), (96, 64, 3)])
def test_frchol_integer_exact(s, r, seed):
    L, piv = integer_ltrue(s, r, seed)
    Li = L.astype(np.int64)
    A = C.int_matmul(Li, Li.T).astype(float)
    # through G: G = [L'; 0] (m >= s) has G'G == A exactly
    G = np.vstack([L.T, np.zeros((max(0, s - r) + 1, s))])
    A2, tr = O.gram(G)
    assert not tr and np.array_equal(A2, A)
    ch = O.full_rank_cholesky(A, O.tolerance(A))
    assert ch.rank == r
    assert np.array_equal(ch.piv, piv)
    assert np.array_equal(ch.L, L)
    assert np.all(ch.dropped == 0.0)
    assert np.array_equal(ch.accepted, np.diag(L[piv]) ** 2)


# ------------------------------------------- P3: unimodular SPD inverse pin
@pytest.mark.parametrize("r,seed", [(8, 0), (12, 1), (16, 2)])
def test_inverse_unimodular(r, seed):
    rng = np.random.default_rng(seed)
    U = np.tril(rng.integers(-1, 2, size=(r, r)), -1) + np.eye(r, dtype=np.int64)
    B = C.int_matmul(U, U.T)
    Ui = np.eye(r, dtype=object)  # exact U^-1 by forward substitution in python ints
    Uo = U.astype(object)
    for i in range(r):
        for j in range(i):
            Ui[i, j] = -sum(Uo[i, k] * Ui[k, j] for k in range(j, i))
    Mx = C.int_matmul(Ui.T, Ui)
    assert np.array_equal(C.int_matmul(B, Mx), np.eye(r, dtype=object))   # exact inverse
    M = O.inverse(B.astype(float))
    assert C.rel_fro(M, Mx.astype(float)) <= 1e-10


# ----------------------------------------- P5: full-rank closed form
@pytest.mark.parametrize("m,n", [(512, 128), (300, 200), (128, 512)])
def test_closed_form_full_rank(m, n):
    G = I.dense_normal(11, m, n).numpy()
    R = O.geninv(G)
    assert R.rank == min(m, n)
    ref = C.closed_form_full_rank(G) if m >= n else C.closed_form_full_rank(G.T).T
    assert C.rel_fro(R.Gp, ref) <= 1e-12


def test_full_rank_L_is_classical_cholesky():
    # SPD input -> L equals the classical Cholesky factor
    G = I.dense_normal(5, 400, 120).numpy()
    A, _ = O.gram(G)
    ch = O.full_rank_cholesky(A, O.tolerance(A))
    assert ch.rank == 120
    assert C.rel_fro(ch.L, np.linalg.cholesky(A)) <= 1e-12


# -------------------------------------------- P6: SVD pseudoinverse (tiny)
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_c1_vs_jacobi_svd(seed):
    cfg = I.CONFIGS["C1"]
    G = I.make_single(cfg, seed).numpy()
    R = O.geninv(G)
    assert R.in_Qstar()
    assert R.rank == cfg.rank
    P = C.jacobi_svd_pinv(G, cfg.rank)
    assert C.rel_fro(R.Gp, P) <= 1e-9
    assert C.rel_fro(R.Gp, np.linalg.pinv(G, rcond=1e-10)) <= 1e-9


@pytest.mark.parametrize("n", [16, 32, 64])
def test_paper_family(n):
    # m = 2n, r = 7n/8, coefficients in [-1, 1]; every Penrose error coefficient < 2e-10
    for seed in range(3):
        G = I.paper_family(n, seed).numpy()
        R = O.geninv(G)
        assert R.rank == 7 * n // 8
        rho, absmax = O.penrose_residuals(G, R.Gp)
        assert absmax < 2e-10 and max(rho) < 1e-10
        P = np.linalg.pinv(G, rcond=1e-10)
        assert np.abs(R.Gp - P).max() <= 1e-8 * max(1.0, np.abs(P).max())


def test_c5_slice_vs_svd_and_batched():
    cfg = I.CONFIGS["C5"]
    Gb = I.make_batch(cfg, 2024, 0, 64).numpy()
    Gp, r, mu_acc, mu_drop = O.geninv_batched(Gb)
    nq = 0
    for b in range(len(Gb)):
        R = O.geninv(Gb[b])
        assert R.rank == r[b]
        if not R.in_Q():
            continue
        nq += 1
        assert r[b] == cfg.rank
        P = np.linalg.pinv(Gb[b], rcond=1e-10)
        assert C.rel_fro(R.Gp, P) <= 1e-9
        assert C.rel_fro(Gp[b], R.Gp) <= 1e-9
    assert nq >= 55


# ------------------------------------------------ P7: Penrose conditions
@pytest.mark.parametrize("seed", [1, 2])
def test_penrose_c1(seed):
    G = I.make_single(I.CONFIGS["C1"], seed).numpy()
    rho, _ = O.penrose_residuals(G, O.geninv(G).Gp)
    assert max(rho) <= 1e-10


# ---------------------------------------------------------- P8: invariants
def test_transpose_invariant_and_branches():
    G = I.low_rank(3, 80, 50, 30).numpy()
    R = O.geninv(G)
    Rt = O.geninv(G.T)
    assert not R.transposed and Rt.transposed
    assert R.rank == Rt.rank == 30
    assert C.rel_fro(Rt.Gp, R.Gp.T) <= 1e-10


def test_duplicate_columns_give_equal_rows():
    # R13: G[:, D] = G[:, S] -> G+[D, :] == G+[S, :] (the factored Gram is G G', fixed by G's rows)
    G = I.low_rank(4, 60, 200, 40).numpy()
    D, S = I.copy_columns(4, 200, 16)
    G[:, D] = G[:, S]
    R = O.geninv(G)
    assert R.transposed and R.rank == 40
    assert np.array_equal(R.Gp[D], R.Gp[S])


def test_involution_and_min_norm():
    G = I.low_rank(8, 70, 45, 20).numpy()
    X = O.geninv(G).Gp
    assert C.rel_fro(O.geninv(X).Gp, G) <= 1e-8
    # minimum norm: solutions are orthogonal to null(G)
    _, sv, Vt = np.linalg.svd(G)
    Z = Vt[20:].T                         # null space basis of G
    W = X @ I.dense_normal(9, 70, 3).numpy()
    for j in range(3):
        w = W[:, j]
        assert np.abs(Z.T @ w).max() <= 1e-8 * np.linalg.norm(w)


def test_rank_equals_constructed_and_determinism():
    for seed in (1, 2, 3):
        G = I.low_rank(seed, 120, 90, 33).numpy()
        R1 = O.geninv(G)
        R2 = O.geninv(G)
        assert R1.rank == 33
        assert np.array_equal(R1.Gp, R2.Gp)


def test_rank_invariant_under_permutation():
    # rank invariant under P A P'
    G = I.low_rank(6, 100, 60, 25).numpy()
    A, _ = O.gram(G)
    p = np.random.default_rng(0).permutation(60)
    r1 = O.full_rank_cholesky(A, O.tolerance(A)).rank
    Ap = A[np.ix_(p, p)]
    r2 = O.full_rank_cholesky(Ap, O.tolerance(Ap)).rank
    assert r1 == r2 == 25


# ----------------------------------------------------- edge cases / readings
def test_strict_greater_tolerance():
    # R3: a pivot equal to tol is dropped (P:124 uses '>')
    A = np.diag([4.0, 1.0])
    ch = O.full_rank_cholesky(A, 1.0)
    assert ch.rank == 1 and list(ch.piv) == [0]
    ch = O.full_rank_cholesky(A, np.nextafter(1.0, 0.0))
    assert ch.rank == 2


def test_tolerance_reading():
    # P:117 tol = min positive diagonal * 1e-9; R2 empty -> 0
    A = np.diag([5.0, 0.0, 2.0, -1.0])
    assert O.tolerance(A) == 2.0 * 1e-9
    assert O.tolerance(np.zeros((3, 3))) == 0.0
    assert O.tolerance(A, tol_abs=0.5) == 0.5


def test_nonfinite_rejected():
    G = np.ones((4, 3))
    G[1, 2] = np.nan
    with pytest.raises(O.OracleError):
        O.geninv(G)


def test_square_takes_n_branch_and_vectors():
    G = I.dense_normal(2, 7, 7).numpy()
    assert not O.geninv(G).transposed
    v = np.array([[3.0], [4.0]])                       # column vector: v+ = v' / |v|^2
    assert np.abs(O.geninv(v).Gp - v.T / 25).max() <= 1e-16
    assert np.abs(O.geninv(v.T).Gp - v / 25).max() <= 1e-16


# ------------------------------------- the pins catch plausible oracle bugs
def test_mutations_are_caught(monkeypatch):
    """Re-run a subset of the pins against deliberately broken oracles."""
    G = I.make_single(I.CONFIGS["C1"], 1).numpy()
    P = C.jacobi_svd_pinv(G, 32)
    Lt, piv = integer_ltrue(40, 25, 7)
    Li = Lt.astype(np.int64)
    Aint = C.int_matmul(Li, Li.T).astype(float)

    def pins_pass():
        try:
            ok1 = C.rel_fro(O.geninv(G).Gp, P) <= 1e-9
            ch = O.full_rank_cholesky(Aint, O.tolerance(Aint))
            ok2 = ch.rank == 25 and np.array_equal(ch.L, Lt)
            ok3 = O.geninv(G.T).rank == 32 and C.rel_fro(O.geninv(G.T).Gp, P.T) <= 1e-9
            return ok1 and ok2 and ok3
        except Exception:
            return False

    assert pins_pass()
    orig_frc = O.full_rank_cholesky
    orig_gram = O.gram
    orig_inv = O.inverse

    def frc_sign(A, tol):                     # wrong sign of the correction term
        return _frc_variant(A, tol, sign=+1)

    def frc_geq(A, tol):                      # >= instead of >
        return _frc_variant(A, tol, geq=True)

    def frc_noscale(A, tol):                  # forgot to divide by the pivot
        return _frc_variant(A, tol, scale=False)

    def gram_transposed(G_):                  # transposed operand in the Gram
        m, n = G_.shape
        return (G_.T @ G_, True) if m < n else (G_ @ G_.T, False)

    def inv_dropped(B):                       # dropped the inverse: M = I
        return np.eye(B.shape[0])

    for name, fn in [("full_rank_cholesky", frc_sign), ("full_rank_cholesky", frc_noscale),
                     ("gram", gram_transposed), ("inverse", inv_dropped)]:
        monkeypatch.setattr(O, name, fn)
        assert not pins_pass(), name
        monkeypatch.setattr(O, "full_rank_cholesky", orig_frc)
        monkeypatch.setattr(O, "gram", orig_gram)
        monkeypatch.setattr(O, "inverse", orig_inv)
    # '>=' differs only on exact ties: check it on the tie pin itself
    assert frc_geq(np.diag([4.0, 1.0]), 1.0).rank == 2 != O.full_rank_cholesky(np.diag([4.0, 1.0]), 1.0).rank


def _frc_variant(A, tol, sign=-1, geq=False, scale=True):
    n = A.shape[0]
    L = np.zeros((n, n))
    r = 0
    piv, acc, drop = [], [], []
    for k in range(n):
        c = A[k:, k] + sign * (L[k:, :r] @ L[k, :r])
        if (c[0] >= tol) if geq else (c[0] > tol):
            d = np.sqrt(c[0])
            L[k, r] = d
            L[k + 1:, r] = c[1:] / d if scale else c[1:]
            piv.append(k)
            acc.append(c[0])
            r += 1
        else:
            drop.append(c[0])
    return O.FullRankCholesky(L[:, :r].copy(), r, tol, np.array(piv, dtype=np.int64), np.array(acc), np.array(drop))


# ------------------------------------------- oracle/extended.py (the spread reference, reading R23)
def test_extended_integer_exact_and_branches():
    from oracle import extended as E
    Lt, piv = integer_ltrue(30, 12, 3)
    G = np.vstack([Lt.T, np.zeros((5, 30))])          # G'G = Lt Lt' exactly; 17 x 30: transpose branch
    Gt = np.ascontiguousarray(G.T)                    # 30 x 17: N branch, Gram = G G' of the above
    for ge, ce in ((True, True), (True, False), (False, True)):
        Y, r, tol = E.geninv_ext(Gt, ge, ce)
        R = O.geninv(Gt)
        assert r == R.rank == 12 and tol == R.tol
        assert C.rel_fro(Y, R.Gp) <= 1e-12
        Yt, rt, _ = E.geninv_ext(G, ge, ce)
        assert rt == 12 and C.rel_fro(Yt, O.geninv(G).Gp) <= 1e-12


def test_extended_matches_oracle_well_conditioned_and_beats_it_ill_conditioned():
    from oracle import extended as E
    G = I.dense_normal(5, 120, 40).numpy()               # cond ~ 3: both evaluations agree to rounding
    assert C.rel_fro(E.geninv_ext(G)[0], O.geninv(G).Gp) <= 1e-13
    # ill-conditioned accepted columns (C5 shape): the extended Gram + Cholesky is at least as close to the
    # SVD pseudoinverse as the FP64 oracle on average over a few matrices
    Gb = I.make_batch(I.CONFIGS["C5"], 3, 0, 24).numpy()
    e_fp64, e_ext = [], []
    for G in Gb:
        R = O.geninv(G)
        P = np.linalg.pinv(G, rcond=1e-10)
        e_fp64.append(C.rel_fro(R.Gp, P))
        e_ext.append(C.rel_fro(E.geninv_ext(G)[0], P))
    assert np.median(e_ext) <= np.median(e_fp64) * 1.5
