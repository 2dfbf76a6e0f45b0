"""CPU oracle for Courrieu's geninv (arXiv 0804.4809) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this module.  The product path (the CUDA library
and its Python binding) never imports, calls or links anything under oracle/.
It shares no code with paper_0804_4809_b200/csrc or the binding; the only
shared module is the seeded input generator (paper_0804_4809_b200/inputs.py),
which holds none of the method's arithmetic.

What it computes: the paper's `geninv` listing (PAPER.md Appendix, lines
105-140), step by step, in the paper's order and notation, in float64 with
numpy.  Library primitives (matmul, matvec, the general inverse `inv`) serve
as single steps exactly where the listing itself calls a Matlab built-in
(`G'*G`, `L(k:n,1:r-1)*L(k,1:r-1)'`, `inv(L'*L)`, `*`).

Citations (PAPER.md line numbers, "P:NN"):
  P:107-115  transpose branch: if m < n, A = G G', n = m; else A = G' G
  P:117      tol = min(dA(dA>0)) * 1e-9
  P:118-132  full-rank Cholesky loop over k = 1..n, accept iff L(k,r) > tol
  P:133      L = L(:, 1:r)
  P:135      M = inv(L' * L)
  P:136-140  Y = G' * L * M * M * L'  (transpose)  or  L * M * M * L' * G'
  P:66       Theorem 1: G+ = L (L'L)^-1 (L'L)^-1 L' G'

Readings where the paper is silent:
  R2  no positive diagonal -> tol = 0, r = 0, G+ = 0.
  R3  strict '>' (pivot == tol is dropped); NaN / negative pivots dropped.
  R4  zeros above every pivot: a dropped column writes nothing into L
      (the Matlab listing leaves stale tentative values; Eq. (1) P:46 says zeros).
  R6  m == n takes the non-transposed branch.
  R7  `inv` is the general inverse (numpy.linalg.inv, LAPACK getrf/getri) --
      the listing's own built-in.  (The CUDA path uses an SPD inverse.)
  R9  the oracle evaluates the product chain in the listing's literal
      left-to-right order (P:137 / P:139); the CUDA path reassociates it.

Parity pinning: every function here is pinned by tests/test_oracle_pins.py
against values the paper / SPEC fix (tests/golden), closed forms, exact
integer constructions and LAPACK's SVD pseudoinverse.  No function is
"parity unpinned".
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

TOL_REL = 1e-9


class OracleError(ValueError):
    pass


@dataclass
class FullRankCholesky:
    L: np.ndarray            # s x r, zeros above each pivot
    rank: int
    tol: float
    piv: np.ndarray          # int64[r]: row index k at which column j was accepted
    accepted: np.ndarray     # c_k of accepted columns (pivot values before sqrt)
    dropped: np.ndarray      # c_k of dropped columns

    @property
    def mu_acc(self) -> float:
        """min accepted pivot / tol (inf if none or tol == 0)."""
        if len(self.accepted) == 0 or self.tol <= 0:
            return float("inf")
        return float(self.accepted.min() / self.tol)

    @property
    def mu_drop(self) -> float:
        """max |dropped pivot| / tol (0 if none dropped)."""
        if len(self.dropped) == 0:
            return 0.0
        if self.tol <= 0:
            return float("inf")
        return float(np.abs(self.dropped).max() / self.tol)

    @property
    def min_pivot(self) -> float:
        allp = np.concatenate([self.accepted, self.dropped])
        return float(allp.min()) if len(allp) else 0.0


@dataclass
class GeninvResult:
    Gp: np.ndarray
    rank: int
    tol: float
    transposed: bool
    chol: FullRankCholesky
    A: np.ndarray | None = None
    M: np.ndarray | None = None
    extra: dict = field(default_factory=dict)

    @property
    def piv(self):
        return self.chol.piv

    @property
    def mu_acc(self):
        return self.chol.mu_acc

    @property
    def mu_drop(self):
        return self.chol.mu_drop

    def in_Q(self) -> bool:
        """SURVEY §8(c4) predicate Q: mu_acc >= 1e4 and mu_drop <= 1e-2 ("far from the tolerance")."""
        return self.mu_acc >= 1e4 and self.mu_drop <= 1e-2

    def in_Qstar(self) -> bool:
        """Predicate Q*: mu_acc >= 1e6 and mu_drop <= 1e-3."""
        return self.mu_acc >= 1e6 and self.mu_drop <= 1e-3


def _check(G: np.ndarray) -> np.ndarray:
    G = np.asarray(G, dtype=np.float64)
    if G.ndim != 2 or G.shape[0] < 1 or G.shape[1] < 1:
        raise OracleError("G must be a non-empty 2-D matrix")
    if not np.isfinite(G).all():
        raise OracleError("G has non-finite entries")
    return G


def gram(G: np.ndarray) -> tuple[np.ndarray, bool]:
    """[m,n]=size(G); if m<n: A=G*G' (transpose) else A=G'*G."""
    m, n = G.shape
    if m < n:
        return G @ G.T, True
    return G.T @ G, False


def tolerance(A: np.ndarray, tol_rel: float = TOL_REL, tol_abs: float | None = None) -> float:
    """dA=diag(A); tol = min(dA(dA>0))*1e-9.  R2: empty set -> tol = 0."""
    if tol_abs is not None and tol_abs >= 0:
        return float(tol_abs)
    dA = np.diag(A)
    pos = dA[dA > 0]
    if pos.size == 0:
        return 0.0
    return float(pos.min() * tol_rel)


def full_rank_cholesky(A: np.ndarray, tol: float) -> FullRankCholesky:
    """P:118-133, the Appendix loop in 0-based indices.

        L = zeros(size(A)); r = 0
        for k = 1..n:
            r = r + 1
            L(k:n, r) = A(k:n, k) - L(k:n, 1:r-1) * L(k, 1:r-1)'
            if L(k, r) > tol:  L(k,r) = sqrt(L(k,r)); L(k+1:n, r) = L(k+1:n, r) / L(k, r)
            else:              r = r - 1
        L = L(:, 1:r)

    Reading R4: the tentative column is held in `c` and written into L only
    on acceptance, so L has zeros above every pivot (Eq. (1)).
    """
    n = A.shape[0]
    L = np.zeros((n, n))
    r = 0
    piv, acc, drop = [], [], []
    for k in range(n):
        c = A[k:, k] - L[k:, :r] @ L[k, :r]          # P:122 (matvec; zero for r == 0)
        if c[0] > tol:                               # P:124, strict '>' (R3)
            d = np.sqrt(c[0])
            L[k, r] = d
            if k < n - 1:
                L[k + 1:, r] = c[1:] / d             # P:127, true division
            piv.append(k)
            acc.append(c[0])
            r += 1
        else:
            drop.append(c[0])                        # r = r - 1 (nothing kept)
    return FullRankCholesky(L[:, :r].copy(), r, tol, np.array(piv, dtype=np.int64),
                            np.array(acc), np.array(drop))


def inverse(B: np.ndarray) -> np.ndarray:
    """M = inv(L'*L) -- the general inverse, as the listing calls it (R7)."""
    return np.linalg.inv(B)


def geninv(G, tol_rel: float = TOL_REL, tol_abs: float | None = None, keep: bool = False) -> GeninvResult:
    """The whole listing.  Returns G+ (n x m), rank and the decision margins."""
    G = _check(G)
    m, n = G.shape
    A, transposed = gram(G)
    tol = tolerance(A, tol_rel, tol_abs)
    ch = full_rank_cholesky(A, tol)
    L = ch.L
    if ch.rank == 0:                                 # R2: L is s x 0, every product is zero
        return GeninvResult(np.zeros((n, m)), 0, tol, transposed, ch, A if keep else None)
    M = inverse(L.T @ L)
    if transposed:                                   # P:137, left to right (R9)
        Y = (((G.T @ L) @ M) @ M) @ L.T
    else:                                            # P:139, left to right
        Y = ((((L @ M) @ M) @ L.T) @ G.T)
    return GeninvResult(Y, ch.rank, tol, transposed, ch, A if keep else None, M if keep else None)


def from_gram(A: np.ndarray, tol_rel: float = TOL_REL, tol_abs: float | None = None):
    """Steps P:117-135 on a given Gram matrix A, plus the left part of the product chain.

    Returns (X, chol) with X = ((L M) M) L' evaluated left to right exactly as the
    listing's P:139 chain before its final `* G'`, so that geninv(G).Gp == apply(X, G)
    for the N branch, bit for bit.  Used for the row-sharded split (A = sum_p G_p'G_p).
    """
    tol = tolerance(A, tol_rel, tol_abs)
    ch = full_rank_cholesky(A, tol)
    if ch.rank == 0:
        return np.zeros_like(A), ch
    L = ch.L
    M = inverse(L.T @ L)
    return (((L @ M) @ M) @ L.T), ch


def solve(G, F, tol_rel: float = TOL_REL, tol_abs: float | None = None) -> tuple[np.ndarray, int]:
    """Minimum-norm least-squares weights W = G+ F (P:22, P:32-34 with the garbled "W = G+ W" read as
    W = G+ F, reading R10; the RBF use of P:96-100): the listing's Y times F.
    Returns (W (n x k), rank)."""
    R = geninv(G, tol_rel, tol_abs)
    return R.Gp @ np.asarray(F, dtype=np.float64), R.rank


def apply(X: np.ndarray, G: np.ndarray) -> np.ndarray:
    """N branch, last product of P:139: Y = X G'."""
    return X @ G.T


def full_rank_cholesky_batched(A, tol):
    """P:118-133 for a stack of independent Gram matrices A (batch, s, s) with per-matrix tol (batch,).

    The loop is that of full_rank_cholesky, vectorised over the independent batch index only;
    columns not yet accepted are zero, so the correction sums over all s columns add exact zeros.
    Returns (L (batch, s, s) with the kept columns first, r int64[batch], min_acc, max_drop,
    min_pivot) -- min_acc = min accepted c_k (+inf if none), max_drop = max |dropped c_k| (0 if
    none), min_pivot = min over all c_k (SURVEY §8(c4) margins).
    """
    A = np.asarray(A, dtype=np.float64)
    tol = np.asarray(tol, dtype=np.float64)
    nb, s, _ = A.shape
    L = np.zeros((nb, s, s))
    r = np.zeros(nb, dtype=np.int64)
    min_acc = np.full(nb, np.inf)
    max_drop = np.zeros(nb)
    min_piv = np.full(nb, np.inf)
    ar = np.arange(nb)
    for k in range(s):
        c = A[:, k:, k] - np.matmul(L[:, k:, :], L[:, k, :, None])[..., 0]
        ok = c[:, 0] > tol                                                    # P:124, strict (R3)
        d = np.sqrt(np.where(ok, c[:, 0], 1.0))
        idx = ar[ok]
        L[idx, k, r[idx]] = d[idx]
        if k < s - 1:
            L[idx, k + 1:, r[idx]] = c[idx, 1:] / d[idx, None]
        min_acc[idx] = np.minimum(min_acc[idx], c[idx, 0])
        nd = ar[~ok]
        max_drop[nd] = np.maximum(max_drop[nd], np.abs(c[nd, 0]))
        min_piv = np.minimum(min_piv, c[:, 0])
        r[idx] += 1
    return L, r, min_acc, max_drop, min_piv


def geninv_batched(Gb, tol_rel: float = TOL_REL):
    """geninv applied independently to each matrix of a (batch, m, n) stack.

    Gram and tolerance per matrix, the Cholesky loop of P:118-133
    through full_rank_cholesky_batched, then P:135-139 per matrix.
    Returns (Gp (batch, n, m), rank int64[batch], mu_acc, mu_drop).
    """
    Gb = np.asarray(Gb, dtype=np.float64)
    if not np.isfinite(Gb).all():
        raise OracleError("G has non-finite entries")
    nb, m, n = Gb.shape
    transposed = m < n
    A = Gb @ np.swapaxes(Gb, 1, 2) if transposed else np.swapaxes(Gb, 1, 2) @ Gb
    dA = np.diagonal(A, axis1=1, axis2=2)
    pos = np.where(dA > 0, dA, np.inf).min(axis=1)
    tol = np.where(np.isfinite(pos), pos * tol_rel, 0.0)
    L, r, min_acc, max_drop, _ = full_rank_cholesky_batched(A, tol)
    Gp = np.zeros((nb, n, m))
    for rv in np.unique(r):
        if rv == 0:
            continue
        sel = np.nonzero(r == rv)[0]
        Ls = L[sel, :, :rv]
        Lt = np.swapaxes(Ls, 1, 2)
        M = np.linalg.inv(Lt @ Ls)
        Gs = Gb[sel]
        Gt = np.swapaxes(Gs, 1, 2)
        if transposed:
            Gp[sel] = (((Gt @ Ls) @ M) @ M) @ Lt
        else:
            Gp[sel] = ((((Ls @ M) @ M) @ Lt) @ Gt)
    with np.errstate(divide="ignore", invalid="ignore"):
        mu_acc = np.where(tol > 0, min_acc / tol, np.inf)
        mu_drop = np.where(max_drop > 0, max_drop / np.where(tol > 0, tol, 1.0), 0.0)
    return Gp, r, mu_acc, mu_drop


def penrose_residuals(G, X):
    """The four Penrose conditions as relative Frobenius residuals, fresh products.

    rho1 = ||G X G - G|| / ||G||,  rho2 = ||X G X - X|| / ||X||,
    rho3 = ||(G X)' - G X|| / ||G X||,  rho4 = ||(X G)' - X G|| / ||X G||.
    Also returns the paper's absolute per-coefficient maximum.
    """
    G = np.asarray(G, dtype=np.float64)
    X = np.asarray(X, dtype=np.float64)
    GX = G @ X
    XG = X @ G
    E = [GX @ G - G, XG @ X - X, GX.T - GX, XG.T - XG]
    den = [np.linalg.norm(G), np.linalg.norm(X), np.linalg.norm(GX), np.linalg.norm(XG)]
    rho = [float(np.linalg.norm(e) / d) if d > 0 else float(np.linalg.norm(e)) for e, d in zip(E, den)]
    absmax = max(float(np.abs(e).max()) for e in E)
    return rho, absmax
