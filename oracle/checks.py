"""Independent checks used to pin the oracle -- TEST INFRASTRUCTURE ONLY.

Nothing here shares code with geninv_oracle.py's method, nor with the CUDA
path.  Only tests/ (and bench.py's reporting) may use it.

* jacobi_svd_pinv: brute-force one-sided (Hestenes) Jacobi SVD pseudoinverse,
  truncated at a given rank (the "SVD method" the paper compares against,
  P:40; SPEC S:278-286 reads it as one-sided Jacobi).  Pure-Python
  loops over column pairs: tiny inputs only.
* closed_form_full_rank: G+ = (G'G)^-1 G' for full column rank,
  computed through Householder QR (numpy.linalg.qr), G+ = R^-1 Q'.
* exact integer helpers for the integer pins.
"""
from __future__ import annotations

import numpy as np


def jacobi_svd(G, sweeps: int = 60, eps: float = 1e-15):
    """One-sided Jacobi: returns U (m x n), sigma (n), V (n x n) with G = U diag(sigma) V', m >= n."""
    A = np.array(G, dtype=np.float64, copy=True)
    m, n = A.shape
    assert m >= n
    V = np.eye(n)
    for _ in range(sweeps):
        off = 0.0
        for p in range(n - 1):
            for q in range(p + 1, n):
                ap, aq = A[:, p], A[:, q]
                alpha = float(ap @ ap)
                beta = float(aq @ aq)
                gamma = float(ap @ aq)
                if alpha == 0.0 or beta == 0.0:
                    continue
                c_ = abs(gamma) / np.sqrt(alpha * beta)
                off = max(off, c_)
                if c_ < eps:
                    continue
                zeta = (beta - alpha) / (2.0 * gamma)
                t = np.sign(zeta) / (abs(zeta) + np.sqrt(1.0 + zeta * zeta)) if zeta != 0 else 1.0
                cs = 1.0 / np.sqrt(1.0 + t * t)
                sn = cs * t
                Ap = A[:, p].copy()
                A[:, p] = cs * Ap - sn * A[:, q]
                A[:, q] = sn * Ap + cs * A[:, q]
                Vp = V[:, p].copy()
                V[:, p] = cs * Vp - sn * V[:, q]
                V[:, q] = sn * Vp + cs * V[:, q]
        if off < eps:
            break
    sigma = np.linalg.norm(A, axis=0)
    U = np.divide(A, sigma, out=np.zeros_like(A), where=sigma > 0)
    return U, sigma, V


def jacobi_svd_pinv(G, rank: int | None = None, rel: float = 1e-10):
    """Pseudoinverse through the Jacobi SVD, truncated at `rank` (or at sigma > rel * sigma_max)."""
    G = np.asarray(G, dtype=np.float64)
    m, n = G.shape
    if m < n:
        return jacobi_svd_pinv(G.T, rank, rel).T
    U, s, V = jacobi_svd(G)
    order = np.argsort(-s)
    s, U, V = s[order], U[:, order], V[:, order]
    if rank is None:
        rank = int((s > rel * (s[0] if s.size else 0.0)).sum()) if s.size and s[0] > 0 else 0
    inv = np.zeros_like(s)
    inv[:rank] = 1.0 / s[:rank]
    return (V * inv) @ U.T


def closed_form_full_rank(G):
    """G+ = (G'G)^-1 G' for full column rank, via Householder QR: G = QR -> G+ = R^-1 Q'."""
    G = np.asarray(G, dtype=np.float64)
    Q, R = np.linalg.qr(G, mode="reduced")
    return np.linalg.solve(R, Q.T)


def int_matmul(A, B):
    """Exact integer product of integer-valued arrays (python ints, no overflow)."""
    A = np.asarray(A, dtype=object)
    B = np.asarray(B, dtype=object)
    return A.dot(B)


def rel_fro(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / nb) if nb > 0 else float(np.linalg.norm(a - b))
