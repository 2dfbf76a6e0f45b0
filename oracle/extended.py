"""The paper's geninv with chosen steps in x87 extended precision -- TEST
INFRASTRUCTURE ONLY (same import rules as geninv_oracle.py; shares no code with it or the CUDA path).

Purpose: a second, equally valid evaluation of the method, used to measure how far two correct
evaluations can differ on a given input (reading R23).  Near the edge of predicate Q the
forward error of the Cholesky route is set by the conditioning of the accepted columns (the Gram
squares it, and L'L squares it again), so the FP64 result is only determined to
roughly eps * kappa; evaluating the Gram and / or the full-rank Cholesky loop
 with numpy.longdouble (64-bit significand) gives another sample of that spread.

The steps follow the listing exactly as geninv_oracle.geninv does (transpose branch P:107-115, tol
P:117, strict '>' P:124, zeros above pivots R4, inv P:135, the literal product order P:137/139); only
the arithmetic type of the selected steps changes.  Pinned in tests/test_oracle_pins.py
(test_extended_*): exact on integer inputs, equal to the FP64 oracle within 1e-12 on well-conditioned
inputs, and closer to the LAPACK SVD pseudoinverse than the FP64 oracle on ill-conditioned ones.
"""
from __future__ import annotations

import numpy as np

LD = np.longdouble


def geninv_ext(G, gram_ext: bool = True, chol_ext: bool = True, tol_rel: float = 1e-9):
    """Returns (G+ as float64 (n x m), rank, tol) with the Gram / Cholesky in extended precision."""
    G = np.asarray(G, dtype=np.float64)
    m, n = G.shape
    H = G.T if m < n else G                                      # A = H'H, H = G' if m < n
    dt = LD if gram_ext else np.float64
    A = (H.astype(dt).T @ H.astype(dt)).astype(np.float64)        # P:111 / P:114, rounded to FP64
    dA = np.diag(A)
    pos = dA[dA > 0]
    tol = float(pos.min() * tol_rel) if pos.size else 0.0
    ct = LD if chol_ext else np.float64
    s = A.shape[0]
    Ac = A.astype(ct)
    L = np.zeros((s, s), dtype=ct)
    r = 0
    for k in range(s):
        c = Ac[k:, k] - L[k:, :r] @ L[k, :r]
        if c[0] > tol:
            d = np.sqrt(c[0])
            L[k, r] = d
            L[k + 1:, r] = c[1:] / d
            r += 1
    L = L[:, :r].astype(np.float64)
    if r == 0:
        return np.zeros((n, m)), 0, tol
    M = np.linalg.inv(L.T @ L)
    if m < n:
        Y = (((G.T @ L) @ M) @ M) @ L.T
    else:
        Y = ((((L @ M) @ M) @ L.T) @ G.T)
    return Y, r, tol
