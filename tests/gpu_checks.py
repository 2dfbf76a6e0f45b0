"""Test-only GPU checkers (torch / cuBLAS FP64), independent of the library under test.

penrose_streamed: the four relative Penrose residuals of a tall G (m x n)
and its G+ (n x m) without m x m temporaries.  T = G+ G is accumulated over 2^12-row chunks whose
partial products are summed PAIRWISE (a binary counter of partial sums), so the checker's own rounding
(each chunk a K = 4096 cuBLAS product, then ~log2(m / 4096) levels of adds) stays well below the
residuals it measures; a single sequential sum over 2^21 rows would not.
"""
import torch


def pairwise_sum_products(left, right, m, chunk=1 << 12):
    """sum over row chunks c of left(c) @ right(c), summed pairwise in a fixed order."""
    stack = []   # (level, partial sum)
    for c0 in range(0, m, chunk):
        c1 = min(m, c0 + chunk)
        t = left(c0, c1) @ right(c0, c1)
        lvl = 0
        while stack and stack[-1][0] == lvl:
            _, u = stack.pop()
            t = u + t
            lvl += 1
        stack.append((lvl, t))
    T = stack.pop()[1]
    while stack:
        T = stack.pop()[1] + T
    return T


def penrose_streamed(G, Gp, block=1 << 18):
    """[rho1, rho2, rho3, rho4] for G (m x n, m >= n) and Gp (n x m), both CUDA float64."""
    m, n = G.shape
    T = pairwise_sum_products(lambda a, b: Gp[:, a:b], lambda a, b: G[a:b], m)      # T = G+ G (n x n)
    rho4 = float(torch.linalg.norm(T.T - T) / torch.linalg.norm(T))
    e1 = e2 = n1 = n2 = 0.0
    for c0 in range(0, m, block):                       # streamed: no m x n temporaries
        c1 = min(m, c0 + block)
        e1 += float(torch.linalg.norm(G[c0:c1] @ T - G[c0:c1]) ** 2)         # G G+ G - G
        n1 += float(torch.linalg.norm(G[c0:c1]) ** 2)
        e2 += float(torch.linalg.norm(T @ Gp[:, c0:c1] - Gp[:, c0:c1]) ** 2)  # G+ G G+ - G+
        n2 += float(torch.linalg.norm(Gp[:, c0:c1]) ** 2)
    rho1, rho2 = (e1 / n1) ** 0.5, (e2 / n2) ** 0.5
    rows = torch.arange(0, m, max(1, m // 8192), device=G.device)[:8192]    # sampled principal block
    GX = G[rows] @ Gp[:, rows]
    rho3 = float(torch.linalg.norm(GX.T - GX) / torch.linalg.norm(GX))
    return [rho1, rho2, rho3, rho4]
