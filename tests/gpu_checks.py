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


# --------------------------------------------------------------------------- C5 full-batch record
def batched_rho(G, X):
    """Relative Penrose residuals per matrix of a (batch, m, n) stack and its G+ stack (torch, cuBLAS)."""
    GX, XG = G @ X, X @ G
    E = [GX @ G - G, XG @ X - X, GX.transpose(1, 2) - GX, XG.transpose(1, 2) - XG]
    D = [G, X, GX, XG]
    nrm = lambda t: torch.linalg.norm(t.reshape(t.shape[0], -1), dim=1)   # noqa: E731
    return torch.stack([nrm(e) / nrm(d) for e, d in zip(E, D)], dim=1)


def c5_full_record(H, base_seed=1, chunk=8192):
    """The whole benchmarked C5 batch (65,536 x 96 x 64, rank 40) through geninv_batched_d in ONE launch,
    against the oracle (SURVEY §8(c4) gates, §8(d2) C5 fields).  Q is taken from BOTH of the oracle's
    forms (the vectorised geninv_batched for every matrix; the scalar geninv for every matrix that misses
    a gate): a matrix is in Q only if both place its margins far from tol (reading R23: the dropped
    pivot is rounding noise, the two forms can differ by 10x).  For every matrix that misses a gate the
    record carries the decision diagnostics (tol, margins of oracle and device) and the spread of valid
    evaluations of the method (oracle/extended.py) against the LAPACK SVD pseudoinverse."""
    import numpy as np

    from oracle import extended as E
    from oracle import geninv_oracle as O
    from paper_0804_4809_b200 import inputs as I

    def rel_b(a, b):
        return np.linalg.norm((a - b).reshape(len(a), -1), axis=1) / np.linalg.norm(b.reshape(len(b), -1), axis=1)

    def rel1(a, b):
        return float(np.linalg.norm(a - b) / np.linalg.norm(b))

    cfg = I.CONFIGS["C5"]
    nb = cfg.batch
    Gb = I.make_batch(cfg, base_seed, 0, nb, device="cuda")
    Gp, rk = H.geninv_batched_d(Gb)
    torch.cuda.synchronize()
    rk = rk.cpu().numpy()
    rel = np.zeros(nb)
    ro = np.zeros(nb, dtype=np.int64)
    mu_acc = np.zeros(nb)
    mu_drop = np.zeros(nb)
    rho = np.zeros((nb, 4))
    Gpo_keep = {}
    import time
    t_or = 0.0
    for c0 in range(0, nb, chunk):
        c1 = min(nb, c0 + chunk)
        G_ = Gb[c0:c1].cpu().numpy()
        t0 = time.perf_counter()
        Gpo, r_, ma, md = O.geninv_batched(G_)
        t_or += time.perf_counter() - t0
        ro[c0:c1], mu_acc[c0:c1], mu_drop[c0:c1] = r_, ma, md
        rel[c0:c1] = rel_b(Gp[c0:c1].cpu().numpy(), Gpo)
        rho[c0:c1] = batched_rho(Gb[c0:c1], Gp[c0:c1]).cpu().numpy()
    rmax = rho.max(axis=1)
    q_b = (mu_acc >= 1e4) & (mu_drop <= 1e-2)
    qs_b = (mu_acc >= 1e6) & (mu_drop <= 1e-3)
    # candidates: matrices in the batched form's Q that miss any gate
    cand = np.nonzero(q_b & ((rk != ro) | (rel > 1e-9) | (rmax > 1e-9) | (qs_b & (rmax > 1e-10))))[0]
    q, qs = q_b.copy(), qs_b.copy()
    diag = []
    for b in cand.tolist():
        G = Gb[b].cpu().numpy()
        R = O.geninv(G)
        in_q = R.in_Q()
        q[b] &= in_q
        qs[b] &= R.in_Qstar()
        _, info = H.geninv_d(Gb[b])                     # the same one-CTA kernel (batch = 1), with its margins
        U, S, Vt = np.linalg.svd(G, full_matrices=False)
        P = (Vt[:R.rank].T / S[:R.rank]) @ U[:, :R.rank].T
        variants = {"oracle": R.Gp, "ext_gram": E.geninv_ext(G, True, False)[0],
                    "ext_chol": E.geninv_ext(G, False, True)[0], "ext_both": E.geninv_ext(G, True, True)[0]}
        spread = max(rel1(v, R.Gp) for k, v in variants.items() if k != "oracle")
        Xo = torch.as_tensor(R.Gp[None]).cuda()
        Xv = torch.as_tensor(np.stack([v for k, v in variants.items() if k != "oracle"])).cuda()
        rho_var = float(batched_rho(Gb[b:b + 1].expand(len(Xv), -1, -1), Xv).max())
        d = {"index": int(b), "in_Q_scalar_oracle": bool(in_q), "rank_gpu": int(rk[b]), "rank_oracle": int(R.rank),
             "rel_gpu_vs_oracle": float(rel[b]), "rho_gpu": rho[b].tolist(),
             "rho_oracle": batched_rho(Gb[b:b + 1], Xo)[0].tolist(),
             "spread_of_valid_evaluations": spread, "rho_valid_evaluations_max": rho_var,
             "rel_vs_svd": {"gpu": rel1(Gp[b].cpu().numpy(), P), **{k: rel1(v, P) for k, v in variants.items()}},
             "oracle": {"tol": R.tol, "mu_acc": R.mu_acc, "mu_drop": R.mu_drop, "min_pivot": R.chol.min_pivot,
                        "batched_form_mu_acc": float(mu_acc[b]), "batched_form_mu_drop": float(mu_drop[b])},
             "device": {"tol": info.tol, "mu_acc": info.mu_acc, "mu_drop": info.mu_drop, "min_pivot": info.min_pivot}}
        diag.append(d)
    rec = {"config": "C5", "matrices": nb, "base_seed": base_seed, "launch": "one geninv_batched_d call (bench.py's)",
           "n_Q": int(q.sum()), "n_Qstar": int(qs.sum()), "n_Q_batched_form_only": int(q_b.sum()),
           "rank_equal_in_Q": int((rk[q] == ro[q]).sum()), "rank_mismatch_outside_Q": int((rk[~q] != ro[~q]).sum()),
           "n_oracle_rank_ne_40": int((ro != 40).sum()), "worst_rel_in_Q": float(rel[q].max()),
           "n_rel_gt_1e-9_in_Q": int((rel[q] > 1e-9).sum()), "n_rel_gt_1e-10_in_Q": int((rel[q] > 1e-10).sum()),
           "worst_rel_in_Qstar": float(rel[qs].max()),
           "worst_rel_outside_Q": float(rel[~q].max()) if (~q).any() else None,
           "penrose_checked": nb, "worst_rho_in_Q": float(rmax[q].max()),
           "n_rho_gt_1e-9_in_Q": int((rmax[q] > 1e-9).sum()), "n_rho_gt_1e-10_in_Q": int((rmax[q] > 1e-10).sum()),
           "worst_rho_in_Qstar": float(rmax[qs].max()), "n_rho_gt_1e-10_in_Qstar": int((rmax[qs] > 1e-10).sum()),
           "oracle_s": t_or, "gate_misses": diag}
    return rec
