"""The whole benchmarked C5 batch (65,536 matrices 96 x 64 of rank 40, base seed 1) against the oracle:
the SURVEY §8(d2) C5 record (n_Q, n_Q*, rank agreement, worst relative G+ differences, Penrose residuals)
plus, for every matrix in Q whose G+ differs from the oracle's by more than 1e-9, the decision
diagnostics SURVEY §8(c4) "Residual risk" asks for: the oracle's and the device's tol and margins, and
how far each side is from an independent truth (LAPACK SVD pseudoinverse truncated at the oracle's rank).

    python tools/c5_full_report.py [out.json]      (GPU; ~1-2 min of host time for the oracle)
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import geninv_oracle as O              # noqa: E402
from paper_0804_4809_b200 import inputs as I       # noqa: E402
from paper_0804_4809_b200.binding import Handle    # noqa: E402


def batched_rho(G, X):
    """Relative Penrose residuals per matrix, cuBLAS batched products (test-only checker)."""
    GX, XG = G @ X, X @ G
    E = [GX @ G - G, XG @ X - X, GX.transpose(1, 2) - GX, XG.transpose(1, 2) - XG]
    D = [G, X, GX, XG]
    nrm = lambda t: torch.linalg.norm(t.reshape(t.shape[0], -1), dim=1)
    return torch.stack([nrm(e) / nrm(d) for e, d in zip(E, D)], dim=1)


def svd_pinv(Gb, ranks):
    U, S, Vt = np.linalg.svd(Gb, full_matrices=False)
    out = np.zeros((Gb.shape[0], Gb.shape[2], Gb.shape[1]))
    for b in range(Gb.shape[0]):
        r = int(ranks[b])
        out[b] = (Vt[b, :r].T / S[b, :r]) @ U[b, :, :r].T
    return out


def rel_batched(a, b):
    return np.linalg.norm((a - b).reshape(len(a), -1), axis=1) / np.linalg.norm(b.reshape(len(b), -1), axis=1)


def run(base_seed=1, chunk=8192):
    cfg = I.CONFIGS["C5"]
    nb = cfg.batch
    H = Handle(0)
    Gb = I.make_batch(cfg, base_seed, 0, nb, device="cuda")
    Gp, rk = H.geninv_batched_d(Gb)                    # the launch bench.py times (whole batch)
    torch.cuda.synchronize()
    rk = rk.cpu().numpy()
    rel = np.zeros(nb)
    ro = np.zeros(nb, dtype=np.int64)
    mu_acc = np.zeros(nb)
    mu_drop = np.zeros(nb)
    rho = torch.zeros(nb, 4, dtype=torch.float64)
    t_oracle = 0.0
    for c0 in range(0, nb, chunk):
        c1 = min(nb, c0 + chunk)
        G_ = Gb[c0:c1].cpu().numpy()
        t0 = time.perf_counter()
        Gpo, r_, ma, md = O.geninv_batched(G_)
        t_oracle += time.perf_counter() - t0
        ro[c0:c1], mu_acc[c0:c1], mu_drop[c0:c1] = r_, ma, md
        rel[c0:c1] = rel_batched(Gp[c0:c1].cpu().numpy(), Gpo)
        rho[c0:c1] = batched_rho(Gb[c0:c1], Gp[c0:c1]).cpu()
    rho = rho.numpy()
    q = (mu_acc >= 1e4) & (mu_drop <= 1e-2)
    qs = (mu_acc >= 1e6) & (mu_drop <= 1e-3)
    rmax = rho.max(axis=1)
    rec = {"config": "C5", "matrices": nb, "base_seed": base_seed, "n_Q": int(q.sum()), "n_Qstar": int(qs.sum()),
           "rank_equal_in_Q": int((rk[q] == ro[q]).sum()), "rank_mismatch_outside_Q": int((rk[~q] != ro[~q]).sum()),
           "n_oracle_rank_ne_40": int((ro != 40).sum()), "worst_rel_in_Q": float(rel[q].max()),
           "n_rel_gt_1e-9_in_Q": int((rel[q] > 1e-9).sum()), "n_rel_gt_1e-10_in_Q": int((rel[q] > 1e-10).sum()),
           "worst_rel_in_Qstar": float(rel[qs].max()),
           "worst_rel_outside_Q": float(rel[~q].max()) if (~q).any() else None,
           "penrose_checked_in_Q": int(q.sum()), "worst_rho_in_Q": float(rmax[q].max()),
           "n_rho_gt_1e-10_in_Q": int((rmax[q] > 1e-10).sum()), "worst_rho_in_Qstar": float(rmax[qs].max()),
           "n_rho_gt_1e-10_in_Qstar": int((rmax[qs] > 1e-10).sum()),
           "oracle_s": t_oracle, "oracle_threads": os.cpu_count()}
    # decision diagnostics for every Q matrix above 1e-9 (and the 8 worst in Q)
    worst = np.argsort(-np.where(q, rel, -1.0))[:8]
    flagged = sorted(set(np.nonzero(q & (rel > 1e-9))[0].tolist()) | set(worst.tolist()))
    diag = []
    G_f = Gb[flagged].cpu().numpy()
    P_svd = svd_pinv(G_f, ro[flagged])
    for i, b in enumerate(flagged):
        R = O.geninv(G_f[i])
        _, info = H.geninv_d(Gb[b])                     # same one-CTA kernel (batch = 1), with its margins
        diag.append({"index": int(b), "rel_gpu_vs_oracle": float(rel[b]),
                     "rel_gpu_vs_svd": float(rel_batched(Gp[b:b + 1].cpu().numpy(), P_svd[i:i + 1])[0]),
                     "rel_oracle_vs_svd": float(rel_batched(R.Gp[None], P_svd[i:i + 1])[0]),
                     "cond_G": float(np.linalg.cond(G_f[i])), "oracle_tol": R.tol, "oracle_mu_acc": R.mu_acc,
                     "oracle_mu_drop": R.mu_drop, "oracle_min_pivot": R.chol.min_pivot, "gpu_tol": info.tol,
                     "gpu_mu_acc": info.mu_acc, "gpu_mu_drop": info.mu_drop, "gpu_min_pivot": info.min_pivot,
                     "rank": int(R.rank), "rho_gpu": rho[b].tolist()})
    rec["flagged"] = diag
    if os.environ.get("GENINV_C5_DUMP"):   # the flagged matrices' G bits and device G+ (offline analysis)
        np.savez(os.environ["GENINV_C5_DUMP"], index=np.array(flagged), G=G_f, Gp=Gp[flagged].cpu().numpy())
    # Penrose outliers in Q: the device's residuals next to the oracle's and the SVD pseudoinverse's (the
    # checker's own floor) on the same matrix
    pen = []
    idx = np.nonzero(q & (rmax > 1e-10))[0]
    idx = idx[np.argsort(-rmax[idx])][:16]
    if len(idx):
        G_p = Gb[idx.tolist()].cpu().numpy()
        P_p = svd_pinv(G_p, ro[idx])
        for i, b in enumerate(idx):
            R = O.geninv(G_p[i])
            Gt = torch.as_tensor(G_p[i:i + 1]).cuda()
            pen.append({"index": int(b), "rho_gpu": rho[b].tolist(),
                        "rho_oracle": batched_rho(Gt, torch.as_tensor(R.Gp[None]).cuda())[0].tolist(),
                        "rho_svd": batched_rho(Gt, torch.as_tensor(P_p[i:i + 1]).cuda())[0].tolist(),
                        "rel_gpu_vs_oracle": float(rel[b]), "batched_oracle_mu_acc": float(mu_acc[b]),
                        "batched_oracle_mu_drop": float(mu_drop[b]), "oracle_mu_acc": R.mu_acc,
                        "oracle_mu_drop": R.mu_drop, "in_Qstar": bool(qs[b]), "rank": int(ro[b])})
    rec["penrose_outliers"] = pen
    return rec


if __name__ == "__main__":
    rec = run()
    out = sys.argv[1] if len(sys.argv) > 1 else None
    s = json.dumps(rec, indent=1)
    print(s)
    if out:
        open(out, "w").write(s + "\n")
