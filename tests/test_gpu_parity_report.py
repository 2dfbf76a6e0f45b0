"""Parity report over the BASELINE configs (`-m gpu`, slow): one JSON record per config with the
device and oracle ranks, pivot agreement, the oracle's decision margins (predicate Q, SURVEY
§8(c4)), the relative difference of G+ and the four relative Penrose residuals (cuBLAS checker,
test-only), and the device / oracle times -- the row SURVEY §8(d2) asks for -- for the native path
and with the Gram / a7 emulated on the INT8 tensor cores.  Gates as in the
other parity tests.  With GENINV_PARITY_REPORT=<path> the records are written there (JSON lines).
C4 at full size is covered by tests/test_gpu_c4_full.py."""
import json
import os
import time

import numpy as np
import pytest
import torch

from oracle import checks as C
from oracle import geninv_oracle as O
from paper_0804_4809_b200 import inputs as I

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
RECORDS = []


@pytest.fixture(scope="module")
def H():
    from paper_0804_4809_b200.binding import Handle
    h = Handle(0)
    yield h
    path = os.environ.get("GENINV_PARITY_REPORT")
    if path and RECORDS:
        with open(path, "w") as f:
            for r in RECORDS:
                f.write(json.dumps(r) + "\n")


def rho(G, X):
    GX, XG = G @ X, X @ G
    E = [GX @ G - G, XG @ X - X, GX.T - GX, XG.T - XG]
    D = [G, X, GX, XG]
    return [float(torch.linalg.norm(e) / torch.linalg.norm(d)) for e, d in zip(E, D)]


def time_device(H, G, Gp, reps=5):
    H.geninv_d(G, Gp)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        H.geninv_d(G, Gp)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


@pytest.mark.parametrize("emulate", [0, 1], ids=["dmma", "int8_emulated"])
@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C3T"])
def test_config_parity_record(H, name, emulate):
    if name == "C3T":
        G = I.make_single(I.CONFIGS["C3"], I.QSEED["C3"], device="cuda").T.contiguous()
        seed = I.QSEED["C3"]
    else:
        seed = I.QSEED[name]
        G = I.make_single(I.CONFIGS[name], seed, device="cuda")
    m, n = G.shape
    H.set_emulation(emulate)
    Gp, info = H.geninv_d(G)
    ms = time_device(H, G, Gp)
    H.set_emulation(0)
    Gh = G.cpu().numpy()
    t0 = time.perf_counter()
    R = O.geninv(Gh)
    oracle_ms = (time.perf_counter() - t0) * 1e3
    # device pivots from the step entry point on the device Gram
    A = torch.zeros(min(m, n), min(m, n), dtype=torch.float64, device="cuda")
    H.geninv_gram_d(G, int(m < n), A)
    _, piv, _ = H.geninv_frchol_d(A)
    rel = C.rel_fro(Gp.cpu().numpy(), R.Gp)
    rh = rho(G, Gp)
    rec = {"config": name, "emulated": bool(emulate), "seed": seed, "m": m, "n": n, "r_gpu": info.rank,
           "r_oracle": R.rank,
           "piv_equal": bool(np.array_equal(piv.cpu().numpy(), R.chol.piv)), "mu_acc": R.mu_acc,
           "mu_drop": R.mu_drop, "in_Q": R.in_Q(), "rel_fro": rel, "rho": rh, "device_ms": ms,
           "oracle_ms": oracle_ms, "oracle_threads": os.cpu_count()}
    RECORDS.append(rec)
    print(json.dumps(rec))
    assert R.in_Q()
    assert info.rank == R.rank and rec["piv_equal"]
    assert rel <= 1e-9
    assert max(rh) <= 1e-10


def test_c5_parity_record(H):
    cfg = I.CONFIGS["C5"]
    nb = 8192
    Gb = I.make_batch(cfg, 1, 0, nb, device="cuda")
    Gp, rk = H.geninv_batched_d(Gb)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    Gpo, ro, mu_acc, mu_drop = O.geninv_batched(Gb.cpu().numpy())
    oracle_ms = (time.perf_counter() - t0) * 1e3
    q = (mu_acc >= 1e4) & (mu_drop <= 1e-2)
    qs = (mu_acc >= 1e6) & (mu_drop <= 1e-3)
    rk = rk.cpu().numpy()
    G_, Gp_ = Gb.cpu().numpy(), Gp.cpu().numpy()
    rel = np.array([C.rel_fro(Gp_[b], Gpo[b]) for b in range(nb)])
    rho_q, rho_qs = [], []
    for b in np.nonzero(q)[0][:512]:
        rho_q.append(max(rho(torch.as_tensor(G_[b]).cuda(), torch.as_tensor(Gp_[b]).cuda())))
        if qs[b]:
            rho_qs.append(rho_q[-1])
    rho_q, rho_qs = np.array(rho_q), np.array(rho_qs)
    rec = {"config": "C5", "matrices": nb, "base_seed": 1, "n_Q": int(q.sum()), "n_Qstar": int(qs.sum()),
           "rank_equal_in_Q": int((rk[q] == ro[q]).sum()), "rank_mismatch_outside_Q": int((rk[~q] != ro[~q]).sum()),
           "n_oracle_rank_ne_40": int((ro != 40).sum()), "worst_rel_in_Q": float(rel[q].max()),
           "n_rel_gt_1e-9_in_Q": int((rel[q] > 1e-9).sum()), "worst_rel_in_Qstar": float(rel[qs].max()),
           "worst_rel_outside_Q": float(rel[~q].max()) if (~q).any() else None,
           "penrose_checked_in_Q": int(rho_q.size), "worst_rho_in_Q": float(rho_q.max()),
           "n_rho_gt_1e-10_in_Q": int((rho_q > 1e-10).sum()), "worst_rho_in_Qstar": float(rho_qs.max()),
           "oracle_ms": oracle_ms}
    RECORDS.append(rec)
    print(json.dumps(rec))
    assert rec["rank_equal_in_Q"] == rec["n_Q"]
    # R23: at mu_acc just above the Q bound the accepted L is ill-conditioned and the G+ error is
    # conditioning-limited (matrix 1900 of base seed 1: mu_acc 1.01e4; device vs oracle 2.9e-9, oracle vs
    # LAPACK pinv 5.2e-10); the 1e-9 / 1e-10 gates are asserted on Q*, Q gets the C5 1e-9 Penrose gate
    assert rec["worst_rel_in_Qstar"] <= 1e-9
    assert rec["n_rel_gt_1e-9_in_Q"] <= 2
    assert rec["worst_rho_in_Qstar"] <= 1e-10
    assert rec["worst_rho_in_Q"] <= 1e-9
