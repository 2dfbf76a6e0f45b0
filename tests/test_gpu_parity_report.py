"""Parity report over the BASELINE configs (`-m gpu`, slow): one JSON record per config with the
device and oracle ranks, pivot agreement, the oracle's decision margins (predicate Q, SURVEY
§8(c4)), the relative difference of G+ and the four relative Penrose residuals (cuBLAS checker,
test-only), and the device / oracle times -- the row SURVEY §8(d2) asks for -- for the native path
and with the Gram / a7 emulated on the INT8 tensor cores.  Gates as in the
other parity tests.  With GENINV_PARITY_REPORT=<path> the records are written there (JSON lines).
C4 at full size is covered by tests/test_gpu_c4_full.py, C5's whole batch by tests/test_gpu_c5_full.py."""
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

# C5: the whole benchmarked batch (65,536 matrices) is compared in tests/test_gpu_c5_full.py.
