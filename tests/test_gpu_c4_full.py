"""C4 at BASELINE.json's full size (2,097,152 x 4096, rank 3584), in the launch configuration bench.py
times (split C ABI: geninv_gram_d -> geninv_from_gram_d -> geninv_apply_d, one GPU), against the oracle.

The oracle runs on the host from the same G bits (copied device -> host): its Gram is numpy's
G'G (the listing's `G'*G`), then its own tolerance / full-rank Cholesky / inverse / product
chain (oracle.from_gram).  Compared: the detected rank and pivot list (exact, inputs in Q),
X = L M M L' (relative), and sampled columns of G+ = X G' (relative); plus full-size Penrose
conditions on the GPU with cuBLAS (tests/gpu_checks.py: torch.matmul with pairwise-summed 4096-row
chunks, a test-only checker independent of the library), gated at 1e-10 as the north star states.
Needs ~130 GiB of HBM and ~70 GiB of host RAM; takes a few minutes.  Run for the native path and
for the INT8-emulated Gram and a7.
"""
import os

import numpy as np
import pytest
import torch

from oracle import checks as C
from oracle import geninv_oracle as O
from paper_0804_4809_b200 import inputs as I
from tests.gpu_checks import penrose_streamed

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.mark.parametrize("emulate", [0, 1], ids=["dmma", "int8_emulated"])
def test_c4_full_size(emulate):
    """emulate = 1: the Gram and a7 on the INT8 tensor cores (geninv_set_emulation)."""
    from paper_0804_4809_b200.binding import Handle
    from paper_0804_4809_b200.sharded import CudaBackend, sharded_geninv

    cfg = I.CONFIGS["C4"]
    m, n = cfg.m, cfg.n
    h = Handle(0)
    h.set_emulation(emulate)
    be = CudaBackend(h)
    seed = int(os.environ.get("GENINV_C4_SEED", I.QSEED["C4"]))   # override: screening candidate seeds
    G = I.make_single(cfg, seed, device="cuda")
    A = torch.zeros(n, n, dtype=torch.float64, device="cuda")
    Gp = torch.empty(n, m, dtype=torch.float64, device="cuda")
    res = sharded_geninv(be, G, A, Gp)                  # world size 1: the bench's step
    torch.cuda.synchronize()
    info = res.info
    assert info.rank == cfg.rank
    # device-side pivot list (same A, untimed step entry point)
    _, piv_gpu, _ = h.geninv_frchol_d(A)
    piv_gpu = piv_gpu.cpu().numpy()
    X_gpu = h.geninv_copy_x().cpu().numpy()

    # ---- oracle from the same G bits
    Gh = G.cpu().numpy()
    A_or = Gh.T @ Gh                                    # P:114, A = G'G
    X_or, ch = O.from_gram(A_or)
    in_q = ch.mu_acc >= 1e4 and ch.mu_drop <= 1e-2
    print(f"C4 seed {seed} device: mu_acc {info.mu_acc:.3g}, mu_drop {info.mu_drop:.3g}")
    print(f"C4 oracle: rank {ch.rank}, mu_acc {ch.mu_acc:.3g}, mu_drop {ch.mu_drop:.3g}, in Q: {in_q}")
    assert ch.rank == info.rank
    assert in_q, f"seed {seed} is not in Q by the oracle's margins (SURVEY §8(c4)); pick another QSEED"
    if in_q:
        assert np.array_equal(piv_gpu, ch.piv)
        assert C.rel_fro(X_gpu, X_or) <= 1e-9
        # sampled columns of G+ (row blocks of G)
        rng = np.random.default_rng(0)
        cols = np.sort(rng.choice(m, size=512, replace=False))
        want = X_or @ Gh[cols].T
        got = Gp[:, torch.as_tensor(cols, device="cuda")].cpu().numpy()
        assert C.rel_fro(got, want) <= 1e-9
    del Gh, A_or
    torch.cuda.empty_cache()

    # ---- full-size Penrose conditions on the GPU (cuBLAS, independent of the library), for the
    #      device's G+ and, with the same checker, for the oracle's G+ = X_or G' (the method's own
    #      rounding floor at this size: G'G squares the conditioning of the accepted columns)
    rho_gpu = penrose_streamed(G, Gp)
    del Gp, res                                         # 64 GiB: make room for the oracle's G+
    torch.cuda.empty_cache()
    Gp_or = torch.as_tensor(X_or, device="cuda") @ G.T
    rho_or = penrose_streamed(G, Gp_or)
    print("C4 Penrose device", rho_gpu)
    print("C4 Penrose oracle", rho_or)
    assert max(rho_gpu) <= 1e-10                        # the north star's gate as written
