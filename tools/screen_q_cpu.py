"""Find, for each GPU parity-test shape, the first seed >= its base whose ORACLE margins are in Q
(mu_acc >= 1e4 and mu_drop <= 1e-2).  CPU only; calls nothing but oracle/ and the
input generator, so the seeds it prints (hard-coded in tests/ with this script named) come from the
oracle, never from the CUDA path.

    python tools/screen_q_cpu.py            # prints a python dict per test
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import geninv_oracle as O          # noqa: E402
from paper_0804_4809_b200 import inputs as I   # noqa: E402


def first_q(m, n, r, base, qstar=False, limit=200):
    for seed in range(base, base + limit):
        R = O.geninv(I.low_rank(seed, m, n, r).numpy())
        if (R.in_Qstar() if qstar else R.in_Q()) and R.rank == r:
            return seed, R.mu_acc, R.mu_drop
    raise RuntimeError((m, n, r, base))


CASES = {
    "test_ragged_shapes": [((m, n, r), m * 31 + n) for (m, n, r) in
                           [(200, 130, 70), (130, 200, 70), (257, 255, 200), (1000, 333, 260), (33, 700, 20),
                            (520, 129, 1), (64, 64, 48), (2050, 530, 400)]],
    "test_low_rank_k_order": [((m, n, r), m * 3 + n) for (m, n, r) in
                              [(4096, 1024, 100), (600, 3000, 50), (20000, 300, 30), (1000, 999, 400),
                               (1000, 32, 12), (3000, 40, 9), (200, 64, 33), (30, 900, 12)]],
    "test_host_buffers_chunked": [((m, n, r), m + 2 * n) for (m, n, r) in [(90000, 300, 250), (300, 90000, 250)]],
    "test_small_path_info": [((m, n, r), m + n) for (m, n, r) in [(64, 48, 32), (40, 90, 17), (128, 64, 64)]],
    "test_small_path_boundary": [((m, n, min(m, n) - 3), m * 7 + n) for (m, n) in
                                 [(64, 64), (128, 64), (64, 128), (129, 64), (64, 65), (65, 64)]],
    "test_async_matches_sync": [((m, n, r), m + 5 * n) for (m, n, r) in [(2000, 500, 350), (500, 2000, 350),
                                                                         (700, 300, 300)]],
    "test_solve_parity": [((m, n, r), m * 7 + n) for (m, n, r) in
                          [(300, 130, 70), (130, 300, 70), (2050, 530, 400), (257, 255, 200), (96, 64, 40),
                           (64, 64, 64)]],
    # the batched kernel's chunk rings and output chunks: both orientations, ragged s and ell, full rank
    "test_batched_shape_sweep": [((m, n, r), m * 13 + n) for (m, n, r) in
                                 [(1, 1, 1), (7, 3, 3), (3, 7, 2), (64, 64, 64), (128, 64, 64), (64, 128, 64),
                                  (100, 63, 41), (63, 100, 41), (128, 17, 17), (17, 128, 9), (96, 64, 40),
                                  (64, 96, 40), (127, 57, 33), (57, 127, 56), (120, 8, 5), (9, 121, 9),
                                  (80, 50, 30), (50, 80, 27)]],
    # full rank (r = s) through X = L^-T L^-1 (R27): s not a multiple of 32 (TRTRI's identity padding), both
    # orientations, and a square case
    "test_full_rank_direct": [((m, n, r), m * 5 + n) for (m, n, r) in
                              [(700, 333, 333), (333, 700, 333), (2050, 97, 97), (97, 2050, 97), (420, 300, 300)]],
    "test_sharded": [((m, n, r), m + 11 * n) for (m, n, r) in [(3000, 400, 300), (400, 3000, 300),
                                                               (9000, 3200, 3000)]],
}

if __name__ == "__main__":
    only = sys.argv[1:]
    for name, cases in CASES.items():
        if only and name not in only:
            continue
        out = {}
        for shape, base in cases:
            seed, ma, md = first_q(*shape, base)
            out[shape] = seed
            print(f"# {name} {shape}: seed {seed} (base {base}, skipped {seed - base}) mu_acc {ma:.3g} mu_drop {md:.3g}",
                  flush=True)
        print(name, "=", out, flush=True)
