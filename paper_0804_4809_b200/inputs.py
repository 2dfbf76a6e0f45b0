"""Seeded synthetic inputs for geninv -- shared by the tests, the oracle runs and bench.py.

This module holds NONE of the method's arithmetic (no Gram, no Cholesky, no
inverse, no product of the method).  It only builds the matrices G that both
the CUDA path and the oracle consume, following the config recipes of
BASELINE.json `configs` and SURVEY.md §8(d1) (reading R15 in DESIGN.md):

* uniforms are counter-based splitmix64: u_i = (mix64(key + (i+1)*GOLDEN) >> 11) * 2^-53,
  so any row chunk / row shard is generated independently;
* normals are Box-Muller over consecutive uniform pairs;
* exact-rank matrices are G = U @ V (U: m x r, V: r x n, N(0,1) entries), formed
  by torch.matmul (cuBLAS on a GPU, the CPU BLAS otherwise) -- input
  construction only, not the product path;
* C3's 512 duplicated columns come from a seeded Fisher-Yates permutation (R13).

The same G bits are fed to both sides; where G is formed on the GPU (C3, C4)
it is copied to the host for the oracle.  Works on CPU and CUDA tensors.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

GOLDEN = 0x9E3779B97F4A7C15
_M64 = (1 << 64) - 1

TAG_U, TAG_V, TAG_DIRECT, TAG_COLS = 1, 2, 3, 4


def _s64(x: int) -> int:
    """uint64 constant -> the int64 with the same bits."""
    x &= _M64
    return x - (1 << 64) if x >= (1 << 63) else x


def _srl(z: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of int64 tensors holding uint64 bits."""
    return (z >> k) & ((1 << (64 - k)) - 1)


def mix64_int(z: int) -> int:
    """splitmix64 finaliser on a python int (uint64 semantics)."""
    z &= _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def _mix64(z: torch.Tensor) -> torch.Tensor:
    z = (z ^ _srl(z, 30)) * _s64(0xBF58476D1CE4E5B9)
    z = (z ^ _srl(z, 27)) * _s64(0x94D049BB133111EB)
    return z ^ _srl(z, 31)


def stream_key(seed: int, tag: int) -> int:
    return mix64_int((seed & _M64) ^ tag)


def uniforms(key: int, start: int, count: int, device="cpu") -> torch.Tensor:
    """u_i for i in [start, start+count): float64 in [0, 1)."""
    i = torch.arange(start + 1, start + count + 1, dtype=torch.int64, device=device)
    z = _s64(key) + i * _s64(GOLDEN)
    z = _mix64(z)
    return _srl(z, 11).to(torch.float64) * (2.0 ** -53)


def normals(key: int, start: int, count: int, device="cpu") -> torch.Tensor:
    """N(0,1) entries e_i, i in [start, start+count); e_{2p}, e_{2p+1} from Box-Muller of (u_{2p}, u_{2p+1})."""
    p0 = start // 2
    p1 = (start + count + 1) // 2
    u = uniforms(key, 2 * p0, 2 * (p1 - p0), device).view(-1, 2)
    rad = torch.sqrt(-2.0 * torch.log1p(-u[:, 0]))
    ang = (2.0 * math.pi) * u[:, 1]
    z = torch.stack((rad * torch.cos(ang), rad * torch.sin(ang)), dim=1).reshape(-1)
    off = start - 2 * p0
    return z[off:off + count]


def normal_matrix(key: int, rows: int, cols: int, row0: int = 0, device="cpu") -> torch.Tensor:
    """rows x cols block (starting at global row row0) of the matrix whose element (i, j) is e_{i*cols+j}."""
    return normals(key, row0 * cols, rows * cols, device).view(rows, cols)


def low_rank(seed: int, m: int, n: int, r: int, device="cpu", row0: int = 0, rows: int | None = None,
             chunk: int = 1 << 14, out: torch.Tensor | None = None) -> torch.Tensor:
    """Rows [row0, row0+rows) of G = U @ V, U: m x r, V: r x n, i.i.d. N(0,1) (configs 1, 3, 4, 5)."""
    rows = m - row0 if rows is None else rows
    V = normal_matrix(stream_key(seed, TAG_V), r, n, 0, device)
    if out is None:
        out = torch.empty(rows, n, dtype=torch.float64, device=device)
    ku = stream_key(seed, TAG_U)
    for c0 in range(0, rows, chunk):
        c1 = min(rows, c0 + chunk)
        U = normal_matrix(ku, c1 - c0, r, row0 + c0, device)
        torch.matmul(U, V, out=out[c0:c1])
        del U
    return out


def dense_normal(seed: int, m: int, n: int, device="cpu") -> torch.Tensor:
    """G with i.i.d. N(0,1) entries (config 2)."""
    return normal_matrix(stream_key(seed, TAG_DIRECT), m, n, 0, device)


def copy_columns(seed: int, n: int, ncopy: int):
    """Seeded Fisher-Yates over 0..n-1; D = perm[:ncopy] (destinations), S = perm[ncopy:2 ncopy] (sources)."""
    key = stream_key(seed, TAG_COLS)
    u = uniforms(key, 0, n, "cpu").tolist()
    perm = list(range(n))
    for i in range(n - 1, 0, -1):
        j = int(u[i] * (i + 1))
        perm[i], perm[j] = perm[j], perm[i]
    return perm[:ncopy], perm[ncopy:2 * ncopy]


def batch_seed(base: int, b: int) -> int:
    return mix64_int((base & _M64) ^ (((b + 1) * GOLDEN) & _M64))


# ---------------------------------------------------------------------------
# The five configs of BASELINE.json.
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Config:
    name: str
    m: int
    n: int
    rank: int          # constructed rank (min(m, n) for full rank)
    batch: int = 1
    ncopy: int = 0     # C3: duplicated columns

    @property
    def s(self):
        return min(self.m, self.n)

    @property
    def ell(self):
        return max(self.m, self.n)


CONFIGS = {
    "C1": Config("C1", 64, 48, 32),
    "C2": Config("C2", 4096, 1024, 1024),
    "C3": Config("C3", 4096, 16384, 3072, ncopy=512),
    "C4": Config("C4", 1 << 21, 4096, 3584),
    "C5": Config("C5", 96, 64, 40, batch=65536),
}

# The seed each single-matrix config is run with (tests and bench.py): the first seed >= 1 whose
# ORACLE decision margins satisfy predicate Q (mu_acc >= 1e4 and mu_drop <= 1e-2),
# pre-screened on the device with tools/screen_seeds.py and confirmed by the oracle in the GPU
# parity tests (which assert Q).  C5 uses fixed per-matrix seeds from base seed 1 (no rejection).
QSEED = {"C1": 1, "C2": 1, "C3": 1, "C4": 5, "C5": 1}
# C4 screen (tools/screen_seeds.py, device margins; profiles/r01_seed_screen_c4.jsonl): seeds 1-4 and 6-9
# fail Q (mu_drop > 1e-2 or mu_acc < 1e4); seed 5: device mu_acc 1.1e5 / mu_drop 9.8e-3, oracle
# mu_acc 1.1e5 / mu_drop 4.6e-3 -> in Q.  C3: seed 1 is in Q (device mu_acc 2.8e5, mu_drop 4.1e-4).


def make_single(cfg: Config, seed: int, device="cpu", row0: int = 0, rows: int | None = None,
                out: torch.Tensor | None = None) -> torch.Tensor:
    """G (or its row block [row0, row0+rows)) for a single-matrix config."""
    if cfg.rank >= cfg.s and cfg.ncopy == 0 and cfg.name == "C2":
        G = dense_normal(seed, cfg.m, cfg.n, device)
        rows = cfg.m - row0 if rows is None else rows
        G = G[row0:row0 + rows]
        if out is not None:
            out.copy_(G)
            return out
        return G.contiguous()
    G = low_rank(seed, cfg.m, cfg.n, cfg.rank, device, row0, rows, out=out)
    if cfg.ncopy:
        D, S = copy_columns(seed, cfg.n, cfg.ncopy)
        G[:, torch.tensor(D, device=G.device)] = G[:, torch.tensor(S, device=G.device)]
    return G


def make_batch(cfg: Config, base_seed: int, b0: int = 0, count: int | None = None, device="cpu") -> torch.Tensor:
    """Matrices [b0, b0+count) of a batched config, shape (count, m, n); matrix b uses seed batch_seed(base, b).

    Each matrix b draws U_b from stream_key(seed_b, TAG_U) and V_b from
    stream_key(seed_b, TAG_V), exactly as low_rank(); this builds all keys at
    once and runs one batched matmul.
    """
    count = cfg.batch - b0 if count is None else count
    m, n, r = cfg.m, cfg.n, cfg.rank
    seeds = [batch_seed(base_seed, b0 + i) for i in range(count)]
    ku = torch.tensor([_s64(stream_key(s, TAG_U)) for s in seeds], dtype=torch.int64, device=device)
    kv = torch.tensor([_s64(stream_key(s, TAG_V)) for s in seeds], dtype=torch.int64, device=device)

    def batched_normals(keys, cnt):
        npair = (cnt + 1) // 2
        idx = torch.arange(1, 2 * npair + 1, dtype=torch.int64, device=device)
        z = keys[:, None] + idx[None, :] * _s64(GOLDEN)
        u = _srl(_mix64(z), 11).to(torch.float64) * (2.0 ** -53)
        u = u.view(len(keys), npair, 2)
        rad = torch.sqrt(-2.0 * torch.log1p(-u[..., 0]))
        ang = (2.0 * math.pi) * u[..., 1]
        e = torch.stack((rad * torch.cos(ang), rad * torch.sin(ang)), dim=-1).reshape(len(keys), -1)
        return e[:, :cnt]

    out = torch.empty(count, m, n, dtype=torch.float64, device=device)
    step = 4096
    for c0 in range(0, count, step):
        c1 = min(count, c0 + step)
        U = batched_normals(ku[c0:c1], m * r).view(-1, m, r)
        V = batched_normals(kv[c0:c1], r * n).view(-1, r, n)
        torch.matmul(U, V, out=out[c0:c1])
    return out


# Seed used for the paper's family at each n (the first seed >= 1 whose ORACLE margins are in Q,
# as for the configs; asserted by tests/test_gpu_paper_family.py).  Seed 1 misses Q at n = 128
# (mu_drop 0.013) and n = 1024 (mu_drop 0.048), where even the oracle's G+ exceeds the paper's
# 2e-10 per-coefficient bound.
PAPER_QSEED = {32: 1, 64: 1, 128: 2, 256: 1, 512: 1, 1024: 2, 2048: 1, 4096: 1, 8192: 1}
# ... and the first seed whose oracle margins are in Q* (mu_acc >= 1e6, mu_drop <= 1e-3): the inputs on
# which the paper's 2e-10 per-coefficient statement is checked (reading R22).
PAPER_QSTAR_SEED = {32: 1, 64: 2, 128: 3, 256: 1, 512: 9, 1024: 17}


def paper_family(n: int, seed: int, device="cpu") -> torch.Tensor:
    """The paper's own test family: m = 2n, rank r = 7n/8, coefficients in [-1, 1].

    The construction is unstated in the paper; reading R16 (after SPEC S:393):
    G = B C with B (2n x r), C (r x n) uniform in [-1, 1], rescaled so that
    max |G| = 1.
    """
    m, r = 2 * n, (7 * n) // 8
    B = uniforms(stream_key(seed, TAG_U), 0, m * r, device).view(m, r) * 2.0 - 1.0
    C = uniforms(stream_key(seed, TAG_V), 0, r * n, device).view(r, n) * 2.0 - 1.0
    G = B @ C
    return G / G.abs().max()
