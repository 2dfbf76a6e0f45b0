"""Sharded geninv (north star "G is row-sharded").

Tall G (C4, m >= n, trans = 0): rank p holds rows [p*m/P, (p+1)*m/P) of G.  One step:

    A_p = G_p' G_p              (a1 on the local rows)        backend.gram
    A   = sum_p A_p             (a8, the one exchange step)   backend.all_reduce
    X   = L M M L' from A       (a2-a6, replicated)           backend.from_gram
    G+[:, rows_p] = X G_p'      (a7, local column block)      backend.apply

Wide G (C3, m < n, trans = 1): rank p holds columns [p*n/P, (p+1)*n/P) of G
(an m x n_p block), A = sum_p G_p G_p' (P:111 summed over column blocks), and
G+[cols_p, :] = G_p' X is the rank's row block of G+ -- the same single exchange.

The arithmetic lives in the backend: on GPUs the C ABI (geninv_gram_d /
geninv_from_gram_d / geninv_apply_d) with an NCCL all-reduce; the CPU tests
inject an oracle-based backend with a gloo all-reduce to cover this
orchestration (partitioning, exchange, replicated factorisation) on CPU.
"""
from __future__ import annotations

from dataclasses import dataclass


def row_range(m: int, world: int, rank: int):
    """Contiguous row (or column) block of rank `rank`: [r0, r1)."""
    per = m // world
    r0 = rank * per
    r1 = m if rank == world - 1 else r0 + per
    return r0, r1


@dataclass
class ShardResult:
    rank: int        # detected rank r (identical on every process)
    info: object     # backend-specific diagnostics
    Gp_local: object  # trans 0: n x rows_p (column block of G+); trans 1: cols_p x m (row block of G+)


def sharded_geninv(backend, G_local, A, Gp_local) -> ShardResult:
    """One sharded geninv step.  A (s x s) and Gp_local are caller-owned buffers."""
    backend.gram(G_local, A)
    backend.all_reduce(A)
    info = backend.from_gram(A)
    backend.apply(G_local, Gp_local)
    return ShardResult(backend.rank_of(info), info, Gp_local)


def batch_range(batch: int, world: int, rank: int):
    """C5 (independent matrices): rank p owns matrices [b0, b1) -- no exchange at all."""
    return row_range(batch, world, rank)


_PHI = -7046029254386353131        # 0x9E3779B97F4A7C15 as int64
_M1 = -4658895280553007687         # 0xBF58476D1CE4E5B9
_M2 = -7723592293110705685         # 0x94D049BB133111EB


def _srl(z, k):
    return (z >> k) & ((1 << (64 - k)) - 1)


def replicated_digest(X, r: int):
    """(r, 64-bit hash of X's bits) as 4 exactly representable float64 values (r, then 3 x 22-bit pieces).
    The hash mixes every element with its position (splitmix64 finaliser), so any differing bit of the
    replicated X = L M M L' changes it.  Works on CPU and CUDA tensors."""
    import torch
    b = X.contiguous().view(-1).view(torch.int64)
    z = b + (torch.arange(1, b.numel() + 1, dtype=torch.int64, device=b.device) * _PHI)
    z = (z ^ _srl(z, 30)) * _M1
    z = (z ^ _srl(z, 27)) * _M2
    z = z ^ _srl(z, 31)
    h = int(z.sum().item()) & ((1 << 64) - 1)
    parts = [float((h >> (22 * k)) & ((1 << 22) - 1)) for k in range(3)]
    return torch.tensor([float(r)] + parts, dtype=torch.float64)


def check_replicated(digest, group=None) -> bool:
    """All-gather every rank's replicated_digest; True iff all ranks hold the same r and X bits (the
    factorisation runs replicated from the all-reduced A: deterministic kernels must give identical bits)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return True
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else torch.device("cpu")
    d = digest.to(dev)
    out = [torch.zeros_like(d) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, d, group=group)
    return all(bool(torch.equal(o, out[0])) for o in out)


class CudaBackend:
    """The C-ABI path (binding.Handle) + torch.distributed (NCCL) for the exchange."""

    def __init__(self, handle, group=None, trans: int = 0):
        self.h = handle
        self.group = group
        self.trans = int(trans)

    def gram(self, G, A):
        # writes the lower triangle; the caller allocates A zeroed so the all-reduced
        # upper triangle stays exactly zero
        self.h.geninv_gram_d(G, self.trans, A)

    def all_reduce(self, A):
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(self.group) > 1:
            dist.all_reduce(A, group=self.group)

    def from_gram(self, A):
        return self.h.geninv_from_gram_d(A)

    def apply(self, G, Gp):
        self.h.geninv_apply_d(G, self.trans, Gp)

    @staticmethod
    def rank_of(info):
        return info.rank
