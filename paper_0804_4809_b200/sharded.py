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
