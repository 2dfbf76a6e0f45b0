"""Multi-process (world_size 2, gloo, CPU) test of the row-sharded path (`-m "not gpu"`).

paper_0804_4809_b200/sharded.py orchestrates the C4 path: local Gram, one
all-reduce, replicated factorisation, local column block of G+.  Here the
arithmetic backend is the oracle (test-only), so the partitioning and the
exchange are checked on CPU: every rank must see the same A, rank and X, and
the gathered column blocks must equal the unsharded oracle G+.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_0804_4809_b200 import inputs as I
from paper_0804_4809_b200.sharded import row_range, sharded_geninv


class OracleBackend:
    def __init__(self, trans=0):
        from oracle import geninv_oracle as O
        self.O = O
        self.X = None
        self.trans = trans

    def gram(self, G, A):
        g = G.numpy()
        if self.trans:          # column block of a wide G: its share of G G'
            A.copy_(torch.from_numpy(g @ g.T))
        else:
            A.copy_(torch.from_numpy(self.O.gram(g)[0]))

    def all_reduce(self, A):
        dist.all_reduce(A)

    def from_gram(self, A):
        X, ch = self.O.from_gram(A.numpy())
        self.X = X
        return ch

    def apply(self, G, Gp):
        if self.trans:          # rows of G+ = G_p' X
            Gp.copy_(torch.from_numpy(G.numpy().T @ self.X))
        else:
            Gp.copy_(torch.from_numpy(self.O.apply(self.X, G.numpy())))

    @staticmethod
    def rank_of(ch):
        return ch.rank


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, m, n, r, q, trans=0):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    G = I.low_rank(21, m, n, r)
    if trans:                   # wide G: column blocks, row blocks of G+
        r0, r1 = row_range(n, world, rank)
        A = torch.zeros(m, m, dtype=torch.float64)
        Gp = torch.zeros(r1 - r0, m, dtype=torch.float64)
        Gl = G[:, r0:r1].contiguous()
    else:
        r0, r1 = row_range(m, world, rank)
        A = torch.zeros(n, n, dtype=torch.float64)
        Gp = torch.zeros(n, r1 - r0, dtype=torch.float64)
        Gl = G[r0:r1].contiguous()
    be = OracleBackend(trans)
    res = sharded_geninv(be, Gl, A, Gp)
    # every rank must hold identical A and X bits (the exchange is the only source of A)
    digest = torch.tensor([float(A.sum()), float(np.abs(be.X).sum()), float(res.rank)], dtype=torch.float64)
    alld = [torch.zeros(3, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(alld, digest)
    blocks = [None] * world
    dist.all_gather_object(blocks, (r0, r1, Gp.numpy()))
    if rank == 0:
        q.put((res.rank, [d.tolist() for d in alld], blocks))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_matches_unsharded(world):
    from oracle import checks as C
    from oracle import geninv_oracle as O
    m, n, r = 600, 120, 80
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(k, world, port, m, n, r, q)) for k in range(world)]
    for p in ps:
        p.start()
    rank, digests, blocks = q.get(timeout=120)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(d == digests[0] for d in digests)        # identical A, X, rank on every rank
    G = I.low_rank(21, m, n, r).numpy()
    R = O.geninv(G)
    assert rank == R.rank == r
    Gp = np.zeros((n, m))
    for r0, r1, blk in blocks:
        Gp[:, r0:r1] = blk
    assert C.rel_fro(Gp, R.Gp) <= 1e-9
    assert max(O.penrose_residuals(G, Gp)[0]) <= 1e-10


@pytest.mark.parametrize("world", [2])
def test_column_sharded_wide_matches_unsharded(world):
    # C3-style wide G sharded by columns; one exchange (A = sum_p G_p G_p')
    from oracle import checks as C
    from oracle import geninv_oracle as O
    m, n, r = 120, 600, 80
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(k, world, port, m, n, r, q, 1)) for k in range(world)]
    for p in ps:
        p.start()
    rank, digests, blocks = q.get(timeout=120)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(d == digests[0] for d in digests)
    G = I.low_rank(21, m, n, r).numpy()
    R = O.geninv(G)
    assert R.transposed and rank == R.rank == r
    Gp = np.zeros((n, m))
    for r0, r1, blk in blocks:
        Gp[r0:r1] = blk
    assert C.rel_fro(Gp, R.Gp) <= 1e-9
    assert max(O.penrose_residuals(G, Gp)[0]) <= 1e-10


def test_row_range_partition():
    for m in (7, 600, 1 << 21):
        for world in (1, 2, 3, 8):
            rr = [row_range(m, world, k) for k in range(world)]
            assert rr[0][0] == 0 and rr[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(rr, rr[1:]))


def test_oracle_split_equals_whole():
    from oracle import geninv_oracle as O
    G = I.low_rank(22, 300, 90, 60).numpy()
    X, ch = O.from_gram(O.gram(G)[0])
    assert np.array_equal(O.apply(X, G), O.geninv(G).Gp)


# ---------------------------------------------------------------- C5 batch split
def _batch_worker(rank, world, port, nb, q):
    from oracle import geninv_oracle as O
    from paper_0804_4809_b200.sharded import batch_range
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b0, b1 = batch_range(nb, world, rank)
    Gb = I.make_batch(I.CONFIGS["C5"], 1, b0, b1 - b0).numpy()   # each rank builds only its own matrices
    Gp, r, _, _ = O.geninv_batched(Gb)                           # independent matrices: no exchange
    parts = [None] * world
    dist.all_gather_object(parts, (b0, b1, Gp, r))
    if rank == 0:
        q.put(parts)
    dist.destroy_process_group()


def test_batch_split_matches_unsharded():
    from oracle import geninv_oracle as O
    nb, world = 37, 2                                # ragged split: 18 + 19 matrices
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_batch_worker, args=(k, world, port, nb, q)) for k in range(world)]
    for p in ps:
        p.start()
    parts = q.get(timeout=120)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    Gb = I.make_batch(I.CONFIGS["C5"], 1, 0, nb).numpy()
    Gp, r, _, _ = O.geninv_batched(Gb)
    got = np.zeros_like(Gp)
    rk = np.zeros_like(r)
    covered = 0
    for b0, b1, gp, rr in parts:
        got[b0:b1], rk[b0:b1] = gp, rr
        covered += b1 - b0
    assert covered == nb and [p[0] for p in parts] == [0, nb // world]
    assert np.array_equal(rk, r)
    assert np.abs(got - Gp).max() <= 1e-13 * np.abs(Gp).max()


# ---------------------------------------------------------------- the cross-rank replication check
def _digest_worker(rank, world, port, perturb, q):
    from oracle import geninv_oracle as O
    from paper_0804_4809_b200.sharded import check_replicated, replicated_digest
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    G = I.low_rank(21, 300, 60, 40).numpy()
    X, ch = O.from_gram(O.gram(G)[0])
    X = torch.from_numpy(X)
    if perturb and rank == 1:                        # one flipped low bit on one rank
        X[7, 3] = torch.nextafter(X[7, 3], torch.tensor(1e300, dtype=torch.float64))
    ok = check_replicated(replicated_digest(X, ch.rank))
    if rank == 0:
        q.put(ok)
    dist.destroy_process_group()


@pytest.mark.parametrize("perturb", [False, True])
def test_check_replicated(perturb):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_digest_worker, args=(k, 2, port, perturb, q)) for k in range(2)]
    for p in ps:
        p.start()
    ok = q.get(timeout=120)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok == (not perturb)


# ---------------------------------------------------------------- consistency across P
def _p_worker(rank, world, port, m, n, r, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    G = I.low_rank(seed, m, n, r)
    r0, r1 = row_range(m, world, rank)
    A = torch.zeros(n, n, dtype=torch.float64)
    Gp = torch.zeros(n, r1 - r0, dtype=torch.float64)
    be = OracleBackend(0)
    res = sharded_geninv(be, G[r0:r1].contiguous(), A, Gp)
    blocks = [None] * world
    dist.all_gather_object(blocks, (r0, r1, Gp.numpy(), res.rank, res.info.piv.tolist()))
    if rank == 0:
        q.put(blocks)
    dist.destroy_process_group()


def test_consistency_across_P():
    # the grouping of the Gram's partial sums changes with P; under Q the decisions (r, piv) must not, and
    # G+ stays within rounding ("identical r and piv, G+ within ~1e-11")
    from oracle import checks as C
    from oracle import geninv_oracle as O
    m, n, r, seed = 900, 120, 80, 21
    G = I.low_rank(seed, m, n, r).numpy()
    R = O.geninv(G)
    assert R.in_Q()
    ctx = mp.get_context("spawn")
    for world in (2, 3):
        q = ctx.Queue()
        port = _free_port()
        ps = [ctx.Process(target=_p_worker, args=(k, world, port, m, n, r, seed, q)) for k in range(world)]
        for p in ps:
            p.start()
        blocks = q.get(timeout=180)
        for p in ps:
            p.join(timeout=60)
            assert p.exitcode == 0
        Gp = np.zeros((n, m))
        for r0, r1, blk, rk, piv in blocks:
            assert rk == R.rank == r and piv == R.piv.tolist()
            Gp[:, r0:r1] = blk
        assert C.rel_fro(Gp, R.Gp) <= 1e-11, world
