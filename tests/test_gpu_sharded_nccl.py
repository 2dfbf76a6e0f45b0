"""geninv_sharded_d through a real NCCL communicator (`-m gpu`).  On the single GPU of the test box
the process group has one rank, so the all-reduce is the identity: the call must reproduce
geninv_d bit for bit, in both sharding modes (rows of a tall G, columns of a wide G), on the DMMA
path and with the Gram / a7 emulated on the INT8 tensor cores.  The
multi-rank orchestration is covered on CPU by tests/test_sharded_gloo.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from oracle import checks as C
from oracle import geninv_oracle as O
from paper_0804_4809_b200 import inputs as I

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    t = torch.ones(1, device="cuda")
    dist.all_reduce(t)
    be = dist.distributed_c10d._get_default_group()._get_backend(torch.device("cuda"))
    yield be._comm_ptr()
    dist.destroy_process_group()


@pytest.fixture(scope="module")
def H():
    from paper_0804_4809_b200.binding import Handle
    return Handle(0)


@pytest.mark.parametrize("emulate", [0, 1], ids=["dmma", "int8_emulated"])
@pytest.mark.parametrize("m,n,r,trans", [(3000, 400, 300, 0), (400, 3000, 300, 1), (9000, 3200, 3000, 0)])
def test_sharded_single_rank_equals_geninv(H, comm, m, n, r, trans, emulate):
    # seed: first >= m + 11n with oracle margins in Q (tools/screen_q_cpu.py, CPU-generated G)
    seed = {(3000, 400, 300): 7400, (400, 3000, 300): 33400, (9000, 3200, 3000): 44200}[(m, n, r)]
    G = I.low_rank(seed, m, n, r).cuda()
    H.set_emulation(emulate)
    whole, info = H.geninv_d(G)
    Gp = torch.empty(n, m, dtype=torch.float64, device="cuda")
    _, sinfo = H.geninv_sharded_d(comm, G, trans, Gp)
    H.set_emulation(0)
    assert sinfo.rank == info.rank == r
    R = O.geninv(G.cpu().numpy())
    assert R.in_Q()
    assert C.rel_fro(Gp.cpu().numpy(), R.Gp) <= 1e-9
    assert C.rel_fro(Gp.cpu().numpy(), whole.cpu().numpy()) <= 1e-12


def test_sharded_local_failure_returns_everywhere(H, comm):
    # a rank whose local checks fail still takes part in the pre-check all-reduce and returns the status
    # (with several ranks the others return it too instead of blocking in the all-reduce of A)
    from paper_0804_4809_b200.binding import _Info, _opts
    import ctypes
    G = torch.zeros(100, 40, dtype=torch.float64, device="cuda")
    Gp = torch.zeros(40, 100, dtype=torch.float64, device="cuda")
    rank, info, o = ctypes.c_int64(), _Info(), _opts()
    st = H._lib.geninv_sharded_d(H._h, ctypes.c_void_p(comm), G.data_ptr(), 100, 40, 40, 0, Gp.data_ptr(), 99,
                                 ctypes.byref(rank), ctypes.byref(o), ctypes.byref(info))
    assert st == 1                                           # GENINV_EINVAL: ldp < m_local
    # the communicator is still usable afterwards: a valid call succeeds
    G = I.low_rank(7400, 3000, 400, 300).cuda()
    Gp = torch.empty(400, 3000, dtype=torch.float64, device="cuda")
    _, sinfo = H.geninv_sharded_d(comm, G, 0, Gp)
    assert sinfo.rank == 300
