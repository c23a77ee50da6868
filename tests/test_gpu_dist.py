"""GPU parity of gcm_modify_dist (column-sharded path) with one rank: the real NCCL
communicator and broadcasts on one device, vs the oracle.  (Multi-rank runs need
several GPUs; their host-side schedule is pinned by tests/test_dist_host.py.)"""
import numpy as np
import pytest

import oracle
import synth
from gcm_testutil import rel_fro, upper

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gd():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1011_1173_b200 import dist
    comm = dist.Comm(0, 1)
    yield dist, comm
    comm.close()


@pytest.mark.parametrize("sigma", [1, -1])
@pytest.mark.parametrize("n,k,nb", [(100, 3, 64), (300, 16, 128), (257, 70, 64)])
def test_dist_single_rank_parity(gd, n, k, nb, sigma):
    import paper_1011_1173_b200 as gcm
    dist, comm = gd
    Lbuf, Vbuf, _ = synth.paper_instance(n, k, sigma, seed=n + k, ldl=n + 5, lower_fill=np.nan)
    Lo, Vo = Lbuf.copy(), Vbuf.copy()
    _, _, oi = oracle.modify_a(Lo, Vo, sigma)
    L = torch.from_numpy(Lbuf).cuda()
    V = torch.from_numpy(Vbuf).cuda()
    info = gcm.new_info("cuda")
    dist.modify_dist(comm, L, V, n, nb, sigma, info=info)
    torch.cuda.synchronize()
    assert gcm.read_info(info)[0] == (oi.code, oi.col, oi.row)
    Lg = L.cpu().numpy()
    assert rel_fro(upper(Lg), upper(Lo)) <= 1e-11
    assert rel_fro(V.cpu().numpy(), Vo) <= 1e-10
    assert np.all(np.isnan(Lg[~np.tril(np.ones(Lg.shape, bool))]))


def test_dist_rejects_bad_block_width(gd):
    dist, comm = gd
    L = torch.zeros(10, 10, dtype=torch.float64, device="cuda")
    V = torch.zeros(1, 10, dtype=torch.float64, device="cuda")
    with pytest.raises(Exception):
        dist.modify_dist(comm, L, V, 10, 48, 1)
