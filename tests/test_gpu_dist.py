"""GPU parity of the column-sharded path (panel.cu) against the oracle.

* gcm_modify_dist_virtual: R = 1..4 ranks whose block-cyclic shards all live on this GPU,
  run by one call on one stream -- the multi-rank logic of gcm_modify_dist (ownership of
  column blocks, the owner's P rows and every rank's coefficient panels written straight
  into the other ranks' buffers, per-rank residual updates / diagonal sweeps / Apply,
  the global failure report), each rank on its own buffers, element-wise vs the oracle;
* gcm_modify_dist with a real one-rank NCCL communicator (the NCCL exchange calls);
* GCM_ALGO_PANEL (the one-rank instance) is also in tests/test_gpu_parity.py's grid.
(The guide forbids standing in for more GPUs with ranks whose kernels wait on each other
on one GPU: the virtual ranks never wait -- their kernels are ordered by one stream.)
"""
import numpy as np
import pytest

import oracle
import synth
from gcm_testutil import col_scaled_max, rel_fro, row_scaled_max, upper

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gd():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1011_1173_b200 as gcm
    from paper_1011_1173_b200 import dist
    return gcm, dist


def run_virtual(gcm, dist, n, k, nb, R, sigma, seed, Lbuf=None, Vbuf=None, ldl_pad=3):
    if Lbuf is None:
        Lbuf, Vbuf, _ = synth.paper_instance(n, k, sigma, seed=seed, ldl=n + ldl_pad, lower_fill=np.nan)
    Lo, Vo = Lbuf.copy(), Vbuf.copy()
    _, _, oi = oracle.modify_a(Lo, Vo, sigma)
    Lf = torch.from_numpy(Lbuf).cuda()
    Vf = torch.from_numpy(Vbuf).cuda()
    shards = dist.shard(Lf, Vf, nb, R)
    info = gcm.new_info("cuda")
    dist.modify_dist_virtual([s[0] for s in shards], [s[1] for s in shards], n, nb, sigma, info=info)
    torch.cuda.synchronize()
    Lg = np.full_like(Lbuf, np.nan)
    Vg = np.zeros_like(Vbuf)
    for Ls, Vs, g in shards:
        Lg[g] = Ls.cpu().numpy()
        Vg[:, g] = Vs.cpu().numpy()
    return Lg, Vg, gcm.read_info(info)[0], Lo, Vo, (oi.code, oi.col, oi.row)


CASES = [(65, 8, 64), (130, 1, 128), (300, 5, 64), (1000, 16, 256), (700, 40, 256), (2113, 32, 512), (1030, 4, 512)]


@pytest.mark.parametrize("R", [1, 2, 3, 4])
@pytest.mark.parametrize("n,k,nb", CASES)
@pytest.mark.parametrize("sigma", [1, -1])
def test_virtual_ranks_parity(gd, R, n, k, nb, sigma):
    gcm, dist = gd
    Lg, Vg, ig, Lo, Vo, io = run_virtual(gcm, dist, n, k, nb, R, sigma, seed=n + 7 * k + R)
    assert ig == io == (0, 0, 0)
    assert rel_fro(upper(Lg), upper(Lo)) <= 1e-11
    assert col_scaled_max(upper(Lg), upper(Lo)) <= 1e-12
    assert row_scaled_max(Vg, Vo) <= 1e-11
    bad = ~np.tril(np.ones(Lg.shape, bool))  # strictly lower part + padding rows: never written
    assert np.all(np.isnan(Lg[bad]))


@pytest.mark.parametrize("R", [2, 3])
def test_virtual_ranks_failure_report(gd, R):
    """An indefinite downdate in column e = 1 at row m (owned by some rank): every rank's
    report reduces to the oracle's lexicographic first failure."""
    gcm, dist = gd
    n, m = 600, 413
    Lbuf, _, _ = synth.paper_instance(n, 1, 1, seed=4, ldl=n + 1, lower_fill=np.nan)
    V = np.stack([np.zeros(n), 1.01 * upper(Lbuf)[m, :], 3.0 * upper(Lbuf)[5, :]])
    *_, ig, _, _, io = run_virtual(gcm, dist, n, 3, 256, R, -1, 0, Lbuf=Lbuf, Vbuf=V)
    assert io == (1, 1, m)
    assert ig == io


@pytest.mark.parametrize("sigma", [1, -1])
def test_panel_algo_moderate(gd, sigma):
    """GCM_ALGO_PANEL through gcm_modify_ex at sizes spanning many column blocks."""
    gcm, _ = gd
    for n, k in [(3000, 16), (2500, 33)]:
        Lbuf, Vbuf, _ = synth.paper_instance(n, k, sigma, seed=n + k, lower_fill=np.nan)
        Lo, Vo = Lbuf.copy(), Vbuf.copy()
        oracle.modify_a(Lo, Vo, sigma)
        L, V = torch.from_numpy(Lbuf).cuda(), torch.from_numpy(Vbuf).cuda()
        gcm.modify(L, V, sigma, algo="panel")
        torch.cuda.synchronize()
        assert rel_fro(upper(L.cpu().numpy()), upper(Lo)) <= 1e-11
        assert col_scaled_max(upper(L.cpu().numpy()), upper(Lo)) <= 1e-12
        assert row_scaled_max(V.cpu().numpy(), Vo) <= 1e-11


@pytest.fixture(scope="module")
def comm1(gd):
    _, dist = gd
    c = dist.Comm(0, 1)
    yield c
    c.close()


@pytest.mark.parametrize("sigma", [1, -1])
@pytest.mark.parametrize("n,k,nb", [(100, 3, 64), (300, 16, 128), (257, 70, 64), (1100, 8, 512)])
def test_dist_single_rank_parity(gd, comm1, n, k, nb, sigma):
    """gcm_modify_dist with a real (one-rank) NCCL communicator: the NCCL exchange path."""
    gcm, dist = gd
    Lbuf, Vbuf, _ = synth.paper_instance(n, k, sigma, seed=n + k, ldl=n + 5, lower_fill=np.nan)
    Lo, Vo = Lbuf.copy(), Vbuf.copy()
    _, _, oi = oracle.modify_a(Lo, Vo, sigma)
    L = torch.from_numpy(Lbuf).cuda()
    V = torch.from_numpy(Vbuf).cuda()
    info = gcm.new_info("cuda")
    dist.modify_dist(comm1, L, V, n, nb, sigma, info=info)
    torch.cuda.synchronize()
    assert gcm.read_info(info)[0] == (oi.code, oi.col, oi.row)
    Lg = L.cpu().numpy()
    assert rel_fro(upper(Lg), upper(Lo)) <= 1e-11
    assert col_scaled_max(upper(Lg), upper(Lo)) <= 1e-12
    assert rel_fro(V.cpu().numpy(), Vo) <= 1e-10
    assert np.all(np.isnan(Lg[~np.tril(np.ones(Lg.shape, bool))]))


def test_dist_rejects_bad_block_width(gd, comm1):
    _, dist = gd
    L = torch.zeros(10, 10, dtype=torch.float64, device="cuda")
    V = torch.zeros(1, 10, dtype=torch.float64, device="cuda")
    with pytest.raises(Exception):
        dist.modify_dist(comm1, L, V, 10, 48, 1)


@pytest.fixture(scope="module")
def comm1_peer(gd):
    _, dist = gd
    c = dist.Comm(0, 1, peer=True)
    yield c
    c.close()


@pytest.mark.parametrize("sigma", [1, -1])
@pytest.mark.parametrize("n,k,nb", [(300, 16, 128), (1100, 40, 512)])
def test_dist_single_rank_peer_mode(gd, comm1_peer, n, k, nb, sigma):
    """gcm_comm_set_peer: the IPC-window exchange (owner stores + system-scope flags, panel
    counters) with one rank, twice in a row (the window and its counters are reused)."""
    gcm, dist = gd
    for rep in range(2):
        Lbuf, Vbuf, _ = synth.paper_instance(n, k, sigma, seed=n + k + rep, ldl=n + 5, lower_fill=np.nan)
        Lo, Vo = Lbuf.copy(), Vbuf.copy()
        _, _, oi = oracle.modify_a(Lo, Vo, sigma)
        L = torch.from_numpy(Lbuf).cuda()
        V = torch.from_numpy(Vbuf).cuda()
        info = gcm.new_info("cuda")
        dist.modify_dist(comm1_peer, L, V, n, nb, sigma, info=info)
        torch.cuda.synchronize()
        assert gcm.read_info(info)[0] == (oi.code, oi.col, oi.row)
        assert col_scaled_max(upper(L.cpu().numpy()), upper(Lo)) <= 1e-12
        assert row_scaled_max(V.cpu().numpy(), Vo) <= 1e-11


@pytest.mark.parametrize("grid", [2, 4])
@pytest.mark.parametrize("n,k", [(3000, 16), (2200, 33), (1500, 5)])
def test_pchain_few_helpers_spill(gd, grid, n, k, monkeypatch):
    """The one-rank persistent chain (GCM_ALGO_PANEL) with its grid capped at 2 / 4 CTAs: one or
    three helpers own every strip, so most residuals live in the spill slots and round-trip
    through res[] between tiles (the default grid only does that at n ~ 1e5)."""
    gcm, _ = gd
    monkeypatch.setenv("GCM_PCHAIN_GRID", str(grid))
    for sigma in (1, -1):
        Lbuf, Vbuf, _ = synth.paper_instance(n, k, sigma, seed=n + k + grid, lower_fill=np.nan)
        Lo, Vo = Lbuf.copy(), Vbuf.copy()
        oracle.modify_a(Lo, Vo, sigma)
        L, V = torch.from_numpy(Lbuf).cuda(), torch.from_numpy(Vbuf).cuda()
        gcm.modify(L, V, sigma, algo="panel")
        torch.cuda.synchronize()
        assert col_scaled_max(upper(L.cpu().numpy()), upper(Lo)) <= 1e-12
        assert row_scaled_max(V.cpu().numpy(), Vo) <= 1e-11


@pytest.mark.parametrize("n,k", [(3000, 16), (2500, 33)])
def test_panel_launch_chain_one_rank(gd, n, k, monkeypatch):
    """GCM_PCHAIN=0: the one-rank panel path through the per-solve-block launches (dsolve,
    lookahead and rest pupdate on the aux stream) -- what AUTO runs at n ~ 1e5."""
    gcm, _ = gd
    monkeypatch.setenv("GCM_PCHAIN", "0")
    for sigma in (1, -1):
        Lbuf, Vbuf, _ = synth.paper_instance(n, k, sigma, seed=n + 3 * k, lower_fill=np.nan)
        Lo, Vo = Lbuf.copy(), Vbuf.copy()
        oracle.modify_a(Lo, Vo, sigma)
        L, V = torch.from_numpy(Lbuf).cuda(), torch.from_numpy(Vbuf).cuda()
        gcm.modify(L, V, sigma, algo="panel")
        torch.cuda.synchronize()
        assert col_scaled_max(upper(L.cpu().numpy()), upper(Lo)) <= 1e-12
        assert row_scaled_max(V.cpu().numpy(), Vo) <= 1e-11


@pytest.mark.parametrize("pchain", ["1", "0"])
def test_panel_two_streams(gd, pchain, monkeypatch):
    """Two GCM_ALGO_PANEL calls in flight at once on two CUDA streams: each call has its own
    workspace and auxiliary stream/events (keyed by device and call stream), so neither waits
    on or overwrites the other's hand-offs."""
    gcm, _ = gd
    monkeypatch.setenv("GCM_PCHAIN", pchain)
    cases = []
    for i, (n, k) in enumerate([(1800, 16), (1500, 9)]):
        Lbuf, Vbuf, _ = synth.paper_instance(n, k, 1, seed=100 + i, lower_fill=np.nan)
        Lo, Vo = Lbuf.copy(), Vbuf.copy()
        oracle.modify_a(Lo, Vo, 1)
        cases.append((torch.from_numpy(Lbuf).cuda(), torch.from_numpy(Vbuf).cuda(), Lo, Vo))
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for (L, V, _, _), st in zip(cases, streams):
        with torch.cuda.stream(st):
            gcm.modify(L, V, 1, algo="panel", stream=st)
    torch.cuda.synchronize()
    for L, V, Lo, Vo in cases:
        assert col_scaled_max(upper(L.cpu().numpy()), upper(Lo)) <= 1e-12
        assert row_scaled_max(V.cpu().numpy(), Vo) <= 1e-11
