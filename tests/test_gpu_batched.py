"""GPU parity of gcm_modify_batched (one CTA per factor) against the oracle, factor by factor."""
import numpy as np
import pytest

import oracle
import synth
from gcm_testutil import rel_fro, upper

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL_L = 1e-11
TOL_V = 1e-10


@pytest.fixture(scope="module")
def gcm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1011_1173_b200 as g
    return g


def run_batch(gcm, batch, n, k, sigma, seed0=100):
    Ls, Vs, _ = synth.batched_instances(batch, n, k, sigma, seed=seed0)
    Lo, Vo, infos = Ls.copy(), Vs.copy(), []
    for f in range(batch):
        _, _, inf = oracle.modify_a(Lo[f], Vo[f], sigma)
        infos.append((inf.code, inf.col, inf.row))
    L = torch.from_numpy(Ls).cuda()
    V = torch.from_numpy(Vs).cuda()
    info = gcm.new_info("cuda", batch)
    gcm.modify_batched(L, V, sigma, info=info)
    torch.cuda.synchronize()
    return L.cpu().numpy(), V.cpu().numpy(), gcm.read_info(info), Lo, Vo, infos


@pytest.mark.parametrize("sigma", [1, -1])
@pytest.mark.parametrize("n,k", [(1, 1), (2, 3), (63, 8), (64, 8), (65, 8), (200, 16), (512, 8), (300, 32),
                                 (130, 33), (1030, 4)])
def test_batched_parity(gcm, n, k, sigma):
    batch = 5 if n < 1000 else 2
    Lg, Vg, ig, Lo, Vo, io = run_batch(gcm, batch, n, k, sigma, seed0=7 * n + k)
    assert ig == io
    for f in range(batch):
        assert rel_fro(upper(Lg[f]), upper(Lo[f])) <= TOL_L
        assert rel_fro(Vg[f], Vo[f]) <= TOL_V


def test_batched_per_factor_failure(gcm):
    """One infeasible factor reports its own failure; the others are unaffected."""
    n, k, batch, m = 128, 2, 4, 77
    Ls, Vs, _ = synth.batched_instances(batch, n, k, -1, seed=3)  # downdate-feasible construction
    Vs[2, 0] = 0.0
    Vs[2, 1] = 1.01 * upper(Ls[2])[m, :]  # factor 2, update column 1 fails at row m
    want = []
    for f in range(batch):
        Lf, Vf = Ls[f].copy(), Vs[f].copy()
        _, _, inf = oracle.modify_a(Lf, Vf, -1)
        want.append((inf.code, inf.col, inf.row))
    L = torch.from_numpy(Ls).cuda()
    V = torch.from_numpy(Vs).cuda()
    info = gcm.new_info("cuda", batch)
    gcm.modify_batched(L, V, -1, info=info)
    got = gcm.read_info(info)
    assert got == want
    assert got[2] == (1, 1, m) and got[0] == (0, 0, 0)


def test_batched_matches_single_calls(gcm):
    n, k, batch = 256, 8, 3
    Ls, Vs, _ = synth.batched_instances(batch, n, k, 1, seed=11)
    L = torch.from_numpy(Ls).cuda()
    V = torch.from_numpy(Vs).cuda()
    gcm.modify_batched(L, V, 1)
    for f in range(batch):
        L1 = torch.from_numpy(Ls[f].copy()).cuda()
        V1 = torch.from_numpy(Vs[f].copy()).cuda()
        gcm.modify(L1, V1, 1)
        assert rel_fro(upper(L[f].cpu().numpy()), upper(L1.cpu().numpy())) <= 1e-13
