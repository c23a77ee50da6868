"""GPU parity of the single-precision path (gcm_modify_f32: the panel-order sweep in fp32)
against the fp32 oracle (oracle.modify_a_f32, itself pinned to the fp64 oracle and to brute
force in tests/test_oracle.py), element by element.

Tolerance (reading R21): two fp32 implementations of the same sweep that round in
different orders (the GPU contracts multiply-adds and uses the scaled 2-FMA Apply, R9/R10)
differ by a few units of eps32 per rotation chain; column-scaled element errors <= 256 eps32
(3.1e-5), and V_exit (which carries the downdate amplification) row-scaled <= 1024 eps32.
"""
import numpy as np
import pytest

import oracle
import synth
from gcm_testutil import col_scaled_max, rel_fro, row_scaled_max, upper

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
EPS32 = float(np.finfo(np.float32).eps)


@pytest.fixture(scope="module")
def gcm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1011_1173_b200 as g
    return g


def run32(gcm, Lbuf, Vbuf, sigma):
    L32, V32 = Lbuf.astype(np.float32), Vbuf.astype(np.float32)
    Lo, Vo = L32.copy(), V32.copy()
    _, _, oi = oracle.modify_a_f32(Lo, Vo, sigma)
    L = torch.from_numpy(L32).cuda()
    V = torch.from_numpy(V32).cuda()
    info = gcm.new_info("cuda")
    gcm.modify_f32(L, V, sigma, info=info)
    torch.cuda.synchronize()
    return L.cpu().numpy(), V.cpu().numpy(), gcm.read_info(info)[0], Lo, Vo, (oi.code, oi.col, oi.row)


@pytest.mark.parametrize("sigma", [1, -1])
@pytest.mark.parametrize("n", [1, 63, 64, 65, 200, 1000])
@pytest.mark.parametrize("k", [1, 16, 40])
def test_f32_parity(gcm, n, k, sigma):
    Lbuf, Vbuf, _ = synth.paper_instance(n, k, sigma, seed=3 * n + k, ldl=n + 1, lower_fill=np.nan)
    Lg, Vg, ig, Lo, Vo, io = run32(gcm, Lbuf, Vbuf, sigma)
    assert ig == io == (0, 0, 0)
    assert col_scaled_max(upper(Lg), upper(Lo)) <= 256 * EPS32
    assert rel_fro(upper(Lg), upper(Lo)) <= 256 * EPS32
    assert row_scaled_max(Vg, Vo) <= 1024 * EPS32
    assert np.all(np.isnan(Lg[~np.tril(np.ones(Lg.shape, bool))]))  # lower part never written


def test_f32_failure_report(gcm):
    n, m = 300, 213
    Lbuf, _, _ = synth.paper_instance(n, 1, 1, seed=4)
    V = np.stack([np.zeros(n), 1.01 * upper(Lbuf)[m, :], 3.0 * upper(Lbuf)[5, :]])
    *_, ig, _, _, io = run32(gcm, Lbuf, V, -1)
    assert io == (1, 1, m) and ig == io


def test_f32_paper_error_metric_close_to_f64(gcm):
    """PAPER.md 111/115: the paper's error max|A~ - L~^T L~| of the fp32 GPU result is within a
    small factor of the fp32 oracle's ("the errors are always very similar")."""
    n, k = 800, 16
    for sigma in (1, -1):
        Lbuf, Vbuf, A = synth.paper_instance(n, k, sigma, seed=n + k)
        Lg, _, ig, Lo, _, io = run32(gcm, Lbuf, Vbuf, sigma)
        At = A + sigma * (Vbuf.T @ Vbuf)
        eg = np.abs(At - upper(Lg).astype(np.float64).T @ upper(Lg).astype(np.float64)).max()
        eo = np.abs(At - upper(Lo).astype(np.float64).T @ upper(Lo).astype(np.float64)).max()
        assert ig == io == (0, 0, 0)
        assert eg <= 4 * eo and eo <= 4 * eg
