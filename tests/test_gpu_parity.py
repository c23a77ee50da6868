"""GPU parity: the CUDA path through the C-ABI vs the CPU oracle, element by
element on the same seeded inputs.

Tolerances: L~ relative Frobenius <= 1e-11 (north_star);
V_exit relative Frobenius <= 1e-10 (V_exit is the rotated residual, a secondary
output whose error carries the downdate amplification).  Beside the
Frobenius bounds every element is checked: |L~_gpu - L~_cpu|_ij <= 1e-12 ||L~_cpu(:, j)||
(column-scaled) and |V_gpu - V_cpu|_ej <= 1e-11 max_j |V_cpu(e, j)| (row-scaled), so a
single wrong tile cannot pass under a large norm.
"""
import numpy as np
import pytest

import oracle
import synth
from gcm_testutil import col_scaled_max, rel_fro, row_scaled_max, upper

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL_L = 1e-11
TOL_V = 1e-10
TOL_L_ELEM = 1e-12  # column-scaled, per element
TOL_V_ELEM = 1e-11  # row-scaled, per element


@pytest.fixture(scope="module")
def gcm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1011_1173_b200 as g
    return g


def run_both(gcm, n, k, sigma, ldl=None, seed=1, algo="auto", instance="paper"):
    ldl = n if ldl is None else ldl
    if instance == "paper":
        Lbuf, Vbuf, _ = synth.paper_instance(n, k, sigma, seed=seed, ldl=ldl, lower_fill=np.nan)
    else:
        Lbuf, Vbuf = synth.direct_instance(n, k, seed=seed, ldl=ldl, lower_fill=np.nan)
    Lo, Vo = Lbuf.copy(), Vbuf.copy()
    _, _, oinfo = oracle.modify_a(Lo, Vo, sigma)
    dev = torch.device("cuda")
    L = torch.from_numpy(Lbuf).to(dev)
    V = torch.from_numpy(Vbuf).to(dev)
    info = gcm.new_info(dev)
    gcm.modify(L, V, sigma, info=info, algo=algo)
    torch.cuda.synchronize()
    return L.cpu().numpy(), V.cpu().numpy(), gcm.read_info(info)[0], Lo, Vo, oinfo


def check(Lg, Vg, ginfo, Lo, Vo, oinfo, n):
    assert ginfo == (oinfo.code, oinfo.col, oinfo.row)
    assert rel_fro(upper(Lg), upper(Lo)) <= TOL_L
    assert col_scaled_max(upper(Lg), upper(Lo)) <= TOL_L_ELEM
    if Vo.size:
        assert rel_fro(Vg, Vo) <= TOL_V
        assert row_scaled_max(Vg, Vo) <= TOL_V_ELEM
    # strictly lower part and padding rows are never written (NaN sentinel)
    bad = ~np.tril(np.ones(Lg.shape, bool))
    assert np.all(np.isnan(Lg[bad]))
    assert np.all(np.isfinite(upper(Lg)))


SIZES = [1, 2, 3, 31, 63, 64, 65, 127, 128, 129, 200]
RANKS = [1, 2, 3, 8, 15, 16, 17, 33, 64, 65]


ALGOS = ["sweep", "blocked", "panel", "auto"]


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("sigma", [1, -1])
@pytest.mark.parametrize("n", SIZES)
def test_parity_grid_sizes(gcm, n, sigma, algo):
    for k in (1, 4, 16):
        check(*run_both(gcm, n, k, sigma, seed=n * 7 + k, algo=algo), n)


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("sigma", [1, -1])
@pytest.mark.parametrize("k", RANKS)
def test_parity_grid_ranks(gcm, k, sigma, algo):
    check(*run_both(gcm, 150, k, sigma, seed=100 + k, algo=algo), 150)


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("ldl_pad", [3, 64])
def test_parity_leading_dimension(gcm, ldl_pad, algo):
    for sigma in (1, -1):
        n = 190
        check(*run_both(gcm, n, 7, sigma, ldl=n + ldl_pad, seed=ldl_pad, algo=algo), n)


def test_parity_direct_instance(gcm):
    """Large-n construction (R18): update, then downdate the result by the same V."""
    n, k = 700, 16
    Lbuf, Vbuf = synth.direct_instance(n, k, seed=3, lower_fill=np.nan)
    dev = torch.device("cuda")
    L = torch.from_numpy(Lbuf).to(dev)
    Lo = Lbuf.copy()
    for sigma in (1, -1):
        Vo = Vbuf.copy()
        _, _, oinfo = oracle.modify_a(Lo, Vo, sigma)
        V = torch.from_numpy(Vbuf).to(dev)
        info = gcm.new_info(dev)
        gcm.modify(L, V, sigma, info=info)
        torch.cuda.synchronize()
        check(L.cpu().numpy(), V.cpu().numpy(), gcm.read_info(info)[0], Lo, Vo, oinfo, n)
        # keep both sides on identical inputs for the downdate
        L = torch.from_numpy(Lo.copy()).to(dev)


@pytest.mark.parametrize("algo", ALGOS)
def test_parity_moderate(gcm, algo):
    for sigma in (1, -1):
        check(*run_both(gcm, 1000, 16, sigma, seed=12, algo=algo), 1000)
        check(*run_both(gcm, 2113, 32, sigma, seed=13, algo=algo), 2113)


def test_zero_update_identity(gcm):
    n, k = 100, 4
    Lbuf, _, _ = synth.paper_instance(n, k, 1, seed=2)
    L = torch.from_numpy(Lbuf).cuda()
    V = torch.zeros(k, n, dtype=torch.float64, device="cuda")
    gcm.modify(L, V, 1)
    torch.cuda.synchronize()
    assert rel_fro(upper(L.cpu().numpy()), upper(Lbuf)) < 1e-15


def test_empty_is_noop(gcm):
    L = torch.ones(5, 5, dtype=torch.float64, device="cuda")
    V = torch.ones(0, 5, dtype=torch.float64, device="cuda")
    info = gcm.new_info("cuda")
    gcm.modify(L, V, 1, info=info)
    assert gcm.read_info(info)[0] == (0, 0, 0)
    assert torch.all(L == 1)
    L0 = torch.ones(0, 1, dtype=torch.float64, device="cuda")
    gcm.modify(L0, torch.ones(3, 0, dtype=torch.float64, device="cuda"), -1)


@pytest.mark.parametrize("algo", ALGOS)
def test_indefinite_downdate_reported(gcm, algo):
    n, m = 150, 97
    Lbuf, _, _ = synth.paper_instance(n, 1, 1, seed=4)
    v = 1.01 * upper(Lbuf)[m, :]
    V = np.stack([np.zeros(n), v, 3.0 * upper(Lbuf)[5, :]])  # second column fails at m
    L = torch.from_numpy(Lbuf).cuda()
    Vt = torch.from_numpy(V).cuda()
    info = gcm.new_info("cuda")
    gcm.modify(L, Vt, -1, info=info, algo=algo)
    Lo, Vo = Lbuf.copy(), V.copy()
    _, _, oi = oracle.modify_a(Lo, Vo, -1)
    assert (oi.code, oi.col, oi.row) == (1, 1, m)
    assert gcm.read_info(info)[0] == (1, 1, m)


@pytest.mark.parametrize("algo", ALGOS)
def test_non_positive_pivot_reported(gcm, algo):
    Lbuf, Vbuf, _ = synth.paper_instance(80, 2, 1, seed=8)
    Lbuf[70, 70] = 0.0
    info = gcm.new_info("cuda")
    gcm.modify(torch.from_numpy(Lbuf).cuda(), torch.from_numpy(Vbuf).cuda(), 1, info=info, algo=algo)
    assert gcm.read_info(info)[0] == (2, 0, 70)


def test_repeated_calls_and_streams(gcm):
    """Workspace reuse across calls and streams; results independent of the stream."""
    n, k = 300, 8
    Lbuf, Vbuf, _ = synth.paper_instance(n, k, 1, seed=10)
    outs = []
    for s in (torch.cuda.current_stream(), torch.cuda.Stream(), torch.cuda.Stream()):
        with torch.cuda.stream(s):  # clones and calls ordered on the same stream
            L = torch.from_numpy(Lbuf).cuda()
            V = torch.from_numpy(Vbuf).cuda()
            for _ in range(3):
                gcm.modify(L, V.clone(), 1)
        torch.cuda.synchronize()
        outs.append(L.cpu().numpy())
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


@pytest.mark.parametrize("n,k", [(257, 9), (600, 16), (600, 40)])  # 1 and 3 256-column copy blocks, ragged; k=40: two passes
def test_host_entry_point(gcm, n, k):
    for sigma in (1, -1):
        Lbuf, Vbuf, _ = synth.paper_instance(n, k, sigma, seed=14, ldl=n + 1)
        Lo, Vo = Lbuf.copy(), Vbuf.copy()
        oracle.modify_a(Lo, Vo, sigma)
        lower = ~np.tril(np.ones(Lbuf.shape, bool))  # strictly lower part + padding row
        Lin = Lbuf.copy()
        Lin[lower] = np.nan  # never read: a NaN there must not reach the factor
        Lh = torch.from_numpy(Lin).pin_memory()
        Vh = torch.from_numpy(Vbuf.copy()).pin_memory()
        assert gcm.modify_host(Lh, Vh, sigma) == (0, 0, 0)
        assert rel_fro(upper(Lh.numpy()), upper(Lo)) <= TOL_L
        assert rel_fro(Vh.numpy(), Vo) <= TOL_V
        assert np.isnan(Lh.numpy()[lower]).all()  # left as the caller had it


@pytest.mark.slow
@pytest.mark.parametrize("k", [1, 4, 64])
def test_parity_k_sweep_config(gcm, k):
    """BASELINE configs[2]: n=5000, k in {1, 4, 64} (k=64 = two rank-32 passes), update and
    downdate, full-size element-wise parity in the launch configuration bench.py times."""
    for sigma in (1, -1):
        check(*run_both(gcm, 5000, k, sigma, seed=synth.SEED_ROOT + k), 5000)


@pytest.mark.slow
def test_parity_headline_config(gcm):
    """BASELINE configs[1]: n=5000, k=16, update and downdate, full-size element-wise parity."""
    for sigma in (1, -1):
        check(*run_both(gcm, 5000, 16, sigma, seed=synth.SEED_ROOT), 5000)


@pytest.mark.parametrize("budget,n,k", [(1 << 18, 700, 16), (1 << 17, 1000, 5), (1 << 15, 1000, 5), (1 << 21, 1300, 32)])  # CI = 2, 4, 16, 2
@pytest.mark.parametrize("sigma", [1, -1])
def test_parity_checkpoint_interval(gcm, monkeypatch, budget, n, k, sigma):
    """A small checkpoint budget forces CI > 1 (the very-large-n Apply walk, bapply_kernel),
    which the default budget (>= 2 GiB, up to a quarter of free memory) never reaches at
    these sizes."""
    monkeypatch.setenv("GCM_CHK_BUDGET", str(budget))
    check(*run_both(gcm, n, k, sigma, seed=n + k, algo="blocked"), n)


@pytest.mark.slow
@pytest.mark.parametrize("n,k", [(24000, 16), (24000, 32)])
def test_large_n_properties(gcm, n, k):
    """Sizes where each strip owner holds several strips (n/32/139 ~ 5, all kept in shared
    memory by default; the spill path is driven by test_gpu_edge.py's GCM_HELP_OWN_CAP cases)
    and the oracle is slow element-wise: full-size pins that hold at any size (SURVEY 8(c) P4,
    P5) -- the column-norm identity ||L~_{:,c}||^2 = ||L_{:,c}||^2 + sigma ||V_{c,:}||^2 on
    every column, and Freivalds' check L~^T L~ x = L^T L x + sigma V V^T x -- for an update
    and the downdate back (direct-L instance, R18, drawn on the device)."""
    dev = torch.device("cuda")
    g = torch.Generator(device=dev)
    g.manual_seed(synth.SEED_ROOT + n + k)
    Lt = torch.empty((n, n), dtype=torch.float64, device=dev)  # row c = column c of L
    Lt.uniform_(-1.0 / n ** 0.5, 1.0 / n ** 0.5, generator=g)
    Lt.diagonal().uniform_(1.0, 2.0, generator=g)
    V0 = torch.rand((k, n), dtype=torch.float64, device=dev, generator=g) / n ** 0.5
    x = torch.rand((n, 2), dtype=torch.float64, device=dev, generator=g)
    for sigma in (1, -1):
        low = torch.tril(Lt)  # L^T (lower), the upper factor's entries only
        col2 = (low ** 2).sum(1)
        ax = low @ (low.T @ x)
        del low
        V = V0.clone()
        gcm.modify(Lt, V, sigma)
        torch.cuda.synchronize()
        low = torch.tril(Lt)
        vn = (V0 ** 2).sum(0)
        rel = ((low ** 2).sum(1) - col2 - sigma * vn).abs() / (low ** 2).sum(1)
        assert rel.max().item() <= 1e-11, f"column-norm identity {rel.max().item():.2e} (sigma={sigma})"
        want = ax + sigma * (V0.T @ (V0 @ x))
        got = low @ (low.T @ x)
        fr = ((got - want).norm() / want.norm()).item()
        assert fr <= 1e-11, f"Freivalds {fr:.2e} (sigma={sigma})"
        del low
