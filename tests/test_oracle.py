"""Pins for the CPU oracle (oracle/oracle.c) against things other than itself.

Each pin is chosen so that a plausible slip in the oracle (a dropped sigma, the
OLD instead of the NEW L_ij in Apply's second line, Compute before the inner
loop, a wrong index or a transposed operand) fails at least one of them:

* worked examples from SPEC.md (exact values, tests/golden/),
* brute force: LAPACK Cholesky of A + sigma V V^T (numpy), n <= 64,
* an independent closed form for rank 1 (the p = L^{-T} v construction of
  Gill, Golub, Murray & Saunders), which also fixes c, s and V_exit,
* invariants: uniqueness under V -> V Q, update/downdate round trip, column
  norms, coefficient ranges, zero update, and the predicted failure row.
"""
import json
import os

import numpy as np
import pytest
from scipy.linalg import solve_triangular

import oracle
import synth
from gcm_testutil import rel_fro, upper

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _random_factor(rng, n, ldl=None, fill=0.0):
    """A well-conditioned random upper factor in an (n, ldl) buffer."""
    ldl = n if ldl is None else ldl
    B = rng.uniform(size=(n, n))
    A = B.T @ B + np.eye(n)
    G = np.linalg.cholesky(A)
    Lbuf = np.full((n, ldl), fill)
    Lbuf[:, :n] = np.where(np.tril(np.ones((n, n), bool)), G, fill)
    return Lbuf, A


def _target(Lbuf, Vbuf, sigma):
    L = upper(Lbuf)
    return L.T @ L + sigma * Vbuf.T @ Vbuf


# --------------------------------------------------------------------------- examples
def test_compute_worked_examples():
    g = json.load(open(os.path.join(GOLDEN, "spec_worked_examples.json")))
    for ex in g["compute"]:
        c, s, w, bad = oracle.compute(ex["Lii"], ex["Vi"], ex["sigma"])
        assert bad == ex["fail"], ex["cite"]
        if not bad:
            assert c == pytest.approx(ex["c"], rel=2e-16, abs=0), ex["cite"]
            assert s == pytest.approx(ex["s"], rel=2e-16, abs=0), ex["cite"]
            assert w == ex["w"], ex["cite"]


def test_apply_worked_examples():
    g = json.load(open(os.path.join(GOLDEN, "spec_worked_examples.json")))
    for ex in g["apply"]:
        l, v = oracle.apply(ex["c"], ex["s"], ex["Lij"], ex["Vj"], ex["sigma"])
        tol = ex.get("tol", 0.0)
        assert abs(l - ex["Lij_new"]) <= tol, ex["cite"]
        assert abs(v - ex["Vj_new"]) <= tol, ex["cite"]


@pytest.mark.parametrize("fn", [oracle.modify_a, oracle.modify_b])
def test_modify_2x2_worked_example(fn):
    ex = json.load(open(os.path.join(GOLDEN, "spec_worked_examples.json")))["modify_2x2"]
    Lbuf = np.ascontiguousarray(np.array(ex["L"]).T)  # row j = column j of L
    Vbuf = np.array([ex["V"]])
    c, s, info = fn(Lbuf, Vbuf, ex["sigma"])
    assert info.code == 0
    np.testing.assert_allclose(upper(Lbuf), np.array(ex["L_new"]), rtol=0, atol=ex["tol"])
    np.testing.assert_allclose(Vbuf[0], ex["V_exit"], rtol=0, atol=ex["tol"])
    assert Lbuf[0, 1] == 0.0  # strictly lower part untouched


# --------------------------------------------------------------------------- brute force
@pytest.mark.parametrize("n,k", [(1, 1), (2, 3), (5, 1), (17, 4), (48, 2), (64, 1)])
@pytest.mark.parametrize("sigma", [1, -1])
def test_brute_force_refactorisation(rng, n, k, sigma):
    """L~ is THE upper factor of A + sigma V V^T: compare with LAPACK."""
    Lbuf, A = _random_factor(rng, n)
    V = rng.uniform(size=(n, k))
    if sigma < 0:  # make the downdate feasible: factor A + V V^T, downdate by V
        A = A + V @ V.T
        G = np.linalg.cholesky(A)
        Lbuf = np.ascontiguousarray(np.tril(G))
    Vbuf = np.ascontiguousarray(V.T)
    target = A + sigma * V @ V.T
    _, _, info = oracle.modify_a(Lbuf, Vbuf, sigma)
    assert info.code == 0
    Lref = np.linalg.cholesky(target).T
    assert rel_fro(upper(Lbuf), Lref) < 1e-13
    assert np.all(np.diag(upper(Lbuf)) > 0)


def test_chol_upper_matches_lapack(rng):
    n = 40
    B = rng.uniform(size=(n, n))
    A = B.T @ B + np.eye(n)
    L = upper(oracle.chol_upper(A))
    assert rel_fro(L, np.linalg.cholesky(A).T) < 1e-14
    with pytest.raises(np.linalg.LinAlgError):
        oracle.chol_upper(-np.eye(3))


def test_paper_config0_update_then_downdate():
    """BASELINE.json configs[0]: n=64, k=1, update then downdate vs brute force."""
    n, k = 64, 1
    Lbuf, Vbuf, A = synth.paper_instance(n, k, +1)
    L0 = Lbuf.copy()
    V0 = Vbuf.copy()
    _, _, info = oracle.modify_a(Lbuf, Vbuf, +1)
    assert info.code == 0
    target = A + V0.T @ V0
    assert rel_fro(upper(Lbuf), upper(oracle.chol_upper(target))) < 1e-13
    Vbuf[:] = V0
    _, _, info = oracle.modify_a(Lbuf, Vbuf, -1)
    assert info.code == 0
    assert rel_fro(upper(Lbuf), upper(L0)) < 1e-13


# --------------------------------------------------------------------------- closed form
def _ggms_rank1(L, v, sigma):
    """Independent rank-1 construction: p = L^{-T} v, t_j = 1 + sigma sum_{m<=j} p_m^2,
    A + sigma v v^T = L^T (I + sigma p p^T) L and chol(I + sigma p p^T) = W with
    W_jj = sqrt(t_j / t_{j-1}), W_jm = sigma p_j p_m / sqrt(t_j t_{j-1}) (m > j).
    The Givens/hyperbolic sweep's coefficients then are c_j = sqrt(t_j/t_{j-1}),
    s_j = p_j / sqrt(t_{j-1}) and its consumed residual V_j = L_jj p_j / sqrt(t_{j-1})."""
    n = L.shape[0]
    p = solve_triangular(L.T, v, lower=True)
    t = 1.0 + sigma * np.cumsum(p * p)
    tprev = np.concatenate([[1.0], t[:-1]])
    W = np.triu(sigma * np.outer(p, p) / np.sqrt(t * tprev)[:, None], 1)
    W[np.diag_indices(n)] = np.sqrt(t / tprev)
    c = np.sqrt(t / tprev)
    s = p / np.sqrt(tprev)
    vexit = np.diag(L) * p / np.sqrt(tprev)
    return W @ L, c, s, vexit


@pytest.mark.parametrize("sigma", [1, -1])
def test_rank_k_matches_closed_form(sigma):
    """Rank k = k sequential rank-1 modifications (PAPER.md 14, 73, 86); each one
    checked against the closed form, including c, s and the consumed V."""
    n, k = 120, 3
    Lbuf, Vbuf, _ = synth.paper_instance(n, k, sigma, seed=77)
    L = upper(Lbuf)
    V = Vbuf.T.copy()
    c, s, info = oracle.modify_a(Lbuf, Vbuf, sigma)
    assert info.code == 0
    for e in range(k):
        L, ce, se, ve = _ggms_rank1(L, V[:, e], sigma)
        assert rel_fro(c[:, e], ce) < 1e-12
        assert rel_fro(s[:, e], se) < 1e-11
        assert rel_fro(Vbuf[e], ve) < 1e-11
    assert rel_fro(upper(Lbuf), L) < 1e-13


# --------------------------------------------------------------------------- invariants
@pytest.mark.parametrize("sigma", [1, -1])
def test_modify_a_equals_modify_b_bitwise(rng, sigma):
    """Both orderings execute the same scalar DAG (SPEC.md 174, acceptance 3)."""
    for trial in range(40):
        n = int(rng.integers(1, 40))
        k = int(rng.integers(1, 5))
        Lbuf, Vbuf, _ = synth.paper_instance(n, k, sigma, seed=1000 + trial)
        La, Va = Lbuf.copy(), Vbuf.copy()
        Lb, Vb = Lbuf.copy(), Vbuf.copy()
        ca, sa, ia = oracle.modify_a(La, Va, sigma)
        cb, sb, ib = oracle.modify_b(Lb, Vb, sigma)
        assert ia == ib
        assert np.array_equal(La, Lb) and np.array_equal(Va, Vb)
        assert np.array_equal(ca, cb) and np.array_equal(sa, sb)


def test_rank_k_equals_sequential_rank_1_bitwise():
    n, k = 33, 5
    for sigma in (1, -1):
        Lbuf, Vbuf, _ = synth.paper_instance(n, k, sigma, seed=5)
        Lk, Vk = Lbuf.copy(), Vbuf.copy()
        oracle.modify_a(Lk, Vk, sigma)
        L1 = Lbuf.copy()
        for e in range(k):
            v = Vbuf[e:e + 1].copy()
            oracle.modify_a(L1, v, sigma)
            assert np.array_equal(v[0], Vk[e])
        assert np.array_equal(L1, Lk)


def test_zero_update_is_identity():
    Lbuf, _, _ = synth.paper_instance(30, 2, 1, seed=9)
    L0 = Lbuf.copy()
    for sigma in (1, -1):
        c, s, info = oracle.modify_a(Lbuf, np.zeros((2, 30)), sigma)
        assert info.code == 0 and np.array_equal(Lbuf, L0)
        assert np.all(c == 1.0) and np.all(s == 0.0)


def test_column_norm_identity():
    """diag(L~^T L~) = diag(L^T L) + sigma rowsq(V): ||L~_{:,i}||^2 = ||L_{:,i}||^2 + sigma ||V_i||^2."""
    for sigma in (1, -1):
        Lbuf, Vbuf, _ = synth.paper_instance(150, 8, sigma, seed=21)
        before = np.sum(upper(Lbuf) ** 2, axis=0)
        vsq = np.sum(Vbuf ** 2, axis=0)
        oracle.modify_a(Lbuf, Vbuf, sigma)
        after = np.sum(upper(Lbuf) ** 2, axis=0)
        np.testing.assert_allclose(after, before + sigma * vsq, rtol=1e-12)


def test_round_trip_update_downdate():
    n, k = 100, 16
    Lbuf, Vbuf, _ = synth.paper_instance(n, k, 1, seed=3)
    L0, V0 = Lbuf.copy(), Vbuf.copy()
    oracle.modify_a(Lbuf, Vbuf, 1)
    oracle.modify_a(Lbuf, V0.copy(), -1)
    assert rel_fro(upper(Lbuf), upper(L0)) < 1e-12


def test_invariant_under_orthogonal_mixing_of_V(rng):
    """The result depends on V only through V V^T (uniqueness of L~)."""
    n, k = 80, 4
    for sigma in (1, -1):
        Lbuf, Vbuf, _ = synth.paper_instance(n, k, sigma, seed=11)
        Q, _ = np.linalg.qr(rng.normal(size=(k, k)))
        variants = [Vbuf.copy(), Q.T @ Vbuf, Vbuf[::-1].copy(), -Vbuf]
        outs = []
        for Vv in variants:
            L = Lbuf.copy()
            oracle.modify_a(L, np.array(Vv, order="C", copy=True), sigma)
            outs.append(upper(L))
        for o in outs[1:]:
            assert rel_fro(o, outs[0]) < 1e-13


def test_coefficient_ranges():
    """sigma=+1 => c >= 1; sigma=-1 => 0 < c <= 1 (SPEC.md 109-110)."""
    for sigma in (1, -1):
        Lbuf, Vbuf, _ = synth.paper_instance(60, 4, sigma, seed=13)
        c, _, _ = oracle.modify_a(Lbuf, Vbuf, sigma)
        if sigma > 0:
            assert np.all(c >= 1.0)
        else:
            assert np.all((c > 0.0) & (c <= 1.0))


def test_residual_paper_construction():
    """||L~^T L~ - (A + sigma V V^T)||_F / ||A||_F <= 1e-12 (north_star)."""
    n, k = 300, 16
    for sigma in (1, -1):
        Lbuf, Vbuf, A = synth.paper_instance(n, k, sigma, seed=31)
        target = A + sigma * Vbuf.T @ Vbuf
        oracle.modify_a(Lbuf, Vbuf, sigma)
        L = upper(Lbuf)
        assert np.linalg.norm(L.T @ L - target) / np.linalg.norm(A) < 1e-12


def test_indefinite_downdate_detected_at_predicted_row():
    """v = 1.01 * (row m of L): rows < m see v_j = 0 so c=1, s=0 exactly; row m has
    L_mm^2 - 1.0201 L_mm^2 < 0 (SPEC.md 407, acceptance 7)."""
    n, m = 25, 11
    Lbuf, _, _ = synth.paper_instance(n, 1, 1, seed=4)
    v = 1.01 * upper(Lbuf)[m, :]
    for fn in (oracle.modify_a, oracle.modify_b):
        L = Lbuf.copy()
        c, s, info = fn(L, v[None, :].copy(), -1)
        assert (info.code, info.col, info.row) == (1, 0, m)
        assert np.all(c[:m, 0] == 1.0) and np.all(s[:m, 0] == 0.0)
    # second update column fails earlier in row order but later lexicographically
    V = np.stack([v, 5.0 * upper(Lbuf)[3, :]])
    L = Lbuf.copy()
    _, _, info = oracle.modify_a(L, V, -1)
    assert (info.code, info.col, info.row) == (1, 0, m)


def test_non_positive_pivot_reported():
    Lbuf, Vbuf, _ = synth.paper_instance(10, 2, 1, seed=8)
    Lbuf[6, 6] = -1.0
    _, _, info = oracle.modify_a(Lbuf, Vbuf, 1)
    assert (info.code, info.col, info.row) == (2, 0, 6)


def test_literal_printed_order_is_wrong():
    """DESIGN.md R1: running ModifyA exactly as printed (Compute BEFORE the inner
    loop, PAPER.md 25-29) does not give the factor of A + v v^T."""
    n = 40
    Lbuf, Vbuf, A = synth.paper_instance(n, 1, 1, seed=2)
    L = upper(Lbuf).copy()
    v = Vbuf[0].copy()
    c = np.zeros(n)
    s = np.zeros(n)
    for i in range(n):
        c[i], s[i], L[i, i], _ = oracle.compute(L[i, i], v[i], 1)  # printed position
        for j in range(i):
            L[j, i], v[i] = oracle.apply(c[j], s[j], L[j, i], v[i], 1)
    Lref = np.linalg.cholesky(A + np.outer(Vbuf[0], Vbuf[0])).T
    assert rel_fro(L, Lref) > 1e-3
    L2 = Lbuf.copy()
    oracle.modify_a(L2, Vbuf.copy(), 1)
    assert rel_fro(upper(L2), Lref) < 1e-13


def test_strictly_lower_and_padding_untouched():
    n, ldl, k = 20, 27, 3
    Lbuf, Vbuf, _ = synth.paper_instance(n, k, 1, seed=6, ldl=ldl, lower_fill=np.nan)
    mask = ~np.tril(np.ones((n, ldl), bool))  # buffer entries (j, i) with i > j: lower part/pad
    mask[:, :n] = ~np.tril(np.ones((n, n), bool))
    oracle.modify_a(Lbuf, Vbuf, 1)
    assert np.all(np.isnan(Lbuf[mask]))
    assert np.all(np.isfinite(Lbuf[~mask]))


# ------------------------------------------------------------------ single precision oracle
EPS32 = float(np.finfo(np.float32).eps)


def test_f32_worked_example_exact():
    """3-4-5 Compute (SPEC.md 125-128) is exact in fp32: L = [3], V = [4] -> L~ = 5, V_exit = 4."""
    L = np.array([[3.0]], dtype=np.float32)
    V = np.array([[4.0]], dtype=np.float32)
    c, s, info = oracle.modify_a_f32(L, V, 1)
    assert info.code == 0 and L[0, 0] == 5.0 and V[0, 0] == 4.0
    assert c[0, 0] == np.float32(5.0) / np.float32(3.0) and s[0, 0] == np.float32(4.0) / np.float32(3.0)


@pytest.mark.parametrize("n,k,sigma", [(64, 1, 1), (64, 1, -1), (200, 16, 1), (200, 16, -1)])
def test_f32_oracle_matches_f64_oracle_and_brute_force(n, k, sigma):
    """The fp32 oracle is the fp64 one rounded to single precision: column-scaled element error
    <= 64 eps32 against the fp64 oracle (measured <= 9 eps32), and the paper's error metric
    max|A~ - L~^T L~| (PAPER.md 111) <= 16 sqrt(n) eps32 max|A~| (measured <= 2 sqrt(n) eps32)."""
    Lbuf, Vbuf, A = synth.paper_instance(n, k, sigma, seed=n + k)
    L64, V64 = Lbuf.copy(), Vbuf.copy()
    oracle.modify_a(L64, V64, sigma)
    L32, V32 = Lbuf.astype(np.float32), Vbuf.astype(np.float32)
    _, _, info = oracle.modify_a_f32(L32, V32, sigma)
    assert info.code == 0
    U64, U32 = upper(L64), upper(L32).astype(np.float64)
    cn = np.linalg.norm(U64, axis=0)
    assert np.max(np.abs(U32 - U64) / cn[None, :]) <= 64 * EPS32
    At = A + sigma * (Vbuf.T @ Vbuf)
    assert np.abs(At - U32.T @ U32).max() <= 16 * np.sqrt(n) * EPS32 * np.abs(At).max()
    assert np.max(np.abs(V32 - V64)) <= 64 * EPS32 * np.abs(V64).max() * np.sqrt(n)


def test_f32_failure_report_matches_f64():
    n, m = 120, 77
    Lbuf, _, _ = synth.paper_instance(n, 1, 1, seed=4)
    V = np.stack([np.zeros(n), 1.01 * upper(Lbuf)[m, :]])
    _, _, i64 = oracle.modify_a(Lbuf.copy(), V.copy(), -1)
    _, _, i32 = oracle.modify_a_f32(Lbuf.astype(np.float32), V.astype(np.float32), -1)
    assert (i32.code, i32.col, i32.row) == (i64.code, i64.col, i64.row) == (1, 1, m)
