import os

import numpy as np

import synth
from gcm_testutil import upper

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_splitmix64_matches_published_sequence():
    want = [int(l, 16) for l in open(os.path.join(GOLDEN, "splitmix64_state0.txt")) if l.startswith("0x")]
    got = synth.raw64(0, 0, np.arange(len(want)))
    assert [int(x) for x in got] == want


def test_uniform_range_and_determinism():
    u = synth.uniform(synth.SEED_ROOT, synth.S_B, 100000)
    assert u.min() >= 0.0 and u.max() < 1.0
    assert abs(u.mean() - 0.5) < 5e-3
    assert np.array_equal(u, synth.uniform(synth.SEED_ROOT, synth.S_B, 100000))
    # counter-based: any window equals the same slice of a longer draw
    assert np.array_equal(synth.uniform(7, 2, 10, offset=500), synth.uniform(7, 2, 600)[500:510])
    # streams differ
    assert not np.array_equal(u[:10], synth.uniform(synth.SEED_ROOT, synth.S_V, 10))


def test_paper_instance_construction():
    """PAPER.md 111: downdate instance's A - V V^T is the update instance's A."""
    n, k = 50, 3
    Lu, Vu, Au = synth.paper_instance(n, k, 1)
    Ld, Vd, Ad = synth.paper_instance(n, k, -1)
    assert np.array_equal(Vu, Vd)
    np.testing.assert_allclose(Ad - Vd.T @ Vd, Au, rtol=1e-13, atol=1e-10)
    for L, A in ((Lu, Au), (Ld, Ad)):
        U = upper(L)
        assert np.all(np.diag(U) > 0)
        np.testing.assert_allclose(U.T @ U, A, rtol=1e-12, atol=1e-9)


def test_direct_instance_shape():
    L, V = synth.direct_instance(64, 4)
    U = upper(L)
    assert np.all(np.diag(U) >= 1.0) and np.all(np.diag(U) < 2.0)
    assert np.all(np.abs(U - np.diag(np.diag(U))) <= 1 / 8)
    assert V.shape == (4, 64) and V.min() >= 0 and V.max() < 1 / 8
