"""Seeded synthetic instances for the rank-k Cholesky modification benchmarks.

This module is shared by the tests, bench.py and smoke(): it produces inputs
only.  It holds none of the method's arithmetic (no Compute/Apply, no sweep);
the initial factor comes from LAPACK's Cholesky (numpy), exactly as the paper's
experiments obtain it ("compute the Cholesky factor L using the LAPACK
algorithm").

Random numbers: a counter-based SplitMix64.  Draw ``idx`` of stream ``stream``
under ``seed`` is

    z = seed ^ (stream << 48)  +  (idx + 1) * 0x9E3779B97F4A7C15     (mod 2^64)
    u = mix64(z) >> 11, scaled by 2^-53  ->  uniform on [0, 1)

which for ``stream = 0`` is exactly Vigna's sequential SplitMix64 started at
state ``seed`` (tests pin the published first outputs).  Uniform on [0, 1)
rather than [0, 1] is DESIGN.md reading R13.

Buffer conventions (same as the C-ABI): ``Lbuf`` has shape ``(n, ldl)`` with
row ``j`` holding column ``j`` of the upper factor; ``Vbuf`` has shape
``(k, n)`` with row ``e`` holding update vector ``e``.
"""
from __future__ import annotations

import numpy as np

GOLDEN_RATIO = np.uint64(0x9E3779B97F4A7C15)
SEED_ROOT = 10111173  # seed root of every bench/test instance

# stream ids (upper 16 bits of the counter word)
S_B, S_V, S_LDIAG, S_LOFF, S_VDIRECT = 1, 2, 3, 4, 5


def mix64(z: np.ndarray) -> np.ndarray:
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def raw64(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    base = np.uint64((seed ^ (stream << 48)) & 0xFFFFFFFFFFFFFFFF)
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return mix64(base + (idx + np.uint64(1)) * GOLDEN_RATIO)


def uniform(seed: int, stream: int, count: int, offset: int = 0) -> np.ndarray:
    """``count`` draws on [0, 1) starting at counter ``offset``."""
    idx = np.arange(offset, offset + count, dtype=np.uint64)
    return (raw64(seed, stream, idx) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def _colmajor(seed: int, stream: int, rows: int, cols: int) -> np.ndarray:
    """rows x cols matrix whose column-major element t is draw t."""
    return uniform(seed, stream, rows * cols).reshape(cols, rows).T


def paper_instance(n: int, k: int, sigma: int, seed: int = SEED_ROOT, ldl: int | None = None,
                   lower_fill: float = 0.0):
    """The paper's experiment.

    B (n x n) and V (n x k) i.i.d. U[0,1); update: A = B^T B + I; downdate:
    A = B^T B + I + V V^T, to be downdated by V.  Returns ``(Lbuf, Vbuf, A)``
    where ``A`` is the matrix ``Lbuf`` factors and the expected result is
    ``A + sigma V V^T``.  ``lower_fill`` is written into the strictly lower
    part of every column and into the padding rows ``n..ldl-1`` (tests use NaN
    to prove they are never read or written).
    """
    ldl = n if ldl is None else ldl
    B = _colmajor(seed, S_B, n, n)
    V = _colmajor(seed, S_V, n, k)
    A = B.T @ B + np.eye(n)
    if sigma < 0:
        A = A + V @ V.T
    G = np.linalg.cholesky(A)  # A = G G^T, G lower  ->  upper factor L = G^T
    Lbuf = np.full((n, ldl), lower_fill)
    # row j of Lbuf = column j of L = row j of G restricted to i <= j
    Lbuf[:, :n] = np.where(np.tril(np.ones((n, n), dtype=bool)), G, lower_fill)
    Vbuf = np.ascontiguousarray(V.T)
    return Lbuf, Vbuf, A


def direct_instance(n: int, k: int, seed: int = SEED_ROOT, ldl: int | None = None,
                    lower_fill: float = 0.0):
    """Large-n instance that avoids the O(n^3) construction (R18).

    L_ii = 1 + U, L_ij = (2U - 1)/sqrt(n) for i < j, V = U/sqrt(n).
    Returns ``(Lbuf, Vbuf)``.
    """
    ldl = n if ldl is None else ldl
    scale = 1.0 / np.sqrt(n)
    Lbuf = np.full((n, ldl), lower_fill)
    for j in range(n):  # column j of L (row j of Lbuf); counters are column-major
        u = uniform(seed, S_LOFF, j, offset=j * n)
        Lbuf[j, :j] = (2.0 * u - 1.0) * scale
        Lbuf[j, j] = 1.0 + uniform(seed, S_LDIAG, 1, offset=j)[0]
    Vbuf = np.ascontiguousarray(_colmajor(seed, S_VDIRECT, n, k).T * scale)
    return Lbuf, Vbuf


def batched_instances(batch: int, n: int, k: int, sigma: int, seed: int = SEED_ROOT, first: int = 0):
    """``batch`` independent paper instances (factor ``b`` uses seed ``seed + first + b``).

    Returns ``(Lbufs, Vbufs, As)`` with shapes (batch, n, n), (batch, k, n), (batch, n, n).
    """
    Ls, Vs, As = [], [], []
    for b in range(batch):
        L, V, A = paper_instance(n, k, sigma, seed=seed + first + b)
        Ls.append(L)
        Vs.append(V)
        As.append(A)
    return np.stack(Ls), np.stack(Vs), np.stack(As)
