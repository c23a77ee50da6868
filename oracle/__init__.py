"""CPU oracle for the rank-k Cholesky modification of arXiv 1011.1173.

TEST INFRASTRUCTURE ONLY: tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` leg may import this package.  The
product path (``paper_1011_1173_b200``) never imports it and shares no code with
it; see ``oracle/oracle.c`` for the algorithm, the passages it follows
 and the readings it takes (R1-R7).

Buffer conventions (the same ones the product's C-ABI uses, restated here
independently):

* ``Lbuf``: float64 array of shape ``(n, ldl)``, C-contiguous; row ``j`` of
  ``Lbuf`` holds column ``j`` of the upper-triangular factor, so the factor
  entry ``L[i, j]`` (``i <= j``) is ``Lbuf[j, i]``.  Only entries with
  ``i <= j`` are read or written.
* ``Vbuf``: float64 array of shape ``(k, n)``, C-contiguous; row ``e`` is
  update vector ``e`` (the ``e``-th column of the paper's ``V``).

Parity status: every function here is pinned by ``tests/test_oracle.py``
(worked examples from SPEC.md, brute-force re-factorisation, closed forms,
invariants); nothing is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

GCC_FLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (plain gcc, no CUDA)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *GCC_FLAGS, _SRC, "-o", _LIB, "-lm"])
    return _LIB


class _Info(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("col", ctypes.c_int32), ("row", ctypes.c_int64)]


@dataclass
class Info:
    code: int  # 0 ok, 1 indefinite downdate, 2 non-positive pivot on entry
    col: int   # update column e of the first failure
    row: int   # row i of the first failure


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        dp = ctypes.POINTER(ctypes.c_double)
        i64 = ctypes.c_int64
        for name in ("gcmo_modify_a", "gcmo_modify_b"):
            f = getattr(lib, name)
            f.argtypes = [dp, i64, i64, dp, i64, ctypes.c_int, dp, dp, ctypes.POINTER(_Info)]
            f.restype = ctypes.c_int
        fp = ctypes.POINTER(ctypes.c_float)
        lib.gcmo_modify_a_f32.argtypes = [fp, i64, i64, fp, i64, ctypes.c_int, fp, fp, ctypes.POINTER(_Info)]
        lib.gcmo_modify_a_f32.restype = ctypes.c_int
        lib.gcmo_chol_upper.argtypes = [dp, i64, i64, dp, i64]
        lib.gcmo_chol_upper.restype = i64
        lib.gcmo_compute.argtypes = [dp, dp, dp, ctypes.c_double, ctypes.c_int]
        lib.gcmo_compute.restype = ctypes.c_int
        lib.gcmo_apply.argtypes = [ctypes.c_double, ctypes.c_double, dp, dp, ctypes.c_int]
        lib.gcmo_apply.restype = None
        _lib = lib
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _check(Lbuf: np.ndarray, Vbuf: np.ndarray):
    if Lbuf.dtype != np.float64 or Vbuf.dtype != np.float64:
        raise TypeError("oracle works in float64 only")
    if not (Lbuf.flags.c_contiguous and Vbuf.flags.c_contiguous):
        raise ValueError("Lbuf and Vbuf must be C-contiguous")
    n, ldl = Lbuf.shape
    if ldl < max(1, n):
        raise ValueError("ldl < n")
    if Vbuf.ndim != 2 or (Vbuf.shape[1] != n and Vbuf.size):
        raise ValueError("Vbuf must have shape (k, n)")
    return n, ldl, Vbuf.shape[0]


def _modify(fname: str, Lbuf: np.ndarray, Vbuf: np.ndarray, sigma: int):
    if sigma not in (1, -1):
        raise ValueError("sigma must be +1 or -1 (PAPER.md line 20)")
    n, ldl, k = _check(Lbuf, Vbuf)
    c = np.zeros((max(n, 1), max(k, 1)))
    s = np.zeros_like(c)
    info = _Info()
    getattr(_load(), fname)(_dp(Lbuf), n, ldl, _dp(Vbuf), k, sigma, _dp(c), _dp(s), ctypes.byref(info))
    return c[:n, :k], s[:n, :k], Info(info.code, info.col, info.row)


def modify_a(Lbuf: np.ndarray, Vbuf: np.ndarray, sigma: int):
    """In-place CholeskyModifyA (PAPER.md 24-30, dependency-corrected).

    Returns ``(c, s, info)`` with ``c``/``s`` of shape ``(n, k)``: the rotation of
    row ``i`` and update column ``e`` is ``(c[i, e], s[i, e])``.  On exit
    ``Vbuf[e, i]`` holds the value Compute(i, e) consumed (PAPER.md 105).
    """
    return _modify("gcmo_modify_a", Lbuf, Vbuf, sigma)


def modify_a_f32(Lbuf: np.ndarray, Vbuf: np.ndarray, sigma: int):
    """CholeskyModifyA in single precision (gcmo_modify_a_f32; PAPER.md 111 ran fp32 too).
    Lbuf (n, ldl) and Vbuf (k, n) float32, C-contiguous; same conventions as modify_a."""
    if sigma not in (1, -1):
        raise ValueError("sigma must be +1 or -1 (PAPER.md line 20)")
    if Lbuf.dtype != np.float32 or Vbuf.dtype != np.float32:
        raise TypeError("modify_a_f32 works in float32")
    if not (Lbuf.flags.c_contiguous and Vbuf.flags.c_contiguous):
        raise ValueError("Lbuf and Vbuf must be C-contiguous")
    n, ldl = Lbuf.shape
    k = Vbuf.shape[0]
    if ldl < max(1, n) or (Vbuf.shape[1] != n and Vbuf.size):
        raise ValueError("Lbuf (n, ldl >= n), Vbuf (k, n)")
    c = np.zeros((max(n, 1), max(k, 1)), dtype=np.float32)
    s = np.zeros_like(c)
    info = _Info()
    fp = ctypes.POINTER(ctypes.c_float)
    _load().gcmo_modify_a_f32(Lbuf.ctypes.data_as(fp), n, ldl, Vbuf.ctypes.data_as(fp), k, sigma,
                              c.ctypes.data_as(fp), s.ctypes.data_as(fp), ctypes.byref(info))
    return c[:n, :k], s[:n, :k], Info(info.code, info.col, info.row)


def modify_b(Lbuf: np.ndarray, Vbuf: np.ndarray, sigma: int):
    """In-place CholeskyModifyB (PAPER.md 34-40) as k sequential rank-1 sweeps."""
    return _modify("gcmo_modify_b", Lbuf, Vbuf, sigma)


def compute(Lii: float, Vi: float, sigma: int):
    """Scalar Compute (PAPER.md 44-49): returns (c, s, w, failed)."""
    c, s, l = ctypes.c_double(), ctypes.c_double(), ctypes.c_double(Lii)
    bad = _load().gcmo_compute(ctypes.byref(c), ctypes.byref(s), ctypes.byref(l), Vi, sigma)
    return c.value, s.value, l.value, bool(bad)


def apply(c: float, s: float, Lij: float, Vj: float, sigma: int):
    """Scalar Apply (PAPER.md 52-54): returns (new L_ij, new V_j)."""
    l, v = ctypes.c_double(Lij), ctypes.c_double(Vj)
    _load().gcmo_apply(c, s, ctypes.byref(l), ctypes.byref(v), sigma)
    return l.value, v.value


def chol_upper(A: np.ndarray, ldl: int | None = None) -> np.ndarray:
    """Textbook Cholesky A = L^T L; returns Lbuf of shape (n, ldl) (lower part 0)."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    n = A.shape[0]
    ldl = n if ldl is None else ldl
    # A is symmetric, so its C-order buffer is also its column-major buffer.
    Lbuf = np.zeros((n, ldl))
    r = _load().gcmo_chol_upper(_dp(A), n, n, _dp(Lbuf), ldl)
    if r:
        raise np.linalg.LinAlgError(f"non-positive pivot at {r - 1}")
    return Lbuf


def factor_of(Lbuf: np.ndarray) -> np.ndarray:
    """The n x n upper-triangular matrix held by ``Lbuf`` (lower part zeroed)."""
    n = Lbuf.shape[0]
    return np.triu(Lbuf[:, :n].T)
