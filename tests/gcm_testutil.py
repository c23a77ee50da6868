"""Shared test helpers (pure numpy)."""
import numpy as np


def rel_fro(a, b):
    """||a - b||_F / ||b||_F (b is the reference)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def upper(Lbuf):
    """The n x n upper-triangular factor held in an (n, ldl) buffer."""
    n = Lbuf.shape[0]
    return np.triu(Lbuf[:, :n].T)


def col_scaled_max(a, b):
    """max_ij |a_ij - b_ij| / ||b_{:,j}||_2 over the upper factor's columns: an element-wise
    bound that a localised error (one wrong tile) cannot hide under a large Frobenius norm."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    cn = np.linalg.norm(b, axis=0)
    cn[cn == 0] = 1.0
    return float(np.max(np.abs(a - b) / cn[None, :])) if b.size else 0.0


def row_scaled_max(a, b):
    """max_ej |a_ej - b_ej| / max_j |b_ej| over the rows of V (one row = one update vector)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if not b.size:
        return 0.0
    rm = np.max(np.abs(b), axis=1)
    rm[rm == 0] = 1.0
    return float(np.max(np.abs(a - b) / rm[:, None]))
