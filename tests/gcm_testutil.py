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
