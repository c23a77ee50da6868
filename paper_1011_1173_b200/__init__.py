"""paper_1011_1173_b200 -- B200-native rank-k Cholesky up/down-dating (arXiv 1011.1173).

Thin Python binding over the C ABI in include/gcm.h (libgcm.so, built for
sm_100a).  Every step of the computation runs in the library's CUDA kernels;
this module only marshals torch tensors (device memory, streams) into plain
pointers and sizes.  There is no CPU fallback: if libgcm.so is missing or the
tensors are not on a CUDA device the calls raise.

Tensor conventions (include/gcm.h):
  L : torch.float64, CUDA, shape (n, ldl), C-contiguous.  Row j of the tensor is
      column j of the upper-triangular factor: factor entry (i, j), i <= j, is
      L[j, i].  Only those entries are read/written.
  V : torch.float64, CUDA, shape (k, n), C-contiguous.  Row e is update vector e.
      Overwritten with V_exit (the residuals Compute consumed, PAPER.md 105).
"""
from __future__ import annotations

import ctypes

from . import _native
from ._native import GcmError, GcmInfo

__all__ = ["modify", "modify_f32", "modify_batched", "modify_host", "modify_host_bytes", "new_info", "read_info", "GcmError", "lib_path",
           "release_workspace", "version"]


def lib_path() -> str:
    return _native.lib_path()


def version() -> str:
    return _native.lib().gcm_version().decode()


def _stream_ptr(stream, device):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return ctypes.c_void_p(stream.cuda_stream)


def _check_L_V(L, V):
    import torch
    if not (isinstance(L, torch.Tensor) and isinstance(V, torch.Tensor)):
        raise TypeError("L and V must be torch tensors")
    if L.dtype != torch.float64 or V.dtype != torch.float64:
        raise TypeError("gcm computes in fp64: L and V must be torch.float64")
    if not (L.is_cuda and V.is_cuda):
        raise ValueError("L and V must be CUDA tensors (no CPU fallback)")
    if L.device != V.device:
        raise ValueError("L and V must be on the same device")
    if not (L.is_contiguous() and V.is_contiguous()):
        raise ValueError("L and V must be contiguous")


def _info_ptr(info, device, count):
    """Device pointer of an info buffer made by new_info (None -> NULL), checked for size/device."""
    if info is None:
        return None
    if not info.is_cuda or info.device != device or info.numel() * info.element_size() < count * ctypes.sizeof(GcmInfo):
        raise ValueError(f"info must be a CUDA buffer on {device} with room for {count} gcm_info_t records")
    return ctypes.c_void_p(info.data_ptr())


def new_info(device, count: int = 1):
    """Device buffer for `count` gcm_info_t records (16 bytes each)."""
    import torch
    return torch.zeros(count * ctypes.sizeof(GcmInfo), dtype=torch.uint8, device=device)


def read_info(info):
    """List of (code, col, row) from a buffer made by new_info (synchronises)."""
    raw = bytes(info.cpu().numpy().tobytes())
    n = len(raw) // ctypes.sizeof(GcmInfo)
    recs = (GcmInfo * n).from_buffer_copy(raw)
    return [(r.code, r.col, r.row) for r in recs]


def modify(L, V, sigma: int, info=None, algo: str = "auto", stream=None) -> None:
    """In place: L~^T L~ = L^T L + sigma V V^T. Asynchronous."""
    _check_L_V(L, V)
    if L.dim() != 2:
        raise ValueError("L must have shape (n, ldl)")
    n, ldl = L.shape
    if ldl < max(1, n):
        raise ValueError("L must be (n, ldl) with ldl >= n")
    k = V.shape[0] if V.dim() == 2 else 0
    if V.dim() != 2 or (V.shape[1] != n and V.numel()):
        raise ValueError("V must have shape (k, n)")
    ip = _info_ptr(info, L.device, 1)
    import torch
    with torch.cuda.device(L.device):  # the library sizes workspaces on the current device
        st = _native.lib().gcm_modify_ex(ctypes.c_void_p(L.data_ptr()), n, ldl, ctypes.c_void_p(V.data_ptr()), k,
                                         int(sigma), ip, _native.ALGO[algo], _stream_ptr(stream, L.device))
    _native.check("gcm_modify_ex", st)


def modify_f32(L, V, sigma: int, info=None, stream=None) -> None:
    """Single-precision in-place modification (gcm_modify_f32): L (n, ldl), V (k, n), float32 CUDA."""
    import torch
    if not (isinstance(L, torch.Tensor) and isinstance(V, torch.Tensor)):
        raise TypeError("L and V must be torch tensors")
    if L.dtype != torch.float32 or V.dtype != torch.float32:
        raise TypeError("modify_f32 takes torch.float32 tensors")
    if not (L.is_cuda and V.is_cuda) or L.device != V.device:
        raise ValueError("L and V must be CUDA tensors on one device (no CPU fallback)")
    if not (L.is_contiguous() and V.is_contiguous()) or L.dim() != 2 or V.dim() != 2:
        raise ValueError("L (n, ldl) and V (k, n) must be contiguous")
    n, ldl = L.shape
    if ldl < max(1, n):
        raise ValueError("L must be (n, ldl) with ldl >= n")
    k = V.shape[0]
    if V.shape[1] != n and V.numel():
        raise ValueError("V must have shape (k, n)")
    ip = _info_ptr(info, L.device, 1)
    with torch.cuda.device(L.device):
        st = _native.lib().gcm_modify_f32(ctypes.c_void_p(L.data_ptr()), n, ldl, ctypes.c_void_p(V.data_ptr()), k,
                                          int(sigma), ip, _stream_ptr(stream, L.device))
    _native.check("gcm_modify_f32", st)


def modify_host(L, V, sigma: int):
    """End-to-end call with HOST (ideally pinned) tensors; synchronous.  Returns (code, col, row)."""
    import torch
    if not (isinstance(L, torch.Tensor) and isinstance(V, torch.Tensor)):
        raise TypeError("L and V must be torch tensors")
    if L.dtype != torch.float64 or V.dtype != torch.float64 or L.is_cuda or V.is_cuda:
        raise ValueError("modify_host takes float64 host tensors")
    # the library copies n*ldl doubles of L and n*k of V through these raw pointers:
    # shapes and contiguity are checked here so it can never read or write past them
    if L.dim() != 2 or V.dim() != 2:
        raise ValueError("L must be (n, ldl) and V (k, n)")
    if not (L.is_contiguous() and V.is_contiguous()):
        raise ValueError("L and V must be contiguous")
    n, ldl = L.shape
    k = V.shape[0]
    if ldl < max(1, n):
        raise ValueError("L must be (n, ldl) with ldl >= n")
    if V.shape[1] != n and V.numel():
        raise ValueError("V must have shape (k, n)")
    info = GcmInfo()
    st = _native.lib().gcm_modify_host(ctypes.c_void_p(L.data_ptr()), n, ldl, ctypes.c_void_p(V.data_ptr()), k,
                                       int(sigma), ctypes.byref(info))
    _native.check("gcm_modify_host", st)
    return (info.code, info.col, info.row)


def modify_host_bytes(n: int, k: int) -> int:
    """Bytes modify_host moves in each direction for (n, k) (gcm_modify_host_bytes)."""
    b = _native.lib().gcm_modify_host_bytes(int(n), int(k))
    if b < 0:
        raise ValueError("n and k must be >= 0")
    return int(b)


def modify_batched(L, V, sigma: int, info=None, stream=None) -> None:
    """Batched in-place modification.  L: (batch, n, ldl), V: (batch, k, n), both contiguous fp64 CUDA."""
    _check_L_V(L, V)
    if L.dim() != 3 or V.dim() != 3:
        raise ValueError("L must be (batch, n, ldl) and V (batch, k, n)")
    batch, n, ldl = L.shape
    k = V.shape[1]
    if V.shape[0] != batch or V.shape[2] != n:
        raise ValueError("V must have shape (batch, k, n)")
    ip = _info_ptr(info, L.device, batch)
    import torch
    with torch.cuda.device(L.device):
        st = _native.lib().gcm_modify_batched(ctypes.c_void_p(L.data_ptr()), n, ldl, n * ldl,
                                              ctypes.c_void_p(V.data_ptr()), k * n, k, int(sigma), batch, ip,
                                              _stream_ptr(stream, L.device))
    _native.check("gcm_modify_batched", st)


def profile_enable(on: bool = True) -> None:
    """Bracket every library kernel launch with CUDA events (measurement hook)."""
    _native.check("gcm_profile_enable", _native.lib().gcm_profile_enable(1 if on else 0))


def profile_read(max_entries: int = 32):
    """{kernel family: (launches, total ms)} since the last read (synchronises)."""
    import numpy as np
    names = ctypes.create_string_buffer(32 * max_entries)
    counts = np.zeros(max_entries, dtype=np.int64)
    ms = np.zeros(max_entries, dtype=np.float64)
    n = _native.lib().gcm_profile_read(names, counts.ctypes.data_as(ctypes.c_void_p),
                                       ms.ctypes.data_as(ctypes.c_void_p), max_entries)
    if n < 0:
        raise GcmError("gcm_profile_read", 2)
    out = {}
    for i in range(n):
        nm = names.raw[32 * i:32 * i + 32].split(b"\0", 1)[0].decode()
        out[nm] = (int(counts[i]), float(ms[i]))
    return out


def profile_launches() -> int:
    """Kernels the library launched while profiling was enabled, since the last call (resets)."""
    return int(_native.lib().gcm_profile_launches())


def release_workspace() -> None:
    _native.check("gcm_release_workspace", _native.lib().gcm_release_workspace())
