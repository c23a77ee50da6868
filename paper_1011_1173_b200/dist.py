"""Column-sharded multi-GPU binding (include/gcm.h: gcm_comm_*, gcm_modify_dist).

One process per GPU.  torch.distributed is used only to share the 128-byte NCCL
unique id; the data path is the library's own NCCL broadcasts of coefficient
panels.  Argument marshalling only.

Layout (block-cyclic columns, width nb, a multiple of 64): rank r owns global
column blocks g = r, r + P, r + 2P, ...; ``L_local`` is a float64 CUDA tensor of
shape (n_local, ldl) whose row c is the (global) column ``global_cols(...)[c]``
of L (all n rows); ``V_local`` is (k, n_local): the V entries of those columns.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from ._native import GcmError


def local_cols(n: int, nb: int, world: int, rank: int) -> int:
    v = _native.lib().gcm_dist_local_cols(n, nb, world, rank)
    if v < 0:
        raise ValueError("invalid block-cyclic layout arguments")
    return int(v)


def global_cols(n: int, nb: int, world: int, rank: int) -> np.ndarray:
    """Global column index of every local column of `rank` (increasing)."""
    nloc = local_cols(n, nb, world, rank)
    lib = _native.lib()
    return np.array([lib.gcm_dist_global_col(nb, world, rank, c) for c in range(nloc)], dtype=np.int64)


class Comm:
    """NCCL communicator of the library.  world == 1 needs no process group."""

    def __init__(self, rank: int, world: int, group=None, peer: bool = False):
        lib = _native.lib()
        uid = ctypes.create_string_buffer(128)
        if rank == 0:
            _native.check("gcm_comm_unique_id", lib.gcm_comm_unique_id(uid))
        if world > 1:
            import torch.distributed as dist
            obj = [uid.raw if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0, group=group)
            uid = ctypes.create_string_buffer(obj[0], 128)
        self._h = ctypes.c_void_p()
        _native.check("gcm_comm_init", lib.gcm_comm_init(ctypes.byref(self._h), uid, world, rank))
        self.rank, self.world = rank, world
        if peer:  # device-initiated exchange through IPC windows (gcm_comm_set_peer)
            _native.check("gcm_comm_set_peer", lib.gcm_comm_set_peer(self._h, 1))

    def close(self):
        if self._h:
            _native.check("gcm_comm_destroy", _native.lib().gcm_comm_destroy(self._h))
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def modify_dist(comm: Comm, L_local, V_local, n: int, nb: int, sigma: int, info=None, stream=None) -> None:
    """Collective in-place modification of the sharded factor (every rank calls it)."""
    import torch
    if L_local.dtype != torch.float64 or V_local.dtype != torch.float64 or not (L_local.is_cuda and V_local.is_cuda):
        raise ValueError("L_local and V_local must be float64 CUDA tensors")
    if not (L_local.is_contiguous() and V_local.is_contiguous()):
        raise ValueError("L_local and V_local must be contiguous")
    nloc = local_cols(n, nb, comm.world, comm.rank)
    if L_local.shape[0] != nloc or (V_local.numel() and V_local.shape[1] != nloc):
        raise ValueError(f"this rank owns {nloc} columns")
    k = V_local.shape[0]
    ldl = L_local.shape[1]
    if stream is None:
        stream = torch.cuda.current_stream(L_local.device)
    ip = ctypes.c_void_p(info.data_ptr()) if info is not None else None
    st = _native.lib().gcm_modify_dist(comm._h, ctypes.c_void_p(L_local.data_ptr()), n, nb, ldl,
                                       ctypes.c_void_p(V_local.data_ptr()), k, int(sigma), ip,
                                       ctypes.c_void_p(stream.cuda_stream))
    _native.check("gcm_modify_dist", st)


def plan(n: int, nb: int, world: int, rank: int, what: str) -> np.ndarray:
    """The work `rank` does in modify_dist (gcm_dist_plan): what = "tiles" -> (b, s) pairs of
    its Apply tiles, "diag" -> its 64-row diagonal blocks, "solve" -> the column blocks whose
    rows of P it solves.  Host only."""
    code = {"tiles": 0, "diag": 1, "solve": 2}[what]
    lib = _native.lib()
    cnt = lib.gcm_dist_plan(n, nb, world, rank, code, None, 0)
    if cnt < 0:
        raise ValueError("invalid block-cyclic layout arguments")
    out = np.zeros(max(cnt, 1), dtype=np.int64)
    lib.gcm_dist_plan(n, nb, world, rank, code, ctypes.c_void_p(out.ctypes.data), cnt)
    out = out[:cnt]
    return out.reshape(-1, 2) if code == 0 else out


def modify_dist_virtual(L_locals, V_locals, n: int, nb: int, sigma: int, info=None, stream=None) -> None:
    """All ranks of a column-sharded job on the current device, in one call (gcm_modify_dist_virtual):
    L_locals[r] (n_local_r, ldl_r) and V_locals[r] (k, n_local_r) as for modify_dist with
    world = len(L_locals), rank = r.  The owner of each column block writes its rows of P, and
    each rank its panels, straight into the other ranks' buffers (device-initiated stores)."""
    import torch
    R = len(L_locals)
    if R != len(V_locals) or not 1 <= R <= 8:
        raise ValueError("1..8 ranks, one L and one V per rank")
    k = V_locals[0].shape[0]
    dev = L_locals[0].device
    for r in range(R):
        L, V = L_locals[r], V_locals[r]
        if L.dtype != torch.float64 or V.dtype != torch.float64 or not (L.is_cuda and V.is_cuda):
            raise ValueError("L_local and V_local must be float64 CUDA tensors")
        if L.device != dev or V.device != dev:
            raise ValueError("virtual ranks share one device")
        if not (L.is_contiguous() and V.is_contiguous()) or L.dim() != 2 or V.dim() != 2:
            raise ValueError("L_local (n_local, ldl) and V_local (k, n_local) must be contiguous")
        nloc = local_cols(n, nb, R, r)
        if L.shape[0] != nloc or V.shape[0] != k or (V.numel() and V.shape[1] != nloc) or L.shape[1] < max(1, n):
            raise ValueError(f"rank {r} owns {nloc} columns")
    Lp = (ctypes.c_void_p * R)(*[L.data_ptr() for L in L_locals])
    Vp = (ctypes.c_void_p * R)(*[V.data_ptr() for V in V_locals])
    ld = (ctypes.c_int64 * R)(*[L.shape[1] for L in L_locals])
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    ip = ctypes.c_void_p(info.data_ptr()) if info is not None else None
    with torch.cuda.device(dev):
        st = _native.lib().gcm_modify_dist_virtual(R, Lp, n, nb, ld, Vp, k, int(sigma), ip,
                                                   ctypes.c_void_p(stream.cuda_stream))
    _native.check("gcm_modify_dist_virtual", st)


def shard(L_full, V_full, nb: int, world: int):
    """Split a (n, ldl) factor buffer and (k, n) V into the block-cyclic shards of `world` ranks
    (row c of a shard = global column global_cols()[c]).  Torch ops; a test/bench helper."""
    n = L_full.shape[0]
    out = []
    for r in range(world):
        g = global_cols(n, nb, world, r)
        import torch
        idx = torch.from_numpy(g).to(L_full.device)
        out.append((L_full.index_select(0, idx).contiguous(), V_full.index_select(1, idx).contiguous(), g))
    return out


__all__ = ["Comm", "modify_dist", "modify_dist_virtual", "plan", "shard", "local_cols", "global_cols", "GcmError"]
