"""ctypes declarations of include/gcm.h (argument marshalling only)."""
from __future__ import annotations

import ctypes
import os

from . import _build

_lib = None


class GcmInfo(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("col", ctypes.c_int32), ("row", ctypes.c_int64)]


STATUS = {0: "GCM_OK", 1: "GCM_EINVAL", 2: "GCM_ECUDA", 3: "GCM_ENOMEM", 4: "GCM_ENCCL", 5: "GCM_ENOTSUP"}
ALGO = {"auto": 0, "sweep": 1, "blocked": 2, "panel": 3}

# every symbol include/gcm.h declares, with (restype, argtypes)
_vp, _i64, _int, _dp = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
SIGNATURES = {
    "gcm_modify": (_int, [_dp, _i64, _i64, _dp, _i64, _int, _vp]),
    "gcm_modify_info": (_int, [_dp, _i64, _i64, _dp, _i64, _int, _vp, _vp]),
    "gcm_modify_ex": (_int, [_dp, _i64, _i64, _dp, _i64, _int, _vp, _int, _vp]),
    "gcm_modify_host": (_int, [_dp, _i64, _i64, _dp, _i64, _int, _vp]),
    "gcm_modify_f32": (_int, [_vp, _i64, _i64, _vp, _i64, _int, _vp, _vp]),
    "gcm_modify_host_bytes": (_i64, [_i64, _i64]),
    "gcm_modify_batched": (_int, [_dp, _i64, _i64, _i64, _dp, _i64, _i64, _int, _i64, _vp, _vp]),
    "gcm_comm_unique_id": (_int, [_vp]),
    "gcm_comm_init": (_int, [ctypes.POINTER(_vp), _vp, _int, _int]),
    "gcm_comm_destroy": (_int, [_vp]),
    "gcm_comm_set_peer": (_int, [_vp, _int]),
    "gcm_dist_local_cols": (_i64, [_i64, _i64, _int, _int]),
    "gcm_dist_global_col": (_i64, [_i64, _int, _int, _i64]),
    "gcm_modify_dist": (_int, [_vp, _dp, _i64, _i64, _i64, _dp, _i64, _int, _vp, _vp]),
    "gcm_modify_dist_virtual": (_int, [_int, _vp, _i64, _i64, _vp, _vp, _i64, _int, _vp, _vp]),
    "gcm_dist_plan": (_i64, [_i64, _i64, _int, _int, _int, _vp, _i64]),
    "gcm_profile_enable": (_int, [_int]),
    "gcm_profile_read": (_int, [ctypes.c_char_p, _vp, _vp, _int]),
    "gcm_profile_launches": (_i64, []),
    "gcm_status_string": (ctypes.c_char_p, [_int]),
    "gcm_release_workspace": (_int, []),
    "gcm_version": (ctypes.c_char_p, []),
}


class GcmError(RuntimeError):
    def __init__(self, fn: str, status: int):
        self.status = status
        msg = lib().gcm_status_string(status).decode()
        super().__init__(f"{fn} failed: {msg}")


def lib_path() -> str:
    return _build.LIB


def lib():
    """Load libgcm.so.  Raises if it is missing: there is no CPU fallback."""
    global _lib
    if _lib is None:
        path = os.environ.get("GCM_LIB_PATH", _build.LIB)  # experiments may point at a variant build
        if not os.path.exists(path):
            raise RuntimeError(
                f"{path} is missing: build it with `python -m paper_1011_1173_b200._build` "
                "(or __graft_entry__.build()); the product path has no CPU fallback")
        h = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(h, name)
            f.restype = res
            f.argtypes = args
        _lib = h
    return _lib


def check(fn: str, status: int):
    if status != 0:
        raise GcmError(fn, status)
