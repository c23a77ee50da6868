"""Build libgcm.so (all CUDA sources, sm_100a) in-tree with nvcc."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libgcm.so")
ROOT = os.path.dirname(HERE)

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
]


def _nccl_paths():
    """NCCL headers/lib: the pip wheel torch ships with (nvidia-nccl-cu12)."""
    try:
        import nvidia.nccl  # type: ignore
        base = list(nvidia.nccl.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    except Exception:
        pass
    for inc, lib in (("/usr/include", "/usr/lib/x86_64-linux-gnu"),):
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    return None, None


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + [
        os.path.join(ROOT, "include", "gcm.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    cmd = ["nvcc", *NVCC_FLAGS, "-I", os.path.join(ROOT, "include")]
    inc, lib = _nccl_paths()
    link = []
    if inc:
        cmd += ["-DGCM_WITH_NCCL=1", "-I", inc]
        so = sorted(glob.glob(os.path.join(lib, "libnccl.so*")))
        if so:
            # link the exact file torch uses; rpath so the loader finds it at run time
            link = ["-L" + lib, "-l:" + os.path.basename(so[0]), "-Xlinker", f"-rpath={lib}"]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    cmd += sources() + link + ["-o", LIB + ".tmp"]
    subprocess.check_call(cmd)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
