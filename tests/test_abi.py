"""CPU-side checks of the C-ABI library: it loads, exports every symbol that
include/gcm.h declares, and rejects invalid arguments synchronously (no
compute call is made; there is no GPU here)."""
import ctypes
import os
import re

import pytest

import paper_1011_1173_b200 as gcm
from paper_1011_1173_b200 import _build, _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gcm.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gcm_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return _native.lib()


def test_library_exports_every_declared_symbol(lib):
    names = header_functions()
    assert "gcm_modify" in names and "gcm_modify_batched" in names and "gcm_modify_dist" in names
    for name in names:
        assert hasattr(lib, name), f"{name} declared in gcm.h but not exported"
    assert set(names) == set(_native.SIGNATURES), "ctypes binding out of sync with gcm.h"


def test_library_is_sm100a_only(lib):
    out = os.popen(f"cuobjdump --list-elf {_build.LIB} 2>&1").read()
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", ""))


def test_version_and_status_strings(lib):
    assert gcm.version().startswith("gcm")
    assert lib.gcm_status_string(1).decode().startswith("GCM_EINVAL")


@pytest.mark.parametrize("args", [
    (-1, 1, 1, 1),   # n < 0
    (4, 3, 1, 1),    # ldl < n
    (4, 4, -1, 1),   # k < 0
    (4, 4, 1, 0),    # sigma not +-1
    (4, 4, 1, 2),
])
def test_invalid_arguments_rejected_synchronously(lib, args):
    n, ldl, k, sigma = args
    dummy = ctypes.c_void_p(16)  # never dereferenced: validation happens first
    st = lib.gcm_modify(dummy, n, ldl, dummy, k, sigma, None)
    assert st == 1


def test_null_pointers_rejected(lib):
    assert lib.gcm_modify(None, 4, 4, None, 2, 1, None) == 1
    assert lib.gcm_modify_batched(None, 4, 4, 16, None, 8, 2, 1, -1, None, None) == 1
    assert lib.gcm_modify_ex(ctypes.c_void_p(16), 4, 4, ctypes.c_void_p(16), 2, 1, None, 7, None) == 1


def test_oracle_not_imported_by_product():
    """The product path never imports the oracle (and has no CPU fallback)."""
    pkg_dir = os.path.dirname(gcm.__file__)
    for dirpath, _, files in os.walk(pkg_dir):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", src), f"{f} mentions the oracle in code"


def test_host_bytes_counts_triangle_blocks(lib):
    """gcm_modify_host_bytes is host-only arithmetic: 256-column blocks, block
    [j0, j1) carrying rows 0..j1-1, plus V; at least the triangle, at most the square."""
    assert lib.gcm_modify_host_bytes(257, 9) == 8 * (256 * 256 + 257 * 1 + 257 * 9)
    assert lib.gcm_modify_host_bytes(0, 0) == 0
    assert lib.gcm_modify_host_bytes(-1, 3) == -1
    for n, k in [(1, 1), (255, 4), (5000, 16), (100000, 32)]:
        b = lib.gcm_modify_host_bytes(n, k) // 8 - n * k
        assert n * (n + 1) // 2 <= b <= n * n
