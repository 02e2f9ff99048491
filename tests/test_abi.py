"""The C-ABI library loads, exports every entry point include/gfb.h declares,
and its descriptor layouts match the ctypes binding (no compute calls)."""
import os
import re

from conftest import REPO
from paper_2509_02197_b200 import _lib as L


def test_library_loads_and_layouts_match():
    lib = L.load()
    assert lib.gfb_abi_version() == L.ABI_VERSION


def test_every_declared_symbol_is_exported():
    header = open(os.path.join(REPO, "include", "gfb.h")).read()
    declared = set(re.findall(r"^\s*(?:int|int64_t|const char \*)\s*\**\s*(gfb_\w+)\(", header, re.M))
    assert declared, "no entry points parsed from gfb.h"
    lib = L.load()
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(L.EXPORTED)


def test_workspace_queries_are_pure_host():
    lib = L.load()
    assert lib.gfb_reduce_workspace_bytes(1 << 20) > 0
    assert lib.gfb_matmul_workspace_bytes(1, 1, 0, 4000, 1, 4000) > 0
    assert lib.gfb_matmul_workspace_bytes(1, 0, 0, 64, 64, 64) == 0


def test_halo_exchange_rejects_malformed_descriptors_without_a_device():
    """K15 (gfb_halo_exchange): descriptor checks happen before NCCL or CUDA
    is touched."""
    import ctypes as C

    lib = L.load()
    d = L.HaloDesc()
    d.n, d.lower, d.upper = 1, -1, 1
    a = d.a[0]
    a.base, a.plane_bytes, a.planes, a.own_lo, a.own_hi, a.width = 0x1000, 64, 10, 0, 8, 2
    assert lib.gfb_halo_exchange(C.byref(d), None, None) == 1  # no communicator
    a.own_hi = 9  # the upper halo would run past the local planes
    assert lib.gfb_halo_exchange(C.byref(d), C.c_void_p(0x10), None) == 1
    d.n = L.MAX_HALO + 1
    assert lib.gfb_halo_exchange(C.byref(d), C.c_void_p(0x10), None) == 1
