"""ORACLE — ctypes binding of the C restatement (stencil_ref.c) of the
jacobi_2d / heat_3d gradient programs. Test / CPU-baseline use only."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def load():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libstencil_ref.so")
        if not os.path.exists(path):
            subprocess.run(["make", "-s"], cwd=_HERE, check=True)
        lib = C.CDLL(path)
        dp = C.POINTER(C.c_double)
        for fn in (lib.heat3d_gradient, lib.jacobi2d_gradient):
            fn.restype = C.c_int
            fn.argtypes = [C.c_int, C.c_int, dp, dp, C.c_double, dp, dp, C.c_int]
        lib.stencil_ref_max_threads.restype = C.c_int
        lib.seidel2d_value.restype = C.c_double
        lib.seidel2d_value.argtypes = [C.c_int, C.c_int, dp]
        _LIB = lib
    return _LIB


def gradient(name: str, params: dict, inputs: dict, *, seed=1.0, threads=0):
    """(value, grad_A) of jacobi_2d / heat_3d, reference program semantics."""
    lib = load()
    n, t = int(params["N"]), int(params["TSTEPS"])
    A = np.ascontiguousarray(inputs["A"], dtype=np.float64)
    B = np.ascontiguousarray(inputs["B"], dtype=np.float64)
    g = np.empty_like(A)
    v = C.c_double(0.0)
    dp = C.POINTER(C.c_double)
    fn = lib.heat3d_gradient if name == "heat_3d" else lib.jacobi2d_gradient
    rc = fn(n, t, A.ctypes.data_as(dp), B.ctypes.data_as(dp), float(seed), C.byref(v), g.ctypes.data_as(dp),
            int(threads))
    if rc:
        raise MemoryError("stencil_ref: allocation failed")
    return v.value, g


def max_threads() -> int:
    return int(load().stencil_ref_max_threads())


def seidel_value(params: dict, A) -> float:
    """Forward value of the corpus seidel_stencil (sequential C restatement)."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    return float(load().seidel2d_value(int(params["N"]), int(params["TSTEPS"]),
                                       A.ctypes.data_as(C.POINTER(C.c_double))))
