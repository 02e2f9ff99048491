"""ctypes binding of libgfb.so (the C ABI declared in include/gfb.h).

The structures below mirror the C layouts field by field; ``load()`` checks
the sizes against ``gfb_struct_sizes`` so a stale build fails loudly. There
is no fallback: if the library is missing the engine raises EngineError.
"""
from __future__ import annotations

import ctypes as C
import os

from .errors import EngineError

P = 8   # GFB_MAX_PARAMS
R = 8   # GFB_MAX_RANK
MAXIN = 8
MAXOUT = 8
MAXCODE = 128
MAXCONST = 24
MAXTAPS = 32
MAXSRCS = 4
ABI_VERSION = 12

F32, F64 = 0, 1
STAR_SKIP_ZCOPY, STAR_SKIP_XCOPY = 1, 2

# bytecode opcodes (enum gfb_op)
OP_IN, OP_CONST, OP_ADD, OP_SUB, OP_MUL, OP_DIV, OP_IDIV, OP_MOD, OP_MIN, OP_MAX, OP_POW = range(11)
OP_NEG, OP_SIN, OP_COS, OP_EXP, OP_LOG, OP_SQRT, OP_TANH, OP_ABS, OP_SIGN = range(11, 20)
BINOP = {"add": OP_ADD, "sub": OP_SUB, "mul": OP_MUL, "div": OP_DIV, "idiv": OP_IDIV, "mod": OP_MOD,
         "min": OP_MIN, "max": OP_MAX, "pow": OP_POW}
UNOP = {"neg": OP_NEG, "sin": OP_SIN, "cos": OP_COS, "exp": OP_EXP, "log": OP_LOG, "sqrt": OP_SQRT,
        "tanh": OP_TANH, "abs": OP_ABS, "sign": OP_SIGN}

EBITS = {0x1: "division by zero", 0x2: "log of non-positive value", 0x4: "sqrt of negative value",
         0x8: "pow outside its domain", 0x10: "floor division by zero", 0x20: "modulo by zero"}

i32, i64, u8, f64, vp = C.c_int32, C.c_int64, C.c_uint8, C.c_double, C.c_void_p


class Space(C.Structure):
    _fields_ = [("nparams", i32), ("triangular", i32), ("lo0", i64 * P), ("hi0", i64 * P), ("step", i64 * P),
                ("loc", (i64 * P) * P), ("hic", (i64 * P) * P), ("box_lo", i64 * P), ("box_ext", i64 * P)]


class Operand(C.Structure):
    _fields_ = [("base", vp), ("dtype", i32), ("_pad", i32), ("c0", i64), ("s", i64 * P)]


class MapDesc(C.Structure):
    _fields_ = [("space", Space), ("n_in", i32), ("n_out", i32), ("compute_f64", i32), ("ncode", i32),
                ("in_", Operand * MAXIN), ("out", Operand * MAXOUT), ("wcr", i32 * MAXOUT),
                ("code_start", i32 * MAXOUT), ("code_len", i32 * MAXOUT), ("code", u8 * MAXCODE),
                ("arg", u8 * MAXCODE), ("consts", f64 * MAXCONST), ("err", vp)]


class Term(C.Structure):
    _fields_ = [("row_of", i32 * P), ("order", i32 * P), ("npiv", i32), ("code_start", i32), ("code_len", i32),
                ("_pad", i32), ("C", (i64 * P) * R), ("off", i64 * R)]


class GatherDesc(C.Structure):
    _fields_ = [("space", Space), ("rank", i32), ("dtype", i32), ("compute_f64", i32), ("n_in", i32),
                ("n_terms", i32), ("clear_mode", i32), ("lanes_on_free", i32), ("nsplit", i32), ("dst", vp),
                ("dst_strides", i64 * R), ("ybox_lo", i64 * R), ("ybox_ext", i64 * R), ("clear_lo", i64 * R),
                ("clear_hi", i64 * R), ("free_lo", i64 * P), ("free_ext", i64 * P), ("in_", Operand * MAXIN),
                ("terms", Term * 4), ("code", u8 * MAXCODE), ("arg", u8 * MAXCODE), ("consts", f64 * MAXCONST),
                ("workspace", vp), ("err", vp)]


class StencilDesc(C.Structure):
    _fields_ = [("rank", i32), ("dtype", i32), ("clear_mode", i32), ("ntaps", i32), ("dst", vp),
                ("src", vp * MAXSRCS), ("dims", i64 * 3), ("lo", i64 * 3), ("hi", i64 * 3),
                ("clear_lo", i64 * 3), ("clear_hi", i64 * 3), ("tap_src", i32 * MAXTAPS),
                ("tap_masked", i32 * MAXTAPS), ("tap_delta", (i64 * 3) * MAXTAPS),
                ("tap_mlo", (i64 * 3) * MAXTAPS), ("tap_mhi", (i64 * 3) * MAXTAPS), ("tap_coef", f64 * MAXTAPS)]


class StarOp(C.Structure):
    _fields_ = [("coef", f64 * 7), ("present", i32), ("masked", i32), ("mode", i32), ("_pad", i32),
                ("mlo", (i64 * 3) * 7), ("mhi", (i64 * 3) * 7), ("lo", i64 * 3), ("hi", i64 * 3),
                ("clo", i64 * 3), ("chi", i64 * 3)]


class StarPairDesc(C.Structure):
    _fields_ = [("rank", i32), ("dtype", i32), ("xwrite", i32), ("flags", i32), ("dims", i64 * 3),
                ("a", StarOp), ("b", StarOp), ("y", vp), ("xold", vp), ("xout", vp), ("zold", vp), ("zout", vp),
                ("dead_lo", i64 * 3), ("dead_hi", i64 * 3), ("plane0", i64), ("zlo", i64), ("zhi", i64),
                ("global_d0", i64), ("tpm_hint", i64)]


class ContractDesc(C.Structure):
    _fields_ = [("dtype", i32), ("clear_mode", i32), ("ncm", i32), ("ncn", i32), ("a_kfast", i32),
                ("b_nfast", i32), ("nsplit", i32), ("mstride", i32), ("nstride", i32), ("kstride", i32),
                ("M", i64), ("N", i64), ("K", i64), ("scale", f64), ("a", vp), ("b", vp), ("d", vp),
                ("mtab", vp), ("ntab", vp), ("ktab", vp), ("lo", i32 * 4), ("hi", i32 * 4), ("workspace", vp)]


class WaveDesc(C.Structure):
    _fields_ = [("map", MapDesc), ("c", i64 * P), ("hmax", i64), ("solve", i32), ("_pad", i32)]


M2DIMS, M2OUTS, M2DEPTH = 8, 4, 6


class M2Operand(C.Structure):
    _fields_ = [("base", vp), ("dtype", i32), ("_pad", i32), ("c0", i64), ("s", i64 * M2DIMS)]


class Map2Desc(C.Structure):
    _fields_ = [("mode", i32), ("compute_f64", i32), ("ndim", i32), ("vec", i32), ("n_in", i32), ("n_out", i32),
                ("clear_mode", i32), ("nsplit", i32), ("ext", i64 * M2DIMS), ("in_", M2Operand * MAXIN),
                ("out", M2Operand * M2OUTS), ("wcr", i32 * M2OUTS), ("code_start", i32 * M2OUTS),
                ("code_len", i32 * M2OUTS), ("code", C.c_uint32 * MAXCODE), ("consts", f64 * MAXCONST),
                ("clear_lo", i64 * M2DIMS), ("clear_hi", i64 * M2DIMS), ("workspace", vp), ("err", vp)]


_LIB = None
_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgfb.so")

# (name, restype, argtypes)
class HaloArray(C.Structure):
    _fields_ = [("base", vp), ("plane_bytes", i64), ("planes", i64), ("own_lo", i64), ("own_hi", i64),
                ("width", i64)]


MAX_HALO = 4


class HaloDesc(C.Structure):
    _fields_ = [("n", i32), ("lower", i32), ("upper", i32), ("_pad", i32), ("a", HaloArray * MAX_HALO)]


_SIGS = [
    ("gfb_abi_version", i32, []),
    ("gfb_last_error", C.c_char_p, []),
    ("gfb_device_sm_count", i32, []),
    ("gfb_struct_sizes", i32, [C.POINTER(i64), i32]),
    ("gfb_map_launch", i32, [C.POINTER(MapDesc), vp]),
    ("gfb_wave_launch", i32, [C.POINTER(WaveDesc), vp]),
    ("gfb_gather_launch", i32, [C.POINTER(GatherDesc), vp]),
    ("gfb_gather_workspace_bytes", i64, [C.POINTER(GatherDesc)]),
    ("gfb_stencil_launch", i32, [C.POINTER(StencilDesc), vp]),
    ("gfb_star_pair_launch", i32, [C.POINTER(StarPairDesc), vp]),
    ("gfb_contract_launch", i32, [C.POINTER(ContractDesc), vp]),
    ("gfb_map2_launch", i32, [C.POINTER(Map2Desc), vp]),
    ("gfb_map2_workspace_bytes", i64, [C.POINTER(Map2Desc)]),
    ("gfb_reduce_workspace_bytes", i64, [i64]),
    ("gfb_reduce_sum", i32, [vp, i32, i64, vp, i32, i32, vp, vp]),
    ("gfb_elementwise", i32, [i32, f64, vp, i64, vp, i64, vp, i64, i32, i32, vp, vp]),
    ("gfb_broadcast", i32, [vp, i32, f64, vp, i64, i32, i32, vp]),
    ("gfb_fill_box", i32, [vp, i32, i32, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64), f64, vp]),
    ("gfb_matmul_workspace_bytes", i64, [i32, i32, i32, i64, i64, i64]),
    ("gfb_matmul", i32, [i32, i32, i32, i64, i64, i64, vp, i64, vp, i64, vp, i64, i32, vp, vp]),
    ("gfb_matvec_pair_workspace_bytes", i64, [i32, i64, i64, i32]),
    ("gfb_matvec_pair_usable", i32, [i32, i64, i64, i64, vp, vp]),
    ("gfb_matvec_pair", i32, [i32, i64, i64, vp, i64, vp, vp, i32, vp, vp, i32, i32, vp, vp]),
    ("gfb_rank2", i32, [i32, i64, i64, vp, vp, vp, vp, vp, i64, i32, vp]),
    ("gfb_copy", i32, [vp, vp, i64, vp]),
    ("gfb_plane_copy", i32, [vp, vp, i64, i32, i64, vp]),
    ("gfb_halo_exchange", i32, [C.POINTER(HaloDesc), vp, vp]),
]

EXPORTED = tuple(name for name, _, _ in _SIGS)


def load(path: str | None = None):
    """Load libgfb.so and bind every entry point (raises EngineError if absent)."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = path or os.environ.get("GFB_LIBRARY", LIB_PATH)
    if not os.path.exists(p):
        raise EngineError(f"CUDA engine library not built: {p} (run __graft_entry__.build())")
    try:
        lib = C.CDLL(p)
    except OSError as exc:
        raise EngineError(f"cannot load {p}: {exc}") from None
    for name, res, args in _SIGS:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.gfb_abi_version() != ABI_VERSION:
        raise EngineError(f"libgfb ABI {lib.gfb_abi_version()} != expected {ABI_VERSION}; rebuild")
    sizes = (i64 * 12)()
    n = lib.gfb_struct_sizes(sizes, 12)
    want = [C.sizeof(Space), C.sizeof(Operand), C.sizeof(MapDesc), C.sizeof(Term), C.sizeof(GatherDesc),
            C.sizeof(StencilDesc), C.sizeof(StarOp), C.sizeof(StarPairDesc), C.sizeof(ContractDesc),
            C.sizeof(Map2Desc), C.sizeof(WaveDesc), C.sizeof(HaloDesc)]
    got = list(sizes[:n])
    if got[: len(want)] != want:
        raise EngineError(f"struct layout mismatch between gfb.h and _lib.py: C {got} vs ctypes {want}")
    if path is None:
        _LIB = lib
    return lib


def check(rc: int, what: str):
    if rc != 0:
        msg = load().gfb_last_error().decode(errors="replace")
        raise EngineError(f"{what} failed (status {rc}): {msg}")
