"""Lowering: reference IR + parameter bindings -> a static launch list.

This replaces the reference's interpretation loop (``Executor``,
interpreter.py:116-550). Because loop headers are resolved from parameters
(the reference's own static-iteration-space rule, SPEC "static iteration
space"), the whole forward+backward execution of one gradient unrolls into a
flat list of kernel launches over preallocated HBM buffers. The runtime
replays that list directly or as one captured CUDA graph.

Per node kind (reference -> here):

* MapNode with one tasklet (``_exec_map``/``_exec_tasklet``,
  interpreter.py:478-507/405-426): subsets are required to be affine in the
  map parameters (probed numerically, checked at several points), bounds are
  checked statically over the whole iteration space (``OutOfBounds``), and
  outputs are split into
    - point-private outputs (injective subsets): one pointwise launch;
    - scatter-add outputs (``wcr="sum"`` with collisions across points):
      one atomic-free *gather* pass per target array (output-stationary);
    - constant-zero clears (the adjoint ``_z`` outputs, autodiff.py:
      996-1004, and ``scale 0.0`` nodes, :901-906): not launched at all but
      recorded as a *pending clear* on the target buffer and folded into the
      next kernel that writes it.
  Linear constant-coefficient bodies over shifted identity subsets (the
  stencils and their adjoints) take the stencil fast path.
* LibraryNode (``_exec_library``, interpreter.py:428-476): reduce / fused
  elementwise / broadcast / matmul launches.
* Tape (``_visit_access``, interpreter.py:371-386) and forwarded reads
  (``_fetch_forwarded``/``_cand_coords``, :511-550): resolved at lowering
  time to tape slots; a slot whose source is never overwritten afterwards
  aliases it instead of copying (zero-cost store).
* Zero-init on first touch (interpreter.py:171-189): every fresh buffer
  starts with a pending whole-array clear, so the first writer overwrites
  instead of accumulating and no memset is issued.
"""
from __future__ import annotations

import ctypes as C
import itertools
import math
import os

import numpy as np

from . import _lib as L
from .errors import (
    DomainError,
    GradflowError,
    MissingInverse,
    MissingTapeValue,
    NonTermination,
    OutOfBounds,
    ShapeMismatch,
    UnboundName,
    UnsupportedConstruct,
)
from .ir import (
    AccessNode,
    Binary,
    Conditional,
    Const,
    Index,
    LibraryNode,
    LoopRegion,
    MapNode,
    Name,
    State,
    Tasklet,
    Unary,
    count_ops,
    eval_int,
    evaluate,
    free_names,
    number_writes,
    schedule,
)

KIND_DTYPE = {"real32": L.F32, "real64": L.F64}
ITEMSIZE = {"real32": 4, "real64": 8}
MAX_UNROLLED_OPS = int(os.environ.get("GFB_MAX_OPS", "200000"))


def default_trip_limit() -> int:
    raw = os.environ.get("GRADFLOW_TRIP_LIMIT")
    return int(raw) if raw else 10**9


# ---------------------------------------------------------------------------
# boxes: tuple of (lo, hi) per dimension, hi exclusive


def box_contains(outer, inner) -> bool:
    return all(ol <= il and ih <= oh for (ol, oh), (il, ih) in zip(outer, inner))


def box_union_bbox(a, b):
    return tuple((min(al, bl), max(ah, bh)) for (al, ah), (bl, bh) in zip(a, b))


def box_size(b) -> int:
    n = 1
    for lo, hi in b:
        n *= max(0, hi - lo)
    return n


def whole_box(shape):
    return tuple((0, d) for d in shape)


# ---------------------------------------------------------------------------
# buffers


class Buffer:
    """One device array (an env entry, a tape slot, or scratch)."""

    _ids = itertools.count()

    def __init__(self, name: str, shape: tuple, kind: str, *, fresh: bool):
        self.bid = next(Buffer._ids)
        self.name = name
        self.shape = tuple(int(s) for s in shape)
        self.kind = kind
        self.dtype = KIND_DTYPE[kind]
        self.itemsize = ITEMSIZE[kind]
        self.numel = int(np.prod(self.shape, dtype=np.int64)) if self.shape else 1
        self.nbytes = self.numel * self.itemsize
        # region known to be zero but not yet written (first touch or a
        # deferred gradient clear); None = contents are materialized
        self.pending = whole_box(self.shape) if fresh else None
        self.alias_of: Buffer | None = None
        self.offset = 0  # element offset into alias_of (slab views)
        self.tensor = None
        self.strides = tuple(int(np.prod(self.shape[d + 1:], dtype=np.int64)) for d in range(len(self.shape)))

    def root(self) -> "Buffer":
        b = self
        while b.alias_of is not None:
            b = b.alias_of
        return b

    def root_offset(self) -> int:
        b, off = self, 0
        while b.alias_of is not None:
            off += b.offset
            b = b.alias_of
        return off

    @property
    def ptr(self) -> int:
        t = self.root().tensor
        if t is None:
            raise RuntimeError(f"buffer '{self.name}' not allocated")
        return t.data_ptr() + self.root_offset() * self.itemsize

    def __repr__(self):
        return f"Buffer({self.name}, {self.shape}, {self.kind})"


# ---------------------------------------------------------------------------
# affine analysis of subsets and ranges

_PROBES = [(3, 7, 11, 13, 17, 19, 23, 29), (-5, 2, 9, -4, 6, 1, -8, 5), (101, 57, -33, 12, 71, -19, 44, 3),
           (2, 2, 2, 2, 2, 2, 2, 2), (-1, -3, -7, -2, -9, -6, -4, -11)]


def affine_form(expr, bind: dict, params: tuple, what: str):
    """(c0, [s_p]) with expr == c0 + sum_p s_p * x_p for integer x."""
    base = dict(bind)
    for p in params:
        base[p] = 0
    try:
        c0 = eval_int(expr, base, what)
        coefs = []
        for p in params:
            b = dict(base)
            b[p] = 1
            coefs.append(eval_int(expr, b, what) - c0)
        if params and (free_names(expr) & set(params)):
            for pt in _PROBES:
                b = dict(bind)
                b.update(zip(params, pt))
                if eval_int(expr, b, what) != c0 + sum(c * v for c, v in zip(coefs, pt)):
                    raise UnsupportedConstruct(f"{what} is not affine in the map parameters")
    except (DomainError, ZeroDivisionError) as exc:
        if params and (free_names(expr) & set(params)):
            raise UnsupportedConstruct(f"{what} is not affine in the map parameters") from exc
        raise
    return c0, coefs


class SpaceInfo:
    """Iteration space of one map with concrete bindings."""

    def __init__(self, params, lo, hi, step):
        self.params = tuple(params)
        self.np = len(params)
        self.lo = lo      # list of (c0, coefs over earlier params)
        self.hi = hi
        self.step = step  # list of int
        self.triangular = any(any(c) for c, in ((f[1],) for f in lo + hi))
        # bounding box (first value, last value) per parameter
        self.first, self.last, self.ext = [], [], []
        for p in range(self.np):
            lo_min = self._interval(lo[p], p)[0]
            hi_max = self._interval(hi[p], p)[1]
            if self.triangular:
                first, last = lo_min, hi_max - 1
                ext = max(0, last - first + 1)
            else:
                n = max(0, -(-(hi[p][0] - lo[p][0]) // step[p]))
                first = lo[p][0]
                last = first + (n - 1) * step[p]
                ext = n
            self.first.append(first)
            self.last.append(last)
            self.ext.append(ext)
        self._npoints = None

    def _interval(self, form, p):
        c0, coefs = form
        lo = hi = c0
        for q in range(p):
            a, b = coefs[q] * self.first[q], coefs[q] * self.last[q]
            lo += min(a, b)
            hi += max(a, b)
        return lo, hi

    @property
    def empty(self) -> bool:
        return any(e <= 0 for e in self.ext)

    def points(self) -> int:
        if self._npoints is None:
            if self.empty:
                self._npoints = 0
            elif not self.triangular:
                self._npoints = int(np.prod(self.ext, dtype=np.int64))
            else:
                self._npoints = int(self.enumerate_count())
        return self._npoints

    def enumerate_count(self) -> int:
        def rec(p, xs):
            if p == self.np:
                return 1
            lo = self.lo[p][0] + sum(c * x for c, x in zip(self.lo[p][1], xs))
            hi = self.hi[p][0] + sum(c * x for c, x in zip(self.hi[p][1], xs))
            if p == self.np - 1:
                return max(0, -(-(hi - lo) // self.step[p]))
            return sum(rec(p + 1, xs + [v]) for v in range(lo, hi, self.step[p]))

        return rec(0, [])

    def range_of(self, form):
        """min/max of c0 + sum s_p x_p over the bounding box."""
        c0, coefs = form
        lo = hi = c0
        for p, s in enumerate(coefs):
            a, b = s * self.first[p], s * self.last[p]
            lo += min(a, b)
            hi += max(a, b)
        return lo, hi

    def box_points(self) -> int:
        return int(np.prod(self.ext, dtype=np.int64)) if self.np else 1

    def fill(self, sp: L.Space):
        sp.nparams = self.np
        sp.triangular = 1 if self.triangular else 0
        for p in range(self.np):
            sp.lo0[p] = self.lo[p][0]
            sp.hi0[p] = self.hi[p][0]
            sp.step[p] = self.step[p]
            for q in range(p):
                sp.loc[p][q] = self.lo[p][1][q]
                sp.hic[p][q] = self.hi[p][1][q]
            sp.box_lo[p] = self.first[p]
            sp.box_ext[p] = self.ext[p]


class Access:
    """One memlet endpoint: buffer + per-dimension affine index forms."""

    def __init__(self, buf: Buffer, forms: list):
        self.buf = buf
        self.forms = forms  # per dim (c0, coefs)

    def flat(self, np_: int):
        c0 = sum(st * f[0] for st, f in zip(self.buf.strides, self.forms))
        s = [sum(st * f[1][p] for st, f in zip(self.buf.strides, self.forms)) for p in range(np_)]
        return c0, s

    def matrix(self, np_):
        return [list(f[1]) for f in self.forms], [f[0] for f in self.forms]

    def key(self):
        return (self.buf.bid, tuple((f[0], tuple(f[1])) for f in self.forms))

    def identity_offset(self, np_):
        """Offsets if dim d == x_d + off_d for every d (and rank == np)."""
        if len(self.forms) != np_:
            return None
        offs = []
        for d, (c0, coefs) in enumerate(self.forms):
            if any(c != (1 if p == d else 0) for p, c in enumerate(coefs)):
                return None
            offs.append(c0)
        return offs


def fill_operand(op: L.Operand, acc: Access, np_: int):
    op.base = acc.buf.ptr
    op.dtype = acc.buf.dtype
    c0, s = acc.flat(np_)
    op.c0 = c0
    for p in range(np_):
        op.s[p] = s[p]


# ---------------------------------------------------------------------------
# tasklet bodies -> bytecode


class Code:
    def __init__(self):
        self.code, self.arg, self.consts = [], [], []

    def const(self, v: float) -> int:
        v = float(v)
        for i, c in enumerate(self.consts):
            if c == v and math.copysign(1, c) == math.copysign(1, v):
                return i
        if len(self.consts) >= L.MAXCONST:
            raise UnsupportedConstruct("tasklet body has too many constants")
        self.consts.append(v)
        return len(self.consts) - 1

    def compile(self, expr, conn_index: dict) -> tuple:
        start = len(self.code)
        depth = self._emit(expr, conn_index, 0)
        if depth > 12:
            raise UnsupportedConstruct("tasklet body too deep for the device evaluator")
        if len(self.code) > L.MAXCODE:
            raise UnsupportedConstruct("tasklet bodies too long for the device evaluator")
        return start, len(self.code) - start

    def _emit(self, e, ci, depth) -> int:
        t = type(e)
        if t is Const:
            self.code.append(L.OP_CONST)
            self.arg.append(self.const(e.value))
            return depth + 1
        if t is Name:
            if e.id not in ci:
                raise UnboundName(f"tasklet body uses unbound connector '{e.id}'")
            self.code.append(L.OP_IN)
            self.arg.append(ci[e.id])
            return depth + 1
        if t is Unary:
            d = self._emit(e.x, ci, depth)
            self.code.append(L.UNOP[e.op])
            self.arg.append(0)
            return d
        if t is Binary:
            if e.op not in L.BINOP:
                raise UnsupportedConstruct(f"operator '{e.op}' is not allowed in tasklet bodies")
            d1 = self._emit(e.x, ci, depth)
            d2 = self._emit(e.y, ci, depth + 1)
            self.code.append(L.BINOP[e.op])
            self.arg.append(0)
            return max(d1, d2)
        raise UnsupportedConstruct(f"cannot evaluate {e!r} in a tasklet")

    def fill(self, desc):
        for i, (c, a) in enumerate(zip(self.code, self.arg)):
            desc.code[i] = c
            desc.arg[i] = a
        for i, v in enumerate(self.consts):
            desc.consts[i] = v


def linearize(expr):
    """(const, {conn: coef}) if expr is an affine combination of connectors
    with constant coefficients, else None."""
    t = type(expr)
    if t is Const:
        return float(expr.value), {}
    if t is Name:
        return 0.0, {expr.id: 1.0}
    if t is Unary:
        if expr.op != "neg":
            return None
        r = linearize(expr.x)
        return None if r is None else (-r[0], {k: -v for k, v in r[1].items()})
    if t is Binary:
        a, b = linearize(expr.x), linearize(expr.y)
        if a is None or b is None:
            return None
        if expr.op in ("add", "sub"):
            sgn = 1.0 if expr.op == "add" else -1.0
            coef = dict(a[1])
            for k, v in b[1].items():
                coef[k] = coef.get(k, 0.0) + sgn * v
            return a[0] + sgn * b[0], coef
        if expr.op == "mul":
            if not a[1]:
                return a[0] * b[0], {k: a[0] * v for k, v in b[1].items()}
            if not b[1]:
                return a[0] * b[0], {k: b[0] * v for k, v in a[1].items()}
            return None
        if expr.op == "div" and not b[1] and b[0] != 0:
            return a[0] / b[0], {k: v / b[0] for k, v in a[1].items()}
        return None
    return None


# ---------------------------------------------------------------------------
# operations


class Op:
    family = "op"
    reads: tuple = ()
    writes: tuple = ()
    full_write = False  # True when the op defines every element of its single write
    _bufs: tuple = ()   # attribute names holding Buffers (remapped by ping-pong)

    def prepare(self, rt):
        pass

    def remap(self, f):
        """Substitute every buffer reference b by f(b) (physical placement)."""
        for name in self._bufs:
            v = getattr(self, name)
            if isinstance(v, Buffer):
                setattr(self, name, f(v))
            elif isinstance(v, list):
                setattr(self, name, [f(x) if isinstance(x, Buffer) else x for x in v])
        self.reads = tuple(f(b) for b in self.reads)
        self.writes = tuple(f(b) for b in self.writes)

    def launch(self, rt, stream):
        raise NotImplementedError

    def algorithmic_bytes(self) -> int:
        return sum(b.nbytes for b in set(self.reads)) + sum(b.nbytes for b in set(self.writes))


class MapOp(Op):
    family = "map_pointwise"

    def __init__(self, space: SpaceInfo, ins: list, outs: list, code: Code, segs: list, compute_f64: bool):
        self.space, self.ins, self.outs, self.code, self.segs = space, ins, outs, code, segs
        self.compute_f64 = compute_f64
        self.reads = tuple(a.buf for a in ins) + tuple(a.buf for a, w in outs if w == 1)
        self.writes = tuple(a.buf for a, _ in outs)

    def remap(self, f):
        for a in self.ins:
            a.buf = f(a.buf)
        for a, _ in self.outs:
            a.buf = f(a.buf)
        self.reads = tuple(f(b) for b in self.reads)
        self.writes = tuple(f(b) for b in self.writes)

    def prepare(self, rt):
        d = L.MapDesc()
        self.space.fill(d.space)
        d.n_in, d.n_out = len(self.ins), len(self.outs)
        d.compute_f64 = 1 if self.compute_f64 else 0
        for k, a in enumerate(self.ins):
            fill_operand(d.in_[k], a, self.space.np)
        for o, (a, w) in enumerate(self.outs):
            fill_operand(d.out[o], a, self.space.np)
            d.wcr[o] = w
            d.code_start[o], d.code_len[o] = self.segs[o]
        self.code.fill(d)
        d.ncode = len(self.code.code)
        d.err = rt.err_ptr
        self.desc = d
        self._ref = C.byref(d)

    def launch(self, rt, stream):
        L.check(rt.lib.gfb_map_launch(self._ref, stream), "map")


class WavefrontOp(Op):
    """A sequential loop nest of one tasklet executed by hyperplanes
    (gfb_wave_launch): ``c`` are the hyperplane coefficients over the
    loops' execution indices, proven dependence-respecting by
    ``ProgramRun._wavefront``."""

    family = "wavefront"

    def __init__(self, space: SpaceInfo, ins: list, outs: list, code: Code, segs: list, compute_f64: bool, c):
        self.space, self.ins, self.outs, self.code, self.segs = space, ins, outs, code, segs
        self.compute_f64 = compute_f64
        self.c = list(c)
        self.reads = tuple(a.buf for a in ins) + tuple(a.buf for a, w in outs if w == 1)
        self.writes = tuple(a.buf for a, _ in outs)

    @property
    def hmax(self) -> int:
        return sum(c * (e - 1) for c, e in zip(self.c, self.space.ext))

    @property
    def solve(self) -> int:
        return max(p for p, c in enumerate(self.c) if c > 0)

    def remap(self, f):
        for a in self.ins:
            a.buf = f(a.buf)
        for a, _ in self.outs:
            a.buf = f(a.buf)
        self.reads = tuple(f(b) for b in self.reads)
        self.writes = tuple(f(b) for b in self.writes)

    def prepare(self, rt):
        w = L.WaveDesc()
        d = w.map
        self.space.fill(d.space)
        d.n_in, d.n_out = len(self.ins), len(self.outs)
        d.compute_f64 = 1 if self.compute_f64 else 0
        for k, a in enumerate(self.ins):
            fill_operand(d.in_[k], a, self.space.np)
        for o, (a, wc) in enumerate(self.outs):
            fill_operand(d.out[o], a, self.space.np)
            d.wcr[o] = wc
            d.code_start[o], d.code_len[o] = self.segs[o]
        self.code.fill(d)
        d.ncode = len(self.code.code)
        d.err = rt.err_ptr
        for p, c in enumerate(self.c):
            w.c[p] = c
        w.hmax = self.hmax
        w.solve = self.solve
        self.desc = w
        self._ref = C.byref(w)

    def launch(self, rt, stream):
        L.check(rt.lib.gfb_wave_launch(self._ref, stream), "wavefront")


def hyperplane(exts, deps):
    """Smallest-span integer hyperplane c (c_p >= 0) with c . d >= 1 for
    every dependence set in ``deps``; None if none with small coefficients.

    A dependence set is (fixed, free): ``fixed`` maps loop position -> the
    fixed difference of execution indices between the later and the earlier
    iteration, ``free`` the positions whose difference is unconstrained
    (iterators absent from the subscripts). Members: every d with those
    components that is lexicographically positive (the later iteration
    really is later) and |d_p| <= ext_p - 1."""
    D = len(exts)

    def ok(c):
        for fixed, free in deps:
            for lead in range(D):
                # d_0..d_{lead-1} = 0, d_lead >= 1, the rest anything allowed
                if any(fixed.get(p, 0) != 0 for p in range(lead) if p not in free):
                    break
                if lead not in free and fixed.get(lead, 0) <= 0:
                    if fixed.get(lead, 0) < 0:
                        break
                    continue
                if lead in free and exts[lead] < 2:
                    continue
                worst = 0
                if lead in free:
                    worst += c[lead] * 1
                else:
                    worst += c[lead] * fixed[lead]
                for p in range(lead + 1, D):
                    if p in free:
                        worst -= c[p] * (exts[p] - 1)
                    else:
                        worst += c[p] * fixed.get(p, 0)
                if worst < 1:
                    return False
                if lead not in free:
                    break  # a fixed positive leading component: no later lead
        return True

    best = None
    rng = range(0, 7)
    for c in itertools.product(rng, repeat=D):
        if not any(c):
            continue
        if ok(c):
            span = sum(ci * (e - 1) for ci, e in zip(c, exts))
            if best is None or span < best[0]:
                best = (span, c)
    return None if best is None else list(best[1])


class GatherOp(Op):
    family = "map_gather"

    def __init__(self, space, dst: Buffer, ybox, clear_mode, clear_box, ins, terms, code, compute_f64,
                 lanes_on_free, nsplit):
        self.space, self.dst, self.ybox = space, dst, ybox
        self.clear_mode, self.clear_box = clear_mode, clear_box
        self.ins, self.terms, self.code = ins, terms, code
        self.compute_f64, self.lanes_on_free, self.nsplit = compute_f64, lanes_on_free, nsplit
        self.reads = tuple(a.buf for a in ins) + ((dst,) if clear_mode in (0, 2) else ())
        self.writes = (dst,)

    def workspace_bytes(self):
        return 0 if self.nsplit <= 1 else self.nsplit * box_size(self.ybox) * (8 if self.compute_f64 else 4)

    def remap(self, f):
        for a in self.ins:
            a.buf = f(a.buf)
        self.dst = f(self.dst)
        self.reads = tuple(f(b) for b in self.reads)
        self.writes = tuple(f(b) for b in self.writes)

    def prepare(self, rt):
        d = L.GatherDesc()
        self.space.fill(d.space)
        d.rank = len(self.dst.shape)
        d.dtype = self.dst.dtype
        d.compute_f64 = 1 if self.compute_f64 else 0
        d.n_in = len(self.ins)
        d.n_terms = len(self.terms)
        d.clear_mode = self.clear_mode
        d.lanes_on_free = self.lanes_on_free
        d.nsplit = self.nsplit
        d.dst = self.dst.ptr
        for r in range(d.rank):
            d.dst_strides[r] = self.dst.strides[r]
            d.ybox_lo[r] = self.ybox[r][0]
            d.ybox_ext[r] = self.ybox[r][1] - self.ybox[r][0]
            if self.clear_box is not None:
                d.clear_lo[r], d.clear_hi[r] = self.clear_box[r]
        for k, a in enumerate(self.ins):
            fill_operand(d.in_[k], a, self.space.np)
        for t, (row_of, order, Cm, off, seg) in enumerate(self.terms):
            tm = d.terms[t]
            for p in range(self.space.np):
                tm.row_of[p] = row_of[p]
            for k, p in enumerate(order):
                tm.order[k] = p
            tm.npiv = len(order)
            tm.code_start, tm.code_len = seg
            for r in range(d.rank):
                tm.off[r] = off[r]
                for p in range(self.space.np):
                    tm.C[r][p] = Cm[r][p]
        self.code.fill(d)
        d.workspace = rt.workspace_ptr if self.nsplit > 1 else None
        d.err = rt.err_ptr
        self.desc = d
        self._ref = C.byref(d)

    def launch(self, rt, stream):
        L.check(rt.lib.gfb_gather_launch(self._ref, stream), "gather")


class StencilOp(Op):
    family = "stencil"
    _bufs = ("dst", "srcs")

    def __init__(self, dst: Buffer, srcs: list, region, clear_mode, clear_box, taps, *, kind="sweep"):
        # taps: (src index, coef, delta tuple, mask box or None)
        self.dst, self.srcs, self.region = dst, srcs, region
        self.clear_mode, self.clear_box, self.taps = clear_mode, clear_box, taps
        self.kind = kind
        self.reads = tuple(srcs) + ((dst,) if clear_mode in (0, 2) else ())
        self.writes = (dst,)

    def prepare(self, rt):
        d = L.StencilDesc()
        rank = len(self.dst.shape)
        d.rank, d.dtype = rank, self.dst.dtype
        d.clear_mode = self.clear_mode
        d.ntaps = len(self.taps)
        d.dst = self.dst.ptr
        for i, s in enumerate(self.srcs):
            d.src[i] = s.ptr
        for r in range(rank):
            d.dims[r] = self.dst.shape[r]
            d.lo[r], d.hi[r] = self.region[r]
            if self.clear_box is not None:
                d.clear_lo[r], d.clear_hi[r] = self.clear_box[r]
        for t, (si, coef, delta, mask) in enumerate(self.taps):
            d.tap_src[t] = si
            d.tap_coef[t] = coef
            d.tap_masked[t] = 0 if mask is None else 1
            for r in range(rank):
                d.tap_delta[t][r] = delta[r]
                if mask is not None:
                    d.tap_mlo[t][r], d.tap_mhi[t][r] = mask[r]
        self.desc = d
        self._ref = C.byref(d)

    def launch(self, rt, stream):
        L.check(rt.lib.gfb_stencil_launch(self._ref, stream), "stencil")

    def algorithmic_bytes(self) -> int:
        pts = box_size(self.region)
        per = self.dst.itemsize
        nsrc = len(self.srcs)
        return pts * per * (nsrc + 1 + (1 if self.clear_mode == 0 else 0))


class FillOp(Op):
    """D[box] = value (materialized pending clear / zero-init)."""

    family = "fill"
    _bufs = ("dst",)

    def __init__(self, dst: Buffer, box, value=0.0):
        self.dst, self.box, self.value = dst, box, value
        self.writes = (dst,)
        self.full_write = box == whole_box(dst.shape)

    def prepare(self, rt):
        rank = len(self.dst.shape)
        self.whole = self.full_write or rank == 0
        if not self.whole and rank > 3:
            raise UnsupportedConstruct("partial clears of arrays with rank > 3")
        self._dims = (L.i64 * max(rank, 1))(*self.dst.shape)
        self._lo = (L.i64 * max(rank, 1))(*[b[0] for b in self.box])
        self._hi = (L.i64 * max(rank, 1))(*[b[1] for b in self.box])

    def launch(self, rt, stream):
        if self.whole:
            L.check(rt.lib.gfb_broadcast(None, 0, self.value, self.dst.ptr, self.dst.numel, self.dst.dtype, 0,
                                         stream), "fill")
        else:
            L.check(rt.lib.gfb_fill_box(self.dst.ptr, self.dst.dtype, len(self.dst.shape), self._dims, self._lo,
                                        self._hi, self.value, stream), "fill_box")


class ReduceOp(Op):
    family = "reduce_sum"
    _bufs = ("x", "out")

    def __init__(self, x: Buffer, out: Buffer, accumulate: bool):
        self.x, self.out, self.accumulate = x, out, accumulate
        self.reads = (x,) + ((out,) if accumulate else ())
        self.writes = (out,)
        self.full_write = not accumulate

    def workspace_bytes(self):
        return int(L.load().gfb_reduce_workspace_bytes(self.x.numel))

    def launch(self, rt, stream):
        L.check(rt.lib.gfb_reduce_sum(self.x.ptr, self.x.dtype, self.x.numel, self.out.ptr, self.out.dtype,
                                      1 if self.accumulate else 0, rt.workspace_ptr, stream), "reduce_sum")


class EwOp(Op):
    family = "elementwise"
    _bufs = ("a", "b", "out")

    def __init__(self, op: int, const: float, a: Buffer, b: Buffer | None, out: Buffer, accumulate: bool):
        self.op, self.const, self.a, self.b, self.out, self.accumulate = op, const, a, b, out, accumulate
        self.reads = (a,) + ((b,) if b is not None else ()) + ((out,) if accumulate else ())
        self.writes = (out,)
        self.full_write = not accumulate

    def launch(self, rt, stream):
        L.check(rt.lib.gfb_elementwise(self.op, self.const, self.a.ptr, self.a.numel,
                                       None if self.b is None else self.b.ptr,
                                       0 if self.b is None else self.b.numel, self.out.ptr, self.out.numel,
                                       self.out.dtype, 1 if self.accumulate else 0, rt.err_ptr, stream),
                "elementwise")


class BroadcastOp(Op):
    family = "broadcast"
    _bufs = ("src", "out")

    def __init__(self, src: Buffer | None, scale: float, out: Buffer, accumulate: bool):
        self.src, self.scale, self.out, self.accumulate = src, scale, out, accumulate
        self.reads = ((src,) if src is not None else ()) + ((out,) if accumulate else ())
        self.writes = (out,)
        self.full_write = not accumulate

    def launch(self, rt, stream):
        L.check(rt.lib.gfb_broadcast(None if self.src is None else self.src.ptr,
                                     0 if self.src is None else self.src.dtype, self.scale, self.out.ptr,
                                     self.out.numel, self.out.dtype, 1 if self.accumulate else 0, stream),
                "broadcast")


class MatmulOp(Op):
    family = "matmul"
    _bufs = ("a", "b", "out")

    def __init__(self, a: Buffer, b: Buffer, out: Buffer, ta: bool, tb: bool, M, N, K, accumulate: bool):
        self.a, self.b, self.out = a, b, out
        self.ta, self.tb, self.M, self.N, self.K = ta, tb, M, N, K
        self.accumulate = accumulate
        self.reads = (a, b) + ((out,) if accumulate else ())
        self.writes = (out,)
        self.full_write = not accumulate
        self.lda = a.shape[1]
        self.ldb = b.shape[1]
        self.ldc = N

    def workspace_bytes(self):
        return int(L.load().gfb_matmul_workspace_bytes(self.out.dtype, int(self.ta), int(self.tb), self.M, self.N,
                                                       self.K))

    def flops(self):
        return 2 * self.M * self.N * self.K

    def launch(self, rt, stream):
        L.check(rt.lib.gfb_matmul(self.out.dtype, int(self.ta), int(self.tb), self.M, self.N, self.K, self.a.ptr,
                                  self.lda, self.b.ptr, self.ldb, self.out.ptr, self.ldc,
                                  1 if self.accumulate else 0, rt.workspace_ptr, stream), "matmul")


def matvec_form(op):
    """(matrix, "row" | "col", vector, out) of a matrix-vector MatmulOp
    (K > 1 and N == 1 or M == 1) over the matrix as stored, row-major [R, C]:
    "row" is out[i] = sum_j mat[i, j] vec[j], "col" is out[j] = sum_i mat[i, j]
    vec[i]. Vectors of these shapes are contiguous."""
    if not isinstance(op, MatmulOp) or op.K <= 1:
        return None
    if op.N == 1:
        return op.a, ("col" if op.ta else "row"), op.b, op.out
    if op.M == 1:
        return op.b, ("row" if op.tb else "col"), op.a, op.out
    return None


def rank1_form(op):
    """(u, v, out) of an outer-product MatmulOp (K == 1): out = u v^T."""
    if not isinstance(op, MatmulOp) or op.K != 1 or op.M < 2 or op.N < 2:
        return None
    return op.a, op.b, op.out


def _span(b: Buffer):
    o = b.root_offset()
    return b.root(), o, o + b.numel


def overlaps(x: Buffer, y: Buffer) -> bool:
    rx, x0, x1 = _span(x)
    ry, y0, y1 = _span(y)
    return rx is ry and x0 < y1 and y0 < x1


def same_buffer(x: Buffer, y: Buffer) -> bool:
    return _span(x) == _span(y) and x.shape == y.shape


class MatvecPairOp(Op):
    """Two matrix-vector library nodes over one matrix in one streaming pass
    (csrc/matvec.cu): r (+)= mat @ u and c (+)= mat^T @ v, v = the new r in
    chain mode (atax forward). Replaces ``parts`` (the original MatmulOps,
    launched in order as the fallback when the placed buffers are not
    16-byte aligned)."""
    family = "matvec"
    _bufs = ("mat", "u", "r", "v", "c")

    def __init__(self, parts, mat, u, r, r_acc, v, c, c_acc, chain):
        self.parts = parts
        self.mat, self.u, self.r, self.v, self.c = mat, u, r, v, c
        self.r_acc, self.c_acc, self.chain = r_acc, c_acc, chain
        self.R, self.C = mat.shape
        reads = [mat, u, v] + ([r] if r_acc else []) + ([c] if c_acc else [])
        self.reads = tuple(b for b in reads if b is not None)
        self.writes = (r, c)
        self.use_parts = False

    def remap(self, f):
        super().remap(f)
        for p in self.parts:
            p.remap(f)

    def workspace_bytes(self):
        lib = L.load()
        ws = int(lib.gfb_matvec_pair_workspace_bytes(self.mat.dtype, self.R, self.C, 1))
        return max([ws] + [p.workspace_bytes() for p in self.parts])

    def flops(self):
        return 4 * self.R * self.C

    def algorithmic_bytes(self) -> int:
        # SURVEY 8(d) counts each matrix-vector pass as a full read of the
        # matrix; one launch performs both passes (as a fused star-pair launch
        # performs two sweeps), so its algorithmic bytes are its parts'
        return sum(p.algorithmic_bytes() for p in self.parts)

    def prepare(self, rt):
        self.use_parts = not L.load().gfb_matvec_pair_usable(self.mat.dtype, self.R, self.C, self.C, self.mat.ptr,
                                                            self.u.ptr)

    def launch(self, rt, stream):
        if self.use_parts:
            for p in self.parts:
                p.launch(rt, stream)
            return
        L.check(rt.lib.gfb_matvec_pair(self.mat.dtype, self.R, self.C, self.mat.ptr, self.C, self.u.ptr, self.r.ptr,
                                       int(self.r_acc), None if self.chain else self.v.ptr, self.c.ptr,
                                       int(self.c_acc), int(self.chain), rt.workspace_ptr, stream), "matvec_pair")


class Rank2Op(Op):
    """Two outer-product adjoint jobs into one matrix gradient in one write
    pass (csrc/matvec.cu gfb_rank2): out (+)= u1 v1^T + u2 v2^T."""
    family = "rank2"
    _bufs = ("u1", "v1", "u2", "v2", "out")

    def __init__(self, parts, u1, v1, u2, v2, out, accumulate):
        self.parts = parts
        self.u1, self.v1, self.u2, self.v2, self.out = u1, v1, u2, v2, out
        self.accumulate = accumulate
        self.M, self.N = out.shape
        self.reads = (u1, v1, u2, v2) + ((out,) if accumulate else ())
        self.writes = (out,)
        self.full_write = not accumulate
        self.use_parts = False

    def remap(self, f):
        super().remap(f)
        for p in self.parts:
            p.remap(f)

    def workspace_bytes(self):
        return max(p.workspace_bytes() for p in self.parts)

    def flops(self):
        return 4 * self.M * self.N

    def prepare(self, rt):
        w = 16 // self.out.itemsize
        self.use_parts = bool(self.N % w or self.out.ptr % 16 or self.v1.ptr % 16 or self.v2.ptr % 16)

    def launch(self, rt, stream):
        if self.use_parts:
            for p in self.parts:
                p.launch(rt, stream)
            return
        L.check(rt.lib.gfb_rank2(self.out.dtype, self.M, self.N, self.u1.ptr, self.v1.ptr, self.u2.ptr, self.v2.ptr,
                                 self.out.ptr, self.N, int(self.accumulate), stream), "rank2")


class CopyOp(Op):
    family = "copy"
    _bufs = ("dst", "src")

    def __init__(self, dst: Buffer, src: Buffer):
        self.dst, self.src = dst, src
        self.reads = (src,)
        self.writes = (dst,)
        self.full_write = True
        self.elided = False

    def launch(self, rt, stream):
        if not self.elided:
            L.check(rt.lib.gfb_copy(self.dst.ptr, self.src.ptr, self.dst.nbytes, stream), "copy")


def packed_code(code: "Code", segs) -> list | None:
    """Bytecode for gfb_map2: op | depth_before << 6 | arg << 10 per
    instruction, or None if a segment needs more than GFB_M2_DEPTH slots."""
    out = [0] * len(code.code)
    for start, n in segs:
        depth = 0
        for pc in range(start, start + n):
            op, arg = code.code[pc], code.arg[pc]
            out[pc] = op | (depth << 6) | (arg << 10)
            if op in (L.OP_IN, L.OP_CONST):
                depth += 1
                if depth > L.M2DEPTH:
                    return None
            elif op < L.OP_NEG:
                depth -= 1
    return out


def fold_loops(space, flats, labels):
    """Loop dimensions of a rectangular space for gfb_map2: parameters in
    the given order (labels[p] groups them; only same-label neighbours
    merge), zero-based coordinates with first/step folded into each
    operand's (c0, strides), extent-1 dimensions dropped, and adjacent
    dimensions merged when every operand's strides allow.
    flats: per operand (c0, [stride per parameter]); labels: per parameter in
    loop order, list of (param, label). Returns (ext, [(c0, strides)], dim labels)."""
    dims = [(p, lab) for p, lab in labels if space.ext[p] > 1]
    ops = []
    for c0, st in flats:
        c0f = c0 + sum(st[p] * space.first[p] for p in range(space.np))
        ops.append([c0f, [st[p] * space.step[p] for p, _ in dims]])
    ext = [space.ext[p] for p, _ in dims]
    labs = [lab for _, lab in dims]
    i = len(ext) - 2
    while i >= 0:
        if labs[i] == labs[i + 1] and all(o[1][i] == ext[i + 1] * o[1][i + 1] for o in ops):
            ext[i] *= ext[i + 1]
            for o in ops:
                o[1][i] = o[1][i + 1]
                del o[1][i + 1]
            del ext[i + 1]
            del labs[i + 1]
        i -= 1
    return ext, ops, labs


def _fits_i32(ext, ops) -> bool:
    """gfb_map2 indexes in int32: point count and every operand offset."""
    if int(np.prod(ext, dtype=np.int64)) >= 2**31 - 4096:
        return False
    for c0, st in ops:
        lo = hi = c0
        for e, v in zip(ext, st):
            a = v * (e - 1)
            lo, hi = lo + min(a, 0), hi + max(a, 0)
        if lo < 0 or hi >= 2**31:
            return False
    return True


class Map2Op(Op):
    """Vectorised pointwise map or one-dimensional reduction (csrc/map2.cu)."""

    def __init__(self, mode, ext, ins, outs, code, segs, compute_f64, *, clear_mode=1, clear_box=None, nsplit=1,
                 family="map_pointwise"):
        # ins: [(Buffer, c0, strides)]; outs: [(Buffer, c0, strides, wcr)]
        self.mode, self.ext, self.ins, self.outs = mode, ext, ins, outs
        self.code, self.segs, self.compute_f64 = code, segs, compute_f64
        self.clear_mode, self.clear_box, self.nsplit = clear_mode, clear_box, nsplit
        self.family = family
        self.vec = 4  # informational: the kernel picks 4 (fp32) / 2 (fp64) points per lane
        self._refresh()

    def _refresh(self):
        self.reads = tuple(b for b, _, _ in self.ins) + tuple(
            b for b, _, _, w in self.outs if w == 1 or (self.mode != 0 and self.clear_mode in (0, 2)))
        self.writes = tuple(b for b, _, _, _ in self.outs)

    def remap(self, f):
        self.ins = [(f(b), c0, st) for b, c0, st in self.ins]
        self.outs = [(f(b), c0, st, w) for b, c0, st, w in self.outs]
        self._refresh()

    def workspace_bytes(self):
        return self.nsplit * self.ext[1] * 8 if self.mode == 2 and self.nsplit > 1 else 0

    def prepare(self, rt):
        d = L.Map2Desc()
        d.mode, d.compute_f64, d.ndim, d.vec = self.mode, 1 if self.compute_f64 else 0, len(self.ext), self.vec
        d.n_in, d.n_out = len(self.ins), len(self.outs)
        d.clear_mode, d.nsplit = self.clear_mode, self.nsplit
        for i, e in enumerate(self.ext):
            d.ext[i] = e
            d.clear_lo[i], d.clear_hi[i] = (self.clear_box[i] if self.clear_box else (0, e))
        for k, (b, c0, st) in enumerate(self.ins):
            o = d.in_[k]
            o.base, o.dtype, o.c0 = b.ptr, b.dtype, c0
            for i, v in enumerate(st):
                o.s[i] = v
        for k, (b, c0, st, w) in enumerate(self.outs):
            o = d.out[k]
            o.base, o.dtype, o.c0 = b.ptr, b.dtype, c0
            for i, v in enumerate(st):
                o.s[i] = v
            d.wcr[k] = w
            d.code_start[k], d.code_len[k] = self.segs[k]
        for i, v in enumerate(self.code_words):
            d.code[i] = v
        for i, v in enumerate(self.code.consts):
            d.consts[i] = v
        d.workspace = rt.workspace_ptr if self.workspace_bytes() else None
        d.err = rt.err_ptr
        self.desc = d
        self._ref = C.byref(d)

    def launch(self, rt, stream):
        L.check(rt.lib.gfb_map2_launch(self._ref, stream), "map2")


def map2_pointwise(space, ins, outs, code, segs, compute_f64):
    """Map2Op for a rectangular pointwise map, or None (generic evaluator).
    ins: [Access]; outs: [(Access, wcr)]."""
    if space.triangular or space.empty or len(outs) > L.M2OUTS or os.environ.get("GFB_MAP2", "1") == "0":
        return None
    if any(w not in (0, 1) for _, w in outs):
        return None
    words = packed_code(code, segs)
    if words is None:
        return None
    np_ = space.np
    in_roots = [a.buf.root().bid for a in ins]
    out_roots = [a.buf.root().bid for a, _ in outs]
    if len(outs) > 1 and (len(set(out_roots)) != len(out_roots) or set(out_roots) & set(in_roots)):
        return None  # read-all-then-write across outputs needs the generic evaluator
    if len(outs) == 1 and out_roots[0] in in_roots:
        fo = outs[0][0].flat(np_)
        if any(a.buf.root().bid == out_roots[0] and (a.flat(np_) != fo or a.buf.root_offset() !=
                                                      outs[0][0].buf.root_offset()) for a in ins):
            return None
    flats = [a.flat(np_) for a in ins] + [a.flat(np_) for a, _ in outs]
    # innermost loop dimension: the parameter with the smallest output stride
    o0 = flats[len(ins)][1]
    order = list(range(np_))
    cand = [p for p in order if o0[p] != 0 and space.ext[p] > 1]
    if cand:
        best = min(cand, key=lambda p: (abs(o0[p]), -p))
        order.remove(best)
        order.append(best)
    ext, ops, _ = fold_loops(space, flats, [(p, 0) for p in order])
    while len(ext) < 2:  # the kernels walk (row, innermost) pairs
        ext = [1] + ext
        ops = [[c0, [0] + st] for c0, st in ops]
    if len(ext) > L.M2DIMS or not _fits_i32(ext, ops):
        return None
    op = Map2Op(0, ext, [(a.buf, c0, st) for a, (c0, st) in zip(ins, ops[:len(ins)])],
                [(a.buf, c0, st, w) for (a, w), (c0, st) in zip(outs, ops[len(ins):])], code, segs, compute_f64)
    op.code_words = words
    return op


def map2_reduce(space, acc, ins, dst, ybox, clear_mode, cbox, code, seg, compute_f64):
    """Map2Op for a single-term gather whose output subset selects
    parameters one-to-one (every other parameter is summed over), when the
    summed parameters fold into one loop dimension; else None."""
    if space.triangular or space.empty or os.environ.get("GFB_MAP2", "1") == "0":
        return None
    np_ = space.np
    Cm, off = acc.matrix(np_)
    kept = {}
    for r, row in enumerate(Cm):
        nz = [p for p, c in enumerate(row) if c != 0]
        if len(nz) != 1 or row[nz[0]] != 1 or nz[0] in kept.values():
            return None
        kept[r] = nz[0]
    # the targets must be exactly the image of the space (no extra clears)
    for r, p in kept.items():
        lo = space.first[p] + off[r]
        if space.step[p] != 1 or ybox[r] != (lo, lo + space.ext[p]):
            return None
    kp = set(kept.values())
    red = [p for p in range(np_) if p not in kp and space.ext[p] > 1]
    if not red:
        return None
    words = packed_code(code, [seg])
    if words is None:
        return None
    flats = [a.flat(np_) for a in ins] + [acc.flat(np_)]
    # innermost contiguous parameter of the reads decides the layout
    smallest = None
    for c0, st in flats[:-1]:
        for p in range(np_):
            if st[p] != 0 and space.ext[p] > 1 and (smallest is None or abs(st[p]) < smallest[0]):
                smallest = (abs(st[p]), p)
    inner_reduced = smallest is None or smallest[1] not in kp
    keptp = [p for p in range(np_) if p in kp]
    labels = ([(p, 0) for p in keptp] + [(p, 1) for p in red]) if inner_reduced else \
        ([(p, 1) for p in red] + [(p, 0) for p in keptp])
    ext, ops, labs = fold_loops(space, flats, labels)
    if labs.count(1) != 1:
        return None
    # clear box in loop coordinates of the kept dimensions
    cl = None
    if clear_mode == 2:
        kept_dims = [p for p, _ in labels if space.ext[p] > 1 and p in kp]
        if len(kept_dims) != labs.count(0):
            return None  # kept dimensions merged: clear box not expressible per dimension
        cl = []
        r_of = {p: r for r, p in kept.items()}
        kd = iter(kept_dims)
        for lab in labs:
            if lab == 1:
                cl.append((0, 0))
                continue
            p = next(kd)
            r = r_of[p]
            base = space.first[p] + off[r]
            cl.append((cbox[r][0] - base, cbox[r][1] - base))
        # kept params of extent 1 must lie inside the clear box
        for r, p in kept.items():
            if space.ext[p] == 1 and not (cbox[r][0] <= space.first[p] + off[r] < cbox[r][1]):
                return None
    if inner_reduced:
        mode = 1
        if labs[-1] != 1:
            return None
        if not ext[:-1]:
            ext = [1] + ext
            ops = [[c0, [0] + st] for c0, st in ops]
            if cl is not None:
                cl = [(0, 1)] + cl
    else:
        mode = 2
        if labs == [1]:
            ext, ops = ext + [1], [[c0, st + [0]] for c0, st in ops]
            if cl is not None:
                cl = cl + [(0, 1)]
            labs = [1, 0]
        if labs != [1, 0]:
            return None
    if len(ext) > L.M2DIMS or not _fits_i32(ext, ops):
        return None
    nsplit = 1
    if mode == 2:
        # column blocks of the launch (128 columns each, csrc/map2_kernels.cuh);
        # row splits fill eight 256-thread CTAs per SM (the finish pass adds
        # the split partials in 32 parallel groups)
        chunks = -(-ext[1] // 128)
        nsplit = int(max(1, min(-(-8 * 148 // chunks), ext[0] // 64, 4096)))
    n_in = len(ins)
    op = Map2Op(mode, ext, [(a.buf, c0, st) for a, (c0, st) in zip(ins, ops[:n_in])],
                [(dst, ops[n_in][0], ops[n_in][1], 0)], code, [seg], compute_f64, clear_mode=clear_mode,
                clear_box=cl, nsplit=nsplit, family="map_reduce")
    op.code_words = words
    return op


def contract_tile(M: int, N: int, f32: bool = True):
    """(BM, BN) of the contraction kernel variant gfb_contract_launch picks."""
    if f32 and 48 < M <= 144 and N <= 32:
        return 144, 32
    if M <= 48 * 4 and N <= 32:
        return 48, 32
    if N <= 16:
        return (256 if f32 else 128), 16
    if N <= 32:
        return (256 if f32 else 128), 32
    return (128, 64) if f32 else (64, 64)


class ContractOp(Op):
    """Product-contraction gather as an implicit GEMM over index tables
    (csrc/contract.cu): D[m, n] = base + scale * sum_k A[.] B[.], see gfb.h."""

    family = "contract"
    _bufs = ("a", "b", "dst")

    def __init__(self, dst, a, b, scale, clear_mode, M, N, K, mtab, ntab, ktab, ncm, ncn, lo, hi, a_kfast,
                 b_nfast, nsplit):
        self.dst, self.a, self.b, self.scale, self.clear_mode = dst, a, b, scale, clear_mode
        self.M, self.N, self.K = M, N, K
        self.mtab, self.ntab, self.ktab = mtab, ntab, ktab
        self.ncm, self.ncn, self.lo, self.hi = ncm, ncn, lo, hi
        self.a_kfast, self.b_nfast, self.nsplit = a_kfast, b_nfast, nsplit
        self.reads = (a, b) + ((dst,) if clear_mode in (0, 2) else ())
        self.writes = (dst,)

    def workspace_bytes(self):
        return 0 if self.nsplit <= 1 else self.nsplit * self.M * self.N * 8

    def flops(self):
        return 2 * self.M * self.N * self.K

    def prepare(self, rt):
        d = L.ContractDesc()
        d.dtype = self.dst.dtype
        d.clear_mode = self.clear_mode
        d.ncm, d.ncn = self.ncm, self.ncn
        d.a_kfast, d.b_nfast, d.nsplit = self.a_kfast, self.b_nfast, self.nsplit
        d.mstride, d.nstride, d.kstride = self.mtab.shape[1], self.ntab.shape[1], self.ktab.shape[1]
        d.M, d.N, d.K = self.M, self.N, self.K
        d.scale = self.scale
        d.a, d.b, d.d = self.a.ptr, self.b.ptr, self.dst.ptr
        d.mtab, d.ntab, d.ktab = rt.upload(self.mtab), rt.upload(self.ntab), rt.upload(self.ktab)
        for c in range(self.ncm + self.ncn):
            d.lo[c], d.hi[c] = self.lo[c], self.hi[c]
        d.workspace = rt.workspace_ptr if self.nsplit > 1 else None
        self.desc = d
        self._ref = C.byref(d)

    def launch(self, rt, stream):
        L.check(rt.lib.gfb_contract_launch(self._ref, stream), "contract")


def product_form(expr):
    """(scale, [connectors]) if expr is a constant times a product of
    connector reads, else None."""
    t = type(expr)
    if t is Const:
        return float(expr.value), []
    if t is Name:
        return 1.0, [expr.id]
    if t is Unary and expr.op == "neg":
        r = product_form(expr.x)
        return None if r is None else (-r[0], r[1])
    if t is Binary and expr.op in ("mul", "div"):
        a, b = product_form(expr.x), product_form(expr.y)
        if a is None or b is None:
            return None
        if expr.op == "mul":
            return a[0] * b[0], a[1] + b[1]
        if b[1] or b[0] == 0:
            return None
        return a[0] / b[0], a[1]
    return None


def pivot_rows(Cm, np_):
    """Solve the output subset for parameters: per output row one pivot
    parameter with coefficient +-1 (preferring one no later row uses); the
    other parameters of a pivot row become free. Returns (row_of, order)."""
    row_of = [-1] * np_
    forced_free = set()
    order = []
    for r in range(len(Cm)):
        cands = [p for p in range(np_) if abs(Cm[r][p]) == 1 and row_of[p] < 0 and p not in forced_free]
        if not cands:
            continue
        later = [p for p in cands if not any(Cm[rr][p] for rr in range(r + 1, len(Cm)))]
        p = (later or cands)[0]
        row_of[p] = r
        order.append(p)
        for q in range(np_):
            if q != p and Cm[r][q] != 0 and row_of[q] < 0:
                forced_free.add(q)
    return row_of, order


def _grid(exts):
    """Row-major coordinates (n_points, len(exts)) of a box of extents."""
    if not exts:
        return np.zeros((1, 0), dtype=np.int64)
    g = np.indices(exts, dtype=np.int64).reshape(len(exts), -1)
    return g.T


INT32_MAX = 2**31 - 1


def _i32(a):
    a = np.asarray(a, dtype=np.int64)
    if a.size and (a.min() < -INT32_MAX or a.max() > INT32_MAX):
        return None
    return np.ascontiguousarray(a.astype(np.int32))


def _quads(fast_off, fast_cons, other_off) -> bool:
    """Four consecutive entries along the fast table form 16-byte quads:
    offsets consecutive and 4-aligned, constraint parts equal within each
    quad, and every other-side offset 4-aligned (count a multiple of 4)."""
    n = len(fast_off)
    if n % 4 or n == 0:
        return False
    q = np.asarray(fast_off, dtype=np.int64).reshape(-1, 4)
    if np.any(q[:, 0] % 4) or np.any(q - q[:, :1] != np.arange(4)):
        return False
    if fast_cons.size:
        c = np.asarray(fast_cons, dtype=np.int64).reshape(-1, 4, fast_cons.shape[1])
        if np.any(c != c[:, :1, :]):
            return False
    return not np.any(np.asarray(other_off, dtype=np.int64) % 4)


def contract_form(space, body, acc, ins, dst, ybox, clear_mode, cbox):
    """Build the ContractOp of a single-term gather whose body is a scaled
    product of two reads, or None when the pass does not have that shape
    (the generic gather then runs it)."""
    if space.triangular or space.np == 0 or any(s != 1 for s in space.step) or space.empty:
        return None
    if os.environ.get("GFB_CONTRACT", "1") == "0":
        return None
    pf = product_form(body)
    if pf is None or len(pf[1]) != 2 or pf[1][0] == pf[1][1]:
        return None
    scale, (ca, cb) = pf
    A, B = ins[ca], ins[cb]
    if A.buf.kind != dst.kind or B.buf.kind != dst.kind:
        return None
    np_ = space.np
    Cm, off = acc.matrix(np_)
    rank = len(Cm)
    if rank == 0:
        return None
    row_of, order = pivot_rows(Cm, np_)
    if sorted(row_of[p] for p in order) != list(range(rank)):
        return None  # an output row without a pivot: generic gather checks it
    free = [p for p in range(np_) if row_of[p] < 0]
    nv = rank + len(free) + 1
    form = {}
    for i, p in enumerate(free):
        v = np.zeros(nv, dtype=np.int64)
        v[rank + i] = 1
        form[p] = v
    for p in order:
        r = row_of[p]
        v = np.zeros(nv, dtype=np.int64)
        v[r] = 1
        v[-1] = -off[r]
        for q in range(np_):
            if q != p and Cm[r][q] != 0:
                if q not in form:
                    return None
                v = v - Cm[r][q] * form[q]
        form[p] = v * Cm[r][p]

    def addr(a):
        c0, st = a.flat(np_)
        v = np.zeros(nv, dtype=np.int64)
        v[-1] = c0
        for p in range(np_):
            v = v + st[p] * form[p]
        return v

    fa, fb = addr(A), addr(B)
    ext = [hi - lo for lo, hi in ybox]
    ya = {r for r in range(rank) if fa[r] != 0}
    yb = {r for r in range(rank) if fb[r] != 0}
    if ya & yb:
        return None  # a batch dimension: no operand reuse, the generic gather is as good
    if int(np.prod([ext[r] for r in yb], dtype=np.int64)) > int(np.prod([ext[r] for r in ya], dtype=np.int64)):
        A, B, fa, fb, ya, yb = B, A, fb, fa, yb, ya
    ndims = sorted(yb)
    mdims = [r for r in range(rank) if r not in yb]
    # pivot-range constraints not implied by the boxes
    yl = [lo for lo, _ in ybox]
    yh = [hi - 1 for _, hi in ybox]
    cons_m, cons_n = [], []
    for p in order:
        v = form[p]
        vmin = vmax = int(v[-1])
        for r in range(rank):
            a, b = int(v[r]) * yl[r], int(v[r]) * yh[r]
            vmin, vmax = vmin + min(a, b), vmax + max(a, b)
        for i, q in enumerate(free):
            a, b = int(v[rank + i]) * space.first[q], int(v[rank + i]) * space.last[q]
            vmin, vmax = vmin + min(a, b), vmax + max(a, b)
        lo_p, hi_p = space.first[p], space.last[p] + 1
        if vmin >= lo_p and vmax < hi_p:
            continue
        dep = {r for r in range(rank) if v[r] != 0}
        if dep <= set(mdims):
            cons_m.append((v, lo_p, hi_p))
        elif dep <= set(ndims):
            cons_n.append((v, lo_p, hi_p))
        else:
            return None
    if len(cons_m) > 2 or len(cons_n) > 2:
        return None
    # k order: free parameters by decreasing |A stride| (innermost contiguous)
    kperm = sorted(range(len(free)), key=lambda i: -abs(int(fa[rank + i])))
    kdims = [free[i] for i in kperm]
    M = int(np.prod([ext[r] for r in mdims], dtype=np.int64))
    N = int(np.prod([ext[r] for r in ndims], dtype=np.int64))
    K = int(np.prod([space.ext[q] for q in kdims], dtype=np.int64))
    if M == 0 or N == 0 or K == 0:
        return None

    def side(dims, f, cons):
        g = _grid([ext[r] for r in dims]) + np.array([yl[r] for r in dims], dtype=np.int64)
        cols = [g @ np.array([f[r] for r in dims], dtype=np.int64),
                g @ np.array([dst.strides[r] for r in dims], dtype=np.int64)]
        if cbox is not None:
            inside = np.ones(g.shape[0], dtype=bool)
            for j, r in enumerate(dims):
                inside &= (g[:, j] >= cbox[r][0]) & (g[:, j] < cbox[r][1])
            cols.append(inside.astype(np.int64))
        else:
            cols.append(np.ones(g.shape[0], dtype=np.int64))
        for v, _, _ in cons:
            cols.append(g @ np.array([v[r] for r in dims], dtype=np.int64))
        return _i32(np.stack(cols, axis=1))

    mtab = side(mdims, fa, cons_m)
    ntab = side(ndims, fb, cons_n)
    gk = _grid([space.ext[q] for q in kdims]) + np.array([space.first[q] for q in kdims], dtype=np.int64)
    fi = [free.index(q) for q in kdims]
    kcols = [gk @ np.array([fa[rank + i] for i in fi], dtype=np.int64) + fa[-1],
             gk @ np.array([fb[rank + i] for i in fi], dtype=np.int64) + fb[-1]]
    for v, _, _ in cons_m + cons_n:
        kcols.append(gk @ np.array([v[rank + i] for i in fi], dtype=np.int64) + v[-1])
    ktab = _i32(np.stack(kcols, axis=1))
    if mtab is None or ntab is None or ktab is None:
        return None
    bounds = [(lo, hi) for _, lo, hi in cons_m + cons_n]
    if any(abs(b) > INT32_MAX for lh in bounds for b in lh):
        return None
    a_kfast = 1 if kdims and abs(int(fa[rank + free.index(kdims[-1])])) == 1 else 0
    b_nfast = 1 if ndims and abs(int(fb[ndims[-1]])) == 1 else 0
    ncm, ncn = len(cons_m), len(cons_n)
    # 16-byte quads along each operand's fast direction (bit 1)
    if a_kfast:
        a_q = _quads(ktab[:, 0], ktab[:, 2:2 + ncm], mtab[:, 0])
    else:
        a_q = _quads(mtab[:, 0], mtab[:, 3:3 + ncm], ktab[:, 0])
    if b_nfast:
        b_q = _quads(ntab[:, 0], ntab[:, 3:3 + ncn], ktab[:, 1])
    else:
        b_q = _quads(ktab[:, 1], ktab[:, 2 + ncm:2 + ncm + ncn], ntab[:, 0])
    a_kfast |= 2 if a_q and A.buf.dtype == L.F32 else 0
    b_nfast |= 2 if b_q and B.buf.dtype == L.F32 else 0
    BM, BN = contract_tile(M, N, A.buf.dtype == L.F32)
    tiles = -(-M // BM) * -(-N // BN)
    nsplit = 1
    # enough CTAs to fill the SMs in one wave: two per SM, four for the
    # 64-thread whole-output tile of the weight adjoints (its register-bound
    # occupancy; eight per SM doubled the split-k partial traffic: 150 vs 188 us)
    per_sm = 4 if (BM, BN) == (144, 32) else 2
    if tiles < per_sm * 148 and K >= 64 * 16:
        nsplit = int(min(-(-per_sm * 148 // tiles), K // (8 * 16), 2048))
    return ContractOp(dst, A.buf, B.buf, scale, clear_mode, M, N, K, mtab, ntab, ktab, len(cons_m), len(cons_n),
                      [lo for lo, _ in bounds], [hi for _, hi in bounds], a_kfast, b_nfast, max(nsplit, 1))


def small_fuse_bytes() -> int:
    """rank-3 arrays below this size stay unfused (GFB_SMALL_FUSE_BYTES)."""
    return int(os.environ.get("GFB_SMALL_FUSE_BYTES", 32 << 20))


STAR_POS = {(0, 0, 0): 0, (-1, 0, 0): 1, (1, 0, 0): 2, (0, -1, 0): 3, (0, 1, 0): 4, (0, 0, -1): 5, (0, 0, 1): 6}


def star_form(op):
    """(source, {position: (coef, mask)}) if a StencilOp is a single-source
    radius-1 star on a rank-2/3 array, else None."""
    if not isinstance(op, StencilOp) or len(op.srcs) != 1:
        return None
    rank = len(op.dst.shape)
    if rank not in (2, 3) or op.srcs[0].shape != op.dst.shape or op.srcs[0].kind != op.dst.kind:
        return None
    taps = {}
    for _si, coef, delta, mask in op.taps:
        d3 = (0,) * (3 - rank) + tuple(delta)
        pos = STAR_POS.get(d3)
        if pos is None or pos in taps:
            return None
        taps[pos] = (coef, mask)
    return op.srcs[0], taps


def _fill_star(so: L.StarOp, op: StencilOp, taps: dict):
    rank = len(op.dst.shape)
    so.mode = op.clear_mode
    for pos, (coef, mask) in taps.items():
        so.present |= 1 << pos
        so.coef[pos] = coef
        if mask is not None:
            so.masked |= 1 << pos
            for r in range(rank):
                so.mlo[pos][r], so.mhi[pos][r] = mask[r]
    for r in range(rank):
        so.lo[r], so.hi[r] = op.region[r]
        if op.clear_box is not None:
            so.clo[r], so.chi[r] = op.clear_box[r]


class StarPairOp(Op):
    """Two consecutive radius-1 star sweeps X = a(Y); Z = b(X) in one
    launch (csrc/star.cu). Physical outputs are assigned by the ping-pong
    placement pass (``xout``/``zout``)."""

    family = "star_pair"

    def __init__(self, a: StencilOp, b: StencilOp, fa, fb, xwrite: bool, dead):
        self.a, self.b, self.fa, self.fb = a, b, fa, fb
        self.X, self.Y, self.Z = a.dst, fa[0], b.dst
        self.xwrite, self.dead = xwrite, dead
        self.xout = self.X
        self.zout = self.Z
        # out-of-region copies already in place in the target twin
        self.skip_zcopy = self.skip_xcopy = False
        # slab placement (decomp.py): global plane of local plane 0, local
        # planes produced, global extent of dim 0; single device: whole array
        self.plane0, self.zrange, self.global_d0 = 0, None, None
        self.tpm_hint = 0  # planes per CTA of the 3-D kernel (0: the launch chooses)
        self._refresh()

    def _refresh(self):
        self.reads = (self.Y, self.X, self.Z)
        self.writes = (self.zout,) + ((self.xout,) if self.xwrite else ())

    def remap(self, f):
        self.X, self.Y, self.Z = f(self.X), f(self.Y), f(self.Z)
        self.xout, self.zout = f(self.xout), f(self.zout)
        self._refresh()

    def algorithmic_bytes(self) -> int:
        # the two map sweeps it replaces, each one read + one write of the array
        return self.a.algorithmic_bytes() + self.b.algorithmic_bytes()

    def prepare(self, rt):
        d = L.StarPairDesc()
        rank = len(self.Z.shape)
        d.rank, d.dtype = rank, self.Z.dtype
        d.xwrite = 1 if self.xwrite else 0
        d.flags = (L.STAR_SKIP_ZCOPY if self.skip_zcopy else 0) | (L.STAR_SKIP_XCOPY if self.skip_xcopy else 0)
        for r in range(rank):
            d.dims[r] = self.Z.shape[r]
        _fill_star(d.a, self.a, self.fa[1])
        _fill_star(d.b, self.b, self.fb[1])
        d.y, d.xold, d.zold = self.Y.ptr, self.X.ptr, self.Z.ptr
        d.xout = self.xout.ptr if self.xwrite else None
        d.zout = self.zout.ptr
        if self.dead is not None:
            for r in range(rank):
                d.dead_lo[r], d.dead_hi[r] = self.dead[r]
        d.plane0 = self.plane0
        d.zlo, d.zhi = self.zrange if self.zrange is not None else (0, self.Z.shape[0])
        d.global_d0 = self.global_d0 if self.global_d0 is not None else self.Z.shape[0]
        d.tpm_hint = self.tpm_hint
        self.desc = d
        self._ref = C.byref(d)

    def launch(self, rt, stream):
        L.check(rt.lib.gfb_star_pair_launch(self._ref, stream), "star_pair")


# ---------------------------------------------------------------------------
# lowering context


class LoopCtx:
    __slots__ = ("label", "iterates", "pos")

    def __init__(self, label, iterates, pos=0):
        self.label, self.iterates, self.pos = label, iterates, pos

    @property
    def current(self):
        return self.iterates[self.pos]


class _Elements:
    """The elements of an array a decision reads (snapshotted one by one
    instead of the whole array): ``x[(Ellipsis, *idx)]`` as numpy would
    index the full array."""

    def __init__(self, shape, idxs, values):
        self.shape = tuple(shape)
        vals = np.asarray(values).reshape(-1)
        self.map = {tuple(idx): vals[k] for k, idx in enumerate(idxs)}

    def __getitem__(self, key):
        idx = tuple(int(i) + (s if int(i) < 0 else 0) for i, s in zip(key[1:], self.shape))
        return self.map[idx]


def _element_view(buf: Buffer, lin: int) -> Buffer:
    """A one-element view of ``buf`` at linear element offset ``lin``."""
    v = Buffer(f"{buf.name}[{lin}]", (), buf.kind, fresh=False)
    v.alias_of = buf
    v.offset = lin
    return v


def static_reads(expr, bind: dict, shapes: dict):
    """Element indices of each array ``expr`` reads (``idx`` nodes) when
    every subscript is fixed by ``bind``; arrays with a data-dependent or
    out-of-range subscript are left out (snapshotted whole). Every ``idx``
    node is evaluated exactly once (``evaluate`` has no short-circuit), so
    this is exactly the set a condition reads."""
    out, whole = {}, set()

    def walk(e):
        t = type(e)
        if t is Index:
            shape = shapes.get(e.base)
            try:
                idx = tuple(int(evaluate(x, bind)) for x in e.indices)
            except GradflowError:
                idx = None
            if shape is None or idx is None or len(idx) != len(shape):
                whole.add(e.base)
            else:
                norm = tuple(i + s if i < 0 else i for i, s in zip(idx, shape))
                if all(0 <= i < s for i, s in zip(norm, shape)):
                    if norm not in out.setdefault(e.base, []):
                        out[e.base].append(norm)
                else:
                    whole.add(e.base)
            for x in e.indices:
                walk(x)
        elif t is Binary:
            walk(e.x)
            walk(e.y)
        elif t is Unary:
            walk(e.x)

    walk(expr)
    return {n: v for n, v in out.items() if n not in whole}


def _host_index(vals: dict, base: str, idx: tuple):
    """``idx`` read in a condition (reference symexpr.py:180-184: numpy
    indexing of the env array, so negative indices wrap)."""
    if base not in vals:
        raise UnboundName(f"no array available for '{base}'")
    return vals[base][(Ellipsis, *idx)]


class LTape:
    """Lowering-time image of the reference Tape (interpreter.py:70-75)."""

    def __init__(self):
        self.values = {}           # (data, version, coords) -> Buffer
        self.branch_trace = {}     # label -> [bool]
        self.iterate_records = {}  # label -> {coords: [int]}


class NeedValues(Exception):
    """Raised while lowering when control flow reads runtime data: a
    data-dependent branch condition (reference interpreter.py:342-347) or a
    loop header bound to a scalar (``_header_bindings``, :210-219).

    ``slots`` maps each data name to a device snapshot taken at that point of
    the launch list. The caller (``api.probe_lower``) runs the launches
    emitted so far, reads the snapshots back and lowers again with the values
    appended to ``Lowering.known``; the finished launch list keeps the
    snapshots, and ``Executable`` re-checks every decision after each run."""

    def __init__(self, slots: dict):
        super().__init__("runtime values needed: " + ", ".join(sorted(slots)))
        self.slots = slots


class Lowering:
    """Accumulates launches for one or more program runs over shared buffers."""

    def __init__(self, *, trip_limit=None, fuse_small=False, known=None):
        self.fuse_small = fuse_small  # fuse small 3-D domains too (slab decomposition needs fused pairs)
        # runtime control-flow values observed by earlier probe runs, in
        # decision order; decisions = [(slots, key_fn, key)] taken this lowering
        self.known: list = list(known or [])
        # incremental prober (api.probe_lower): runs the launches emitted
        # since the previous decision and returns the snapshot values, so a
        # decision no longer restarts the lowering (None: raise NeedValues)
        self.probe = getattr(known, "probe", None)
        self.decisions: list = []
        self.entry_inputs: dict = {}  # caller name -> Buffer (for probe runs of a prefix)
        self.entry_seed = None
        self.ops: list[Op] = []
        self.buffers: list[Buffer] = []
        self.flops = 0
        self.trip_limit = trip_limit if trip_limit is not None else default_trip_limit()

    def new_buffer(self, name, shape, kind, *, fresh=True) -> Buffer:
        b = Buffer(name, shape, kind, fresh=fresh)
        self.buffers.append(b)
        return b

    def emit(self, op: Op):
        if len(self.ops) >= MAX_UNROLLED_OPS:
            raise UnsupportedConstruct(
                f"program unrolls to more than {MAX_UNROLLED_OPS} launches (sequential scalar loop nest); "
                "express the parallel work as a map")
        self.ops.append(op)

    # -- pending clears -------------------------------------------------------

    def materialize(self, buf: Buffer):
        if buf.pending is not None:
            box = buf.pending
            buf.pending = None
            if box_size(box) > 0:
                self.emit(FillOp(buf, box))

    def add_clear(self, buf: Buffer, box):
        if box_size(box) == 0:
            return
        if buf.pending is None or box_contains(box, buf.pending):
            buf.pending = box
        elif box_contains(buf.pending, box):
            pass
        else:
            self.materialize(buf)
            buf.pending = box

    # -- post passes -------------------------------------------------------------

    def finish(self, observed: list):
        for b in observed:
            self.materialize(b)
        if os.environ.get("GFB_FUSE", "1") != "0":
            self._fuse_star_pairs(observed)
            if os.environ.get("GFB_SYNC_ELIDE", "1") != "0":
                self._elide_synced_copies()
        if os.environ.get("GFB_FUSE_MV", "1") != "0":
            self._fuse_matvec_pairs()
            self._fuse_rank2()
        self._stencil_copies()
        self._elide_copies()

    def resolve(self, buf: Buffer) -> Buffer:
        """Physical buffer holding ``buf``'s final value (after ping-pong)."""
        return self.final.get(buf.bid, buf) if hasattr(self, "final") else buf

    def _fuse_star_pairs(self, observed):
        """Fuse adjacent radius-1 star sweeps X = a(Y); Z = b(X) into one
        launch, then place ping-pong physical buffers."""
        ops = self.ops
        obs = {b.bid for b in observed}
        small_bytes = 0 if self.fuse_small else small_fuse_bytes()
        fused, i = [], 0
        while i < len(ops):
            a = ops[i]
            b = ops[i + 1] if i + 1 < len(ops) else None
            fa, fb = star_form(a), star_form(b) if b is not None else None
            # small 3-D domains stay unfused: they are L2-resident, so fusion
            # saves no DRAM traffic, while a short march pays the fused
            # kernel's dim-0 halo recompute (C2 heat_3d, N = 70: 3.1 vs 3.8 ms)
            small3d = fa is not None and len(a.dst.shape) == 3 and a.dst.nbytes < small_bytes
            if (fa and fb and not small3d and a.dst.shape == b.dst.shape and a.dst.kind == b.dst.kind
                    and fb[0] is a.dst and fa[0] is not a.dst and b.dst is not a.dst):
                xwrite, dead = self._x_liveness(a.dst, i + 2, obs)
                fused.append(StarPairOp(a, b, fa, fb, xwrite, dead))
                i += 2
            else:
                fused.append(a)
                i += 1
        if len(fused) == len(ops):
            return
        # placement: every fused pair writes Z (and a live X) into the other
        # physical buffer of a two-buffer ring when the old value is still
        # being read by neighbouring CTAs during the launch
        cur, alt = {}, {}

        def phys(b):
            return cur.get(b.bid, b)

        def other(logical: Buffer, now: Buffer) -> Buffer:
            ring = alt.get(logical.bid)
            if ring is None:
                twin = self.new_buffer(logical.name + "~pp", logical.shape, logical.kind, fresh=False)
                ring = alt[logical.bid] = (logical, twin)
            return ring[1] if now is ring[0] else ring[0]

        for op in fused:
            if isinstance(op, StarPairOp):
                X, Y, Z = op.X, op.Y, op.Z
                op.remap(phys)
                if Z is Y:
                    op.zout = other(Z, op.Z)
                    cur[Z.bid] = op.zout
                if op.xwrite:
                    op.xout = other(X, op.X)
                    cur[X.bid] = op.xout
                op._refresh()
            else:
                op.remap(phys)
        self.final = dict(cur)
        self.ops = fused

    def _elide_synced_copies(self):
        """Outside its region a fused sweep copies the old value into the
        ping-pong twin. Track, in launch order, which twin pairs are known to
        hold equal values outside which region; a copy into a twin that
        already holds it is skipped (heat_3d / jacobi_2d: every timestep after
        the first two). Any other write to a buffer forgets its pairs."""
        synced = set()  # (frozenset of two root bids, region)

        def forget(b):
            r = b.root().bid
            for e in [e for e in synced if r in e[0]]:
                synced.discard(e)

        for op in self.ops:
            if not isinstance(op, StarPairOp):
                for b in op.writes:
                    forget(b)
                continue
            Z, zout = op.Z.root(), op.zout.root()
            X, xout = op.X.root(), op.xout.root()
            if zout is not Z:
                key = (frozenset((Z.bid, zout.bid)), tuple(op.b.region))
                op.skip_zcopy = key in synced
            if op.xwrite and xout is not X:
                xkey = (frozenset((X.bid, xout.bid)), tuple(op.a.region))
                op.skip_xcopy = xkey in synced
            # after the launch: the targets changed inside the regions, and
            # hold their old twins' values outside
            forget(op.zout)
            if zout is not Z:
                synced.add((frozenset((Z.bid, zout.bid)), tuple(op.b.region)))
            if op.xwrite:
                forget(op.xout)
                full = op.dead is None or box_contains(op.a.region, op.dead)
                if xout is not X and full:
                    synced.add((frozenset((X.bid, xout.bid)), tuple(op.a.region)))

    def _stencil_copies(self):
        """A one-tap identity sweep over the whole array that overwrites its
        target (the adjoint of `h = z + b` into a fresh z__grad) is a copy;
        as a CopyOp it can become an alias (_elide_copies) instead of a launch."""
        for i, op in enumerate(self.ops):
            if not (isinstance(op, StencilOp) and len(op.taps) == 1):
                continue
            whole = whole_box(op.dst.shape)
            overwrite = op.clear_mode in (1, 3) or (op.clear_mode == 2 and op.clear_box is not None
                                                    and box_contains(op.clear_box, whole))
            if not overwrite:
                continue
            si, coef, delta, mask = op.taps[0]
            src = op.srcs[si]
            if (coef == 1.0 and mask is None and not any(delta) and src is not op.dst and src.shape == op.dst.shape
                    and src.kind == op.dst.kind and box_contains(op.region, whole)):
                self.ops[i] = CopyOp(op.dst, src)

    def _fuse_matvec_pairs(self):
        """Pair a row-dot and a column-sum matmul node over the same matrix
        into one MatvecPairOp at the earlier position (one read of the matrix
        instead of two). Legal when the later node's operands are not written
        and its output not touched in between, and neither output aliases an
        operand; the chain form (column sums of the row-dot result, atax) needs
        the row dots first."""
        ops = self.ops
        out, used = [], set()
        for i, a in enumerate(ops):
            if i in used:
                continue
            fa = matvec_form(a)
            if fa is None:
                out.append(a)
                continue
            pair = None
            for j in range(i + 1, len(ops)):
                if j in used:
                    continue
                b = ops[j]
                fb = matvec_form(b)
                if fb is not None and same_buffer(fa[0], fb[0]) and {fa[1], fb[1]} == {"row", "col"}:
                    if self._pair_legal(a, fa, b, fb, ops[i + 1:j]):
                        pair = (j, b, fb)
                    break
                # stop at anything that rewrites the matrix
                if any(overlaps(w, fa[0]) for w in b.writes):
                    break
            if pair is None:
                out.append(a)
                continue
            j, b, fb = pair
            used.add(j)
            row, col = (a, b) if fa[1] == "row" else (b, a)
            fr, fc = matvec_form(row), matvec_form(col)
            chain = fc[2] is fr[3]
            out.append(MatvecPairOp([a, b], fr[0], fr[2], fr[3], row.accumulate, None if chain else fc[2], fc[3],
                                    col.accumulate, chain))
        self.ops = out

    @staticmethod
    def _pair_legal(a, fa, b, fb, between) -> bool:
        mat = fa[0]
        chain = fb[2] is fa[3]
        if chain and fa[1] != "row":
            return False
        ins_a, ins_b = [fa[0], fa[2]], [fb[0]] + ([] if chain else [fb[2]])
        if overlaps(fa[3], fb[3]):
            return False
        for o in (fa[3], fb[3]):
            if any(overlaps(o, x) for x in ins_a + ins_b):
                return False
        if not chain and overlaps(fb[2], fa[3]):
            return False
        for op in between:
            for w in op.writes:
                if overlaps(w, mat) or overlaps(w, fb[3]) or any(overlaps(w, x) for x in ins_b):
                    return False
                if chain and overlaps(w, fa[3]):
                    return False
            if any(overlaps(rd, fb[3]) for rd in op.reads):
                return False
        return True

    def _fuse_rank2(self):
        """Merge two outer-product nodes into the same matrix (the second one
        accumulating) into one Rank2Op at the later position, when nothing in
        between touches the target or rewrites the first node's vectors."""
        ops = self.ops
        drop, repl = set(), {}
        for i, a in enumerate(ops):
            fa = rank1_form(a)
            if fa is None or i in drop:
                continue
            if any(overlaps(fa[2], x) for x in fa[:2]):
                continue
            for j in range(i + 1, len(ops)):
                b = ops[j]
                fb = rank1_form(b)
                if fb is not None and same_buffer(fb[2], fa[2]) and b.accumulate and j not in repl:
                    if not any(overlaps(fb[2], x) for x in fb[:2]):
                        drop.add(i)
                        repl[j] = Rank2Op([a, b], fa[0], fa[1], fb[0], fb[1], fa[2], a.accumulate)
                    break
                if any(overlaps(w, x) for w in b.writes for x in fa) or any(overlaps(rd, fa[2]) for rd in b.reads):
                    break
        self.ops = [repl.get(k, op) for k, op in enumerate(ops) if k not in drop]

    def _x_liveness(self, X: Buffer, start: int, obs: set):
        """(write X back?, dead box) for the intermediate of a fused pair."""
        whole = whole_box(X.shape)
        for op in self.ops[start:]:
            touches_read = any(b is X for b in op.reads)
            touches_write = any(b is X for b in op.writes)
            if not (touches_read or touches_write):
                continue
            if isinstance(op, StencilOp) and op.dst is X and not any(s is X for s in op.srcs):
                if op.clear_mode in (1, 3):
                    dead = op.region
                elif op.clear_mode == 2:
                    dead = op.clear_box
                else:
                    return True, None
                if box_contains(dead, whole):
                    return False, None
                return True, dead
            return True, None
        return (X.bid in obs), None

    def _elide_copies(self):
        """Copies whose source and destination are never written afterwards
        (tape snapshots, plan keep-copies) become aliases."""
        # keyed by root buffer: a write through a view writes its root
        last_write = {}
        first_touch = {}
        for i, op in enumerate(self.ops):
            for b in op.writes:
                last_write[b.root().bid] = i
            for b in tuple(op.reads) + tuple(op.writes):
                first_touch.setdefault(b.root().bid, i)
        for i, op in enumerate(self.ops):
            if not isinstance(op, CopyOp):
                continue
            src, dst = op.src, op.dst
            if last_write.get(src.root().bid, -1) > i or last_write.get(dst.root().bid, -1) > i:
                continue
            if first_touch.get(dst.root().bid, i) < i or dst.alias_of is not None:
                continue
            if src.root() is dst.root():
                continue
            dst.alias_of = src
            op.elided = True


class ProgramRun:
    """Lowers one program execution (the reference Executor.run)."""

    def __init__(self, low: Lowering, program, params: dict, env: dict, *, record=None, tape: LTape | None = None,
                 src_tape: LTape | None = None, forwarding=None, versions=None):
        self.low = low
        self.program = program
        self.params = dict(params)
        self.bind = dict(params)
        self.env = env
        self.record = record
        self.tape = tape
        self.src_tape = src_tape
        self.forwarding = forwarding or {}
        self.versions = versions  # (version_of, loops_of) or None
        self.ctx = {}
        self.ctx_stack = []
        self.branch_down = {}
        self._shapes = {}

    # -- env -------------------------------------------------------------------

    def shape_of(self, name) -> tuple:
        s = self._shapes.get(name)
        if s is None:
            desc = self.program.descriptors[name]
            s = tuple(eval_int(d, self.params, f"dimension of '{name}'") for d in desc.shape)
            self._shapes[name] = s
        return s

    def read(self, name: str) -> Buffer:
        b = self.env.get(name)
        if b is not None:
            return b
        if name in self.forwarding:
            return self.fetch_forwarded(name)
        desc = self.program.descriptors.get(name)
        if desc is None or desc.role == "input":
            raise UnboundName(f"no value for input '{name}'")
        return self._fresh(name)

    def write(self, name: str) -> Buffer:
        b = self.env.get(name)
        if b is None:
            if name not in self.program.descriptors:
                raise UnboundName(f"'{name}' is not declared")
            b = self._fresh(name)
        return b

    def _fresh(self, name) -> Buffer:
        desc = self.program.descriptors[name]
        b = self.low.new_buffer(name, self.shape_of(name), desc.element_kind, fresh=True)
        self.env[name] = b
        return b

    def fetch_forwarded(self, name) -> Buffer:
        entry = self.forwarding[name]
        if self.src_tape is None:
            raise MissingTapeValue(f"'{name}' requested but no tape is attached")
        for cand in entry.candidates:
            coords = self._cand_coords(cand.directives)
            if coords is None:
                continue
            slot = self.src_tape.values.get((entry.data, cand.version, coords))
            if slot is not None:
                return slot
        raise MissingTapeValue(f"no recorded instance of '{entry.data}' matches '{name}' here")

    def _cand_coords(self, directives):
        coords = []
        for j, (label, kind) in enumerate(directives):
            ctx = self.ctx.get(label)
            if kind == "cur":
                if ctx is None:
                    return None
                coords.append(ctx.current)
            elif kind == "prev":
                if ctx is None or ctx.pos == 0:
                    return None
                coords.append(ctx.iterates[ctx.pos - 1])
            elif kind == "last":
                if ctx is not None:
                    coords.append(ctx.iterates[-1])
                else:
                    recs = (self.src_tape.iterate_records if self.src_tape else {}).get(label)
                    if not recs:
                        return None
                    seq = recs.get(tuple(coords[:j]))
                    if not seq:
                        return None
                    coords.append(seq[-1])
        return tuple(coords)

    # -- control flow ----------------------------------------------------------

    def run(self):
        self.region(self.program.region)

    def region(self, blocks):
        for b in blocks:
            if isinstance(b, State):
                self.state(b)
            elif isinstance(b, LoopRegion):
                self.loop(b)
            else:
                self.branch(b)

    def runtime_values(self, names, key_fn, reads=None) -> dict:
        """Host values of the data ``names`` at this point of the program.

        Emits a device snapshot of each (so later writes do not disturb it)
        and returns the values a probe run observed for this decision. With a
        prober (``Lowering.probe``) the launches emitted so far run now;
        without one, ``NeedValues`` is raised for the caller to probe and
        lower again. ``key_fn(values)`` is what the decision depends on (a
        branch outcome, a loop's header scalars): the executable re-evaluates
        it from the snapshots after every run and rebuilds when it changes.

        ``reads`` maps an array name to the element indices the decision
        reads (static under the current bindings): only those elements are
        snapshotted, and ``key_fn`` sees them through ``_Elements``; other
        names are snapshotted whole."""
        low = self.low
        slots, specs = {}, {}
        i = len(low.decisions)
        for n in sorted(names):
            src = self.env.get(n)
            if src is None:
                continue  # unbound: evaluation raises UnboundName as in the reference
            low.materialize(src)
            idxs = (reads or {}).get(n)
            if idxs is not None and src.shape:
                slot = low.new_buffer(f"{n}@probe{i}", (len(idxs),), src.kind, fresh=False)
                for k, idx in enumerate(idxs):
                    lin = int(sum(int(x) * st for x, st in zip(idx, src.strides)))
                    low.emit(CopyOp(_element_view(slot, k), _element_view(src, lin)))
                specs[n] = (src.shape, idxs)
            else:
                slot = low.new_buffer(f"{n}@probe{i}", src.shape, src.kind, fresh=False)
                low.emit(CopyOp(slot, src))
            slots[n] = slot
        if specs:
            inner = key_fn

            def key_fn(raw, inner=inner, specs=specs):
                return inner({n: _Elements(*specs[n], v) if n in specs else v for n, v in raw.items()})

        if i >= len(low.known):
            if low.probe is None:
                nv = NeedValues(slots)
                nv.low = low
                raise nv
            low.known.append(low.probe(low, slots))
        raw = low.known[i]
        low.decisions.append((slots, key_fn, key_fn(raw)))
        return {n: _Elements(*specs[n], v) if n in specs else v for n, v in raw.items()}

    def _header_bind(self, loop):
        need = (free_names(loop.init) | free_names(loop.bound) | free_names(loop.update)) - {loop.iterator}
        data = {n for n in need if n not in self.bind and n in self.program.descriptors
                and self.program.descriptors[n].rank == 0}
        if not data:
            return dict(self.bind)
        label = loop.label

        def key(vals, label=label):
            out = []
            for n in sorted(vals):
                f = float(vals[n].reshape(-1)[0])
                if not f.is_integer():
                    raise DomainError(f"scalar '{n}' in a loop header evaluated to non-integer {f} "
                                      f"(loop '{label}')")
                out.append(int(f))
            return tuple(out)

        vals = self.runtime_values(data, key)
        b = dict(self.bind)
        b.update(zip(sorted(vals), key(vals)))
        return b

    def simulate(self, loop) -> list:
        b = self._header_bind(loop)
        out = []
        i = eval_int(loop.init, b, f"init of '{loop.label}'")
        lt = loop.cmp == "<"
        while True:
            bound = eval_int(loop.bound, b, f"bound of '{loop.label}'")
            if not (i < bound if lt else i > bound):
                break
            out.append(i)
            if len(out) > self.low.trip_limit:
                raise NonTermination(f"loop '{loop.label}' exceeded the trip limit of {self.low.trip_limit}")
            b[loop.iterator] = i
            i = eval_int(loop.update, b, f"update of '{loop.label}'")
        return out

    # nests of at least this many iterations are tried as hyperplane wavefronts
    WAVE_MIN = int(os.environ.get("GFB_WAVE_MIN", "256"))

    def _wavefront(self, loop) -> bool:
        """A perfectly nested loop nest whose innermost body is one state with
        one scalar tasklet (the reference visits it point by point in loop
        order, interpreter.py:221-330, 396-426), lowered to ONE launch that
        runs hyperplanes of the iteration space in order (WavefrontOp).

        Every array the tasklet writes must be accessed (read and written)
        through subsets of the form x_p + const along each dimension (one
        loop iterator per dimension, shared by all its accesses). Two
        iterations X1 before X2 touch one element through accesses o1, o2
        iff X2 - X1 = o1 - o2 on the subscripted iterators; iterators absent
        from the subscripts (the time loop) are unconstrained. A hyperplane
        sum_p c_p k_p (k_p = execution index of loop p) with c . (X2 - X1) >= 1
        for all such pairs, at least one of the two a write, orders every
        conflicting pair as the sequential nest does (hyperplane()). Returns
        False (the caller unrolls) when the shape or the proof fails."""
        nest, cur = [], loop
        while True:
            if (not isinstance(cur, LoopRegion) or cur.replay_of is not None or cur.reversed_simulate
                    or cur.label in self.ctx):
                return False
            nest.append(cur)
            if len(cur.body) != 1:
                return False
            inner = cur.body[0]
            if isinstance(inner, State):
                state = inner
                break
            cur = inner
        if len(nest) > 4:  # the hyperplane search is exhaustive over small coefficients
            return False
        comp = [n for n in state.graph.nodes if not isinstance(n, AccessNode)]
        if len(comp) != 1 or not isinstance(comp[0], Tasklet):
            return False
        t = comp[0]
        iters = [lp.iterator for lp in nest]
        if len(set(iters)) != len(iters) or any(i in self.bind for i in iters):
            return False
        for lp in nest:
            names = free_names(lp.init) | free_names(lp.bound) | free_names(lp.update)
            if names & (set(iters) - {lp.iterator}):
                return False  # not rectangular
        # recorded values inside the nest (tape) need the per-point walk
        if self.tape is not None and self.versions is not None and self.record:
            version_of, _ = self.versions
            for n in state.graph.nodes:
                if isinstance(n, AccessNode):
                    v = version_of.get((state.label, n.id))
                    if v is not None and self._want(n.data, v):
                        return False
        seqs = [self.simulate(lp) for lp in nest]
        lo, hi, step = [], [], []
        for sq in seqs:
            if not sq:
                return False
            st = sq[1] - sq[0] if len(sq) > 1 else 1
            if st == 0 or any(b - a != st for a, b in zip(sq, sq[1:])):
                return False
            lo.append((sq[0], [0] * len(nest)))
            hi.append((sq[0] + st * len(sq), [0] * len(nest)))
            step.append(st)
        total = int(np.prod([len(sq) for sq in seqs], dtype=np.int64))
        if total < self.WAVE_MIN:
            return False
        space = SpaceInfo(iters, lo, hi, step)
        in_edges, out_edges = state.graph.in_edges(t.id), state.graph.out_edges(t.id)
        written = {e.data for e in out_edges}
        # per written array: every access is dim d = x_{p(d)} + off_d
        accs = {}
        for e, is_w in [(e, False) for e in in_edges] + [(e, True) for e in out_edges]:
            if e.data not in written:
                continue
            forms = [affine_form(x, self.bind, tuple(iters), f"subset of '{e.data}'") for x in (e.subset or ())]
            pos, offs = [], []
            for c0, coefs in forms:
                nz = [p for p, v in enumerate(coefs) if v != 0]
                if len(nz) > 1 or (nz and coefs[nz[0]] != 1):
                    return False
                pos.append(nz[0] if nz else None)
                offs.append(c0)
            accs.setdefault(e.data, []).append((tuple(pos), tuple(offs), is_w))
        deps = []
        D = len(nest)
        for data, lst in accs.items():
            shapes = {a[0] for a in lst}
            if len(shapes) != 1:
                return False
            pos = next(iter(shapes))
            used = [p for p in pos if p is not None]
            if len(used) != len(set(used)):
                return False
            free = frozenset(p for p in range(D) if p not in used)
            for (_, o1, w1), (_, o2, w2) in itertools.product(lst, lst):
                if not (w1 or w2):
                    continue
                # constant subscripts must agree for the element to be shared
                if any(pp is None and a != b for pp, a, b in zip(pos, o1, o2)):
                    continue
                fixed = {}
                for pp, a, b in zip(pos, o1, o2):
                    if pp is None:
                        continue
                    dx = a - b  # X2 - X1 in iterator units
                    if dx % step[pp]:
                        fixed = None
                        break
                    fixed[pp] = dx // step[pp]
                if fixed is None:
                    continue
                deps.append((fixed, free))
        c = hyperplane([len(sq) for sq in seqs], deps)
        if c is None:
            return False
        # operands (bounds-checked over the whole nest) and the body code
        ins = {e.dst_conn: self.access(self.read(e.data), e.subset, space, f"loop nest '{loop.label}'")
               for e in in_edges}
        outs = [(e.src_conn, self.access(self.write(e.data), e.subset, space, f"loop nest '{loop.label}'"), e.wcr)
                for e in out_edges]
        self.low.flops += sum(count_ops(t.body[e.src_conn]) for e in out_edges) * total
        for a in list(ins.values()) + [a for _, a, _ in outs]:
            self.low.materialize(a.buf)
        conns = list(ins)
        if len(conns) > L.MAXIN or len(outs) > L.MAXOUT:
            return False
        code = Code()
        ci = {cn: k for k, cn in enumerate(conns)}
        segs = [code.compile(t.body[conn], ci) for conn, _, _ in outs]
        compute_f64 = any(a.buf.kind == "real64" for a in ins.values()) or not ins
        op = WavefrontOp(space, [ins[cn] for cn in conns], [(a, 1 if w == "sum" else 0) for _, a, w in outs],
                         code, segs, compute_f64, c)
        self.low.emit(op)
        if self.tape is not None:
            # the iterate records the per-point walk leaves for a reverse pass
            # that replays loops (reference Tape.iterate_records); constant-
            # step headers reverse in closed form, so only bounded record sets
            # are kept (a replay that needs more raises MissingTapeValue)
            key0 = tuple(cc.current for cc in self.ctx_stack)
            n_outer = 1
            for depth, lp in enumerate(nest):
                if n_outer > 4096:
                    break
                recs = self.tape.iterate_records.setdefault(lp.label, {})
                for outer in itertools.product(*seqs[:depth]):
                    recs[key0 + tuple(outer)] = list(seqs[depth])
                n_outer *= len(seqs[depth])
        return True

    def loop(self, loop):
        if os.environ.get("GFB_WAVEFRONT", "1") != "0" and self._wavefront(loop):
            return
        if loop.replay_of is not None:
            if self.src_tape is None:
                raise MissingInverse(
                    f"loop '{loop.replay_of}' has a non-affine header and no declared inverse; "
                    "reversing it requires recorded iterates")
            key = tuple(c.current for c in self.ctx_stack)
            recs = self.src_tape.iterate_records.get(loop.replay_of, {})
            if key not in recs:
                raise MissingTapeValue(f"no recorded iterates for loop '{loop.replay_of}' at {key}")
            self.iterates(loop, recs[key], loop.replay_of, reverse=True)
        elif loop.reversed_simulate:
            fwd = self.simulate(loop)
            self.inverse(loop, fwd, loop.reverse_of or loop.label)
        elif loop.reverse_of is not None:
            order = self.simulate(loop)
            self.iterates(loop, order[::-1], loop.reverse_of, reverse=True)
        else:
            its = self.simulate(loop)
            if self.tape is not None:
                key = tuple(c.current for c in self.ctx_stack)
                self.tape.iterate_records.setdefault(loop.label, {})[key] = list(its)
            self.iterates(loop, its, loop.label, reverse=False)

    def _enter(self, loop, label, fwd):
        ctx = LoopCtx(label, fwd)
        self.ctx[label] = ctx
        self.ctx_stack.append(ctx)
        return ctx, loop.iterator in self.bind, self.bind.get(loop.iterator)

    def _leave(self, loop, label, had, saved):
        self.ctx_stack.pop()
        del self.ctx[label]
        if had:
            self.bind[loop.iterator] = saved
        else:
            self.bind.pop(loop.iterator, None)

    def iterates(self, loop, fwd, label, reverse):
        ctx, had, saved = self._enter(loop, label, fwd)
        try:
            positions = range(len(fwd) - 1, -1, -1) if reverse else range(len(fwd))
            for pos in positions:
                ctx.pos = pos
                self.bind[loop.iterator] = fwd[pos]
                self.region(loop.body)
        finally:
            self._leave(loop, label, had, saved)

    def inverse(self, loop, fwd, label):
        if not fwd:
            return
        ctx, had, saved = self._enter(loop, label, fwd)
        try:
            i = fwd[-1]
            for pos in range(len(fwd) - 1, -1, -1):
                ctx.pos = pos
                if i != fwd[pos]:
                    raise DomainError(f"declared inverse of loop '{loop.label}' diverges: expected {fwd[pos]}, got {i}")
                self.bind[loop.iterator] = i
                self.region(loop.body)
                if pos > 0:
                    i = eval_int(loop.inverse, dict(self.bind), f"inverse of '{loop.label}'")
        finally:
            self._leave(loop, label, had, saved)

    def branch(self, br):
        if br.trace_ref is not None:
            outcomes = (self.src_tape.branch_trace if self.src_tape else {}).get(br.trace_ref)
            if not outcomes:
                raise MissingTapeValue(f"no recorded outcomes for branch '{br.trace_ref}'")
            cursor = self.branch_down.get(br.trace_ref, len(outcomes)) - 1
            if cursor < 0:
                raise MissingTapeValue(f"branch trace of '{br.trace_ref}' exhausted")
            self.branch_down[br.trace_ref] = cursor
            outcome = outcomes[cursor]
        else:
            data = (free_names(br.condition) & set(self.program.descriptors)) - set(self.bind)
            if data:
                cond, label = br.condition, br.label
                descs = self.program.descriptors

                # the bindings that hold at the decision point (loop iterators
                # included): the key is re-evaluated after lowering, when the
                # live self.bind no longer holds them
                def key(vals, cond=cond, label=label, bind=dict(self.bind)):
                    b = dict(bind)
                    b.update({n: v.reshape(()).item() for n, v in vals.items() if descs[n].rank == 0})
                    return bool(evaluate(cond, b, lambda base, idx: _host_index(vals, base, idx)))

                shapes = {n: self.env[n].shape for n in data if n in self.env}
                outcome = key(self.runtime_values(data, key, static_reads(cond, self.bind, shapes)))
            else:
                outcome = bool(evaluate(br.condition, dict(self.bind)))
            if self.tape is not None:
                self.tape.branch_trace.setdefault(br.label, []).append(outcome)
        self.region(br.then_body if outcome else br.else_body)

    # -- states -----------------------------------------------------------------

    def state(self, st: State):
        by_id = {n.id: n for n in st.graph.nodes}
        for nid in schedule(st.graph):
            node = by_id[nid]
            if isinstance(node, AccessNode):
                self.visit_access(st.label, node)
            elif isinstance(node, Tasklet):
                self.map_like(None, node, st.graph)
            elif isinstance(node, LibraryNode):
                self.library(node, st.graph)
            else:
                self.map_node(node)

    def visit_access(self, label, node):
        if self.tape is None or self.versions is None or self.record is None:
            return
        version_of, loops_of = self.versions
        v = version_of.get((label, node.id))
        if v is None or not self._want(node.data, v):
            return
        coords = tuple(self.ctx[l].current for l in loops_of[(node.data, v)])
        self.snapshot(node.data, v, coords)

    def _want(self, data, v):
        return self.record == "all" or (data, v) in self.record

    def snapshot(self, data, v, coords):
        src = self.read(data)
        self.low.materialize(src)
        slot = self.low.new_buffer(f"{data}@v{v}{list(coords) if coords else ''}", src.shape, src.kind, fresh=False)
        self.low.emit(CopyOp(slot, src))
        self.tape.values[(data, v, coords)] = slot

    # -- maps and tasklets --------------------------------------------------------

    def build_space(self, node: MapNode) -> SpaceInfo:
        lo, hi, step = [], [], []
        params = node.params
        for k, (start, stop, st) in enumerate(node.ranges):
            lo.append(affine_form(start, self.bind, params[:k], f"map '{node.id}' start"))
            hi.append(affine_form(stop, self.bind, params[:k], f"map '{node.id}' stop"))
            s = affine_form(st, self.bind, params[:k], f"map '{node.id}' step")
            if any(s[1]):
                raise UnsupportedConstruct(f"map '{node.id}' step depends on map parameters")
            if s[0] <= 0:
                raise DomainError(f"map '{node.id}' step must be positive, got {s[0]}")
            step.append(s[0])
        return SpaceInfo(params, lo, hi, step)

    def map_node(self, node: MapNode):
        computes = [n for n in node.body.nodes if not isinstance(n, AccessNode)]
        if len(computes) != 1 or not isinstance(computes[0], Tasklet):
            raise UnsupportedConstruct(f"map '{node.id}': the engine lowers single-tasklet map bodies")
        space = self.build_space(node)
        saved = {p: self.bind[p] for p in node.params if p in self.bind}
        try:
            self.map_like(space, computes[0], node.body, node_id=node.id)
        finally:
            for p in node.params:
                self.bind.pop(p, None)
            self.bind.update(saved)

    def access(self, buf: Buffer, subset, space: SpaceInfo, what: str) -> Access:
        params = space.params if space else ()
        rank = len(buf.shape)
        if subset is None or len(subset) != rank:
            raise UnsupportedConstruct(f"{what}: element subset of rank {rank} required")
        forms = [affine_form(e, self.bind, params, f"subset of '{buf.name}'") for e in subset]
        # static bounds check over the whole iteration space (reference
        # checks each access at run time, interpreter.py:396-403)
        for k, f in enumerate(forms):
            if space is None:
                lo = hi = f[0]
            else:
                lo, hi = space.range_of(f)
            if lo < 0 or hi >= buf.shape[k]:
                if space is not None and space.triangular and space.box_points() <= (1 << 22):
                    lo, hi = self._exact_range(space, f)
                if lo < 0 or hi >= buf.shape[k]:
                    bad = lo if lo < 0 else hi
                    raise OutOfBounds(f"'{buf.name}' index {bad} outside dimension of size {buf.shape[k]}")
        return Access(buf, forms)

    @staticmethod
    def _exact_range(space: SpaceInfo, form):
        grids = np.meshgrid(*[np.arange(f, l + 1) for f, l in zip(space.first, space.last)], indexing="ij")
        pts = np.stack([g.reshape(-1) for g in grids], axis=1)
        ok = np.ones(len(pts), dtype=bool)
        for p in range(space.np):
            lo = space.lo[p][0] + sum(c * pts[:, q] for q, c in enumerate(space.lo[p][1]))
            hi = space.hi[p][0] + sum(c * pts[:, q] for q, c in enumerate(space.hi[p][1]))
            ok &= (pts[:, p] >= lo) & (pts[:, p] < hi) & ((pts[:, p] - lo) % space.step[p] == 0)
        v = form[0] + pts[ok] @ np.asarray(form[1], dtype=np.int64)
        return (int(v.min()), int(v.max())) if v.size else (0, 0)

    def map_like(self, space, t: Tasklet, df, node_id=None):
        """Lower one tasklet, at state level (space None: a single point) or
        as the body of a map over ``space``."""
        what = f"map '{node_id}'" if node_id else f"tasklet '{t.id}'"
        if space is None:
            space = SpaceInfo((), [], [], [])
        npts = space.points()
        in_edges = df.in_edges(t.id)
        out_edges = df.out_edges(t.id)
        self.low.flops += sum(count_ops(t.body[e.src_conn]) for e in out_edges) * npts
        if npts == 0:
            return
        np_ = space.np
        ins = {}
        for e in in_edges:
            buf = self.read(e.data)
            ins[e.dst_conn] = self.access(buf, e.subset, space, what)
        outs = []
        for e in out_edges:
            buf = self.write(e.data)
            outs.append((e.src_conn, self.access(buf, e.subset, space, what), e.wcr))
        in_f64 = any(a.buf.kind == "real64" for a in ins.values())
        compute_f64 = in_f64 or not ins

        # classify outputs per target buffer
        by_buf = {}
        for conn, acc, wcr in outs:
            by_buf.setdefault(acc.buf.bid, []).append((conn, acc, wcr))
        read_bids = {a.buf.bid for a in ins.values()}
        pointwise, gathers = [], []
        if npts == 1 and any(len(g) > 1 for g in by_buf.values()):
            # one point writing one array several times: a single thread
            # applies the outputs in declaration order, like the reference
            for conn, acc, wcr in outs:
                self.low.materialize(acc.buf)
            for c in ins:
                self.low.materialize(ins[c].buf)
            self.lower_pointwise(space, t, outs, ins, compute_f64, what)
            return
        for bid, group in by_buf.items():
            inj = len(group) == 1 and self._injective(group[0][1], space)
            if bid in read_bids and npts > 1:
                # self-update: only the same element may be read and written
                wkeys = {g[1].key() for g in group}
                rkeys = {a.key() for a in ins.values() if a.buf.bid == bid}
                if not inj or rkeys != wkeys:
                    raise UnsupportedConstruct(
                        f"{what} reads and writes '{group[0][1].buf.name}' at different points "
                        "(cross-point dependence is not a parallel map)")
            if inj:
                pointwise.append(group[0])
            else:
                if any(w != "sum" for _, _, w in group):
                    raise UnsupportedConstruct(
                        f"{what} overwrites elements of '{group[0][1].buf.name}' from several points")
                gathers.append(group)
        gather_bids = {g[0][1].buf.bid for g in gathers}
        for group in gathers:
            used = self._used_inputs([t.body[c] for c, _, _ in group], ins)
            if any(ins[c].buf.bid in gather_bids for c in used):
                raise UnsupportedConstruct(f"{what}: a scatter-add target is also read by another scatter")
        pw_used = self._used_inputs([t.body[c] for c, _, _ in pointwise], ins)
        if any(ins[c].buf.bid in gather_bids for c in pw_used):
            raise UnsupportedConstruct(f"{what}: a scatter-add target is read by a pointwise output")

        # everything read must be materialized (pending clears resolved)
        for c in set(pw_used) | {c for g in gathers for c in self._used_inputs([t.body[x] for x, _, _ in g], ins)}:
            self.low.materialize(ins[c].buf)

        for group in gathers:
            self.lower_gather(space, t, group, ins, compute_f64, what)

        clears = []
        rest = []
        for conn, acc, wcr in pointwise:
            body = t.body[conn]
            if wcr is None and isinstance(body, Const) and float(body.value) == 0.0:
                img = self._image_box(acc, space)
                if img is not None:
                    clears.append((acc.buf, img))
                    continue
            rest.append((conn, acc, wcr))
        if rest:
            self.lower_pointwise(space, t, rest, ins, compute_f64, what)
        for buf, img in clears:
            self.low.add_clear(buf, img)

    @staticmethod
    def _used_inputs(exprs, ins):
        used = set()
        for e in exprs:
            used |= free_names(e)
        return [c for c in ins if c in used]

    @staticmethod
    def _injective(acc: Access, space: SpaceInfo) -> bool:
        live = [p for p in range(space.np) if space.ext[p] > 1]
        if not live:
            return True
        m = np.array([[f[1][p] for p in live] for f in acc.forms], dtype=np.float64).reshape(len(acc.forms), len(live))
        return int(np.linalg.matrix_rank(m)) == len(live) if m.size else False

    @staticmethod
    def _image_box(acc: Access, space: SpaceInfo):
        """Exact image of an injective access if it is a box, else None."""
        if space.triangular or any(s != 1 for s in space.step):
            return None if space.np else tuple((f[0], f[0] + 1) for f in acc.forms)
        used = set()
        box = []
        for c0, coefs in acc.forms:
            nz = [p for p, c in enumerate(coefs) if c != 0 and space.ext[p] > 1]
            if not nz:
                v = c0 + sum(c * space.first[p] for p, c in enumerate(coefs))
                box.append((v, v + 1))
                continue
            if len(nz) != 1 or abs(coefs[nz[0]]) != 1 or nz[0] in used:
                return None
            used.add(nz[0])
            lo, hi = space.range_of((c0, coefs))
            box.append((lo, hi + 1))
        return tuple(box)

    # -- pointwise ---------------------------------------------------------------

    def lower_pointwise(self, space, t, outs, ins, compute_f64, what):
        # stencil fast path: a single linear output over identity+offset subsets
        if len(outs) == 1:
            op = self._broadcast_pointwise(space, t, outs[0], ins) or self._stencil_pointwise(space, t, outs[0], ins)
            if op is not None:
                self.low.emit(op)
                return
        conns = list(ins)
        if len(conns) > L.MAXIN or len(outs) > L.MAXOUT:
            raise UnsupportedConstruct(f"{what}: too many connectors for the device evaluator")
        code = Code()
        ci = {c: k for k, c in enumerate(conns)}
        segs, out_specs = [], []
        for conn, acc, wcr in outs:
            segs.append(code.compile(t.body[conn], ci))
            w = 1 if wcr == "sum" else 0
            buf = acc.buf
            if buf.pending is not None:
                img = self._image_box(acc, space)
                if w == 0 and img is not None and box_contains(img, buf.pending):
                    buf.pending = None
                elif w == 1 and img is not None and img == buf.pending:
                    buf.pending = None
                    w = 0
                else:
                    self.low.materialize(buf)
            out_specs.append((acc, w))
        op = map2_pointwise(space, [ins[c] for c in conns], out_specs, code, segs, compute_f64)
        self.low.emit(op or MapOp(space, [ins[c] for c in conns], out_specs, code, segs, compute_f64))

    def _broadcast_pointwise(self, space, t, out, ins):
        """`out[all] (+)= c * scalar` (the reduce_sum adjoint map,
        autodiff.py:940-960) as one streaming fill."""
        conn, acc, wcr = out
        if space.np == 0:
            return None
        lin = linearize(t.body[conn])
        if lin is None or len(lin[1]) > 1 or (lin[1] and lin[0] != 0.0):
            return None
        src, scale = None, lin[0]
        if lin[1]:
            (c, scale), = lin[1].items()
            if ins[c].buf.shape != () or ins[c].buf.kind != acc.buf.kind:
                return None
            src = ins[c].buf
        dst = acc.buf
        if self._image_box(acc, space) != whole_box(dst.shape) or not self._injective(acc, space):
            return None
        accumulate = wcr == "sum"
        if dst.pending is not None:
            if dst.pending == whole_box(dst.shape):
                accumulate = False
                dst.pending = None
            else:
                self.low.materialize(dst)
        if not accumulate:
            dst.pending = None
        return BroadcastOp(src, scale, dst, accumulate)

    def _stencil_pointwise(self, space, t, out, ins):
        conn, acc, wcr = out
        if space.triangular or space.np == 0 or space.np > 3 or any(s != 1 for s in space.step):
            return None
        lin = linearize(t.body[conn])
        if lin is None or lin[0] != 0.0 or not lin[1]:
            return None
        dst = acc.buf
        ooff = acc.identity_offset(space.np)
        if ooff is None or len(dst.shape) != space.np:
            return None
        srcs, taps = [], []
        for c, coef in lin[1].items():
            a = ins[c]
            if a.buf.shape != dst.shape or a.buf.kind != dst.kind or a.buf.bid == dst.bid:
                return None
            doff = a.identity_offset(space.np)
            if doff is None:
                return None
            if a.buf not in srcs:
                srcs.append(a.buf)
            if len(srcs) > L.MAXSRCS:
                return None
            taps.append((srcs.index(a.buf), coef, tuple(d - o for d, o in zip(doff, ooff)), None))
        if len(taps) > L.MAXTAPS:
            return None
        region = tuple((f + o, l + o + 1) for f, l, o in zip(space.first, space.last, ooff))
        mode, cbox = (3 if wcr is None else 0), None
        if dst.pending is not None:
            if mode == 3 and box_contains(region, dst.pending):
                dst.pending = None
            elif mode == 0 and box_contains(region, dst.pending):
                mode, cbox = 2, dst.pending
                dst.pending = None
            else:
                self.low.materialize(dst)
        return StencilOp(dst, srcs, region, mode, cbox, taps, kind="sweep")

    # -- gather -------------------------------------------------------------------

    def lower_gather(self, space, t, group, ins, compute_f64, what):
        dst = group[0][1].buf
        rank = len(dst.shape)
        ybox = None
        for _, acc, _ in group:
            b = tuple((lo, hi + 1) for lo, hi in (space.range_of(f) for f in acc.forms))
            ybox = b if ybox is None else box_union_bbox(ybox, b)
        ybox = tuple((max(0, lo), min(d, hi)) for (lo, hi), d in zip(ybox, dst.shape))
        clear_mode, cbox = 0, None
        if dst.pending is not None:
            ybox = box_union_bbox(ybox, dst.pending)
            cbox = dst.pending
            clear_mode = 1 if cbox == ybox else 2
            dst.pending = None
        op = self._stencil_gather(space, t, group, ins, dst, ybox, clear_mode, cbox)
        if op is None and len(group) == 1:
            op = contract_form(space, t.body[group[0][0]], group[0][1], ins, dst, ybox, clear_mode, cbox)
        if op is not None:
            self.low.emit(op)
            return
        if len(group) > 4:
            # more than 4 terms: split into several passes (later ones accumulate)
            for k in range(0, len(group), 4):
                sub = group[k:k + 4]
                self._emit_gather(space, t, sub, ins, dst, ybox, clear_mode if k == 0 else 0,
                                  cbox if k == 0 else None, compute_f64, what)
            return
        self._emit_gather(space, t, group, ins, dst, ybox, clear_mode, cbox, compute_f64, what)

    def _emit_gather(self, space, t, group, ins, dst, ybox, clear_mode, cbox, compute_f64, what):
        used = self._used_inputs([t.body[c] for c, _, _ in group], ins)
        if len(used) > L.MAXIN:
            raise UnsupportedConstruct(f"{what}: too many inputs for the gather evaluator")
        ci = {c: k for k, c in enumerate(used)}
        code = Code()
        terms = []
        np_ = space.np
        for conn, acc, _ in group:
            seg = code.compile(t.body[conn], ci)
            Cm, off = acc.matrix(np_)
            row_of, order = pivot_rows(Cm, np_)
            terms.append((row_of, order, Cm, off, seg))
        if len(group) == 1:
            op = map2_reduce(space, group[0][1], [ins[c] for c in used], dst, ybox, clear_mode, cbox, code,
                             terms[0][4], compute_f64)
            if op is not None:
                self.low.emit(op)
                return
        # work shape: free iterations per target
        F = max(int(np.prod([space.ext[p] for p in range(np_) if rof[p] < 0], dtype=np.int64))
                for rof, *_ in terms)
        ny = box_size(ybox)
        inner_free = [p for p in range(np_) if terms[0][0][p] < 0]
        lanes = 0
        if inner_free and F >= 32:
            pin = inner_free[-1]
            if any(abs(ins[c].flat(np_)[1][pin]) == 1 for c in used):
                lanes = 1
        threads = ny * (32 if lanes else 1)
        want = max(1, -(-(148 * 1024) // max(threads, 1)))
        cap = max(1, F // ((32 if lanes else 1) * 16))
        nsplit = int(min(want, cap, 4096))
        op = GatherOp(space, dst, ybox, clear_mode, cbox, [ins[c] for c in used], terms, code, compute_f64,
                      lanes, nsplit)
        self.low.emit(op)

    def _stencil_gather(self, space, t, group, ins, dst, ybox, clear_mode, cbox):
        if space.triangular or space.np == 0 or space.np > 3 or any(s != 1 for s in space.step):
            return None
        if len(dst.shape) != space.np:
            return None
        box = tuple((f, l + 1) for f, l in zip(space.first, space.last))
        srcs, taps = [], []
        for conn, acc, _ in group:
            lin = linearize(t.body[conn])
            if lin is None or lin[0] != 0.0:
                return None
            ooff = acc.identity_offset(space.np)
            if ooff is None:
                return None
            mask = tuple((lo + o, hi + o) for (lo, hi), o in zip(box, ooff))
            for c, coef in lin[1].items():
                a = ins[c]
                if a.buf.shape != dst.shape or a.buf.kind != dst.kind:
                    return None
                doff = a.identity_offset(space.np)
                if doff is None:
                    return None
                if a.buf not in srcs:
                    srcs.append(a.buf)
                if len(srcs) > L.MAXSRCS:
                    return None
                taps.append((srcs.index(a.buf), coef, tuple(d - o for d, o in zip(doff, ooff)), mask))
        if len(taps) > L.MAXTAPS:
            return None
        return StencilOp(dst, srcs, ybox, clear_mode, cbox, taps, kind="adjoint")

    # -- library nodes -------------------------------------------------------------

    def library(self, node: LibraryNode, df):
        ins = {e.dst_conn: e.data for e in df.in_edges(node.id)}
        outs = df.out_edges(node.id)
        shapes = {c: self.shape_of(d) for c, d in ins.items()}
        bufs = {c: self.read(d) for c, d in ins.items()}
        kind = node.kind
        if lower_scale_zero(node) and all(e.wcr is None for e in outs):
            # gradient clear `scale 0.0` (autodiff.py:901-906): deferred and
            # folded into the next writer instead of a separate pass
            n = int(np.prod(shapes["x"], dtype=np.int64)) if shapes["x"] else 1
            self.low.flops += n
            for e in outs:
                out = self._lib_out(e, shapes["x"], node)
                self.low.add_clear(out, whole_box(out.shape))
            return
        for b in bufs.values():
            self.low.materialize(b)
        if kind == "matmul":
            sa, sb = shapes["a"], shapes["b"]
            if len(sa) != 2 or len(sb) != 2:
                raise UnsupportedConstruct(f"matmul '{node.id}': operands must be 2-D")
            a_eff = sa[::-1] if node.ta else sa
            b_eff = sb[::-1] if node.tb else sb
            if a_eff[1] != b_eff[0]:
                raise ShapeMismatch(f"matmul '{node.id}': inner dims {a_eff[1]} vs {b_eff[0]}")
            M, K, N = a_eff[0], a_eff[1], b_eff[1]
            self.low.flops += 2 * M * K * N
            for e in outs:
                out = self._lib_out(e, (M, N), node)
                acc = self._accumulate(e, out)
                if bufs["a"].kind != out.kind or bufs["b"].kind != out.kind:
                    raise UnsupportedConstruct(f"matmul '{node.id}': mixed element kinds")
                if out.bid in (bufs["a"].bid, bufs["b"].bid):
                    raise UnsupportedConstruct(f"matmul '{node.id}': output aliases an operand")
                self.low.emit(MatmulOp(bufs["a"], bufs["b"], out, node.ta, node.tb, M, N, K, acc))
        elif kind == "reduce_sum":
            x = bufs["x"]
            n = x.numel if shapes["x"] else 1
            self.low.flops += n if shapes["x"] else 0
            for e in outs:
                out = self._lib_out(e, (), node)
                acc = self._accumulate(e, out)
                self.low.emit(ReduceOp(x, out, acc))
        elif kind == "ew_unary":
            x = bufs["x"]
            n = int(np.prod(shapes["x"], dtype=np.int64)) if shapes["x"] else 1
            op, const = self._unary_code(node)
            self.low.flops += (0 if node.op == "copy" else 1) * n
            for e in outs:
                out = self._lib_out(e, shapes["x"], node)
                acc = self._accumulate(e, out)
                if out.kind != x.kind:
                    raise UnsupportedConstruct(f"'{node.id}': element kind conversion")
                if node.op == "copy" and not acc:
                    self.low.emit(CopyOp(out, x))
                else:
                    self.low.emit(EwOp(op, const, x, None, out, acc))
        else:
            a, b = bufs["a"], bufs["b"]
            if shapes["a"] != shapes["b"]:
                raise ShapeMismatch(f"'{node.id}': operand shapes {shapes['a']} vs {shapes['b']}")
            n = int(np.prod(shapes["a"], dtype=np.int64)) if shapes["a"] else 1
            self.low.flops += n
            if node.op not in L.BINOP or node.op in ("idiv", "mod", "pow"):
                raise UnsupportedConstruct(f"'{node.id}': unknown elementwise op '{node.op}'")
            for e in outs:
                out = self._lib_out(e, shapes["a"], node)
                acc = self._accumulate(e, out)
                if not (a.kind == b.kind == out.kind):
                    raise UnsupportedConstruct(f"'{node.id}': element kind conversion")
                self.low.emit(EwOp(L.BINOP[node.op], 0.0, a, b, out, acc))

    def _unary_code(self, node):
        op = node.op
        if op == "copy":
            return L.OP_IN, 0.0
        if op == "scale":
            return L.OP_MUL, float(node.const)
        if op in L.UNOP:
            return L.UNOP[op], 0.0
        raise DomainError(f"unknown elementwise op '{op}'")

    def _lib_out(self, e, res_shape, node) -> Buffer:
        want = self.shape_of(e.data)
        if tuple(res_shape) != tuple(want) and not (len(res_shape) == 0 and e.wcr is None):
            raise ShapeMismatch(f"'{node.id}': result shape {tuple(res_shape)} does not match '{e.data}' {want}")
        if tuple(res_shape) != tuple(want):
            raise UnsupportedConstruct(f"'{node.id}': broadcasting a scalar result into '{e.data}'")
        return self.write(e.data)

    def _accumulate(self, e, out: Buffer) -> bool:
        """wcr=sum accumulates unless the target is known zero (first touch
        or a pending whole-array clear): then it is a plain overwrite."""
        if e.wcr == "sum":
            if out.pending is not None and out.pending == whole_box(out.shape):
                out.pending = None
                return False
            self.low.materialize(out)
            return True
        out.pending = None  # overwrite (the reference rebinds the array)
        return False


def lower_scale_zero(node) -> bool:
    return node.kind == "ew_unary" and node.op == "scale" and float(node.const) == 0.0


def required_record(forwarding) -> set:
    out = set()
    for e in forwarding.values():
        for c in e.candidates:
            out.add((e.data, c.version))
    return out


__all__ = ["Lowering", "ProgramRun", "LTape", "Buffer", "number_writes", "lower_scale_zero"]
