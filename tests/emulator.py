"""CPU emulation of libgfb launch descriptors — TEST INFRASTRUCTURE ONLY.

Executes a lowered launch list on numpy arrays by interpreting the exact
ctypes descriptors the engine would pass to libgfb.so (gfb_map_desc,
gfb_gather_desc, gfb_stencil_desc, and the scalar-argument entry points).
This checks the host lowering and descriptor packing on the CPU-only build
machine; the CUDA kernels themselves are checked by the `-m gpu` tests.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from paper_2509_02197_b200 import _lib as L
from paper_2509_02197_b200.lowering import (
    BroadcastOp,
    ContractOp,
    Map2Op,
    CopyOp,
    EwOp,
    FillOp,
    GatherOp,
    MapOp,
    MatmulOp,
    MatvecPairOp,
    Rank2Op,
    ReduceOp,
    StarPairOp,
    StencilOp,
    WavefrontOp,
)

NPT = {L.F32: np.float32, L.F64: np.float64}


class _Shim:
    """Stands in for a torch tensor: exposes data_ptr() of a numpy array."""

    def __init__(self, arr):
        self.arr = arr

    def data_ptr(self):
        return self.arr.ctypes.data

    def numel(self):
        return self.arr.size

    def element_size(self):
        return self.arr.itemsize


class Memory:
    def __init__(self):
        self.arrays = []

    def alloc(self, n, dtype):
        a = np.zeros(max(n, 1), dtype=dtype)
        self.arrays.append(a)
        return a

    def resolve(self, ptr):
        """(flat array, element offset) for a pointer into one allocation."""
        for a in self.arrays:
            base = a.ctypes.data
            if base <= ptr < base + a.nbytes:
                return a, (ptr - base) // a.itemsize
        raise KeyError(hex(ptr))


def _np_floordiv(a, b):
    return np.floor_divide(a, b)


def _vm(code, arg, start, n, consts, fetch, T, err):
    st = []
    for pc in range(start, start + n):
        op = code[pc]
        if op == L.OP_IN:
            st.append(fetch(arg[pc]))
        elif op == L.OP_CONST:
            st.append(T(consts[arg[pc]]))
        elif op >= L.OP_NEG:
            x = st.pop()
            if op == L.OP_NEG:
                r = -x
            elif op == L.OP_SIN:
                r = np.sin(x)
            elif op == L.OP_COS:
                r = np.cos(x)
            elif op == L.OP_EXP:
                r = np.exp(x)
            elif op == L.OP_LOG:
                if np.any(~(x > 0)):
                    err[0] |= 0x2
                r = np.log(np.where(x > 0, x, 1))
            elif op == L.OP_SQRT:
                if np.any(x < 0):
                    err[0] |= 0x4
                r = np.sqrt(np.where(x < 0, 0, x))
            elif op == L.OP_TANH:
                r = np.tanh(x)
            elif op == L.OP_ABS:
                r = np.abs(x)
            else:
                r = np.sign(x)
            st.append(np.asarray(r, dtype=T))
        else:
            b = st.pop()
            a = st.pop()
            if op == L.OP_ADD:
                r = a + b
            elif op == L.OP_SUB:
                r = a - b
            elif op == L.OP_MUL:
                r = a * b
            elif op in (L.OP_DIV, L.OP_IDIV, L.OP_MOD):
                if np.any(np.equal(b, 0)):
                    err[0] |= {L.OP_DIV: 0x1, L.OP_IDIV: 0x10, L.OP_MOD: 0x20}[op]
                bs = np.where(np.equal(b, 0), 1, b)
                r = a / bs if op == L.OP_DIV else (_np_floordiv(a, bs) if op == L.OP_IDIV else np.mod(a, bs))
            elif op == L.OP_MIN:
                r = np.where(b < a, b, a)
            elif op == L.OP_MAX:
                r = np.where(b > a, b, a)
            else:
                r = np.power(a, b)
            st.append(np.asarray(r, dtype=T))
    return st[0]


def _space_points(sp):
    """All member points of a gfb_space as an (np, npts) int64 array."""
    npar = sp.nparams
    if npar == 0:
        return np.zeros((0, 1), dtype=np.int64)
    axes = []
    for p in range(npar):
        k = np.arange(sp.box_ext[p], dtype=np.int64)
        axes.append(sp.box_lo[p] + (k if sp.triangular else k * sp.step[p]))
    grids = np.meshgrid(*axes, indexing="ij")
    x = np.stack([g.reshape(-1) for g in grids])
    if sp.triangular:
        x = x[:, _member(sp, x)]
    return x


def _member(sp, x):
    ok = np.ones(x.shape[1], dtype=bool)
    for p in range(sp.nparams):
        lo = sp.lo0[p] + sum(sp.loc[p][q] * x[q] for q in range(p))
        hi = sp.hi0[p] + sum(sp.hic[p][q] * x[q] for q in range(p))
        lo = np.broadcast_to(lo, x.shape[1:])
        hi = np.broadcast_to(hi, x.shape[1:])
        ok &= (x[p] >= lo) & (x[p] < hi)
        if sp.step[p] != 1:
            ok &= ((x[p] - lo) % sp.step[p]) == 0
    return ok


def _offsets(opnd, x, npar):
    off = np.full(x.shape[1] if x.ndim > 1 else 1, opnd.c0, dtype=np.int64)
    for p in range(npar):
        off = off + opnd.s[p] * x[p]
    return off


class Emulator:
    def __init__(self, mem: Memory):
        self.mem = mem
        self.err = np.zeros(1, dtype=np.uint32)

    def arr(self, ptr, dtype=None):
        a, o = self.mem.resolve(ptr)
        return a, o

    def run_op(self, op):
        if isinstance(getattr(op, "edges", None), list):  # decomp.EdgeOp: its star pairs in order
            for p in op.edges:
                self.run_op(p)
        elif isinstance(op, WavefrontOp):
            self.wave(op.desc)
        elif isinstance(op, MapOp):
            self.map(op.desc)
        elif isinstance(op, GatherOp):
            self.gather(op.desc)
        elif isinstance(op, StencilOp):
            self.stencil(op.desc)
        elif isinstance(op, StarPairOp):
            self.star_pair(op.desc)
        elif isinstance(op, ContractOp):
            self.contract(op.desc)
        elif isinstance(op, Map2Op):
            self.map2(op.desc)
        elif isinstance(op, FillOp):
            a, o = self.arr(op.dst.ptr)
            if op.whole:
                a[o:o + op.dst.numel] = op.value
            else:
                v = a[o:o + op.dst.numel].reshape(op.dst.shape)
                v[tuple(slice(lo, hi) for lo, hi in op.box)] = op.value
        elif isinstance(op, ReduceOp):
            xa, xo = self.arr(op.x.ptr)
            s = np.sum(xa[xo:xo + op.x.numel].astype(np.float64))
            oa, oo = self.arr(op.out.ptr)
            oa[oo] = (oa[oo] + s) if op.accumulate else s
        elif isinstance(op, EwOp):
            T = NPT[op.out.dtype]
            aa, ao = self.arr(op.a.ptr)
            a = aa[ao:ao + op.a.numel]
            b = None
            if op.b is not None:
                ba, bo = self.arr(op.b.ptr)
                b = ba[bo:bo + op.b.numel]
            if b is None:
                if op.op == L.OP_IN:
                    r = a.copy()
                elif op.op == L.OP_MUL:
                    r = a * T(op.const)
                else:
                    r = _vm([L.OP_IN, op.op], [0, 0], 0, 2, [], lambda k: a, T, self.err)
            else:
                r = _vm([L.OP_IN, L.OP_IN, op.op], [0, 1, 0], 0, 3, [], lambda k: (a, b)[k], T, self.err)
            oa, oo = self.arr(op.out.ptr)
            sl = slice(oo, oo + op.out.numel)
            oa[sl] = (oa[sl] + r) if op.accumulate else r
        elif isinstance(op, BroadcastOp):
            v = op.scale
            if op.src is not None:
                sa, so = self.arr(op.src.ptr)
                v = v * float(sa[so])
            oa, oo = self.arr(op.out.ptr)
            sl = slice(oo, oo + op.out.numel)
            oa[sl] = (oa[sl] + v) if op.accumulate else v
        elif isinstance(op, MatmulOp):
            aa, ao = self.arr(op.a.ptr)
            ba, bo = self.arr(op.b.ptr)
            A = aa[ao:ao + op.a.numel].reshape(op.a.shape)
            B = ba[bo:bo + op.b.numel].reshape(op.b.shape)
            A = A.T if op.ta else A
            B = B.T if op.tb else B
            r = A @ B
            oa, oo = self.arr(op.out.ptr)
            sl = slice(oo, oo + op.out.numel)
            oa[sl] = (oa[sl] + r.reshape(-1)) if op.accumulate else r.reshape(-1)
        elif isinstance(op, (MatvecPairOp, Rank2Op)):
            # the fused op is, by construction, the parts run in order
            for part in op.parts:
                self.run_op(part)
        elif isinstance(op, CopyOp):
            if not op.elided:
                sa, so = self.arr(op.src.ptr)
                da, do = self.arr(op.dst.ptr)
                da[do:do + op.dst.numel] = sa[so:so + op.src.numel]
        else:
            raise NotImplementedError(type(op))

    def table(self, ptr, n, stride):
        a, o = self.arr(ptr)
        return a[o:o + n * stride * 4].view(np.int32).reshape(n, stride) if a.dtype == np.uint8 else \
            a[o:o + n * stride].reshape(n, stride)

    def contract(self, d):
        T = NPT[d.dtype]
        M, N, K = d.M, d.N, d.K
        mt, nt, kt = self.table(d.mtab, M, d.mstride), self.table(d.ntab, N, d.nstride), self.table(d.ktab, K, d.kstride)
        aa, ao = self.arr(d.a)
        ba, bo = self.arr(d.b)
        ia = ao + mt[:, 0].astype(np.int64)[:, None] + kt[:, 0].astype(np.int64)[None, :]
        ok = np.ones((M, K), dtype=bool)
        for c in range(d.ncm):
            v = mt[:, 3 + c].astype(np.int64)[:, None] + kt[:, 2 + c].astype(np.int64)[None, :]
            ok &= (v >= d.lo[c]) & (v < d.hi[c])
        Am = np.where(ok, aa[np.where(ok, ia, ao)], 0).astype(T)
        ib = bo + kt[:, 1].astype(np.int64)[:, None] + nt[:, 0].astype(np.int64)[None, :]
        okb = np.ones((K, N), dtype=bool)
        for c in range(d.ncn):
            v = nt[:, 3 + c].astype(np.int64)[None, :] + kt[:, 2 + d.ncm + c].astype(np.int64)[:, None]
            okb &= (v >= d.lo[d.ncm + c]) & (v < d.hi[d.ncm + c])
        Bm = np.where(okb, ba[np.where(okb, ib, bo)], 0).astype(T)
        acc = (Am.astype(np.float64) @ Bm.astype(np.float64)) * d.scale
        da, do = self.arr(d.d)
        off = do + mt[:, 1].astype(np.int64)[:, None] + nt[:, 1].astype(np.int64)[None, :]
        if d.clear_mode in (1, 3):
            base = 0
        elif d.clear_mode == 2:
            inside = (mt[:, 2][:, None] != 0) & (nt[:, 2][None, :] != 0)
            base = np.where(inside, 0, da[off])
        else:
            base = da[off]
        da[off] = (base + acc).astype(da.dtype)

    def map2(self, d):
        T = np.float64 if d.compute_f64 else np.float32
        nd = d.ndim
        ext = [d.ext[i] for i in range(nd)]
        k = np.indices(ext, dtype=np.int64).reshape(nd, -1)

        def offs(o):
            return o.c0 + sum(o.s[i] * k[i] for i in range(nd))

        def fetch(j):
            o = d.in_[j]
            a, base = self.arr(o.base)
            return a[base + offs(o)].astype(T)

        words = list(d.code)
        code = [w & 63 for w in words]
        arg = [w >> 10 for w in words]
        consts = list(d.consts)
        vals = [np.broadcast_to(np.asarray(_vm(code, arg, d.code_start[o], d.code_len[o], consts, fetch, T, self.err),
                                           dtype=T), k.shape[1:]) for o in range(d.n_out)]
        if d.mode == 0:
            for o in range(d.n_out):
                w = d.out[o]
                a, base = self.arr(w.base)
                idx = base + offs(w)
                a[idx] = vals[o] if d.wcr[o] == 0 else a[idx] + vals[o]
            return
        w = d.out[0]
        a, base = self.arr(w.base)
        idx = (base + offs(w)).reshape(ext)
        v = vals[0].reshape(ext)
        if d.mode == 1:
            acc, tgt = v.sum(axis=-1, dtype=T), idx[..., 0]
            kk = k.reshape([nd] + ext)[:-1, ..., 0]
            inside = np.ones(tgt.shape, dtype=bool)
            for i in range(nd - 1):
                inside &= (kk[i] >= d.clear_lo[i]) & (kk[i] < d.clear_hi[i])
        else:
            acc, tgt = v.sum(axis=0, dtype=T), idx[0]
            kk = np.arange(ext[1])
            inside = (kk >= d.clear_lo[1]) & (kk < d.clear_hi[1])
        if d.clear_mode in (1, 3):
            base_v = 0
        elif d.clear_mode == 2:
            base_v = np.where(inside, 0, a[tgt])
        else:
            base_v = a[tgt]
        a[tgt] = base_v + acc

    def map(self, d):
        T = np.float64 if d.compute_f64 else np.float32
        x = _space_points(d.space)
        npar = d.space.nparams

        def fetch(k):
            o = d.in_[k]
            a, base = self.arr(o.base)
            return a[base + _offsets(o, x, npar)].astype(T)

        vals = [_vm(list(d.code), list(d.arg), d.code_start[o], d.code_len[o], list(d.consts), fetch, T, self.err)
                for o in range(d.n_out)]
        for o in range(d.n_out):
            w = d.out[o]
            a, base = self.arr(w.base)
            idx = base + _offsets(w, x, npar)
            v = np.broadcast_to(np.asarray(vals[o]), idx.shape)
            if d.wcr[o] == 0:
                a[idx] = v
            elif d.wcr[o] == 1:
                a[idx] = a[idx] + v
            else:
                np.add.at(a, idx, v)

    def wave(self, w):
        """gfb_wave_launch: hyperplanes in order, each one's points at once
        (read all, then write); asserts the points of a hyperplane never
        write one element twice (the host's dependence proof)."""
        d = w.map
        T = np.float64 if d.compute_f64 else np.float32
        sp = d.space
        npar = sp.nparams
        ks = np.stack([g.reshape(-1) for g in np.meshgrid(*[np.arange(sp.box_ext[p]) for p in range(npar)],
                                                          indexing="ij")])
        h = sum(int(w.c[p]) * ks[p] for p in range(npar))
        xs = np.stack([sp.box_lo[p] + ks[p] * sp.step[p] for p in range(npar)])
        for hv in range(int(w.hmax) + 1):
            sel = np.nonzero(h == hv)[0]
            if sel.size == 0:
                continue
            x = xs[:, sel]

            def fetch(k):
                o = d.in_[k]
                a, base = self.arr(o.base)
                return a[base + _offsets(o, x, npar)].astype(T)

            vals = [_vm(list(d.code), list(d.arg), d.code_start[o], d.code_len[o], list(d.consts), fetch, T,
                        self.err) for o in range(d.n_out)]
            writers = {}  # element -> the one point of this hyperplane that writes it
            for o in range(d.n_out):
                q = d.out[o]
                a, base = self.arr(q.base)
                idx = base + _offsets(q, x, npar)
                for pt, e in enumerate(np.broadcast_to(idx, (x.shape[1],)).tolist()):
                    assert writers.setdefault((q.base, e), pt) == pt, "two points of one hyperplane write one element"
                v = np.broadcast_to(np.asarray(vals[o]), idx.shape)
                if d.wcr[o] == 0:
                    a[idx] = v
                else:
                    a[idx] = a[idx] + v

    def gather(self, d):
        T = np.float64 if d.compute_f64 else np.float32
        sp = d.space
        npar = sp.nparams
        rank = d.rank
        ext = [d.ybox_ext[r] for r in range(rank)]
        ys = np.stack([g.reshape(-1) for g in np.meshgrid(*[d.ybox_lo[r] + np.arange(ext[r]) for r in range(rank)],
                                                          indexing="ij")]) if rank else np.zeros((0, 1), np.int64)
        ny = ys.shape[1]
        acc = np.zeros(ny, dtype=T)
        for t in range(d.n_terms):
            tm = d.terms[t]
            free = [p for p in range(npar) if tm.row_of[p] < 0]
            faxes = [sp.box_lo[p] + (np.arange(sp.box_ext[p]) if sp.triangular else
                                     np.arange(sp.box_ext[p]) * sp.step[p]) for p in free]
            fgrid = np.stack([g.reshape(-1) for g in np.meshgrid(*faxes, indexing="ij")]) if free else \
                np.zeros((0, 1), np.int64)
            nf = fgrid.shape[1]
            x = np.zeros((npar, ny, nf), dtype=np.int64)
            for k, p in enumerate(free):
                x[p] = fgrid[k][None, :]
            for k in range(tm.npiv):
                p = tm.order[k]
                r = tm.row_of[p]
                v = ys[r][:, None] - tm.off[r]
                for q in range(npar):
                    if q != p:
                        v = v - tm.C[r][q] * x[q]
                x[p] = v * tm.C[r][p]
            ok = np.ones((ny, nf), dtype=bool)
            for r in range(rank):
                v = np.full((ny, nf), tm.off[r], dtype=np.int64)
                for q in range(npar):
                    v = v + tm.C[r][q] * x[q]
                ok &= v == ys[r][:, None]
            flat = x.reshape(npar, -1)
            okf = ok.reshape(-1) & _member(sp, flat)
            if not okf.any():
                continue
            xs = flat[:, okf]

            def fetch(k, xs=xs):
                o = d.in_[k]
                a, base = self.arr(o.base)
                return a[base + _offsets(o, xs, npar)].astype(T)

            vals = _vm(list(d.code), list(d.arg), tm.code_start, tm.code_len, list(d.consts), fetch, T, self.err)
            vals = np.broadcast_to(np.asarray(vals, dtype=T), (xs.shape[1],))
            owner = np.nonzero(okf)[0] // nf
            np.add.at(acc, owner, vals)
        a, base = self.arr(d.dst)
        off = base + sum(ys[r] * d.dst_strides[r] for r in range(rank)) if rank else np.array([base])
        cur = a[off].astype(T)
        if d.clear_mode in (1, 3):
            cur = np.zeros_like(cur)
        elif d.clear_mode == 2:
            inside = np.ones(ny, dtype=bool)
            for r in range(rank):
                inside &= (ys[r] >= d.clear_lo[r]) & (ys[r] < d.clear_hi[r])
            cur = np.where(inside, 0, cur)
        a[off] = cur + acc

    def star_pair(self, d):
        rank = d.rank
        dims = [d.dims[r] for r in range(rank)]
        n = int(np.prod(dims))

        def view(ptr):
            a, o = self.arr(ptr)
            return a[o:o + n].reshape(dims)

        Y, Xo, Zo = view(d.y), view(d.xold), view(d.zold)
        Y, Xo, Zo = Y.copy(), Xo.copy(), Zo.copy()
        p0 = d.plane0 if rank == 3 else 0
        zlo, zhi = (d.zlo, d.zhi) if rank == 3 else (0, dims[0])
        Xn = _star_apply(d.a, Y, Xo, rank, dims, p0)
        Zn = _star_apply(d.b, Xn, Zo, rank, dims, p0)
        zv = view(d.zout)
        ys = list(np.meshgrid(*[np.arange(k) for k in dims], indexing="ij"))
        ys[0] = ys[0] + p0

        def inside(lo, hi):
            m = np.ones(ys[0].shape, dtype=bool)
            for r in range(rank):
                m &= (ys[r] >= lo[r]) & (ys[r] < hi[r])
            return m

        zsel = np.zeros(ys[0].shape, dtype=bool)
        zsel[zlo:zhi] = True
        if d.flags & L.STAR_SKIP_ZCOPY:  # out-of-region copies are left to the twin
            zsel &= inside(d.b.lo, d.b.hi)
        zv[zsel] = Zn[zsel]
        if d.xwrite:
            ys = list(np.meshgrid(*[np.arange(k) for k in dims], indexing="ij"))
            ys[0] = ys[0] + p0
            dead = np.ones(ys[0].shape, dtype=bool)
            for r in range(rank):
                dead &= (ys[r] >= d.dead_lo[r]) & (ys[r] < d.dead_hi[r])
            if not any(d.dead_hi[r] > d.dead_lo[r] for r in range(rank)):
                dead[...] = False
            own = np.zeros(ys[0].shape, dtype=bool)
            own[zlo:zhi] = True
            out = view(d.xout)
            sel = ~dead & own
            if d.flags & L.STAR_SKIP_XCOPY:
                sel &= inside(d.a.lo, d.a.hi)
            out[sel] = Xn[sel]

    def stencil(self, d):
        rank = d.rank
        a, base = self.arr(d.dst)
        dims = [d.dims[r] for r in range(rank)]
        n = int(np.prod(dims))
        D = a[base:base + n].reshape(dims)
        T = D.dtype.type
        sl = tuple(slice(d.lo[r], d.hi[r]) for r in range(rank))
        ys = np.meshgrid(*[np.arange(d.lo[r], d.hi[r]) for r in range(rank)], indexing="ij")
        if d.clear_mode == 0:
            acc = D[sl].astype(T).copy()
        elif d.clear_mode == 2:
            inside = np.ones(ys[0].shape, dtype=bool)
            for r in range(rank):
                inside &= (ys[r] >= d.clear_lo[r]) & (ys[r] < d.clear_hi[r])
            acc = np.where(inside, 0, D[sl]).astype(T)
        else:
            acc = np.zeros(ys[0].shape, dtype=T)
        srcs = []
        for i in range(L.MAXSRCS):
            if d.src[i]:
                sa, so = self.arr(d.src[i])
                srcs.append(sa[so:so + n].reshape(dims))
            else:
                srcs.append(None)
        for t in range(d.ntaps):
            S = srcs[d.tap_src[t]]
            idx = tuple(ys[r] + d.tap_delta[t][r] for r in range(rank))
            m = np.ones(ys[0].shape, dtype=bool)
            if d.tap_masked[t]:
                for r in range(rank):
                    m &= (ys[r] >= d.tap_mlo[t][r]) & (ys[r] < d.tap_mhi[t][r])
            safe = tuple(np.where(m, ix, 0) for ix in idx)
            acc = acc + np.where(m, T(d.tap_coef[t]) * S[safe], 0).astype(T)
        D[sl] = acc


_STAR = [(0, 0, 0), (-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)]


def _star_apply(so, src, old, rank, dims, p0=0):
    """One radius-1 star op over the whole (local) array (values outside its
    region keep `old`); p0 = global index of local plane 0."""
    T = old.dtype.type
    ys = list(np.meshgrid(*[np.arange(n) for n in dims], indexing="ij"))
    ys[0] = ys[0] + p0
    loc0 = ys[0] - p0
    pad = 3 - rank

    def inb(lo, hi):
        m = np.ones(ys[0].shape, dtype=bool)
        for r in range(rank):
            m &= (ys[r] >= lo[r]) & (ys[r] < hi[r])
        return m

    region = inb(so.lo, so.hi)
    if so.mode == 0:
        acc = old.copy()
    elif so.mode == 2:
        acc = np.where(inb(so.clo, so.chi), 0, old).astype(T)
    else:
        acc = np.zeros_like(old)
    for pos in range(7):
        if not (so.present >> pos) & 1:
            continue
        delta = _STAR[pos][pad:]
        m = region.copy()
        if (so.masked >> pos) & 1:
            m &= inb(so.mlo[pos], so.mhi[pos])
        idx = tuple(np.clip((loc0 if r == 0 else ys[r]) + delta[r], 0, dims[r] - 1) for r in range(rank))
        acc = acc + np.where(m, T(so.coef[pos]) * src[idx], 0).astype(T)
    return np.where(region, acc, old).astype(T)


def execute(exe_builder_low, inputs: dict, input_bufs: dict, seed_buf=None, seed=1.0):
    """Allocate every buffer of a Lowering in numpy, prepare the descriptors
    and run the launch list on the emulator. Returns (emulator, views)."""
    low = exe_builder_low
    mem = Memory()
    for b in low.buffers:
        if b.alias_of is None and b.tensor is None:
            b.tensor = _Shim(mem.alloc(b.numel, NPT[b.dtype]))

    class RT:
        pass

    rt = RT()

    def upload(arr):
        a = mem.alloc(arr.size, arr.dtype)
        a[:] = arr.reshape(-1)
        return a.ctypes.data

    rt.upload = upload
    ws = mem.alloc(1 << 16, np.uint8)
    rt.workspace_ptr = ws.ctypes.data
    em = Emulator(mem)
    rt.err_ptr = em.err.ctypes.data
    rt.lib = None
    for op in low.ops:
        op.prepare(rt)
    for name, b in input_bufs.items():
        t = b.root().tensor.arr
        t[:b.numel] = np.asarray(inputs[name], dtype=t.dtype).reshape(-1)
    if seed_buf is not None:
        seed_buf.root().tensor.arr[0] = seed
    for op in low.ops:
        em.run_op(op)

    def view(b):
        t = b.root().tensor.arr
        o = b.root_offset()
        return t[o:o + b.numel].reshape(b.shape) if b.shape else t[o:o + 1].reshape(())

    return em, view
