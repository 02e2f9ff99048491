// Fused radius-1 "star" stencil sweeps (the jacobi_2d / heat_3d hot path).
//
// One timestep of those programs is two map sweeps, X = S_a(Y) then
// Z = S_b(X) (forward: B = S(A), A = S(B); reverse: the two gather-form
// adjoint sweeps of autodiff.py:962-1081 with their `_z` clears folded in).
// gfb_star_pair evaluates both in one pass over HBM: each CTA computes X on
// its tile plus a one-point halo into a rolling three-plane shared-memory
// window and applies S_b from there, so per timestep Y is read once and Z is
// written once (plus X where it is still live) instead of 2 reads + 2
// writes. Z goes to a ping-pong buffer because neighbouring CTAs still read
// Y (== the old Z) for their halos.
//
// Positions: 0 centre, 1 (-1,0,0), 2 (+1,0,0), 3 (0,-1,0), 4 (0,+1,0),
// 5 (0,0,-1), 6 (0,0,+1) on a row-major [d0][d1][d2] array (rank 2 arrays
// are padded with d0 = 1).
#include <cstdlib>
#include "gfb_internal.h"
#include "star_common.cuh"

namespace gfb {

template <typename T, bool HAS_I>
struct StarTaps {
  T v[7];
  __device__ __forceinline__ void load(const T *__restrict__ y, int ps, int rs) {
    v[0] = __ldg(y);
    v[3] = __ldg(y - rs);
    v[4] = __ldg(y + rs);
    v[5] = __ldg(y - 1);
    v[6] = __ldg(y + 1);
    if (HAS_I) {
      v[1] = __ldg(y - ps);
      v[2] = __ldg(y + ps);
    }
  }
  // predicated load: tap e only if bit e of `m` is set (out-of-array taps
  // are never admitted by the predicate words, so no load goes out of bounds)
  __device__ __forceinline__ void load_masked(const T *__restrict__ y, int ps, int rs, uint32_t m) {
    v[0] = (m & 1u) ? __ldg(y) : T(0);
    v[3] = (m & 8u) ? __ldg(y - rs) : T(0);
    v[4] = (m & 16u) ? __ldg(y + rs) : T(0);
    v[5] = (m & 32u) ? __ldg(y - 1) : T(0);
    v[6] = (m & 64u) ? __ldg(y + 1) : T(0);
    if (HAS_I) {
      v[1] = (m & 2u) ? __ldg(y - ps) : T(0);
      v[2] = (m & 4u) ? __ldg(y + ps) : T(0);
    }
  }
  __device__ __forceinline__ T dot(const T (&c)[7], T acc) const {
    acc += c[0] * v[0];
    if (HAS_I) {
      acc += c[1] * v[1];
      acc += c[2] * v[2];
    }
    acc += c[3] * v[3];
    acc += c[4] * v[4];
    acc += c[5] * v[5];
    acc += c[6] * v[6];
    return acc;
  }
};

template <typename T, bool HAS_I>
__device__ __forceinline__ void star_pair_fast(const StarPairDev &d, T (*xs)[kPY + 2][kPX + 2], uint32_t aA,
                                               uint32_t aB, int i0, int i1, int tid, int hj0, int hk0, int hj1,
                                               int hk1, bool has1, bool core0, bool core1, int rel0, int rel1,
                                               int zrel, const T (&ca)[7], const T (&cb)[7]) {
  const T *__restrict__ Y = (const T *)d.y;
  const T *__restrict__ Xo = (const T *)d.xold;
  const T *__restrict__ Zo = (const T *)d.zold;
  T *__restrict__ Xn = (T *)d.xout;
  T *__restrict__ Zn = (T *)d.zout;
  const int ps = d.ps, rs = d.rs;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const bool xbase = d.a.mode == 0 || (d.a.mode == 2 && !(aA & kClear));
  const bool zbase = d.b.mode == 0 || (d.b.mode == 2 && !(aB & kClear));
  const bool xw = d.xwrite && !(aA & kDead);
  const bool xw0 = xw && core0, xw1 = xw && core1;
  const int qbeg = HAS_I ? i0 - 1 : 0, qend = HAS_I ? i1 : 0;
  StarTaps<T, HAS_I> r0, r1;
  r0.load(Y + (qbeg * ps + rel0), ps, rs);
  if (has1) r1.load(Y + (qbeg * ps + rel1), ps, rs);
  for (int q = qbeg; q <= qend; ++q) {
    const int slot = q & 3;
    const bool own = q >= i0 && q < i1;
    {
      const int off = q * ps + rel0;
      const T acc = r0.dot(ca, xbase ? Xo[off] : T(0));
      if (own && xw0) Xn[off] = acc;
      xs[slot][hj0][hk0] = acc;
    }
    if (has1) {
      const int off = q * ps + rel1;
      const T acc = r1.dot(ca, xbase ? Xo[off] : T(0));
      if (own && xw1) Xn[off] = acc;
      xs[slot][hj1][hk1] = acc;
    }
    if (q < qend) {  // prefetch the next plane across the barrier
      r0.load(Y + ((q + 1) * ps + rel0), ps, rs);
      if (has1) r1.load(Y + ((q + 1) * ps + rel1), ps, rs);
    }
    __syncthreads();
    const int i = HAS_I ? q - 1 : q;
    if (i >= i0) {
      const int off = i * ps + zrel;
      const int sc = i & 3, sm = (i - 1) & 3, sp = (i + 1) & 3;
      T w = zbase ? Zo[off] : T(0);
      w += cb[0] * xs[sc][ty + 1][tx + 1];
      if (HAS_I) {
        w += cb[1] * xs[sm][ty + 1][tx + 1];
        w += cb[2] * xs[sp][ty + 1][tx + 1];
      }
      w += cb[3] * xs[sc][ty][tx + 1];
      w += cb[4] * xs[sc][ty + 2][tx + 1];
      w += cb[5] * xs[sc][ty + 1][tx];
      w += cb[6] * xs[sc][ty + 1][tx + 2];
      Zn[off] = w;
    }
  }
}

// Boundary CTAs: the same pipelined loop with per-point predicate words
// (array / region / clear / dead bits and per-tap mask bits), all branch-free
// selects around predicated loads.
template <typename T, bool HAS_I>
__device__ __forceinline__ void star_pair_checked(const StarPairDev &d, T (*xs)[kPY + 2][kPX + 2],
                                                  const uint32_t *ai, const uint32_t *bi, int i0, int i1,
                                                  uint32_t mjk0, uint32_t mjk1, uint32_t mzjk, int hj0, int hk0,
                                                  int hj1, int hk1, bool has1, bool core0, bool core1, int rel0,
                                                  int rel1, int zrel, const T (&ca)[7], const T (&cb)[7]) {
  const T *__restrict__ Y = (const T *)d.y;
  const T *__restrict__ Xo = (const T *)d.xold;
  const T *__restrict__ Zo = (const T *)d.zold;
  T *__restrict__ Xn = (T *)d.xout;
  T *__restrict__ Zn = (T *)d.zout;
  const int ps = d.ps, rs = d.rs;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const uint32_t apres = d.a.present, bpres = d.b.present;
  const int amode = d.a.mode, bmode = d.b.mode;
  const int qbeg = HAS_I ? max(i0 - 1, 0) : 0, qend = HAS_I ? i1 : 0;
  StarTaps<T, HAS_I> r0, r1;
  auto xmask = [&](int q, uint32_t mjk) { return ai[q - i0 + 1] & mjk; };
  auto prefetch = [&](int q) {
    const uint32_t m0 = xmask(q, mjk0);
    if ((m0 & (kArray | kRegion)) == (kArray | kRegion)) r0.load_masked(Y + (q * ps + rel0), ps, rs, m0 & apres);
    if (has1) {
      const uint32_t m1 = xmask(q, mjk1);
      if ((m1 & (kArray | kRegion)) == (kArray | kRegion)) r1.load_masked(Y + (q * ps + rel1), ps, rs, m1 & apres);
    }
  };
  auto xpoint = [&](const StarTaps<T, HAS_I> &r, uint32_t m, int off, bool own, bool core) -> T {
    if (!(m & kArray)) return T(0);
    T v;
    if (m & kRegion) {
      const bool base = amode == 0 || (amode == 2 && !(m & kClear));
      v = r.dot(ca, base ? Xo[off] : T(0));
    } else {
      v = Xo[off];
    }
    if (own && core && d.xwrite && !(m & kDead) && !(d.skipx && !(m & kRegion))) Xn[off] = v;
    return v;
  };
  prefetch(qbeg);
  for (int q = qbeg; q <= qend; ++q) {
    // X(q) exists only inside the local array; the Z plane that would read
    // X(d0) at the array end has that tap masked off by b's predicates
    if (q < d.d0) {
      const int slot = q & 3;
      const bool own = q >= i0 && q < i1;
      const T v0 = xpoint(r0, xmask(q, mjk0), q * ps + rel0, own, core0);
      xs[slot][hj0][hk0] = v0;
      if (has1) {
        const T v1 = xpoint(r1, xmask(q, mjk1), q * ps + rel1, own, core1);
        xs[slot][hj1][hk1] = v1;
      }
      if (q < qend && q + 1 < d.d0) prefetch(q + 1);
    }
    __syncthreads();
    const int i = HAS_I ? q - 1 : q;
    if (i >= i0 && i < i1) {
      const uint32_t m = bi[i - i0] & mzjk;
      if (m & kArray) {
        const int off = i * ps + zrel;
        T w;
        if (m & kRegion) {
          const bool base = bmode == 0 || (bmode == 2 && !(m & kClear));
          w = base ? Zo[off] : T(0);
          const uint32_t on = bpres & m;
          const int sc = i & 3, sm = (i - 1) & 3, sp = (i + 1) & 3;
          w += (on & 1u) ? cb[0] * xs[sc][ty + 1][tx + 1] : T(0);
          if (HAS_I) {
            w += (on & 2u) ? cb[1] * xs[sm][ty + 1][tx + 1] : T(0);
            w += (on & 4u) ? cb[2] * xs[sp][ty + 1][tx + 1] : T(0);
          }
          w += (on & 8u) ? cb[3] * xs[sc][ty][tx + 1] : T(0);
          w += (on & 16u) ? cb[4] * xs[sc][ty + 2][tx + 1] : T(0);
          w += (on & 32u) ? cb[5] * xs[sc][ty + 1][tx] : T(0);
          w += (on & 64u) ? cb[6] * xs[sc][ty + 1][tx + 2] : T(0);
        } else {
          if (d.skipz) continue;
          w = Zo[off];
        }
        Zn[off] = w;
      }
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(kPX *kPY, 2) star_pair_kernel(const __grid_constant__ StarPairDev d) {
  constexpr int HX = kPX + 2, HW = (kPY + 2) * HX, NT = kPX * kPY;
  __shared__ T xs[4][kPY + 2][HX];
  __shared__ uint32_t aj[kPY + 2], ak[HX], bj[kPY], bk[kPX], ai[kPM + 2], bi[kPM];
  __shared__ uint32_t s_and_a, s_or_a, s_and_b, s_or_b;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * kPX + tx;
  const int k0 = blockIdx.x * kPX, j0 = blockIdx.y * kPY;
  const int i0 = d.zlo + blockIdx.z * kPM, i1 = min(i0 + kPM, d.zhi);
  star_prologue(d, i0, i1, tid, aj, ak, bj, bk, ai, bi, s_and_a, s_or_a, s_and_b, s_or_b);  // descriptor only
  pdl_wait();
  pdl_trigger();  // after the wait: at most one launch waits ahead of the running one
  const int rs = d.rs;
  T ca[7], cb[7];
#pragma unroll
  for (int p = 0; p < 7; ++p) {
    ca[p] = (T)d.a.coef[p];
    cb[p] = (T)d.b.coef[p];
  }
  const uint32_t apres = d.a.present, bpres = d.b.present;
  // the (at most two) halo-window points this thread computes per plane
  const int hj0 = tid / HX, hk0 = tid - hj0 * HX;
  const int p1 = tid + NT;
  const bool has1 = p1 < HW;
  const int hj1 = p1 / HX, hk1 = p1 - hj1 * HX;
  const uint32_t mjk0 = aj[hj0] & ak[hk0];
  const uint32_t mjk1 = has1 ? (aj[hj1] & ak[hk1]) : 0u;
  const bool core0 = hj0 >= 1 && hj0 <= kPY && hk0 >= 1 && hk0 <= kPX;
  const bool core1 = has1 && hj1 >= 1 && hj1 <= kPY && hk1 >= 1 && hk1 <= kPX;
  const int rel0 = (j0 - 1 + hj0) * rs + (k0 - 1 + hk0);
  const int rel1 = (j0 - 1 + hj1) * rs + (k0 - 1 + hk1);
  const uint32_t mzjk = bj[ty] & bk[tx];
  const int zrel = (j0 + ty) * rs + (k0 + tx);
  {
    // interior fast path: every window point inside the array and both
    // regions, every tap admitted, clear / dead predicates uniform, and both
    // ops full stars (all positions of the array's rank present)
    const uint32_t full = d.d0 > 1 ? 0x7fu : 0x79u;
    const uint32_t fa = full | kRegion | kArray, fb = full | kRegion | kArray;
    const uint32_t aA = s_and_a, oA = s_or_a, aB = s_and_b, oB = s_or_b;
    const bool fast = apres == full && bpres == full && (aA & fa) == fa && (aB & fb) == fb &&
                      ((aA ^ oA) & (kClear | kDead)) == 0 && ((aB ^ oB) & kClear) == 0 &&
                      (d.d0 == 1 || (i0 >= 1 && i1 + 1 <= d.d0));
    if (fast) {
      if (d.d0 > 1)
        star_pair_fast<T, true>(d, xs, aA, aB, i0, i1, tid, hj0, hk0, hj1, hk1, has1, core0, core1, rel0, rel1,
                                zrel, ca, cb);
      else
        star_pair_fast<T, false>(d, xs, aA, aB, i0, i1, tid, hj0, hk0, hj1, hk1, has1, core0, core1, rel0, rel1,
                                 zrel, ca, cb);
      return;
    }
  }
  if (d.d0 > 1)
    star_pair_checked<T, true>(d, xs, ai, bi, i0, i1, mjk0, mjk1, mzjk, hj0, hk0, hj1, hk1, has1, core0, core1, rel0,
                               rel1, zrel, ca, cb);
  else
    star_pair_checked<T, false>(d, xs, ai, bi, i0, i1, mjk0, mjk1, mzjk, hj0, hk0, hj1, hk1, has1, core0, core1,
                                rel0, rel1, zrel, ca, cb);
}

namespace tile32 {
bool star_tma_usable(const StarPairDev &d, int dtype);
int launch_star_pair_tma(const StarPairDev &d, int dtype, dim3 grid, cudaStream_t st);
}  // namespace tile32
namespace small {
bool star_tma_usable(const StarPairDev &d, int dtype);
int launch_star_pair_tma(const StarPairDev &d, int dtype, dim3 grid, cudaStream_t st);
}  // namespace small

static int fill_star_op(StarOpDev &o, const gfb_star_op &s, int pad) {
  o.present = s.present;
  o.masked = s.masked;
  o.mode = s.mode;
  for (int p = 0; p < 7; ++p) {
    o.coef[p] = s.coef[p];
    o.fcoef[p] = (float)s.coef[p];
    for (int r = 0; r < 3; ++r) {
      bool padded = r < pad;
      o.mlo[p][r] = padded ? -(1 << 30) : (int32_t)s.mlo[p][r - pad];
      o.mhi[p][r] = padded ? (1 << 30) : (int32_t)s.mhi[p][r - pad];
    }
  }
  // detect the source-mask form of the tap masks (host side, once per launch)
  static const int kDelta[7][3] = {{0, 0, 0}, {-1, 0, 0}, {1, 0, 0}, {0, -1, 0}, {0, 1, 0}, {0, 0, -1}, {0, 0, 1}};
  o.srcmask = s.masked == 0 ? 0 : 1;
  bool first = true;
  for (int p = 0; p < 7 && o.srcmask == 1; ++p) {
    if (!((s.present >> p) & 1)) continue;
    if (!((s.masked >> p) & 1)) {
      o.srcmask = -1;
      break;
    }
    for (int r = 0; r < 3; ++r) {
      const int32_t lo = o.mlo[p][r] + (r < pad ? 0 : kDelta[p][r]);
      const int32_t hi = o.mhi[p][r] + (r < pad ? 0 : kDelta[p][r]);
      if (first) {
        o.smlo[r] = lo;
        o.smhi[r] = hi;
      } else if (o.smlo[r] != lo || o.smhi[r] != hi) {
        o.srcmask = -1;
      }
    }
    first = false;
  }
  if (o.srcmask != 1)
    for (int r = 0; r < 3; ++r) {
      o.smlo[r] = -(1 << 30);
      o.smhi[r] = 1 << 30;
    }
  for (int r = 0; r < 3; ++r) {
    bool padded = r < pad;
    o.lo[r] = padded ? 0 : (int32_t)s.lo[r - pad];
    o.hi[r] = padded ? 1 : (int32_t)s.hi[r - pad];
    o.clo[r] = padded ? -(1 << 30) : (int32_t)s.clo[r - pad];
    o.chi[r] = padded ? (1 << 30) : (int32_t)s.chi[r - pad];
  }
  return 0;
}

}  // namespace gfb

using namespace gfb;

extern "C" int gfb_star_pair_launch(const gfb_star_pair_desc *s, void *stream) {
  if (!s || s->rank < 2 || s->rank > 3 || !s->y || !s->xold || !s->zout)
    return set_error(GFB_EINVAL, "gfb_star_pair_launch: bad descriptor");
  StarPairDev d;
  const int pad = 3 - s->rank;
  int64_t dims[3] = {1, 1, 1};
  for (int r = 0; r < s->rank; ++r) dims[pad + r] = s->dims[r];
  if (dims[0] * dims[1] * dims[2] >= ((int64_t)1 << 31) || dims[1] >= (1 << 30) || dims[2] >= (1 << 30))
    return set_error(GFB_EUNSUPPORTED, "gfb_star_pair_launch: array too large for 32-bit coordinates");
  d.d0 = (int32_t)dims[0];
  d.d1 = (int32_t)dims[1];
  d.d2 = (int32_t)dims[2];
  d.ps = (int32_t)(dims[1] * dims[2]);
  d.rs = (int32_t)dims[2];
  d.xwrite = s->xwrite;
  d.skipz = (s->flags & GFB_STAR_SKIP_ZCOPY) ? 1 : 0;
  d.skipx = (s->flags & GFB_STAR_SKIP_XCOPY) ? 1 : 0;
  if (s->rank == 3) {
    d.p0 = (int32_t)s->plane0;
    d.gd0 = (int32_t)(s->global_d0 > 0 ? s->global_d0 : dims[0]);
    d.zlo = (int32_t)s->zlo;
    d.zhi = (int32_t)(s->zhi > s->zlo ? s->zhi : dims[0]);
  } else {
    d.p0 = 0;
    d.gd0 = 1;
    d.zlo = 0;
    d.zhi = 1;
  }
  if (d.zlo < 0 || d.zhi > d.d0 || d.zlo >= d.zhi) return set_error(GFB_EINVAL, "gfb_star_pair_launch: bad plane range");
  d.tpm = (int32_t)(s->tpm_hint > 0 && s->tpm_hint < (1 << 20) ? s->tpm_hint : 0);
  fill_star_op(d.a, s->a, pad);
  fill_star_op(d.b, s->b, pad);
  d.y = s->y;
  d.xold = s->xold;
  d.xout = s->xout;
  d.zold = s->zold;
  d.zout = s->zout;
  for (int r = 0; r < 3; ++r) {
    bool padded = r < pad;
    d.dlo[r] = padded ? -(1 << 30) : (int32_t)s->dead_lo[r - pad];
    d.dhi[r] = padded ? (1 << 30) : (int32_t)s->dead_hi[r - pad];
  }
  dim3 block(kPX, kPY);
  dim3 grid((unsigned)ceil_div(d.d2, kPX), (unsigned)ceil_div(d.d1, kPY), (unsigned)ceil_div(d.zhi - d.zlo, kPM));
  cudaStream_t st = (cudaStream_t)stream;
  // the TMA kernel runs masks as data (source-mask form); general masks use the L1 kernel
  if (d.a.srcmask >= 0 && d.b.srcmask >= 0) {
    // small 2-D domains (fewer 32 x 32 tiles than SMs): half-height tiles
    const bool small2d = d.d0 == 1 && ceil_div(d.d1, 32) * ceil_div(d.d2, 32) < sm_count() &&
                         getenv("GFB_STAR_NO_SMALL") == nullptr;
    if (small2d && small::star_tma_usable(d, s->dtype)) return small::launch_star_pair_tma(d, s->dtype, grid, st);
    if (tile32::star_tma_usable(d, s->dtype)) return tile32::launch_star_pair_tma(d, s->dtype, grid, st);
  }
  if (s->dtype == GFB_F64)
    launch_pdl(star_pair_kernel<double>, grid, block, 0, st, d);
  else
    launch_pdl(star_pair_kernel<float>, grid, block, 0, st, d);
  return check_launch("star_pair");
}
