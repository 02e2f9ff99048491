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
#include "gfb_common.cuh"
#include "gfb_internal.h"

namespace gfb {

constexpr int kPX = 32, kPY = 8, kPM = 16;  // tile (k, j) and planes per CTA

struct StarOpDev {
  double coef[7];
  int32_t present;  // bit p: a tap at position p
  int32_t masked;   // bit p: the tap has a mask box
  int32_t mode;     // base: 0 old[y], 1/3 zero, 2 zero inside clear box else old[y]
  int32_t _pad;
  int32_t mlo[7][3], mhi[7][3];
  int32_t lo[3], hi[3];
  int32_t clo[3], chi[3];
};

struct StarPairDev {
  int32_t d0, d1, d2;
  int32_t xwrite;  // write X back (outside the dead box)
  int64_t ps, rs;  // plane / row strides
  StarOpDev a, b;
  const void *y;      // source of a
  const void *xold;   // old X (base of a, value outside a's region)
  void *xout;         // X write-back target (ping-pong)
  const void *zold;   // old Z (base of b, value outside b's region)
  void *zout;         // Z target
  int32_t dlo[3], dhi[3];  // dead box of X (not written back)
};

__device__ __forceinline__ bool in_box(const int32_t *lo, const int32_t *hi, int i, int j, int k) {
  return i >= lo[0] && i < hi[0] && j >= lo[1] && j < hi[1] && k >= lo[2] && k < hi[2];
}

template <typename T>
__device__ __forceinline__ T star_base(const StarOpDev &o, const T *__restrict__ old, int64_t off, int i, int j,
                                       int k) {
  if (o.mode == 0) return old[off];
  if (o.mode == 2) return in_box(o.clo, o.chi, i, j, k) ? T(0) : old[off];
  return T(0);
}

// op a at one point from global memory (tap sources read through L1)
template <typename T>
__device__ __forceinline__ T star_eval_global(const StarOpDev &o, const T *__restrict__ src,
                                              const T *__restrict__ old, int64_t off, int64_t ps, int64_t rs, int i,
                                              int j, int k) {
  T acc = star_base<T>(o, old, off, i, j, k);
  const int64_t doff[7] = {0, -ps, ps, -rs, rs, -1, 1};
  T v[7];
#pragma unroll
  for (int p = 0; p < 7; ++p) {
    bool on = (o.present >> p) & 1;
    if (on && ((o.masked >> p) & 1)) on = in_box(o.mlo[p], o.mhi[p], i, j, k);
    v[p] = on ? __ldg(src + off + doff[p]) : T(0);
  }
#pragma unroll
  for (int p = 0; p < 7; ++p)
    if ((o.present >> p) & 1) acc += (T)o.coef[p] * v[p];
  return acc;
}

template <typename T>
__global__ void __launch_bounds__(kPX *kPY) star_pair_kernel(const __grid_constant__ StarPairDev d) {
  __shared__ T xs[3][kPY + 2][kPX + 2];
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * kPX + tx;
  const int k0 = blockIdx.x * kPX, j0 = blockIdx.y * kPY;
  const int i0 = blockIdx.z * kPM, i1 = min(i0 + kPM, d.d0);
  const T *__restrict__ Y = (const T *)d.y;
  const T *__restrict__ Xo = (const T *)d.xold;
  const T *__restrict__ Zo = (const T *)d.zold;
  T *Xn = (T *)d.xout;
  T *Zn = (T *)d.zout;
  constexpr int HW = (kPY + 2) * (kPX + 2);
  for (int q = i0 - 1; q <= i1; ++q) {
    const int slot = (q + 3) % 3;
    if (q >= 0 && q < d.d0) {
      for (int p = tid; p < HW; p += kPX * kPY) {
        const int hj = p / (kPX + 2), hk = p - hj * (kPX + 2);
        const int j = j0 - 1 + hj, k = k0 - 1 + hk;
        T v = T(0);
        if (j >= 0 && j < d.d1 && k >= 0 && k < d.d2) {
          const int64_t off = (int64_t)q * d.ps + (int64_t)j * d.rs + k;
          if (in_box(d.a.lo, d.a.hi, q, j, k))
            v = star_eval_global<T>(d.a, Y, Xo, off, d.ps, d.rs, q, j, k);
          else
            v = Xo[off];
          if (d.xwrite && q >= i0 && q < i1 && hj >= 1 && hj <= kPY && hk >= 1 && hk <= kPX &&
              !in_box(d.dlo, d.dhi, q, j, k))
            Xn[off] = v;
        }
        xs[slot][hj][hk] = v;
      }
    }
    __syncthreads();
    const int i = q - 1;
    if (i >= i0 && i < i1) {
      const int j = j0 + ty, k = k0 + tx;
      if (j < d.d1 && k < d.d2) {
        const int64_t off = (int64_t)i * d.ps + (int64_t)j * d.rs + k;
        T w;
        if (in_box(d.b.lo, d.b.hi, i, j, k)) {
          w = star_base<T>(d.b, Zo, off, i, j, k);
          const int sc = (i + 3) % 3, sm = (i + 2) % 3, sp = (i + 4) % 3;
          T v[7];
          v[0] = xs[sc][ty + 1][tx + 1];
          v[1] = xs[sm][ty + 1][tx + 1];
          v[2] = xs[sp][ty + 1][tx + 1];
          v[3] = xs[sc][ty][tx + 1];
          v[4] = xs[sc][ty + 2][tx + 1];
          v[5] = xs[sc][ty + 1][tx];
          v[6] = xs[sc][ty + 1][tx + 2];
#pragma unroll
          for (int p = 0; p < 7; ++p) {
            bool on = (d.b.present >> p) & 1;
            if (on && ((d.b.masked >> p) & 1)) on = in_box(d.b.mlo[p], d.b.mhi[p], i, j, k);
            if (on) w += (T)d.b.coef[p] * v[p];
          }
        } else {
          w = Zo[off];
        }
        Zn[off] = w;
      }
    }
    __syncthreads();
  }
}

static int fill_star_op(StarOpDev &o, const gfb_star_op &s, int pad) {
  o.present = s.present;
  o.masked = s.masked;
  o.mode = s.mode;
  for (int p = 0; p < 7; ++p) {
    o.coef[p] = s.coef[p];
    for (int r = 0; r < 3; ++r) {
      bool padded = r < pad;
      o.mlo[p][r] = padded ? -(1 << 30) : (int32_t)s.mlo[p][r - pad];
      o.mhi[p][r] = padded ? (1 << 30) : (int32_t)s.mhi[p][r - pad];
    }
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
  d.ps = dims[1] * dims[2];
  d.rs = dims[2];
  d.xwrite = s->xwrite;
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
  dim3 grid((unsigned)ceil_div(d.d2, kPX), (unsigned)ceil_div(d.d1, kPY), (unsigned)ceil_div(d.d0, kPM));
  cudaStream_t st = (cudaStream_t)stream;
  if (s->dtype == GFB_F64)
    star_pair_kernel<double><<<grid, block, 0, st>>>(d);
  else
    star_pair_kernel<float><<<grid, block, 0, st>>>(d);
  return check_launch("star_pair");
}
