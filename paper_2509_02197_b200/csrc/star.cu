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

constexpr int kPX = 32, kPY = 16, kPM = 16;  // tile (k, j), planes per CTA; 512 threads

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
  int32_t ps, rs;  // plane / row strides (arrays < 2^31 elements)
  StarOpDev a, b;
  const void *y;      // source of a
  const void *xold;   // old X (base of a, value outside a's region)
  void *xout;         // X write-back target (ping-pong)
  const void *zold;   // old Z (base of b, value outside b's region)
  void *zout;         // Z target
  int32_t dlo[3], dhi[3];  // dead box of X (not written back)
};

// Per-coordinate predicate bits. For a point (i, j, k) the predicate word is
// M0[i] & M1[j] & M2[k]: bits 0..6 = tap p's mask box admits the point,
// bit 7 = inside the op's region, bit 8 = inside its clear box, bit 9 = in
// the dead box (op a only), bit 10 = inside the array.
enum : uint32_t { kRegion = 1u << 7, kClear = 1u << 8, kDead = 1u << 9, kArray = 1u << 10 };

__device__ __forceinline__ uint32_t coord_bits(const StarOpDev &o, int dim, int c, int extent, const int32_t *dlo,
                                               const int32_t *dhi) {
  uint32_t b = 0;
#pragma unroll
  for (int p = 0; p < 7; ++p) {
    bool ok = !((o.masked >> p) & 1) || (c >= o.mlo[p][dim] && c < o.mhi[p][dim]);
    b |= (uint32_t)ok << p;
  }
  if (c >= o.lo[dim] && c < o.hi[dim]) b |= kRegion;
  if (c >= o.clo[dim] && c < o.chi[dim]) b |= kClear;
  if (dlo && c >= dlo[dim] && c < dhi[dim]) b |= kDead;
  if (c >= 0 && c < extent) b |= kArray;
  return b;
}

template <typename T>
__global__ void __launch_bounds__(kPX *kPY) star_pair_kernel(const __grid_constant__ StarPairDev d) {
  __shared__ T xs[3][kPY + 2][kPX + 2];
  __shared__ uint32_t aj[kPY + 2], ak[kPX + 2], bj[kPY], bk[kPX];
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * kPX + tx;
  const int k0 = blockIdx.x * kPX, j0 = blockIdx.y * kPY;
  const int i0 = blockIdx.z * kPM, i1 = min(i0 + kPM, d.d0);
  if (tid < kPY + 2) aj[tid] = coord_bits(d.a, 1, j0 - 1 + tid, d.d1, d.dlo, d.dhi);
  if (tid >= 32 && tid < 32 + kPX + 2) ak[tid - 32] = coord_bits(d.a, 2, k0 - 1 + (tid - 32), d.d2, d.dlo, d.dhi);
  if (tid >= 96 && tid < 96 + kPY) bj[tid - 96] = coord_bits(d.b, 1, j0 + (tid - 96), d.d1, nullptr, nullptr);
  if (tid >= 128 && tid < 128 + kPX) bk[tid - 128] = coord_bits(d.b, 2, k0 + (tid - 128), d.d2, nullptr, nullptr);
  __syncthreads();
  const T *__restrict__ Y = (const T *)d.y;
  const T *__restrict__ Xo = (const T *)d.xold;
  const T *__restrict__ Zo = (const T *)d.zold;
  T *Xn = (T *)d.xout;
  T *Zn = (T *)d.zout;
  const int ps = d.ps, rs = d.rs;
  T ca[7], cb[7];
#pragma unroll
  for (int p = 0; p < 7; ++p) {
    ca[p] = (T)d.a.coef[p];
    cb[p] = (T)d.b.coef[p];
  }
  const uint32_t apres = d.a.present, bpres = d.b.present;
  constexpr int HW = (kPY + 2) * (kPX + 2);
  for (int q = i0 - 1; q <= i1; ++q) {
    const int slot = (q + 3) % 3;
    if (q >= 0 && q < d.d0) {
      const uint32_t mi = coord_bits(d.a, 0, q, d.d0, d.dlo, d.dhi);
      const bool own = q >= i0 && q < i1;
      for (int p = tid; p < HW; p += kPX * kPY) {
        const int hj = p / (kPX + 2), hk = p - hj * (kPX + 2);
        const uint32_t m = mi & aj[hj] & ak[hk];
        T v = T(0);
        if (m & kArray) {
          const int off = q * ps + (j0 - 1 + hj) * rs + (k0 - 1 + hk);
          if (m & kRegion) {
            T acc;
            if (d.a.mode == 0 || (d.a.mode == 2 && !(m & kClear)))
              acc = Xo[off];
            else
              acc = T(0);
            const int doff[7] = {0, -ps, ps, -rs, rs, -1, 1};
            T t[7];
#pragma unroll
            for (int e = 0; e < 7; ++e) t[e] = (((apres & m) >> e) & 1) ? __ldg(Y + off + doff[e]) : T(0);
#pragma unroll
            for (int e = 0; e < 7; ++e) acc += ca[e] * t[e];
            v = acc;
          } else {
            v = Xo[off];
          }
          if (d.xwrite && own && hj >= 1 && hj <= kPY && hk >= 1 && hk <= kPX && !(m & kDead)) Xn[off] = v;
        }
        xs[slot][hj][hk] = v;
      }
    }
    __syncthreads();
    const int i = q - 1;
    if (i >= i0 && i < i1) {
      const uint32_t m = coord_bits(d.b, 0, i, d.d0, nullptr, nullptr) & bj[ty] & bk[tx];
      if (m & kArray) {
        const int off = i * ps + (j0 + ty) * rs + (k0 + tx);
        T w;
        if (m & kRegion) {
          if (d.b.mode == 0 || (d.b.mode == 2 && !(m & kClear)))
            w = Zo[off];
          else
            w = T(0);
          const int sc = (i + 3) % 3, sm = (i + 2) % 3, sp = (i + 4) % 3;
          T t[7];
          t[0] = xs[sc][ty + 1][tx + 1];
          t[1] = xs[sm][ty + 1][tx + 1];
          t[2] = xs[sp][ty + 1][tx + 1];
          t[3] = xs[sc][ty][tx + 1];
          t[4] = xs[sc][ty + 2][tx + 1];
          t[5] = xs[sc][ty + 1][tx];
          t[6] = xs[sc][ty + 1][tx + 2];
          const uint32_t on = bpres & m;
#pragma unroll
          for (int e = 0; e < 7; ++e)
            if ((on >> e) & 1) w += cb[e] * t[e];
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
  d.ps = (int32_t)(dims[1] * dims[2]);
  d.rs = (int32_t)dims[2];
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
