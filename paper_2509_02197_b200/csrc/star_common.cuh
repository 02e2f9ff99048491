// Shared definitions of the star-pair stencil kernels (star.cu, star_tma.cu).
#pragma once

#include "gfb_common.cuh"

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
  // source mask: every masked tap p admits y iff y + e_p lies in [smlo, smhi)
  // (the form the adjoint gather produces: "source point inside the map box")
  int32_t srcmask;  // 0: taps unmasked, 1: source-mask form, -1: general masks
  int32_t smlo[3], smhi[3];
  float fcoef[7];   // coef rounded to fp32 (fp32 kernels)
};

struct StarPairDev {
  int32_t d0, d1, d2;   // local extents
  int32_t p0, gd0;      // global index of local plane 0, global extent of dim 0
  int32_t zlo, zhi;     // local planes to produce
  int32_t xwrite;  // write X back (outside the dead box)
  int32_t skipz, skipx;  // out-of-region Z copy / X write-back already in place
  int32_t tpm;           // planes per CTA (TMA kernel)
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
enum : uint32_t { kRegion = 1u << 7, kClear = 1u << 8, kDead = 1u << 9, kArray = 1u << 10, kSrcB = 1u << 11 };

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

// Fill the CTA's per-coordinate predicate words and the block-uniform AND /
// OR summaries (a: X halo window, b: Z core) used to pick the fast path.
__device__ __forceinline__ void star_prologue(const StarPairDev &d, int i0, int i1, int tid, uint32_t *aj,
                                              uint32_t *ak, uint32_t *bj, uint32_t *bk, uint32_t *ai, uint32_t *bi,
                                              uint32_t &s_and_a, uint32_t &s_or_a, uint32_t &s_and_b,
                                              uint32_t &s_or_b) {
  constexpr int HX = kPX + 2;
  const int k0 = blockIdx.x * kPX, j0 = blockIdx.y * kPY;
  // per-coordinate predicate words, once per CTA
  // op-a words carry kSrcB: the X point lies in op b's source mask
  auto srcb = [&](int dim, int c) { return (c >= d.b.smlo[dim] && c < d.b.smhi[dim]) ? kSrcB : 0u; };
  if (tid < kPY + 2) aj[tid] = coord_bits(d.a, 1, j0 - 1 + tid, d.d1, d.dlo, d.dhi) | srcb(1, j0 - 1 + tid);
  if (tid >= 32 && tid < 32 + HX)
    ak[tid - 32] = coord_bits(d.a, 2, k0 - 1 + (tid - 32), d.d2, d.dlo, d.dhi) | srcb(2, k0 - 1 + (tid - 32));
  if (tid >= 96 && tid < 96 + kPY) bj[tid - 96] = coord_bits(d.b, 1, j0 + (tid - 96), d.d1, nullptr, nullptr);
  if (tid >= 128 && tid < 128 + kPX) bk[tid - 128] = coord_bits(d.b, 2, k0 + (tid - 128), d.d2, nullptr, nullptr);
  if (tid >= 192 && tid < 192 + kPM + 2)
    ai[tid - 192] = coord_bits(d.a, 0, i0 - 1 + (tid - 192) + d.p0, d.gd0, d.dlo, d.dhi) |
                    srcb(0, i0 - 1 + (tid - 192) + d.p0);
  if (tid >= 224 && tid < 224 + kPM) bi[tid - 224] = coord_bits(d.b, 0, i0 + (tid - 224) + d.p0, d.gd0, nullptr, nullptr);
  if (tid == 0) {
    s_and_a = s_and_b = 0xffffffffu;
    s_or_a = s_or_b = 0u;
  }
  __syncthreads();
  // block-uniform summary: AND / OR of the predicate words over the CTA's
  // window (a: halo window of X, b: core of Z) -> interior fast path
  {
    const int na = min(i1 + 1, d.d0) - max(i0 - 1, 0);
    uint32_t wa = 0xffffffffu, oa = 0u, wb = 0xffffffffu, ob = 0u;
    if (tid < kPY + 2) { wa &= aj[tid]; oa |= aj[tid]; }
    if (tid < HX) { wa &= ak[tid]; oa |= ak[tid]; }
    if (tid < na) { const uint32_t v = ai[max(i0 - 1, 0) - (i0 - 1) + tid]; wa &= v; oa |= v; }
    if (tid < kPY) { wb &= bj[tid]; ob |= bj[tid]; }
    if (tid < kPX) { wb &= bk[tid]; ob |= bk[tid]; }
    if (tid < i1 - i0) { wb &= bi[tid]; ob |= bi[tid]; }
    if (tid < 64) {
      atomicAnd(&s_and_a, wa);
      atomicOr(&s_or_a, oa);
      atomicAnd(&s_and_b, wb);
      atomicOr(&s_or_b, ob);
    }
  }
  __syncthreads();
}

}  // namespace gfb
