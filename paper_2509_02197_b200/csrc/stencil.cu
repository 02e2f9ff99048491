// Linear stencil sweeps: the forward stencil maps of jacobi_2d / heat_3d and
// the gather (transposed-stencil) form of their adjoints.
//
// Reference: the forward map is Executor._exec_map over a single tasklet
// (interpreter.py:478-507); its adjoint is the scatter-add map emitted by
// adj_map (autodiff.py:962-1081) with `_z` clears (autodiff.py:996-1004).
// The host lowering rewrites the scatter into a gather over the target array
// (one output per thread, no atomics) and folds pending clears into the same
// pass (clear_mode 2), so each sweep reads each source once and writes the
// target once.
//
// Data layout: row-major, innermost dimension contiguous; rank <= 3 (lower
// ranks are padded with leading unit dimensions). Threads map the innermost
// dimension to the warp (coalesced 256 B fp64 rows), the middle dimension to
// the block's y, and each block marches MARCH consecutive outer planes so
// neighbour planes are re-read from L1/L2 rather than HBM.
#include "gfb_common.cuh"
#include "gfb_internal.h"

namespace gfb {

constexpr int kSX = 32, kSY = 8, kMarch = 8;

struct StencilGeom {
  int64_t d1, d2;                // padded dims of the two inner dimensions
  int64_t lo0, lo1, lo2, e0, e1, e2;
  int64_t tap_off[GFB_MAX_TAPS];  // linear offset of each tap
  const void *tap_base[GFB_MAX_TAPS];  // source pointer pre-shifted by the tap offset
  int64_t mlo[GFB_MAX_TAPS][3], mhi[GFB_MAX_TAPS][3];
  int64_t clo[3], chi[3];
  int64_t march;      // planes per CTA along dim 0
  int32_t any_masked; // some tap has a mask box (else the predicate logic is skipped)
};

// Taps are unrolled up to MAXT (compile-time) and their box masks are split
// per dimension: the j/k part is evaluated once per thread, the i part once
// per plane (block-uniform), so the inner loop is predicate + load + FMA.
// NTC > 0: the tap count at compile time; CM: 1 = overwrite with no masked
// tap (forward sweeps), 2 = folded clear with masked taps (adjoint sweeps),
// 0 = read both from the descriptor
template <typename T, int MAXT, int NTC = 0, int CM = 0>
__global__ void __launch_bounds__(kSX *kSY) stencil_kernel(const __grid_constant__ gfb_stencil_desc d,
                                                           const __grid_constant__ StencilGeom g) {
  // launched with programmatic dependent launch: everything before the
  // wait overlaps the previous launch's drain; global memory after it. The
  // successor is released only as CTAs finish (an early trigger lets its
  // waiting CTAs take the slots of this grid's later waves)
  pdl_wait();
  const int64_t k = g.lo2 + (int64_t)blockIdx.x * kSX + threadIdx.x;
  const int64_t j = g.lo1 + (int64_t)blockIdx.y * kSY + threadIdx.y;
  if (k >= g.lo2 + g.e2 || j >= g.lo1 + g.e1) return;
  const int64_t i_begin = g.lo0 + (int64_t)blockIdx.z * g.march;
  const int64_t i_end = min(i_begin + g.march, g.lo0 + g.e0);
  const int nt = NTC > 0 ? NTC : d.ntaps;
  const bool any_masked = CM == 1 ? false : (CM == 2 ? true : g.any_masked != 0);
  const int clear_mode = CM == 1 ? 1 : (CM == 2 ? 2 : d.clear_mode);
  uint32_t mjk = any_masked ? 0u : 0xffffffffu;
#pragma unroll
  for (int t = 0; t < MAXT; ++t) {
    if (t < nt && any_masked) {
      bool ok = !d.tap_masked[t] ||
                (j >= g.mlo[t][1] && j < g.mhi[t][1] && k >= g.mlo[t][2] && k < g.mhi[t][2]);
      mjk |= (uint32_t)ok << t;
    }
  }
  const bool crow = j >= g.clo[1] && j < g.chi[1] && k >= g.clo[2] && k < g.chi[2];
  T *dst = (T *)d.dst;
  for (int64_t i = i_begin; i < i_end; ++i) {
    uint32_t m = mjk;
    if (any_masked) {
#pragma unroll
      for (int t = 0; t < MAXT; ++t)
        if (t < nt && d.tap_masked[t] && (i < g.mlo[t][0] || i >= g.mhi[t][0])) m &= ~(1u << t);
    }
    const int64_t off = (i * g.d1 + j) * g.d2 + k;
    T acc;
    if (clear_mode == 0) {
      acc = dst[off];
    } else if (clear_mode == 2) {
      const bool in = crow && i >= g.clo[0] && i < g.chi[0];
      acc = in ? T(0) : dst[off];
    } else {
      acc = T(0);
    }
    // all tap loads first (independent, issued back to back), then the FMAs
    T v[MAXT];
#pragma unroll
    for (int t = 0; t < MAXT; ++t)
      v[t] = (t < nt && ((m >> t) & 1u)) ? __ldg((const T *)g.tap_base[t] + off) : T(0);
#pragma unroll
    for (int t = 0; t < MAXT; ++t)
      if (t < nt) acc += (T)d.tap_coef[t] * v[t];
    dst[off] = acc;
  }
  pdl_trigger();
}

}  // namespace gfb

using namespace gfb;

extern "C" int gfb_stencil_launch(const gfb_stencil_desc *d, void *stream) {
  if (!d || d->rank < 1 || d->rank > 3 || d->ntaps < 0 || d->ntaps > GFB_MAX_TAPS || !d->dst)
    return set_error(GFB_EINVAL, "gfb_stencil_launch: bad descriptor");
  StencilGeom g;
  int64_t dims[3] = {1, 1, 1}, lo[3] = {0, 0, 0}, hi[3] = {1, 1, 1};
  const int pad = 3 - d->rank;
  for (int r = 0; r < d->rank; ++r) {
    dims[pad + r] = d->dims[r];
    lo[pad + r] = d->lo[r];
    hi[pad + r] = d->hi[r];
  }
  g.d1 = dims[1];
  g.d2 = dims[2];
  g.lo0 = lo[0];
  g.lo1 = lo[1];
  g.lo2 = lo[2];
  g.e0 = hi[0] - lo[0];
  g.e1 = hi[1] - lo[1];
  g.e2 = hi[2] - lo[2];
  if (g.e0 <= 0 || g.e1 <= 0 || g.e2 <= 0) return GFB_OK;
  for (int t = 0; t < d->ntaps; ++t) {
    int64_t dl[3] = {0, 0, 0};
    for (int r = 0; r < d->rank; ++r) dl[pad + r] = d->tap_delta[t][r];
    g.tap_off[t] = (dl[0] * g.d1 + dl[1]) * g.d2 + dl[2];
    const int64_t esz = d->dtype == GFB_F64 ? 8 : 4;
    g.tap_base[t] = (const char *)d->src[d->tap_src[t]] + g.tap_off[t] * esz;
    for (int r = 0; r < 3; ++r) {
      g.mlo[t][r] = r < pad ? INT64_MIN / 4 : d->tap_mlo[t][r - pad];
      g.mhi[t][r] = r < pad ? INT64_MAX / 4 : d->tap_mhi[t][r - pad];
    }
  }
  g.any_masked = 0;
  for (int t = 0; t < d->ntaps; ++t) g.any_masked |= d->tap_masked[t] ? 1 : 0;
  for (int r = 0; r < 3; ++r) {
    g.clo[r] = r < pad ? INT64_MIN / 4 : d->clear_lo[r - pad];
    g.chi[r] = r < pad ? INT64_MAX / 4 : d->clear_hi[r - pad];
  }
  dim3 block(kSX, kSY);
  // planes per CTA: kMarch on large domains; small (L2-resident) domains
  // march fewer planes so a thread's serial chain of plane loads stays short
  // and the grid still fills the SMs (C2 heat_3d, 70^3)
  const int64_t tiles = ceil_div(g.e2, kSX) * ceil_div(g.e1, kSY);
  g.march = kMarch;
  while (g.march > 2 && tiles * ceil_div(g.e0, g.march) < (int64_t)sm_count() * 4) g.march /= 2;
  dim3 grid((unsigned)ceil_div(g.e2, kSX), (unsigned)ceil_div(g.e1, kSY), (unsigned)ceil_div(g.e0, g.march));
  if (grid.y > 65535 || grid.z > 65535) return set_error(GFB_EUNSUPPORTED, "gfb_stencil_launch: extent too large");
  cudaStream_t st = (cudaStream_t)stream;
#define GFB_STENCIL_LAUNCH(MT)                                      \
  if (d->dtype == GFB_F64)                                          \
    launch_pdl(stencil_kernel<double, MT>, grid, block, 0, st, *d, g); \
  else                                                              \
    launch_pdl(stencil_kernel<float, MT>, grid, block, 0, st, *d, g);
  const bool cm1 = (d->clear_mode == 1 || d->clear_mode == 3) && !g.any_masked;
  const bool cm2 = d->clear_mode == 2 && g.any_masked;
  if (d->ntaps == 7 && (cm1 || cm2)) {  // heat_3d sweeps (forward / adjoint)
    if (d->dtype == GFB_F64) {
      if (cm1) launch_pdl(stencil_kernel<double, 8, 7, 1>, grid, block, 0, st, *d, g);
      else launch_pdl(stencil_kernel<double, 8, 7, 2>, grid, block, 0, st, *d, g);
    } else {
      if (cm1) launch_pdl(stencil_kernel<float, 8, 7, 1>, grid, block, 0, st, *d, g);
      else launch_pdl(stencil_kernel<float, 8, 7, 2>, grid, block, 0, st, *d, g);
    }
  } else if (d->ntaps <= 8) {
    GFB_STENCIL_LAUNCH(8)
  } else if (d->ntaps <= 16) {
    GFB_STENCIL_LAUNCH(16)
  } else {
    GFB_STENCIL_LAUNCH(32)
  }
#undef GFB_STENCIL_LAUNCH
  return check_launch("stencil");
}
