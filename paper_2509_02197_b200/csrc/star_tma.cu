// TMA-fed variant of the fused star-pair kernel (see star.cu for the
// algorithm). The source planes Y(q) are moved into a shared-memory ring by
// the Tensor Memory Accelerator (cp.async.bulk.tensor, one elected thread,
// mbarrier transaction counts), kDist planes ahead of use, with the one-
// point halo window [j0-2, j0+kPY+2) x [k0-2, k0+kPX+2) per plane; TMA
// zero-fills the parts that fall outside the array. Every tap of the first
// sweep is then one shared-memory load at an immediate offset, the global
// traffic is bulk and asynchronous, and the SMs spend their issue slots on
// the arithmetic.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "gfb_internal.h"
#include "star_common.cuh"

namespace gfb {

constexpr int YK = kPX + 4, YJ = kPY + 4;  // Y window: halo 2 in (j, k)
constexpr int kDist = 5;                    // planes in flight ahead of use
constexpr int NSY = kDist + 3;              // Y ring slots (8: index by mask)
static_assert((NSY & (NSY - 1)) == 0, "Y ring must be a power of two");

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

template <typename T>
__host__ __device__ constexpr size_t star_tma_smem_bytes() {
  return (size_t)NSY * YJ * YK * sizeof(T) + (size_t)4 * (kPY + 2) * (kPX + 2) * sizeof(T) + NSY * sizeof(uint64_t);
}

constexpr int kTT = kPX * kPY / 2;  // 256 threads: each owns two Z rows (ty, ty + 8)
constexpr int kXP = 3;              // halo-window X points per thread per plane (612 over 256)

template <typename T, bool HAS_I>
__device__ __forceinline__ void star_tma_body(const CUtensorMap *ymap, const StarPairDev &d, T (*ys)[YJ][YK],
                                              T (*xs)[kPY + 2][kPX + 2], uint64_t *mbar, const uint32_t *aj,
                                              const uint32_t *ak, const uint32_t *bj, const uint32_t *bk,
                                              const uint32_t *ai, const uint32_t *bi, bool fast, uint32_t aA,
                                              uint32_t aB, int i0, int i1) {
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * kPX + tx;
  const int k0 = blockIdx.x * kPX, j0 = blockIdx.y * kPY;
  constexpr int HX = kPX + 2, HW = (kPY + 2) * HX;
  constexpr int YS = YJ * YK, XS = (kPY + 2) * HX;
  const T *__restrict__ Xo = (const T *)d.xold;
  const T *__restrict__ Zo = (const T *)d.zold;
  T *__restrict__ Xn = (T *)d.xout;
  T *__restrict__ Zn = (T *)d.zout;
  const int ps = d.ps, rs = d.rs;
  T ca[7], cb[7];
#pragma unroll
  for (int p = 0; p < 7; ++p) {
    ca[p] = (T)d.a.coef[p];
    cb[p] = (T)d.b.coef[p];
  }
  const uint32_t apres = d.a.present, bpres = d.b.present;
  const int amode = d.a.mode, bmode = d.b.mode;
  // planes: X(q) for q in [qbeg, min(qend, d0 - 1)], Y needed on [ylo, yhi]
  const int qbeg = HAS_I ? max(i0 - 1, 0) : 0, qend = HAS_I ? i1 : 0;
  const int ylo = HAS_I ? max(qbeg - 1, 0) : 0;
  const int yhi = HAS_I ? min(min(qend, d.d0 - 1) + 1, d.d0 - 1) : 0;
  constexpr uint32_t kTx = (uint32_t)(YJ * YK * sizeof(T));
  auto issue = [&](int p) {
    const int r = p - ylo, slot = r & (NSY - 1);
    mbar_expect_tx(&mbar[slot], kTx);
    tma_load_3d(&ys[slot][0][0], ymap, &mbar[slot], k0 - 2, j0 - 2, p);
  };
  auto wait_plane = [&](int p) {
    const int r = p - ylo;
    mbar_wait(&mbar[r & (NSY - 1)], (uint32_t)((r / NSY) & 1));
  };
  if (tid == 0) {
    for (int s = 0; s < NSY; ++s) mbar_init(&mbar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int pre_hi = min(ylo + kDist + 1, yhi);
  if (tid == 0)
    for (int p = ylo; p <= pre_hi; ++p) issue(p);
  // thread -> halo-window X points p = tid + m * kTT (m < kXP, p < HW)
  int hj[kXP], hk[kXP], yo[kXP], xo[kXP], rel[kXP];
  bool has[kXP], core[kXP];
  uint32_t mjk[kXP];
#pragma unroll
  for (int m = 0; m < kXP; ++m) {
    const int p = tid + m * kTT;
    has[m] = p < HW;
    hj[m] = has[m] ? p / HX : 0;
    hk[m] = has[m] ? p - hj[m] * HX : 0;
    yo[m] = (hj[m] + 1) * YK + hk[m] + 1;
    xo[m] = hj[m] * HX + hk[m];
    rel[m] = (j0 - 1 + hj[m]) * rs + (k0 - 1 + hk[m]);
    core[m] = has[m] && hj[m] >= 1 && hj[m] <= kPY && hk[m] >= 1 && hk[m] <= kPX;
    mjk[m] = has[m] ? (aj[hj[m]] & ak[hk[m]]) : 0u;
  }
  // Z rows ty and ty + 8
  const int zrel0 = (j0 + ty) * rs + (k0 + tx), zrel1 = zrel0 + 8 * rs;
  const int zo0 = (ty + 1) * HX + tx + 1, zo1 = zo0 + 8 * HX;
  const uint32_t mz0 = bj[ty] & bk[tx], mz1 = bj[ty + 8] & bk[tx];
  const bool xbase_f = amode == 0 || (amode == 2 && !(aA & kClear));
  const bool zbase_f = bmode == 0 || (bmode == 2 && !(aB & kClear));
  const bool xw_f = d.xwrite && !(aA & kDead);
  for (int p = ylo; p <= min(qbeg, yhi); ++p) wait_plane(p);
  const T *ysf = &ys[0][0][0];
  T *xsf = &xs[0][0][0];

  if (fast && !xbase_f && !zbase_f && !xw_f) {
    // Interior CTA: every tap admitted, bases vanish, no X write-back. The
    // plane loop is shared-memory arithmetic plus coalesced Z stores.
    const T a0 = ca[0], a1 = ca[1], a2 = ca[2], a3 = ca[3], a4 = ca[4], a5 = ca[5], a6 = ca[6];
    const T b0 = cb[0], b1 = cb[1], b2 = cb[2], b3 = cb[3], b4 = cb[4], b5 = cb[5], b6 = cb[6];
    T *zp = Zn + (int64_t)(qbeg - 1) * ps;
    int r = qbeg - ylo;
    for (int q = qbeg; q <= qend; ++q, ++r, zp += ps) {
      if (tid == 0) {
        const int pn = q + 1 + kDist;
        if (pn > pre_hi && pn <= yhi) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue(pn);
        }
      }
      if (HAS_I && q + 1 <= yhi && q + 1 > qbeg) wait_plane(q + 1);
      const T *yc = ysf + (r & (NSY - 1)) * YS;
      const T *ym = ysf + ((r - 1) & (NSY - 1)) * YS;
      const T *yp = ysf + ((r + 1) & (NSY - 1)) * YS;
      T *xw = xsf + (q & 3) * XS;
#pragma unroll
      for (int m = 0; m < kXP; ++m) {
        if (m == kXP - 1 && !has[m]) break;
        const T *c = yc + yo[m];
        T acc = a0 * c[0];
        if (HAS_I) acc = fma(a1, ym[yo[m]], fma(a2, yp[yo[m]], acc));
        acc = fma(a3, c[-YK], acc);
        acc = fma(a4, c[YK], acc);
        acc = fma(a5, c[-1], acc);
        acc = fma(a6, c[1], acc);
        xw[xo[m]] = acc;
      }
      __syncthreads();
      if (!HAS_I || q >= i0 + 1) {  // Z(i) for i = q - 1 in [i0, i1)
        const int i = HAS_I ? q - 1 : q;
        const T *xc = xsf + (i & 3) * XS;
        const T *xm = xsf + ((i - 1) & 3) * XS;
        const T *xp = xsf + ((i + 1) & 3) * XS;
        T *zrow = HAS_I ? zp : zp + ps;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int zo = h ? zo1 : zo0;
          const T *c = xc + zo;
          T w = b0 * c[0];
          if (HAS_I) w = fma(b1, xm[zo], fma(b2, xp[zo], w));
          w = fma(b3, c[-HX], w);
          w = fma(b4, c[HX], w);
          w = fma(b5, c[-1], w);
          w = fma(b6, c[1], w);
          zrow[h ? zrel1 : zrel0] = w;
        }
      }
    }
    return;
  }

  // boundary / general CTA: per-point predicate words, branch-free selects
  for (int q = qbeg; q <= qend; ++q) {
    if (q < d.d0) {
      if (tid == 0) {
        const int pn = q + 1 + kDist;
        if (pn > pre_hi && pn <= yhi) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue(pn);
        }
      }
      if (HAS_I && q + 1 <= yhi && q + 1 > qbeg) wait_plane(q + 1);
      const int r = q - ylo;
      const T *yc = ysf + (r & (NSY - 1)) * YS;
      const T *ym = ysf + ((r - 1) & (NSY - 1)) * YS;  // never filled: taps masked
      const T *yp = ysf + ((r + 1) & (NSY - 1)) * YS;
      T *xw = xsf + (q & 3) * XS;
      const bool own = q >= i0 && q < i1;
      const uint32_t mi = ai[q - i0 + 1];
#pragma unroll
      for (int m = 0; m < kXP; ++m) {
        if (!has[m]) continue;
        const uint32_t mm = mi & mjk[m];
        T v = T(0);
        if (mm & kArray) {
          const int off = q * ps + rel[m];
          if (mm & kRegion) {
            const bool base = amode == 0 || (amode == 2 && !(mm & kClear));
            T acc = base ? Xo[off] : T(0);
            const uint32_t on = apres & mm;
            const T *c = yc + yo[m];
            acc += (on & 1u) ? ca[0] * c[0] : T(0);
            if (HAS_I) {
              acc += (on & 2u) ? ca[1] * ym[yo[m]] : T(0);
              acc += (on & 4u) ? ca[2] * yp[yo[m]] : T(0);
            }
            acc += (on & 8u) ? ca[3] * c[-YK] : T(0);
            acc += (on & 16u) ? ca[4] * c[YK] : T(0);
            acc += (on & 32u) ? ca[5] * c[-1] : T(0);
            acc += (on & 64u) ? ca[6] * c[1] : T(0);
            v = acc;
          } else {
            v = Xo[off];
          }
          if (own && core[m] && d.xwrite && !(mm & kDead)) Xn[off] = v;
        }
        xw[xo[m]] = v;
      }
    }
    __syncthreads();
    const int i = HAS_I ? q - 1 : q;
    if (i >= i0 && i < i1) {
      const T *xc = xsf + (i & 3) * XS;
      const T *xm = xsf + ((i - 1) & 3) * XS;
      const T *xp = xsf + ((i + 1) & 3) * XS;
      const uint32_t mi = bi[i - i0];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t m = mi & (h ? mz1 : mz0);
        if (!(m & kArray)) continue;
        const int off = i * ps + (h ? zrel1 : zrel0);
        T w;
        if (m & kRegion) {
          const bool base = bmode == 0 || (bmode == 2 && !(m & kClear));
          w = base ? Zo[off] : T(0);
          const uint32_t on = bpres & m;
          const int zo = h ? zo1 : zo0;
          const T *c = xc + zo;
          w += (on & 1u) ? cb[0] * c[0] : T(0);
          if (HAS_I) {
            w += (on & 2u) ? cb[1] * xm[zo] : T(0);
            w += (on & 4u) ? cb[2] * xp[zo] : T(0);
          }
          w += (on & 8u) ? cb[3] * c[-HX] : T(0);
          w += (on & 16u) ? cb[4] * c[HX] : T(0);
          w += (on & 32u) ? cb[5] * c[-1] : T(0);
          w += (on & 64u) ? cb[6] * c[1] : T(0);
        } else {
          w = Zo[off];
        }
        Zn[off] = w;
      }
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(kTT, 3)
    star_pair_tma_kernel(const __grid_constant__ CUtensorMap ymap, const __grid_constant__ StarPairDev d) {
  extern __shared__ __align__(128) unsigned char smem[];
  T(*ys)[YJ][YK] = reinterpret_cast<T(*)[YJ][YK]>(smem);
  T(*xs)[kPY + 2][kPX + 2] = reinterpret_cast<T(*)[kPY + 2][kPX + 2]>(smem + (size_t)NSY * YJ * YK * sizeof(T));
  uint64_t *mbar = reinterpret_cast<uint64_t *>(smem + (size_t)NSY * YJ * YK * sizeof(T) +
                                                (size_t)4 * (kPY + 2) * (kPX + 2) * sizeof(T));
  __shared__ uint32_t aj[kPY + 2], ak[kPX + 2], bj[kPY], bk[kPX], ai[kPM + 2], bi[kPM];
  __shared__ uint32_t s_and_a, s_or_a, s_and_b, s_or_b;
  const int tid = threadIdx.y * kPX + threadIdx.x;
  const int i0 = d.zlo + blockIdx.z * kPM, i1 = min(i0 + kPM, d.zhi);
  star_prologue(d, i0, i1, tid, aj, ak, bj, bk, ai, bi, s_and_a, s_or_a, s_and_b, s_or_b);
  const uint32_t apres = d.a.present, bpres = d.b.present;
  const uint32_t full = d.d0 > 1 ? 0x7fu : 0x79u;
  const uint32_t fa = full | kRegion | kArray, fb = full | kRegion | kArray;
  const uint32_t aA = s_and_a, oA = s_or_a, aB = s_and_b, oB = s_or_b;
  const bool fast = apres == full && bpres == full && (aA & fa) == fa && (aB & fb) == fb &&
                    ((aA ^ oA) & (kClear | kDead)) == 0 && ((aB ^ oB) & kClear) == 0 &&
                    (d.d0 == 1 || (i0 >= 2 && i1 <= d.d0 - 2));
  if (d.d0 > 1)
    star_tma_body<T, true>(&ymap, d, ys, xs, mbar, aj, ak, bj, bk, ai, bi, fast, aA, aB, i0, i1);
  else
    star_tma_body<T, false>(&ymap, d, ys, xs, mbar, aj, ak, bj, bk, ai, bi, fast, aA, aB, i0, i1);
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

bool star_tma_usable(const StarPairDev &d, int dtype) {
  const int64_t es = dtype == GFB_F64 ? 8 : 4;
  return encode_fn() != nullptr && ((int64_t)d.d2 * es) % 16 == 0 && ((uintptr_t)d.y % 16) == 0 &&
         getenv("GFB_NO_TMA") == nullptr;
}

int launch_star_pair_tma(const StarPairDev &d, int dtype, dim3 grid, cudaStream_t st) {
  const int64_t es = dtype == GFB_F64 ? 8 : 4;
  CUtensorMap map;
  cuuint64_t dims[3] = {(cuuint64_t)d.d2, (cuuint64_t)d.d1, (cuuint64_t)d.d0};
  cuuint64_t strides[2] = {(cuuint64_t)(d.d2 * es), (cuuint64_t)((int64_t)d.d1 * d.d2 * es)};
  cuuint32_t box[3] = {(cuuint32_t)YK, (cuuint32_t)YJ, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode_fn()(&map, dtype == GFB_F64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                           3, const_cast<void *>(d.y), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(GFB_ECUDA, "cuTensorMapEncodeTiled failed for the star-pair source");
  dim3 block(kPX, kPY / 2);
  if (dtype == GFB_F64) {
    static bool attr = false;
    const size_t sm = star_tma_smem_bytes<double>();
    if (!attr) {
      cudaFuncSetAttribute(star_pair_tma_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      attr = true;
    }
    star_pair_tma_kernel<double><<<grid, block, sm, st>>>(map, d);
  } else {
    static bool attr = false;
    const size_t sm = star_tma_smem_bytes<float>();
    if (!attr) {
      cudaFuncSetAttribute(star_pair_tma_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      attr = true;
    }
    star_pair_tma_kernel<float><<<grid, block, sm, st>>>(map, d);
  }
  return check_launch("star_pair_tma");
}

}  // namespace gfb
