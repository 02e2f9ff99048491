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

#include <type_traits>

#include "gfb_internal.h"
#include "star_common.cuh"

namespace gfb {

// Y window: halo 2 in (j, k). The row pitch is padded so that a column of
// the window (the edge X points) spreads over more shared-memory banks; the
// TMA box inner extent must stay a multiple of 16 bytes.
constexpr int YJ = kPY + 4;
template <typename T>
__host__ __device__ constexpr int ypitch() {
  return sizeof(T) == 8 ? kPX + 6 : kPX + 4;
}
constexpr int kDist = 5;        // planes in flight ahead of use
constexpr int NSY = kDist + 3;  // Y ring slots (8: index by mask)
static_assert((NSY & (NSY - 1)) == 0, "Y ring must be a power of two");
constexpr int HX = kPX + 2;           // X~ window pitch (halo 1)
constexpr int XS = (kPY + 2) * HX;    // X~ window plane
constexpr int kTT = kPX * kPY / 2;    // 256 threads: each owns two adjacent Z rows

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

// ring slot stride (elements): TMA destinations must be 128-byte aligned
template <typename T>
__host__ __device__ constexpr int yslot() {
  return (int)(((size_t)YJ * ypitch<T>() * sizeof(T) + 127) / 128 * 128 / sizeof(T));
}
template <typename T>
__host__ __device__ constexpr size_t star_tma_smem_bytes() {
  return (size_t)NSY * yslot<T>() * sizeof(T) + (size_t)4 * XS * sizeof(T) + NSY * sizeof(uint64_t);
}

template <typename T>
__device__ __forceinline__ T coef(const StarOpDev &o, int p);
template <>
__device__ __forceinline__ double coef<double>(const StarOpDev &o, int p) {
  return o.coef[p];
}
template <>
__device__ __forceinline__ float coef<float>(const StarOpDev &o, int p) {
  return o.fcoef[p];
}

// One CTA: a (kPY x kPX) column of Z over planes [i0, i1), marching along
// dim 0. Per plane q: X(q) = a(Y) on the CTA's halo window, then Z(q - 1) =
// b(X). Thread (tx, ty) owns the Z points (2ty, tx), (2ty + 1, tx) and the X
// points at the same positions, so the dim-0 taps of both sweeps and the
// shared j-neighbour come from registers rolled along the march; only the
// remaining in-plane neighbours are shared-memory loads. Warps 0..3 also
// compute one point each of the X halo ring (rows 0 / kPY + 1, columns
// 0 / kPX + 1). Shared-memory wavefronts, not HBM, bound this kernel, so
// every load removed here is time.
//
// Masks are data: op a's taps are in source-mask form (every masked tap
// reads "source inside M_a"), so values outside M_a are zeroed in the Y ring
// once per plane and every tap runs unmasked; op b's source mask is applied
// when X is stored (X~ = X inside M_b, else 0). Points whose region / base /
// write-back status differs from the CTA's common case take a fix-up branch.
template <typename T, bool HAS_I>
__device__ __forceinline__ void star_tma_body(const CUtensorMap *ymap, const StarPairDev &d, T *ys, T *xs,
                                              uint64_t *mbar, const uint32_t *aj, const uint32_t *ak,
                                              const uint32_t *bj, const uint32_t *bk, const uint32_t *ai,
                                              const uint32_t *bi, int i0, int i1) {
  constexpr int YK = ypitch<T>();
  constexpr int YS = YJ * YK, YSS = yslot<T>();
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * kPX + tx;
  const int k0 = blockIdx.x * kPX, j0 = blockIdx.y * kPY;
  const T *__restrict__ Xo = (const T *)d.xold;
  const T *__restrict__ Zo = (const T *)d.zold;
  T *__restrict__ Xn = (T *)d.xout;
  T *__restrict__ Zn = (T *)d.zout;
  const int ps = d.ps, rs = d.rs;
  const int amode = d.a.mode, bmode = d.b.mode;
  // planes: X(q) for q in [qbeg, min(qend, d0 - 1)], Y needed on [ylo, yhi]
  const int qbeg = HAS_I ? max(i0 - 1, 0) : 0, qend = HAS_I ? i1 : 0;
  const int ylo = HAS_I ? max(qbeg - 1, 0) : 0;
  const int yhi = HAS_I ? min(min(qend, d.d0 - 1) + 1, d.d0 - 1) : 0;
  constexpr uint32_t kTx = (uint32_t)(YS * sizeof(T));
  auto slot_of = [&](int p) { return ys + ((p - ylo) & (NSY - 1)) * YSS; };
  auto issue = [&](int p) {
    const int sl = (p - ylo) & (NSY - 1);
    mbar_expect_tx(&mbar[sl], kTx);
    tma_load_3d(ys + sl * YSS, ymap, &mbar[sl], k0 - 2, j0 - 2, p);
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

  // this thread's points (window coordinates: X~ halo 1, Y halo 2)
  const int hj0 = 2 * ty + 1, hk = tx + 1;
  int rj = -1, rk = 0;  // halo-ring X point
  if (ty == 0) {
    rj = 0;
    rk = hk;
  } else if (ty == 1) {
    rj = kPY + 1;
    rk = hk;
  } else if (ty == 2 && tx < kPY + 2) {
    rj = tx;
    rk = 0;
  } else if (ty == 3 && tx < kPY + 2) {
    rj = tx;
    rk = kPX + 1;
  }
  const bool ring = rj >= 0;
  const int yo0 = (hj0 + 1) * YK + hk + 1, yo1 = yo0 + YK;
  const int yor = ring ? (rj + 1) * YK + rk + 1 : yo0;
  const int xo0 = hj0 * HX + hk, xo1 = xo0 + HX;
  const int xor_ = ring ? rj * HX + rk : xo0;
  const int rel0 = (j0 + 2 * ty) * rs + (k0 + tx), rel1 = rel0 + rs;
  const int relr = (j0 - 1 + rj) * rs + (k0 - 1 + rk);
  const uint32_t mx0 = aj[hj0] & ak[hk], mx1 = aj[hj0 + 1] & ak[hk];
  const uint32_t mxr = ring ? (aj[rj] & ak[rk]) : 0u;
  const uint32_t mz0 = bj[2 * ty] & bk[tx], mz1 = bj[2 * ty + 1] & bk[tx];

  const bool ysrc = d.a.srcmask == 1;
  const bool yj_in = j0 - 2 >= d.a.smlo[1] && j0 + kPY + 2 <= d.a.smhi[1];
  const bool yk_in = k0 - 2 >= d.a.smlo[2] && k0 + kPX + 2 <= d.a.smhi[2];
  auto prepare_plane = [&](int p) {
    // zero what the taps must not see: planes never loaded (outside the
    // local array) and, in source-mask form, values outside M_a
    T *slot = slot_of(p);
    const int pg = p + d.p0;
    const bool outside = p < 0 || p >= d.d0 || (ysrc && (pg < d.a.smlo[0] || pg >= d.a.smhi[0]));
    if (outside) {
      for (int e = tid; e < YS; e += kTT) slot[e] = T(0);
    } else if (ysrc && !(yj_in && yk_in)) {
      for (int e = tid; e < YS; e += kTT) {
        const int jj = e / YK, kk = e - jj * YK;
        const int j = j0 - 2 + jj, k = k0 - 2 + kk;
        if (j < d.a.smlo[1] || j >= d.a.smhi[1] || k < d.a.smlo[2] || k >= d.a.smhi[2]) slot[e] = T(0);
      }
    }
  };
  // common-case predicate patterns (block-uniform)
  const uint32_t xmask = kArray | kRegion | (amode == 2 ? kClear : 0u) | (d.xwrite ? kDead : 0u);
  const uint32_t xval = amode == 0 ? 0xffffffffu : xmask;  // mode 0: base always added -> fix-up
  const uint32_t zmask = kArray | kRegion | (bmode == 2 ? kClear : 0u);
  const uint32_t zval = bmode == 0 ? 0xffffffffu : zmask;
  // X~ of one point from its tap sum; abnormal points take the fix-up
  auto x_tilde = [&](T acc, uint32_t w, int rel, bool wb, int q) -> T {
    if ((w & xmask) != xval) {
      if (!(w & kArray)) {
        acc = T(0);
      } else {
        const int off = q * ps + rel;
        if (!(w & kRegion))
          acc = Xo[off];
        else if (amode == 0 || (amode == 2 && !(w & kClear)))
          acc += Xo[off];
        if (wb && d.xwrite && !(w & kDead)) Xn[off] = acc;
      }
    }
    return (w & kSrcB) ? acc : T(0);
  };
  const T a0 = coef<T>(d.a, 0), a1 = coef<T>(d.a, 1), a2 = coef<T>(d.a, 2), a3 = coef<T>(d.a, 3),
          a4 = coef<T>(d.a, 4), a5 = coef<T>(d.a, 5), a6 = coef<T>(d.a, 6);
  const T b0 = coef<T>(d.b, 0), b1 = coef<T>(d.b, 1), b2 = coef<T>(d.b, 2), b3 = coef<T>(d.b, 3),
          b4 = coef<T>(d.b, 4), b5 = coef<T>(d.b, 5), b6 = coef<T>(d.b, 6);

  // CTA-uniform "every point normal" tests: AND of the (j, k) predicate
  // words over the X window / Z tile; per plane the dim-0 word completes it
  __shared__ uint32_t s_jk[2];
  if (ty == 0) {
    uint32_t va = ak[tx] & (tx < kPY + 2 ? aj[tx] : ~0u) & (tx + 32 < HX ? ak[tx + 32] : ~0u);
    uint32_t vb = bk[tx] & (tx < kPY ? bj[tx] : ~0u);
    va = __reduce_and_sync(0xffffffffu, va);
    vb = __reduce_and_sync(0xffffffffu, vb);
    if (tx == 0) {
      s_jk[0] = va;
      s_jk[1] = vb;
    }
  }
  const uint32_t xfast_m = xmask | kSrcB;

  for (int p = ylo; p <= min(qbeg + 1, yhi); ++p) wait_plane(p);
  if (HAS_I) {
    for (int p = qbeg - 1; p <= qbeg + 1; ++p) prepare_plane(p);
  } else {
    prepare_plane(0);
  }
  __syncthreads();
  const uint32_t jka = (amode == 0) ? 0u : s_jk[0], jkb = (bmode == 0) ? 0u : s_jk[1];

  // Registers rolled along the march, rotated by index (three live planes):
  // y*[.] = Y centre values at the own (0, 1) and ring (r) X points,
  // x*[.] = X~ at the own Z points. Step s of the unrolled loop finds
  // Y(q - 1), Y(q) in slots s, s + 1 and loads Y(q + 1) into slot s + 2
  // (mod 3); X~(q - 2), X~(q - 1) likewise and X~(q) goes to slot s + 2.
  T y0[3], y1[3], yr[3], x0[3], x1[3];
#pragma unroll
  for (int u = 0; u < 3; ++u) y0[u] = y1[u] = yr[u] = x0[u] = x1[u] = T(0);
  {
    const T *yq = slot_of(qbeg);
    y0[1] = yq[yo0];
    y1[1] = yq[yo1];
    yr[1] = yq[yor];
    if (HAS_I) {
      const T *yqm = slot_of(qbeg - 1);
      y0[0] = yqm[yo0];
      y1[0] = yqm[yo1];
      yr[0] = yqm[yor];
    }
  }

  auto step = [&](auto S, int q) {
    constexpr int M = decltype(S)::value, C = (M + 1) % 3, P = (M + 2) % 3;
    x0[P] = T(0);
    x1[P] = T(0);
    if (q < d.d0) {
      if (tid == 0) {
        const int pn = q + 1 + kDist;
        if (pn > pre_hi && pn <= yhi) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue(pn);
        }
      }
      if (HAS_I) {
        // plane q + 2 is needed by X(q + 1): land it and mask it now; the
        // barrier below orders this before any read of it
        const int pn = q + 2;
        if (pn <= yhi && pn > qbeg + 1) wait_plane(pn);
        if (pn <= qend + 1 && pn > qbeg + 1) prepare_plane(pn);
      }
      const T *yc = slot_of(q);
      const T *yp = slot_of(q + 1);
      T *xw = xs + (q & 3) * XS;
      const uint32_t mi = ai[q - i0 + 1];
      if (HAS_I) {
        y0[P] = yp[yo0];
        y1[P] = yp[yo1];
      }
      // short dependency chains: four partial sums per point
      T p0 = a0 * y0[C], p1 = a0 * y1[C];
      if (HAS_I) {
        p0 = fma(a1, y0[M], p0);
        p1 = fma(a1, y1[M], p1);
      }
      T q0 = a4 * y1[C], q1 = a3 * y0[C];
      if (HAS_I) {
        q0 = fma(a2, y0[P], q0);
        q1 = fma(a2, y1[P], q1);
      }
      const T r0 = fma(a5, yc[yo0 - 1], a3 * yc[yo0 - YK]);
      const T r1 = fma(a5, yc[yo1 - 1], a4 * yc[yo1 + YK]);
      p0 = fma(a6, yc[yo0 + 1], p0);
      p1 = fma(a6, yc[yo1 + 1], p1);
      T acc0 = (p0 + q0) + r0, acc1 = (p1 + q1) + r1;
      const bool fast = ((mi & jka) & xfast_m) == xfast_m;
      if (!fast) {
        const bool own = q >= i0 && q < i1;
        acc0 = x_tilde(acc0, mi & mx0, rel0, own, q);
        acc1 = x_tilde(acc1, mi & mx1, rel1, own, q);
      }
      x0[P] = acc0;
      x1[P] = acc1;
      xw[xo0] = acc0;
      xw[xo1] = acc1;
      if (ring) {
        const T yrp = HAS_I ? yp[yor] : T(0);
        T pr = a0 * yr[C];
        if (HAS_I) pr = fma(a1, yr[M], fma(a2, yrp, pr));
        const T qr = fma(a3, yc[yor - YK], a4 * yc[yor + YK]);
        const T rr = fma(a5, yc[yor - 1], a6 * yc[yor + 1]);
        T acc = (pr + qr) + rr;
        if (!fast) acc = x_tilde(acc, mi & mxr, relr, false, q);
        xw[xor_] = acc;
        yr[P] = yrp;
      }
    }
    __syncthreads();
    const int i = HAS_I ? q - 1 : q;
    if (i >= i0 && i < i1) {
      const T *xc = xs + (i & 3) * XS;
      // centre values: X~(i) and, along dim 0, X~(i -/+ 1) from registers
      const T c0 = HAS_I ? x0[C] : x0[P], c1 = HAS_I ? x1[C] : x1[P];
      T p0 = b0 * c0, p1 = b0 * c1;
      if (HAS_I) {
        p0 = fma(b1, x0[M], p0);
        p1 = fma(b1, x1[M], p1);
      }
      T q0 = b4 * c1, q1 = b3 * c0;
      if (HAS_I) {
        q0 = fma(b2, x0[P], q0);
        q1 = fma(b2, x1[P], q1);
      }
      const T r0 = fma(b5, xc[xo0 - 1], b3 * xc[xo0 - HX]);
      const T r1 = fma(b5, xc[xo1 - 1], b4 * xc[xo1 + HX]);
      p0 = fma(b6, xc[xo0 + 1], p0);
      p1 = fma(b6, xc[xo1 + 1], p1);
      T z0 = (p0 + q0) + r0, z1 = (p1 + q1) + r1;
      T *zrow = Zn + (size_t)i * ps + rel0;
      const uint32_t mi = bi[i - i0];
      if (((mi & jkb) & zmask) == zmask) {
        zrow[0] = z0;
        zrow[rs] = z1;
      } else {
        const T *zold = Zo + (size_t)i * ps + rel0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t w = mi & (h ? mz1 : mz0);
          T z = h ? z1 : z0;
          const int o = h ? rs : 0;
          if ((w & zmask) != zval) {
            if (!(w & kArray)) continue;
            if (!(w & kRegion))
              z = zold[o];
            else if (bmode == 0 || (bmode == 2 && !(w & kClear)))
              z += zold[o];
          }
          zrow[o] = z;
        }
      }
    }
  };
  using I0 = std::integral_constant<int, 0>;
  using I1 = std::integral_constant<int, 1>;
  using I2 = std::integral_constant<int, 2>;
  for (int q = qbeg; q <= qend; q += 3) {
    step(I0{}, q);
    if (q + 1 > qend) break;
    step(I1{}, q + 1);
    if (q + 2 > qend) break;
    step(I2{}, q + 2);
  }
}

template <typename T>
__global__ void __launch_bounds__(kTT, 3)
    star_pair_tma_kernel(const __grid_constant__ CUtensorMap ymap, const __grid_constant__ StarPairDev d) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr size_t ybytes = (size_t)NSY * yslot<T>() * sizeof(T);
  T *ys = reinterpret_cast<T *>(smem);
  T *xs = reinterpret_cast<T *>(smem + ybytes);
  uint64_t *mbar = reinterpret_cast<uint64_t *>(smem + ybytes + (size_t)4 * XS * sizeof(T));
  __shared__ uint32_t aj[kPY + 2], ak[kPX + 2], bj[kPY], bk[kPX], ai[kPM + 2], bi[kPM];
  __shared__ uint32_t s_and_a, s_or_a, s_and_b, s_or_b;
  const int tid = threadIdx.y * kPX + threadIdx.x;
  const int i0 = d.zlo + blockIdx.z * kPM, i1 = min(i0 + kPM, d.zhi);
  star_prologue(d, i0, i1, tid, aj, ak, bj, bk, ai, bi, s_and_a, s_or_a, s_and_b, s_or_b);
  if (d.d0 > 1)
    star_tma_body<T, true>(&ymap, d, ys, xs, mbar, aj, ak, bj, bk, ai, bi, i0, i1);
  else
    star_tma_body<T, false>(&ymap, d, ys, xs, mbar, aj, ak, bj, bk, ai, bi, i0, i1);
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
  cuuint32_t box[3] = {(cuuint32_t)(dtype == GFB_F64 ? ypitch<double>() : ypitch<float>()), (cuuint32_t)YJ, 1};
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
