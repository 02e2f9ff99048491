// TMA-fed variant of the fused star-pair kernel (see star.cu for the
// algorithm: X = a(Y); Z = b(X), two radius-1 star sweeps in one launch).
//
// One CTA owns a (tPY x tPX) = 32 x 32 column of Z over up to tPM planes and
// marches along dim 0. The source planes Y(q), with a two-point halo in
// (j, k), are moved into a shared-memory ring by the Tensor Memory
// Accelerator (cp.async.bulk.tensor, one elected thread, mbarrier
// transaction counts) kDist planes ahead of use; TMA zero-fills whatever
// falls outside the array. Per plane q the CTA computes X(q) on its one-point
// halo window (kept as X~ in a 3-slot shared ring), then Z(q - 1).
//
// Thread (tx, ty) owns the four Z points (4ty + u, tx), u < 4, and the X
// points at the same positions. The dim-0 taps of both sweeps and the
// j-neighbours inside the thread's four rows come from registers rolled
// along the march, so per point only the +-k neighbours (and one j-neighbour
// per four rows) are shared-memory loads. Warps 0..4 also compute one point
// each of the X halo ring. The CTA-uniform overhead of a plane (ring
// issue, barrier, predicates) is spread over 1024 points.
//
// Masks are data: op a's taps are in source-mask form (every masked tap
// reads "source inside M_a"), so values outside M_a are zeroed in the Y ring
// once per plane and every tap runs unmasked; op b's source mask is applied
// when X is stored (X~ = X inside M_b, else 0). Points whose region / base /
// write-back status differs from the plane's common case take a fix-up
// branch; a plane whose whole window is common takes none.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <type_traits>

#include "gfb_internal.h"
#include "star_common.cuh"

// Compiled twice (Makefile): the default 32 x 32 tile, and a 32 x 16 tile
// with two rows per thread (namespace small) for small 2-D domains whose
// launches are short latency chains (C1 jacobi_2d 200^2: 49 CTAs -> 98)
#ifndef GFB_STAR_NS
#define GFB_STAR_NS tile32
#endif

namespace gfb {
namespace GFB_STAR_NS {

#ifndef GFB_STAR_TPY
#define GFB_STAR_TPY 32
#endif
#ifndef GFB_STAR_KR
#define GFB_STAR_KR 4
#endif
#ifndef GFB_STAR_TPM
#define GFB_STAR_TPM 32
#endif
#ifndef GFB_STAR_UNROLL
#define GFB_STAR_UNROLL 1
#endif
// tap sums as one fma chain per point (7 fp64 ops; the thread's four points
// and the ring point give the scheduler independent chains) instead of three
// partial sums (9 ops)
#ifndef GFB_STAR_CHAIN
#define GFB_STAR_CHAIN 1
#endif
#ifndef GFB_STAR_BRANCHFREE
#define GFB_STAR_BRANCHFREE 1
#endif
#ifndef GFB_STAR_WARPFAST
#define GFB_STAR_WARPFAST 1
#endif
#ifndef GFB_STAR_STEADY
#define GFB_STAR_STEADY 1
#endif
constexpr int tPX = 32, tPY = GFB_STAR_TPY, tPM = GFB_STAR_TPM;  // CTA tile (k, j) and planes
constexpr int kR = GFB_STAR_KR;                                   // Z rows per thread
constexpr int tThreads = tPX * (tPY / kR);
static_assert(tPY % kR == 0 && tThreads % 32 == 0 && tThreads <= 512, "tile / thread mismatch");
static_assert(2 * (tPY + 2) <= tThreads - 64, "halo-ring columns need warps 2..");
constexpr int YJ = tPY + 4;                  // Y window rows (halo 2)
// Y window pitch: halo 2 in k; padded so an edge column spreads over more
// shared-memory banks (the TMA box inner extent stays a multiple of 16 B)
template <typename T>
__host__ __device__ constexpr int ypitch() {
  return sizeof(T) == 8 ? tPX + 6 : tPX + 4;
}
constexpr int NSY = 6;         // Y ring slots
constexpr int kDist = NSY - 2; // planes issued ahead (slot of Y(q-1) is free at step q)
constexpr int HX = tPX + 2;    // X~ window pitch (halo 1)
constexpr int XS = (tPY + 2) * HX;
constexpr int NXS = 3;         // X~ ring slots

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

// Ampere-style asynchronous copy of one element into shared memory: the
// old-value loads of fix-up points are issued one plane ahead, so their
// DRAM latency overlaps a whole march step instead of stalling it.
template <typename T>
__device__ __forceinline__ void cp_async_elem(T *dst, const T *src) {
  if constexpr (sizeof(T) == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// ring slot stride (elements): TMA destinations must be 128-byte aligned
template <typename T>
__host__ __device__ constexpr int yslot() {
  return (int)(((size_t)YJ * ypitch<T>() * sizeof(T) + 127) / 128 * 128 / sizeof(T));
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

// Per-coordinate predicate words of the CTA (star_common.cuh coord_bits;
// op-a words also carry kSrcB = "inside op b's source mask").
struct TmaWords {
  uint32_t aj[tPY + 2], ak[tPX + 2], bj[tPY], bk[tPX], ai[tPM + 2], bi[tPM];
  uint32_t jk[2];  // AND over the X window / Z tile of the (j, k) words
};

__device__ __forceinline__ void tma_prologue(const StarPairDev &d, int i0, int j0, int k0, int tid, TmaWords &w) {
  auto srcb = [&](int dim, int c) { return (c >= d.b.smlo[dim] && c < d.b.smhi[dim]) ? kSrcB : 0u; };
  const int tpm = d.tpm;  // planes per CTA (launch-time choice, <= tPM)
  constexpr int nA = tPY + 2, nB = nA + tPX + 2, nC = nB + tPY, nD = nC + tPX;
  const int nE = nD + tpm + 2, nF = nE + tpm;
  for (int e = tid; e < nF; e += tThreads) {
    if (e < nA) {
      w.aj[e] = coord_bits(d.a, 1, j0 - 1 + e, d.d1, d.dlo, d.dhi) | srcb(1, j0 - 1 + e);
    } else if (e < nB) {
      const int c = k0 - 1 + (e - nA);
      w.ak[e - nA] = coord_bits(d.a, 2, c, d.d2, d.dlo, d.dhi) | srcb(2, c);
    } else if (e < nC) {
      w.bj[e - nB] = coord_bits(d.b, 1, j0 + (e - nB), d.d1, nullptr, nullptr);
    } else if (e < nD) {
      w.bk[e - nC] = coord_bits(d.b, 2, k0 + (e - nC), d.d2, nullptr, nullptr);
    } else if (e < nE) {
      const int c = i0 - 1 + (e - nD) + d.p0;
      w.ai[e - nD] = coord_bits(d.a, 0, c, d.gd0, d.dlo, d.dhi) | srcb(0, c);
    } else {
      w.bi[e - nE] = coord_bits(d.b, 0, i0 + (e - nE) + d.p0, d.gd0, nullptr, nullptr);
    }
  }
  __syncthreads();
  if (tid < 32) {
    uint32_t va = ~0u, vb = ~0u;
    for (int e = tid; e < tPY + 2; e += 32) va &= w.aj[e];
    for (int e = tid; e < tPX + 2; e += 32) va &= w.ak[e];
    for (int e = tid; e < tPY; e += 32) vb &= w.bj[e];
    for (int e = tid; e < tPX; e += 32) vb &= w.bk[e];
    va = __reduce_and_sync(0xffffffffu, va);
    vb = __reduce_and_sync(0xffffffffu, vb);
    if (tid == 0) {
      w.jk[0] = va;
      w.jk[1] = vb;
    }
  }
}

template <typename T, bool HAS_I, int MODES>
__device__ __forceinline__ void star_tma_body(const CUtensorMap *ymap, const StarPairDev &d, T *ys, T *xs,
                                              uint64_t *mbar, const TmaWords &W, T (*xst)[kR + 1][tThreads],
                                              int i0, int i1) {
  constexpr int YK = ypitch<T>();
  constexpr int YS = YJ * YK, YSS = yslot<T>();
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * tPX + tx;
  const int k0 = blockIdx.x * tPX, j0 = blockIdx.y * tPY;
  const T *__restrict__ Xo = (const T *)d.xold;
  const T *__restrict__ Zo = (const T *)d.zold;
  T *__restrict__ Xn = (T *)d.xout;
  T *__restrict__ Zn = (T *)d.zout;
  const int ps = d.ps, rs = d.rs;
  // MODES >= 0: the two sweeps' base modes and the X write-back fixed at
  // compile time (16 xwrite + 4 a + b)
  const int amode = MODES >= 0 ? (MODES / 4) % 4 : d.a.mode, bmode = MODES >= 0 ? MODES % 4 : d.b.mode;
  const bool xwrite = MODES >= 0 ? ((MODES / 16) & 1) != 0 : d.xwrite != 0;
  // planes: X(q) for q in [qbeg, min(qend, d0 - 1)], Y needed on [ylo, yhi]
  const int qbeg = HAS_I ? max(i0 - 1, 0) : 0, qend = HAS_I ? i1 : 0;
  const int ylo = HAS_I ? max(qbeg - 1, 0) : 0;
  const int yhi = HAS_I ? min(min(qend, d.d0 - 1) + 1, d.d0 - 1) : 0;
  constexpr uint32_t kTx = (uint32_t)(YS * sizeof(T));
  auto slot_of = [&](int p) { return ys + ((unsigned)(p - ylo + NSY) % (unsigned)NSY) * YSS; };
  auto issue = [&](int p) {
    const int sl = (int)((unsigned)(p - ylo) % (unsigned)NSY);
    mbar_expect_tx(&mbar[sl], kTx);
    tma_load_3d(ys + sl * YSS, ymap, &mbar[sl], k0 - 2, j0 - 2, p);
  };
  auto wait_plane = [&](int p) {
    const int r = p - ylo;
    mbar_wait(&mbar[(unsigned)r % (unsigned)NSY], ((unsigned)r / (unsigned)NSY) & 1u);
  };
  if (tid == 0) {
    for (int s = 0; s < NSY; ++s) mbar_init(&mbar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // planes issued before the march: the loop issues q + 1 + kDist from
  // q = qbeg on; when the march starts at plane 0 the slot of plane -1 (a
  // zero plane) must stay free, hence qbeg + kDist rather than a full ring
  const int pre_hi = min(qbeg + kDist, yhi);
  if (tid == 0)
    for (int p = ylo; p <= pre_hi; ++p) issue(p);

  // this thread's points (window coordinates: X~ halo 1, Y halo 2)
  const int hj0 = kR * ty + 1, hk = tx + 1;
  int rj = -1, rk = 0;  // halo-ring X point: warps 0, 1 the end rows, then the end columns
  if (ty == 0) {
    rj = 0;
    rk = hk;
  } else if (ty == 1) {
    rj = tPY + 1;
    rk = hk;
  } else {
    const int g = (ty - 2) * 32 + tx;
    if (g < 2 * (tPY + 2)) {
      rj = g % (tPY + 2);
      rk = g < tPY + 2 ? 0 : tPX + 1;
    }
  }
  const bool ring = rj >= 0;
  const int yo0 = (hj0 + 1) * YK + hk + 1;  // Y offset of row u: yo0 + u * YK
  const int yor = ring ? (rj + 1) * YK + rk + 1 : yo0;
  const int xo0 = hj0 * HX + hk;  // X~ offset of row u: xo0 + u * HX
  const int xor_ = ring ? rj * HX + rk : xo0;
  const int rel0 = (j0 + kR * ty) * rs + (k0 + tx);  // global offset of row u: rel0 + u * rs
  const int relr = (j0 - 1 + rj) * rs + (k0 - 1 + rk);
  uint32_t mx[kR], mz[kR];
#pragma unroll
  for (int u = 0; u < kR; ++u) {
    mx[u] = W.aj[hj0 + u] & W.ak[hk];
    mz[u] = W.bj[kR * ty + u] & W.bk[tx];
  }
  const uint32_t mxr = ring ? (W.aj[rj] & W.ak[rk]) : 0u;
#if GFB_STAR_WARPFAST
  // per-warp common-case words: AND of the (j, k) words of the warp's points
  // (ring point included); a plane whose word keeps every common bit for all
  // of them skips the fix-ups warp-uniformly (on a tile at a j face only the
  // warp owning the face rows and the ring warps take them)
  uint32_t mxall = ring ? mxr : ~0u, mzall = ~0u;
#pragma unroll
  for (int u = 0; u < kR; ++u) {
    mxall &= mx[u];
    mzall &= mz[u];
  }
  mxall = __reduce_and_sync(0xffffffffu, mxall);
  mzall = __reduce_and_sync(0xffffffffu, mzall);
#endif
  const bool ysrc = MODES >= 0 ? ((MODES / 32) & 1) != 0 : d.a.srcmask == 1;
  const bool yj_in = j0 - 2 >= d.a.smlo[1] && j0 + tPY + 2 <= d.a.smhi[1];
  const bool yk_in = k0 - 2 >= d.a.smlo[2] && k0 + tPX + 2 <= d.a.smhi[2];
  // window elements e = tid + n * tThreads this thread zeroes on a loaded
  // plane in source-mask form: (j, k) outside M_a (fixed per tile, so found
  // once; on a tile at the domain faces most threads have none)
  constexpr int kZN = (YS + tThreads - 1) / tThreads;
  static_assert(kZN <= 32, "zero-bit mask");
  uint32_t zbits = 0;
  if (ysrc && !(yj_in && yk_in)) {
#pragma unroll
    for (int n = 0; n < kZN; ++n) {
      const int e = tid + n * tThreads;
      const int jj = e / YK, kk = e - jj * YK;
      const int j = j0 - 2 + jj, k = k0 - 2 + kk;
      if (e < YS && (j < d.a.smlo[1] || j >= d.a.smhi[1] || k < d.a.smlo[2] || k >= d.a.smhi[2])) zbits |= 1u << n;
    }
  }
  auto prepare_plane = [&](int p) {
    // zero what the taps must not see: planes never loaded (outside the
    // local array) and, in source-mask form, values outside M_a
    T *slot = slot_of(p);
    const int pg = p + d.p0;
    const bool outside = p < 0 || p >= d.d0 || (ysrc && (pg < d.a.smlo[0] || pg >= d.a.smhi[0]));
    if (outside) {
      for (int e = tid; e < YS; e += tThreads) slot[e] = T(0);
    } else {
      for (uint32_t b = zbits; b; b &= b - 1) slot[tid + (__ffs(b) - 1) * tThreads] = T(0);
    }
  };
  // planes whose preparation is a no-op for this CTA: loaded (inside the
  // local array), inside M_a along dim 0, and a window wholly inside M_a in
  // (j, k) -- one compare per step instead of the full test
  const bool jk_clean = !ysrc || (yj_in && yk_in);
  const int clean_lo = jk_clean ? (ysrc ? max(0, d.a.smlo[0] - d.p0) : 0) : 1;
  const int clean_hi = jk_clean ? (ysrc ? min(d.d0, d.a.smhi[0] - d.p0) : d.d0) : 0;
#if GFB_STAR_WARPFAST
  const uint32_t jka = (amode == 0) ? 0u : mxall, jkb = (bmode == 0) ? 0u : mzall;
#else
  const uint32_t jka = (amode == 0) ? 0u : W.jk[0], jkb = (bmode == 0) ? 0u : W.jk[1];
#endif
  // common-case predicate patterns
  const uint32_t xmask = kArray | kRegion | (amode == 2 ? kClear : 0u) | (xwrite ? kDead : 0u);
  [[maybe_unused]] const uint32_t xval = amode == 0 ? 0xffffffffu : xmask;  // mode 0: base always added -> fix-up
  const uint32_t zmask = kArray | kRegion | (bmode == 2 ? kClear : 0u);
  const uint32_t zval = bmode == 0 ? 0xffffffffu : zmask;
  const uint32_t xfast_m = xmask | kSrcB;
  // old X values a point's fix-up needs: outside op a's region (copy) or
  // where the base is added (mode 0, mode 2 outside the clear box)
  auto needs_xo = [&](uint32_t w) {
    return (w & kArray) && (!(w & kRegion) || amode == 0 || (amode == 2 && !(w & kClear)));
  };
  // stage plane q's old values of this thread's fix-up points (slot u < kR:
  // own rows, kR: ring point) into xst[q & 1]; nothing for a common plane
  auto prefetch_xo = [&](int q) {
    if (q > min(qend, d.d0 - 1)) return;
    const uint32_t mi = W.ai[q - i0 + 1];
    if (((mi & jka) & xfast_m) == xfast_m && amode != 0) return;
    const T *src = Xo + (size_t)q * ps;
#pragma unroll
    for (int u = 0; u < kR; ++u)
      if (needs_xo(mi & mx[u])) cp_async_elem(&xst[q & 1][u][tid], src + rel0 + u * rs);
    if (ring && needs_xo(mi & mxr)) cp_async_elem(&xst[q & 1][kR][tid], src + relr);
    cp_async_commit();
  };
  // X~ of one point from its tap sum; abnormal points take the fix-up
#if GFB_STAR_BRANCHFREE
  // branch-free fix-up: selects instead of nested branches (the boundary
  // tiles run it for every point of every plane); the staged old value is
  // read unconditionally and discarded by the selects where not staged
  auto x_tilde = [&](T acc, uint32_t w, int slot, int rel, bool wb, int q) -> T {
    const bool arr = (w & kArray) != 0, reg = (w & kRegion) != 0;
    const bool add = amode == 0 || (amode == 2 && !(w & kClear));
    const T xo = xst[q & 1][slot][tid];
    T r = reg ? (add ? acc + xo : acc) : xo;
    r = arr ? r : T(0);
    if (wb && xwrite && arr && !(w & kDead) && !(d.skipx && !reg)) Xn[(size_t)q * ps + rel] = r;
    return (w & kSrcB) ? r : T(0);
  };
#else
  auto x_tilde = [&](T acc, uint32_t w, int slot, int rel, bool wb, int q) -> T {
    if ((w & xmask) != xval) {
      if (!(w & kArray)) {
        acc = T(0);
      } else {
        if (!(w & kRegion))
          acc = xst[q & 1][slot][tid];
        else if (amode == 0 || (amode == 2 && !(w & kClear)))
          acc += xst[q & 1][slot][tid];
        if (wb && xwrite && !(w & kDead) && !(d.skipx && !(w & kRegion))) Xn[(size_t)q * ps + rel] = acc;
      }
    }
    return (w & kSrcB) ? acc : T(0);
  };
#endif
  const T a0 = coef<T>(d.a, 0), a1 = coef<T>(d.a, 1), a2 = coef<T>(d.a, 2), a3 = coef<T>(d.a, 3),
          a4 = coef<T>(d.a, 4), a5 = coef<T>(d.a, 5), a6 = coef<T>(d.a, 6);
  const T b0 = coef<T>(d.b, 0), b1 = coef<T>(d.b, 1), b2 = coef<T>(d.b, 2), b3 = coef<T>(d.b, 3),
          b4 = coef<T>(d.b, 4), b5 = coef<T>(d.b, 5), b6 = coef<T>(d.b, 6);

  prefetch_xo(qbeg);
  for (int p = ylo; p <= min(qbeg + 1, yhi); ++p) wait_plane(p);
  if (HAS_I) {
    for (int p = qbeg - 1; p <= qbeg + 1; ++p) prepare_plane(p);
  } else {
    prepare_plane(0);
  }
  __syncthreads();

  // Registers rolled along the march, rotated by index (three live planes):
  // yv[u][.] = Y centre values at the own X points (row u), yr[.] at the
  // ring point, xv[u][.] = X~ at the own Z points. Step S of the unrolled
  // march finds Y(q - 1), Y(q) in slots S, S + 1 and loads Y(q + 1) into
  // slot S + 2 (mod 3); X~(q - 2), X~(q - 1) likewise, X~(q) goes to S + 2.
  T yv[kR][3], yr[3], xv[kR][3];
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    yr[s] = T(0);
#pragma unroll
    for (int u = 0; u < kR; ++u) yv[u][s] = xv[u][s] = T(0);
  }
  {
    const T *yq = slot_of(qbeg);
#pragma unroll
    for (int u = 0; u < kR; ++u) yv[u][1] = yq[yo0 + u * YK];
    yr[1] = yq[yor];
    if (HAS_I) {
      const T *yqm = slot_of(qbeg - 1);
#pragma unroll
      for (int u = 0; u < kR; ++u) yv[u][0] = yqm[yo0 + u * YK];
      yr[0] = yqm[yor];
    }
  }

  // Y ring slot of plane q and slot / phase of plane q + 2, advanced once per
  // step (no modulo in the march)
  unsigned ysl = (unsigned)(qbeg - ylo + NSY) % (unsigned)NSY;
  unsigned wsl = (unsigned)(qbeg + 2 - ylo) % (unsigned)NSY;
  uint32_t wph = ((unsigned)(qbeg + 2 - ylo) / (unsigned)NSY) & 1u;
  // Z fix-ups that add the old value as a base (op b in mode 0, or mode 2
  // outside its clear box: the adjoint sweeps) prefetch it into registers at
  // the start of the step; other instantiations load it in the fix-up (only
  // the out-of-region copies of the first timesteps need it)
  constexpr bool kZPre = MODES < 0 || (MODES % 4) == 0 || (MODES % 4) == 2;
  // ST (steady): a plane inside the segment's steady range [qs, qe) --
  // common X and Z planes, owned, loaded and clean, TMA issue in range -- so
  // every guard of the general step folds away at compile time
  int qe_steady = 0;
  auto step = [&](auto S, int q, auto ST) {
    constexpr int M = decltype(S)::value, C = (M + 1) % 3, P = (M + 2) % 3;
    constexpr bool steady = decltype(ST)::value;
    if (!steady) {
#pragma unroll
      for (int u = 0; u < kR; ++u) xv[u][P] = T(0);
    }
    // old Z values the fix-ups of Z(i) need (plane not common): loaded
    // before the X sweep so their latency overlaps it
    const int i = HAS_I ? q - 1 : q;
    const bool zon = steady || (i >= i0 && i < i1);
    const uint32_t mzi = (!steady && zon) ? W.bi[i - i0] : 0u;
    const bool zfast = steady || ((mzi & jkb) & zmask) == zmask;
    T zo[kR];
#pragma unroll
    for (int u = 0; u < kR; ++u) zo[u] = T(0);
    if (!steady && kZPre && zon && !zfast) {
      const T *zold = Zo + (size_t)i * ps + rel0;
#pragma unroll
      for (int u = 0; u < kR; ++u) {
        const uint32_t w = mzi & mz[u];
        const bool need = (w & zmask) != zval && (w & kArray) &&
                          ((w & kRegion) ? (bmode == 0 || (bmode == 2 && !(w & kClear))) : !d.skipz);
        if (need) zo[u] = zold[u * rs];
      }
    }
    if (steady || q < d.d0) {
      if (tid == 0) {
        const int pn = q + 1 + kDist;
        if (steady || (pn > pre_hi && pn <= yhi)) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue(pn);
        }
      }
      if (HAS_I) {
        // plane q + 2 is needed by X(q + 1): land it and mask it now; the
        // barrier below orders this before any read of it
        const int pn = q + 2;
        if (steady || (pn <= yhi && pn > qbeg + 1)) mbar_wait(&mbar[wsl], wph);
        if (!steady && pn <= qend + 1 && pn > qbeg + 1 && (pn < clean_lo || pn >= clean_hi)) prepare_plane(pn);
      }
      const T *yc = ys + ysl * YSS;
      const T *yp = ys + (ysl + 1 == (unsigned)NSY ? 0u : ysl + 1) * YSS;
      // X~ ring slots relative to the march start: compile-time in the
      // unrolled march (step M handles planes q = qbeg + 3n + M)
#if GFB_STAR_UNROLL
      T *xw = xs + M * XS;
#else
      T *xw = xs + ((unsigned)(q - qbeg) % (unsigned)NXS) * XS;
#endif
      const uint32_t mi = steady ? 0u : W.ai[q - i0 + 1];
      const bool fast = steady || ((mi & jka) & xfast_m) == xfast_m;
      const bool own = steady || (q >= i0 && q < i1);
      if (!fast) cp_async_wait_all();  // this thread's staged old values of plane q
      if (!steady || q + 1 >= qe_steady) prefetch_xo(q + 1);
      if (HAS_I) {
#pragma unroll
        for (int u = 0; u < kR; ++u) yv[u][P] = yp[yo0 + u * YK];
      }
      const T up = yc[yo0 - YK], dn = yc[yo0 + kR * YK];
#pragma unroll
      for (int u = 0; u < kR; ++u) {
        const T jm = u == 0 ? up : yv[u - 1][C];
        const T jp = u == kR - 1 ? dn : yv[u + 1][C];
#if GFB_STAR_CHAIN
        T acc = a0 * yv[u][C];
        if (HAS_I) {
          acc = fma(a1, yv[u][M], acc);
          acc = fma(a2, yv[u][P], acc);
        }
        acc = fma(a3, jm, acc);
        acc = fma(a4, jp, acc);
        acc = fma(a5, yc[yo0 + u * YK - 1], acc);
        acc = fma(a6, yc[yo0 + u * YK + 1], acc);
#else
        // short dependency chains: three partial sums per point
        T p0 = a0 * yv[u][C];
        T p1 = a4 * jp;
        if (HAS_I) {
          p0 = fma(a1, yv[u][M], p0);
          p1 = fma(a2, yv[u][P], p1);
        }
        const T p2 = fma(a5, yc[yo0 + u * YK - 1], a3 * jm);
        p0 = fma(a6, yc[yo0 + u * YK + 1], p0);
        T acc = (p0 + p1) + p2;
#endif
        if (!fast) acc = x_tilde(acc, mi & mx[u], u, rel0 + u * rs, own, q);
        xv[u][P] = acc;
        xw[xo0 + u * HX] = acc;
      }
      if (ring) {
        const T yrp = HAS_I ? yp[yor] : T(0);
#if GFB_STAR_CHAIN
        T acc = a0 * yr[C];
        if (HAS_I) acc = fma(a2, yrp, fma(a1, yr[M], acc));
        acc = fma(a3, yc[yor - YK], acc);
        acc = fma(a4, yc[yor + YK], acc);
        acc = fma(a5, yc[yor - 1], acc);
        acc = fma(a6, yc[yor + 1], acc);
#else
        T pr = a0 * yr[C];
        if (HAS_I) pr = fma(a1, yr[M], fma(a2, yrp, pr));
        const T qr = fma(a3, yc[yor - YK], a4 * yc[yor + YK]);
        const T rr = fma(a5, yc[yor - 1], a6 * yc[yor + 1]);
        T acc = (pr + qr) + rr;
#endif
        if (!fast) acc = x_tilde(acc, mi & mxr, kR, relr, false, q);
        xw[xor_] = acc;
        yr[P] = yrp;
      }
    }
    __syncthreads();
    if (zon) {
#if GFB_STAR_UNROLL
      const T *xc = xs + (HAS_I ? (M + 2) % 3 : M) * XS;
#else
      const T *xc = xs + ((unsigned)(i - qbeg + NXS) % (unsigned)NXS) * XS;
#endif
      const T up = xc[xo0 - HX], dn = xc[xo0 + kR * HX];
      T z[kR];
#pragma unroll
      for (int u = 0; u < kR; ++u) {
        // centre values: X~(i) and, along dim 0, X~(i -/+ 1) from registers
        const T cu = HAS_I ? xv[u][C] : xv[u][P];
        const T jm = u == 0 ? up : (HAS_I ? xv[u - 1][C] : xv[u - 1][P]);
        const T jp = u == kR - 1 ? dn : (HAS_I ? xv[u + 1][C] : xv[u + 1][P]);
#if GFB_STAR_CHAIN
        T acc = b0 * cu;
        if (HAS_I) {
          acc = fma(b1, xv[u][M], acc);
          acc = fma(b2, xv[u][P], acc);
        }
        acc = fma(b3, jm, acc);
        acc = fma(b4, jp, acc);
        acc = fma(b5, xc[xo0 + u * HX - 1], acc);
        z[u] = fma(b6, xc[xo0 + u * HX + 1], acc);
#else
        T p0 = b0 * cu;
        T p1 = b4 * jp;
        if (HAS_I) {
          p0 = fma(b1, xv[u][M], p0);
          p1 = fma(b2, xv[u][P], p1);
        }
        const T p2 = fma(b5, xc[xo0 + u * HX - 1], b3 * jm);
        p0 = fma(b6, xc[xo0 + u * HX + 1], p0);
        z[u] = (p0 + p1) + p2;
#endif
      }
      T *zrow = Zn + (size_t)i * ps + rel0;
      if (zfast) {
#pragma unroll
        for (int u = 0; u < kR; ++u) zrow[u * rs] = z[u];
      } else {
#if GFB_STAR_BRANCHFREE
#pragma unroll
        for (int u = 0; u < kR; ++u) {
          const uint32_t w = mzi & mz[u];
          const bool arr = (w & kArray) != 0, reg = (w & kRegion) != 0;
          const bool add = bmode == 0 || (bmode == 2 && !(w & kClear));
          T old = zo[u];
          if (!kZPre && !reg && arr && !d.skipz) old = Zo[(size_t)i * ps + rel0 + u * rs];
          const T zz = reg ? (add ? z[u] + old : z[u]) : old;
          if (arr && (reg || !d.skipz)) zrow[u * rs] = zz;  // out of region: the twin may hold the copy
        }
#else
#pragma unroll
        for (int u = 0; u < kR; ++u) {
          const uint32_t w = mzi & mz[u];
          T zz = z[u];
          if ((w & zmask) != zval) {
            if (!(w & kArray)) continue;
            if (!(w & kRegion) && d.skipz) continue;  // the twin already holds this copy
            const T old = kZPre ? zo[u] : Zo[(size_t)i * ps + rel0 + u * rs];
            if (!(w & kRegion))
              zz = old;
            else if (bmode == 0 || (bmode == 2 && !(w & kClear)))
              zz += old;
          }
          zrow[u * rs] = zz;
        }
#endif
      }
    }
    ysl = ysl + 1 == (unsigned)NSY ? 0u : ysl + 1;
    if (++wsl == (unsigned)NSY) {
      wsl = 0;
      wph ^= 1u;
    }
  };
  using I0 = std::integral_constant<int, 0>;
  using I1 = std::integral_constant<int, 1>;
  using I2 = std::integral_constant<int, 2>;
#if GFB_STAR_UNROLL
  // steady range: X plane q and Z plane q - 1 common (warp-uniform words),
  // q owned, its TMA issue and wait inside the segment's ranges, plane q + 2
  // clean. Each warp finds it with ballots over 32 planes at a time (all
  // warps agree: the words are the CTA's plane words AND the warp's own).
  int qs = qbeg, qe = qbeg;
  if (HAS_I && GFB_STAR_STEADY) {
    const int lo = max(max(i0 + 1, qbeg), clean_lo - 2);
    const int hi = min(min(min(i1, d.d0), yhi - kDist), clean_hi - 2);  // exclusive
    const int lane = threadIdx.x & 31;
    bool found = false;
    for (int c = lo; c < hi; c += 32) {
      const int q = c + lane;
      bool ok = q < hi;
      if (ok) {
        const uint32_t mi = W.ai[q - i0 + 1], mz = W.bi[q - 1 - i0];
        ok = ((mi & jka) & xfast_m) == xfast_m && ((mz & jkb) & zmask) == zmask;
      }
      const uint32_t bad = __ballot_sync(0xffffffffu, !ok && q < hi), good = __ballot_sync(0xffffffffu, ok);
      if (!found) {
        if (good) {
          qs = c + __ffs(good) - 1;
          found = true;
          const uint32_t after = bad & ~((2u << (__ffs(good) - 1)) - 1u);  // failures past the first good
          if (after) {
            qe = c + __ffs(after) - 1;
            break;
          }
          qe = min(c + 32, hi);
        }
      } else {
        if (bad) {
          qe = c + __ffs(bad) - 1;
          break;
        }
        qe = min(c + 32, hi);
      }
    }
    // align to the 3-step unroll (slot indices are compile-time)
    qs = qbeg + (qs - qbeg + 2) / 3 * 3;
    qe = qe > qs ? qs + (qe - qs) / 3 * 3 : qs;
  }
  qe_steady = qe;
  // one loop, two bodies: steady 3-blocks inside [qs, qe), general otherwise
  for (int q = qbeg; q <= qend; q += 3) {
    if (q >= qs && q + 3 <= qe) {
      step(I0{}, q, std::true_type{});
      step(I1{}, q + 1, std::true_type{});
      step(I2{}, q + 2, std::true_type{});
      continue;
    }
    step(I0{}, q, std::false_type{});
    if (q + 1 > qend) break;
    step(I1{}, q + 1, std::false_type{});
    if (q + 2 > qend) break;
    step(I2{}, q + 2, std::false_type{});
  }
#else
  // one step body, registers rotated by moves (smaller code)
  for (int q = qbeg; q <= qend; ++q) {
    step(I0{}, q, std::false_type{});
#pragma unroll
    for (int u = 0; u < kR; ++u) {
      yv[u][0] = yv[u][1];
      yv[u][1] = yv[u][2];
      xv[u][0] = xv[u][1];
      xv[u][1] = xv[u][2];
    }
    yr[0] = yr[1];
    yr[1] = yr[2];
  }
  (void)I1{};
  (void)I2{};
#endif
}

// 2-D arrays (d0 == 1, HAS_I false) march a single plane: one Y slot and one
// X~ slot, a kernel of its own (its own register allocation) so more CTAs
// fit an SM and short launches are one wave
template <typename T, bool HAS_I>
__host__ __device__ constexpr size_t star_tma_dyn_bytes() {
  return (size_t)(HAS_I ? NSY : 1) * yslot<T>() * sizeof(T) + (size_t)(HAS_I ? NXS : 1) * XS * sizeof(T) +
         NSY * sizeof(uint64_t);
}

template <typename T, bool HAS_I, int MODES>
__global__ void __launch_bounds__(tThreads, HAS_I ? 512 / tThreads : 768 / tThreads)
    star_pair_tma_kernel(const __grid_constant__ CUtensorMap ymap, const __grid_constant__ StarPairDev d) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr size_t ybytes = (size_t)(HAS_I ? NSY : 1) * yslot<T>() * sizeof(T);
  T *ys = reinterpret_cast<T *>(smem);
  T *xs = reinterpret_cast<T *>(smem + ybytes);
  uint64_t *mbar = reinterpret_cast<uint64_t *>(smem + ybytes + (size_t)(HAS_I ? NXS : 1) * XS * sizeof(T));
  __shared__ TmaWords words;
  __shared__ T xst[2][kR + 1][tThreads];  // staged old X values (fix-up points), by plane parity
  const int tid = threadIdx.y * tPX + threadIdx.x;
  const int i0 = d.zlo + blockIdx.z * d.tpm, i1 = min(i0 + d.tpm, d.zhi);
  tma_prologue(d, i0, blockIdx.y * tPY, blockIdx.x * tPX, tid, words);  // descriptor only
  pdl_wait();
  pdl_trigger();  // after the wait: at most one launch waits ahead of the running one
  star_tma_body<T, HAS_I, MODES>(&ymap, d, ys, xs, mbar, words, xst, i0, i1);
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

template <typename T, bool HAS_I, int MODES>
static int launch_tma_m(const CUtensorMap &map, const StarPairDev &d, cudaStream_t st) {
  const size_t sm = star_tma_dyn_bytes<T, HAS_I>();
  ensure_smem(star_pair_tma_kernel<T, HAS_I, MODES>, sm);
  // planes per CTA: the longest march (up to tPM) that still puts every
  // tile-column segment in one wave of resident CTAs (2 per SM); small
  // domains get short marches rather than idle SMs or a straggler wave
  StarPairDev dd = d;
  const int64_t tiles = ceil_div(d.d2, tPX) * ceil_div(d.d1, tPY), planes = d.zhi - d.zlo;
  const int64_t slots = 2 * (int64_t)sm_count();
  dd.tpm = d.tpm >= 2 ? std::min<int32_t>(d.tpm, tPM)  // the caller's choice (slab interiors)
                      : (int32_t)std::max<int64_t>(2, std::min<int64_t>(tPM, ceil_div(planes * tiles, slots)));
  dim3 grid((unsigned)ceil_div(d.d2, tPX), (unsigned)ceil_div(d.d1, tPY), (unsigned)ceil_div(planes, dd.tpm));
  launch_pdl(star_pair_tma_kernel<T, HAS_I, MODES>, grid, dim3(tPX, tPY / kR), sm, st, map, dd);
  return check_launch("star_pair_tma");
}

// the base-mode pairs of the fused timesteps (forward 3/3, adjoint 2/2 and
// 1/2) get instantiations of their own; anything else reads the modes
template <typename T, bool HAS_I>
static int launch_tma(const CUtensorMap &map, const StarPairDev &d, cudaStream_t st) {
  // 32 source-mask form + 16 X write-back + 4 a + b
  const int m = (d.a.srcmask == 1 ? 32 : 0) + (d.xwrite ? 16 : 0) + d.a.mode * 4 + d.b.mode;
  switch (m) {
    case 16 + 3 * 4 + 3: return launch_tma_m<T, HAS_I, 16 + 3 * 4 + 3>(map, d, st);       // forward
    case 3 * 4 + 3: return launch_tma_m<T, HAS_I, 3 * 4 + 3>(map, d, st);                 // last forward
    case 32 + 16 + 2 * 4 + 2: return launch_tma_m<T, HAS_I, 32 + 16 + 2 * 4 + 2>(map, d, st);  // adjoint
    case 32 + 16 + 1 * 4 + 2: return launch_tma_m<T, HAS_I, 32 + 16 + 1 * 4 + 2>(map, d, st);  // first adjoint
    case 32 + 2 * 4 + 2: return launch_tma_m<T, HAS_I, 32 + 2 * 4 + 2>(map, d, st);       // last adjoint
    default: return launch_tma_m<T, HAS_I, -1>(map, d, st);
  }
}

int launch_star_pair_tma(const StarPairDev &d, int dtype, dim3, cudaStream_t st) {
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
  if (d.d0 > 1) return dtype == GFB_F64 ? launch_tma<double, true>(map, d, st) : launch_tma<float, true>(map, d, st);
  return dtype == GFB_F64 ? launch_tma<double, false>(map, d, st) : launch_tma<float, false>(map, d, st);
}

}  // namespace GFB_STAR_NS
}  // namespace gfb
