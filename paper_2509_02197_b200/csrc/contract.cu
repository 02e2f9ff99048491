// Affine product contraction: implicit GEMM over index tables (gfb.h,
// gfb_contract_desc).
//
// Replaces the per-target free-loop of the generic gather pass (map.cu) for
// wcr="sum" maps whose tasklet is `scale * a * b` with affine subsets — the
// reference's convolution forward sum and the two adjoint scatters
// (autodiff.py:962-1081 emits them; interpreter.py:422-423 accumulates them
// point by point). Output coordinates split into m (those A depends on) and
// n (those only B depends on); the free parameters flatten into k. Every
// element address is a table lookup plus an add, so one CTA stages a
// (BM x BK) slab of A and a (BK x BN) slab of B in shared memory and runs a
// register-blocked outer product, exactly like a GEMM whose operand rows are
// gathered. Constraints (pivot parameters of a reparameterised scatter that
// must stay in their box) zero the staged element.
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "gfb_common.cuh"
#include "gfb_internal.h"

namespace gfb {

template <typename T, int BM, int BN, int BK, int TM, int TN>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
    contract_kernel(const __grid_constant__ gfb_contract_desc d) {
  constexpr int NX = BN / TN, NY = BM / TM, NT = NX * NY;
  constexpr int AP = BM + 16 / (int)sizeof(T), BP = BN + 16 / (int)sizeof(T);  // 16-byte aligned rows
  static_assert((BM * BK) % NT == 0 && (BN * BK) % NT == 0, "tile / thread mismatch");
  __shared__ __align__(16) T As[BK][AP];
  __shared__ __align__(16) T Bs[BK][BP];
  __shared__ int32_t sma[BM], smc[2][BM];
  __shared__ int32_t snb[BN], snc[2][BN];
  __shared__ int32_t ska[BK], skb[BK], skc[4][BK];
  const int tid = threadIdx.x;
  const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
  const int ncm = d.ncm, ncn = d.ncn;
  const int64_t M = d.M, N = d.N, K = d.K;
  const int s = blockIdx.z;
  // split boundaries on BK multiples (16-byte k-quads never straddle two splits)
  const int64_t kchunk = (K + (int64_t)d.nsplit * BK - 1) / ((int64_t)d.nsplit * BK) * BK;
  const int64_t kb = min((int64_t)s * kchunk, K), ke = min(kb + kchunk, K);
  const T *__restrict__ Ag = (const T *)d.a;
  const T *__restrict__ Bg = (const T *)d.b;
  const bool aq = sizeof(T) == 4 && (d.a_kfast & 2) && (reinterpret_cast<uintptr_t>(Ag) & 15) == 0;
  const bool bq = sizeof(T) == 4 && (d.b_nfast & 2) && (reinterpret_cast<uintptr_t>(Bg) & 15) == 0;

  for (int i = tid; i < BM; i += NT) {
    const int64_t m = m0 + i;
    if (m < M) {
      const int32_t *e = d.mtab + m * d.mstride;
      sma[i] = e[0];
      smc[0][i] = ncm > 0 ? e[3] : 0;
      smc[1][i] = ncm > 1 ? e[4] : 0;
    }
  }
  for (int i = tid; i < BN; i += NT) {
    const int64_t n = n0 + i;
    if (n < N) {
      const int32_t *e = d.ntab + n * d.nstride;
      snb[i] = e[0];
      snc[0][i] = ncn > 0 ? e[3] : 0;
      snc[1][i] = ncn > 1 ? e[4] : 0;
    }
  }

  T acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = T(0);
  const int tx = tid % NX, ty = tid / NX;

  for (int64_t k0 = kb; k0 < ke; k0 += BK) {
    __syncthreads();  // previous tile consumed (and the m / n tables written)
    for (int i = tid; i < BK; i += NT) {
      const int64_t k = k0 + i;
      if (k < ke) {
        const int32_t *e = d.ktab + k * d.kstride;
        ska[i] = e[0];
        skb[i] = e[1];
        for (int c = 0; c < ncm + ncn; ++c) skc[c][i] = e[2 + c];
      }
    }
    __syncthreads();
    // A slab: As[kk][mm] = A(m, k) or 0
    auto a_elem = [&](int mm, int kk) -> T {
      const int64_t m = m0 + mm, k = k0 + kk;
      if (m >= M || k >= ke) return T(0);
      bool ok = true;
      for (int c = 0; c < ncm; ++c) {
        const int32_t v = smc[c][mm] + skc[c][kk];
        ok &= v >= d.lo[c] && v < d.hi[c];
      }
      return ok ? Ag[(int64_t)sma[mm] + ska[kk]] : T(0);
    };
    auto b_elem = [&](int nn, int kk) -> T {
      const int64_t n = n0 + nn, k = k0 + kk;
      if (n >= N || k >= ke) return T(0);
      bool ok = true;
      for (int c = 0; c < ncn; ++c) {
        const int32_t v = snc[c][nn] + skc[ncm + c][kk];
        ok &= v >= d.lo[ncm + c] && v < d.hi[ncm + c];
      }
      return ok ? Bg[(int64_t)snb[nn] + skb[kk]] : T(0);
    };
    // 16-byte quads (bit 1 of a_kfast / b_nfast, fp32): the host proved
    // four consecutive elements along the fast direction contiguous, aligned
    // and under equal constraints, so one check and one vector load serve four
    auto a_quad_ok = [&](int mm, int kk) -> bool {  // element (mm, kk) starts a quad
      if (m0 + mm >= M || k0 + kk >= ke) return false;
      bool ok = true;
      for (int c = 0; c < ncm; ++c) {
        const int32_t v = smc[c][mm] + skc[c][kk];
        ok &= v >= d.lo[c] && v < d.hi[c];
      }
      return ok;
    };
    auto b_quad_ok = [&](int nn, int kk) -> bool {
      if (n0 + nn >= N || k0 + kk >= ke) return false;
      bool ok = true;
      for (int c = 0; c < ncn; ++c) {
        const int32_t v = snc[c][nn] + skc[ncm + c][kk];
        ok &= v >= d.lo[ncm + c] && v < d.hi[ncm + c];
      }
      return ok;
    };
    if constexpr (sizeof(T) == 4) {
      if (aq) {
        if (d.a_kfast & 1) {
          for (int e = tid; e < BM * BK / 4; e += NT) {
            const int kq = e % (BK / 4), mm = e / (BK / 4), kk = 4 * kq;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (a_quad_ok(mm, kk)) v = *reinterpret_cast<const float4 *>(Ag + (int64_t)sma[mm] + ska[kk]);
            As[kk][mm] = v.x;
            As[kk + 1][mm] = v.y;
            As[kk + 2][mm] = v.z;
            As[kk + 3][mm] = v.w;
          }
        } else {
          for (int e = tid; e < BM * BK / 4; e += NT) {
            const int mq = e % (BM / 4), kk = e / (BM / 4), mm = 4 * mq;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (a_quad_ok(mm, kk)) v = *reinterpret_cast<const float4 *>(Ag + (int64_t)sma[mm] + ska[kk]);
            *reinterpret_cast<float4 *>(&As[kk][mm]) = v;
          }
        }
      }
      if (bq) {
        if (d.b_nfast & 1) {
          for (int e = tid; e < BN * BK / 4; e += NT) {
            const int nq = e % (BN / 4), kk = e / (BN / 4), nn = 4 * nq;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (b_quad_ok(nn, kk)) v = *reinterpret_cast<const float4 *>(Bg + (int64_t)snb[nn] + skb[kk]);
            *reinterpret_cast<float4 *>(&Bs[kk][nn]) = v;
          }
        } else {
          for (int e = tid; e < BN * BK / 4; e += NT) {
            const int kq = e % (BK / 4), nn = e / (BK / 4), kk = 4 * kq;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (b_quad_ok(nn, kk)) v = *reinterpret_cast<const float4 *>(Bg + (int64_t)snb[nn] + skb[kk]);
            Bs[kk][nn] = v.x;
            Bs[kk + 1][nn] = v.y;
            Bs[kk + 2][nn] = v.z;
            Bs[kk + 3][nn] = v.w;
          }
        }
      }
    }
    if (!aq) {
      if (d.a_kfast & 1) {
#pragma unroll
        for (int r = 0; r < BM * BK / NT; ++r) {
          const int e = tid + r * NT, kk = e % BK, mm = e / BK;
          As[kk][mm] = a_elem(mm, kk);
        }
      } else {
#pragma unroll
        for (int r = 0; r < BM * BK / NT; ++r) {
          const int e = tid + r * NT, mm = e % BM, kk = e / BM;
          As[kk][mm] = a_elem(mm, kk);
        }
      }
    }
    if (!bq) {
      if (d.b_nfast & 1) {
#pragma unroll
        for (int r = 0; r < BN * BK / NT; ++r) {
          const int e = tid + r * NT, nn = e % BN, kk = e / BN;
          Bs[kk][nn] = b_elem(nn, kk);
        }
      } else {
#pragma unroll
        for (int r = 0; r < BN * BK / NT; ++r) {
          const int e = tid + r * NT, kk = e % BK, nn = e / BK;
          Bs[kk][nn] = b_elem(nn, kk);
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      T a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[kk][ty * TM + i];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Bs[kk][tx * TN + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
  }

  // epilogue
  T *__restrict__ Dg = (T *)d.d;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int64_t m = m0 + ty * TM + i;
    if (m >= M) continue;
    const int32_t *me = d.mtab + m * d.mstride;
    const int32_t dm = me[1], mclr = me[2];
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int64_t n = n0 + tx * TN + j;
      if (n >= N) continue;
      if (d.nsplit > 1) {
        ((double *)d.workspace)[((int64_t)s * M + m) * N + n] = (double)acc[i][j];
        continue;
      }
      const int32_t *ne = d.ntab + n * d.nstride;
      const int64_t off = (int64_t)dm + ne[1];
      const T v = (T)d.scale * acc[i][j];
      T base = T(0);
      if (d.clear_mode == 0 || (d.clear_mode == 2 && !(mclr && ne[2]))) base = Dg[off];
      Dg[off] = base + v;
    }
  }
}

// Double-buffered variant: the global gathers of slab t + 1 go to registers
// before slab t is multiplied, so their latency hides behind the FMAs; one
// barrier per slab (slab and k-table buffers alternate); TM x TN register
// tiles read with 16-byte shared-memory loads.
// LAYOUT fixes the staging layout at compile time so the staging code carries
// no layout branches: 1 = A quads along k (convolution forward and input
// adjoint), 2 = A quads along m and B quads along n (weight adjoint); 0 reads
// the layout flags from the descriptor
template <typename T, int BM, int BN, int BK, int TM, int TN, int LAYOUT = 0>
__global__ void __launch_bounds__((BM / TM) * (BN / TN), (BM / TM) * (BN / TN) >= 256 ? 2 : 4)
    contract2_kernel(const __grid_constant__ gfb_contract_desc d) {
  constexpr int NX = BN / TN, NY = BM / TM, NT = NX * NY;
  constexpr int PAD = 16 / (int)sizeof(T);
  constexpr int AP = BM + PAD, BP = BN + PAD;
  constexpr int EA = BM * BK / NT, EB = BN * BK / NT;  // staged elements per thread
  static_assert((BM * BK) % NT == 0 && (BN * BK) % NT == 0, "tile / thread mismatch");
  __shared__ __align__(16) T As[2][BK][AP];
  __shared__ __align__(16) T Bs[2][BK][BP];
  __shared__ int32_t sma[BM], smc[2][BM];
  __shared__ int32_t snb[BN], snc[2][BN];
  __shared__ int32_t ska[2][BK], skb[2][BK], skc[2][4][BK];
  const int tid = threadIdx.x;
  const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
  const int ncm = d.ncm, ncn = d.ncn;
  const int64_t M = d.M, N = d.N, K = d.K;
  const int s = blockIdx.z;
  const int64_t kchunk = (K + (int64_t)d.nsplit * BK - 1) / ((int64_t)d.nsplit * BK) * BK;
  const int64_t kb = min((int64_t)s * kchunk, K), ke = min(kb + kchunk, K);
  const int nslab = (int)((ke - kb + BK - 1) / BK);
  const T *__restrict__ Ag = (const T *)d.a;
  const T *__restrict__ Bg = (const T *)d.b;
  const bool akf = LAYOUT == 1 ? true : (LAYOUT == 2 ? false : (d.a_kfast & 1) != 0);
  const bool bnf = LAYOUT == 2 ? true : (d.b_nfast & 1) != 0;
  const bool aq = LAYOUT != 0 || (sizeof(T) == 4 && (d.a_kfast & 2) && (reinterpret_cast<uintptr_t>(Ag) & 15) == 0 &&
                                  EA % 4 == 0);
  const bool bq = LAYOUT == 2 || (sizeof(T) == 4 && (d.b_nfast & 2) && (reinterpret_cast<uintptr_t>(Bg) & 15) == 0 &&
                                  EB % 4 == 0);

  for (int i = tid; i < BM; i += NT) {
    const int64_t m = m0 + i;
    if (m < M) {
      const int32_t *e = d.mtab + m * d.mstride;
      sma[i] = e[0];
      smc[0][i] = ncm > 0 ? e[3] : 0;
      smc[1][i] = ncm > 1 ? e[4] : 0;
    }
  }
  for (int i = tid; i < BN; i += NT) {
    const int64_t n = n0 + i;
    if (n < N) {
      const int32_t *e = d.ntab + n * d.nstride;
      snb[i] = e[0];
      snc[0][i] = ncn > 0 ? e[3] : 0;
      snc[1][i] = ncn > 1 ? e[4] : 0;
    }
  }
  auto load_ktab = [&](int t, int buf) {
    const int64_t k0 = kb + (int64_t)t * BK;
    for (int i = tid; i < BK; i += NT) {
      const int64_t k = k0 + i;
      if (k < ke) {
        const int32_t *e = d.ktab + k * d.kstride;
        ska[buf][i] = e[0];
        skb[buf][i] = e[1];
        for (int c = 0; c < ncm + ncn; ++c) skc[buf][c][i] = e[2 + c];
      }
    }
  };
  auto a_ok = [&](int mm, int kk, int kbuf, int64_t k0) -> bool {
    if (m0 + mm >= M || k0 + kk >= ke) return false;
    bool ok = true;
    for (int c = 0; c < ncm; ++c) {
      const int32_t v = smc[c][mm] + skc[kbuf][c][kk];
      ok &= v >= d.lo[c] && v < d.hi[c];
    }
    return ok;
  };
  auto b_ok = [&](int nn, int kk, int kbuf, int64_t k0) -> bool {
    if (n0 + nn >= N || k0 + kk >= ke) return false;
    bool ok = true;
    for (int c = 0; c < ncn; ++c) {
      const int32_t v = snc[c][nn] + skc[kbuf][ncm + c][kk];
      ok &= v >= d.lo[ncm + c] && v < d.hi[ncm + c];
    }
    return ok;
  };
  // element (or quad) e of a slab -> (row, kk)
  auto a_coord = [&](int e, bool quad, int &mm, int &kk) {
    if (quad) {
      if (akf) { kk = 4 * (e % (BK / 4)); mm = e / (BK / 4); }
      else { mm = 4 * (e % (BM / 4)); kk = e / (BM / 4); }
    } else {
      if (akf) { kk = e % BK; mm = e / BK; }
      else { mm = e % BM; kk = e / BM; }
    }
  };
  auto b_coord = [&](int e, bool quad, int &nn, int &kk) {
    if (quad) {
      if (bnf) { nn = 4 * (e % (BN / 4)); kk = e / (BN / 4); }
      else { kk = 4 * (e % (BK / 4)); nn = e / (BK / 4); }
    } else {
      if (bnf) { nn = e % BN; kk = e / BN; }
      else { kk = e % BK; nn = e / BK; }
    }
  };
  T ra[EA], rb[EB];
  // A quads: each thread stages the same (row, kk) positions every slab, so
  // row offsets and row-side constraint terms are hoisted into registers; a
  // row whose constraints hold for every k of this CTA's range skips the
  // per-element checks (interior points of a convolution)
  constexpr int SA = EA / 4 > 0 ? EA / 4 : 1;
  int32_t q_off[SA], q_cb0[SA], q_cb1[SA];
  int q_mm[SA], q_kk[SA];
  bool q_in[SA], q_mv[SA];
  if (aq) {
    __shared__ int32_t kext[2][4];  // min / max of the k-side constraint terms
    if (tid < 4) {
      kext[0][tid] = INT32_MAX;
      kext[1][tid] = INT32_MIN;
    }
    __syncthreads();
    if (ncm > 0) {
      int32_t lo_[2] = {INT32_MAX, INT32_MAX}, hi_[2] = {INT32_MIN, INT32_MIN};
      for (int64_t k = kb + tid; k < ke; k += NT) {
        const int32_t *e = d.ktab + k * d.kstride;
        for (int c = 0; c < ncm; ++c) {
          lo_[c] = min(lo_[c], e[2 + c]);
          hi_[c] = max(hi_[c], e[2 + c]);
        }
      }
      for (int c = 0; c < ncm; ++c) {
        atomicMin(&kext[0][c], lo_[c]);
        atomicMax(&kext[1][c], hi_[c]);
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < SA; ++i) {
      int mm, kk;
      a_coord(tid + i * NT, true, mm, kk);
      q_mm[i] = mm;
      q_kk[i] = kk;
      q_mv[i] = m0 + mm < M;
      q_off[i] = q_mv[i] ? sma[mm] : 0;
      q_cb0[i] = ncm > 0 ? smc[0][mm] : 0;
      q_cb1[i] = ncm > 1 ? smc[1][mm] : 0;
      bool in = q_mv[i];
      for (int c = 0; c < ncm; ++c) {
        const int32_t cb = c == 0 ? q_cb0[i] : q_cb1[i];
        in &= cb + kext[0][c] >= d.lo[c] && cb + kext[1][c] < d.hi[c];
      }
      q_in[i] = in;
    }
  }
  auto gload = [&](int t) {
    const int kbuf = t & 1;
    const int64_t k0 = kb + (int64_t)t * BK;
    if (aq) {
#pragma unroll
      for (int i = 0; i < EA / 4; ++i) {
        const int kk = q_kk[i];
        bool ok = k0 + kk < ke;
        if (!q_in[i]) {
          ok &= q_mv[i];
          if (ncm > 0) {
            const int32_t v0 = q_cb0[i] + skc[kbuf][0][kk];
            ok &= v0 >= d.lo[0] && v0 < d.hi[0];
          }
          if (ncm > 1) {
            const int32_t v1 = q_cb1[i] + skc[kbuf][1][kk];
            ok &= v1 >= d.lo[1] && v1 < d.hi[1];
          }
        }
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (ok) v = *reinterpret_cast<const float4 *>(Ag + (int64_t)q_off[i] + ska[kbuf][kk]);
        ra[4 * i] = v.x, ra[4 * i + 1] = v.y, ra[4 * i + 2] = v.z, ra[4 * i + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < EA; ++i) {
        int mm, kk;
        a_coord(tid + i * NT, false, mm, kk);
        ra[i] = a_ok(mm, kk, kbuf, k0) ? Ag[(int64_t)sma[mm] + ska[kbuf][kk]] : T(0);
      }
    }
    if (bq) {
#pragma unroll
      for (int i = 0; i < EB / 4; ++i) {
        int nn, kk;
        b_coord(tid + i * NT, true, nn, kk);
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (b_ok(nn, kk, kbuf, k0)) v = *reinterpret_cast<const float4 *>(Bg + (int64_t)snb[nn] + skb[kbuf][kk]);
        rb[4 * i] = v.x, rb[4 * i + 1] = v.y, rb[4 * i + 2] = v.z, rb[4 * i + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < EB; ++i) {
        int nn, kk;
        b_coord(tid + i * NT, false, nn, kk);
        rb[i] = b_ok(nn, kk, kbuf, k0) ? Bg[(int64_t)snb[nn] + skb[kbuf][kk]] : T(0);
      }
    }
  };
  auto sstore = [&](int buf) {
    if (aq) {
#pragma unroll
      for (int i = 0; i < EA / 4; ++i) {
        const int mm = q_mm[i], kk = q_kk[i];
        if (akf) {
#pragma unroll
          for (int j = 0; j < 4; ++j) As[buf][kk + j][mm] = ra[4 * i + j];
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) As[buf][kk][mm + j] = ra[4 * i + j];
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < EA; ++i) {
        int mm, kk;
        a_coord(tid + i * NT, false, mm, kk);
        As[buf][kk][mm] = ra[i];
      }
    }
    if (bq) {
#pragma unroll
      for (int i = 0; i < EB / 4; ++i) {
        int nn, kk;
        b_coord(tid + i * NT, true, nn, kk);
        if (bnf) {
#pragma unroll
          for (int j = 0; j < 4; ++j) Bs[buf][kk][nn + j] = rb[4 * i + j];
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) Bs[buf][kk + j][nn] = rb[4 * i + j];
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < EB; ++i) {
        int nn, kk;
        b_coord(tid + i * NT, false, nn, kk);
        Bs[buf][kk][nn] = rb[i];
      }
    }
  };

  T acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = T(0);
  const int tx = tid % NX, ty = tid / NX;

  // prologue: tables of slabs 0 and 1, slab 0 staged
  load_ktab(0, 0);
  if (nslab > 1) load_ktab(1, 1);
  __syncthreads();
  if (nslab > 0) {
    gload(0);
    sstore(0);
  }
  __syncthreads();
  for (int t = 0; t < nslab; ++t) {
    const int buf = t & 1;
    if (t + 1 < nslab) gload(t + 1);         // tables of t + 1 are in buffer (t + 1) & 1
    if (t + 2 < nslab) load_ktab(t + 2, buf);  // buffer of t's tables is free (t's gathers are done)
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      T a[TM], b[TN];
      if constexpr (sizeof(T) == 4 && TM % 4 == 0) {
#pragma unroll
        for (int i = 0; i < TM; i += 4) {
          const float4 v = *reinterpret_cast<const float4 *>(&As[buf][kk][ty * TM + i]);
          a[i] = v.x, a[i + 1] = v.y, a[i + 2] = v.z, a[i + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < TM; ++i) a[i] = As[buf][kk][ty * TM + i];
      }
      if constexpr (sizeof(T) == 4 && TN % 4 == 0) {
#pragma unroll
        for (int j = 0; j < TN; j += 4) {
          const float4 v = *reinterpret_cast<const float4 *>(&Bs[buf][kk][tx * TN + j]);
          b[j] = v.x, b[j + 1] = v.y, b[j + 2] = v.z, b[j + 3] = v.w;
        }
      } else if constexpr (sizeof(T) == 4 && TN == 2) {
        const float2 v = *reinterpret_cast<const float2 *>(&Bs[buf][kk][tx * TN]);
        b[0] = v.x, b[1] = v.y;
      } else {
#pragma unroll
        for (int j = 0; j < TN; ++j) b[j] = Bs[buf][kk][tx * TN + j];
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    if (t + 1 < nslab) sstore(buf ^ 1);  // its previous readers passed the last barrier
    __syncthreads();
  }

  T *__restrict__ Dg = (T *)d.d;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int64_t m = m0 + ty * TM + i;
    if (m >= M) continue;
    const int32_t *me = d.mtab + m * d.mstride;
    const int32_t dm = me[1], mclr = me[2];
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int64_t n = n0 + tx * TN + j;
      if (n >= N) continue;
      if (d.nsplit > 1) {
        ((double *)d.workspace)[((int64_t)s * M + m) * N + n] = (double)acc[i][j];
        continue;
      }
      const int32_t *ne = d.ntab + n * d.nstride;
      const int64_t off = (int64_t)dm + ne[1];
      const T v = (T)d.scale * acc[i][j];
      T base = T(0);
      if (d.clear_mode == 0 || (d.clear_mode == 2 && !(mclr && ne[2]))) base = Dg[off];
      Dg[off] = base + v;
    }
  }
}

// split-k: fixed-order fp64 sum of the partials, then the base as above
template <typename T>
__global__ void __launch_bounds__(1024) contract_finish_kernel(const __grid_constant__ gfb_contract_desc d) {
  // 32 outputs x 32 split groups per CTA: each group sums every 32nd split,
  // then the groups are added in order (deterministic)
  __shared__ double red[32][33];
  const int64_t M = d.M, N = d.N, MN = M * N;
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t e = (int64_t)blockIdx.x * 32 + lane;
  const double *ws = (const double *)d.workspace;
  double s4[4] = {0.0, 0.0, 0.0, 0.0};
  if (e < MN) {
    int s = g;
    for (; s + 96 < d.nsplit; s += 128) {
#pragma unroll
      for (int u = 0; u < 4; ++u) s4[u] += ws[(int64_t)(s + 32 * u) * MN + e];
    }
    for (; s < d.nsplit; s += 32) s4[0] += ws[(int64_t)s * MN + e];
  }
  red[g][lane] = (s4[0] + s4[1]) + (s4[2] + s4[3]);
  __syncthreads();
  if (g != 0 || e >= MN) return;
  double sum = 0.0;
#pragma unroll
  for (int q = 0; q < 32; ++q) sum += red[q][lane];
  const int64_t m = e / N, n = e - m * N;
  const int32_t *me = d.mtab + m * d.mstride, *ne = d.ntab + n * d.nstride;
  const int64_t off = (int64_t)me[1] + ne[1];
  T *Dg = (T *)d.d;
  T base = T(0);
  if (d.clear_mode == 0 || (d.clear_mode == 2 && !(me[2] && ne[2]))) base = Dg[off];
  Dg[off] = base + (T)(d.scale * sum);
}

template <typename T, int BM, int BN, int TM, int TN, int BK = 16>
static void launch_contract(const gfb_contract_desc &d, cudaStream_t st) {
  dim3 grid((unsigned)ceil_div(d.M, BM), (unsigned)ceil_div(d.N, BN), (unsigned)d.nsplit);
  contract_kernel<T, BM, BN, BK, TM, TN><<<grid, (BM / TM) * (BN / TN), 0, st>>>(d);
}

template <typename T, int BM, int BN, int TM, int TN, int BK = 16>
static void launch_contract2(const gfb_contract_desc &d, cudaStream_t st) {
  dim3 grid((unsigned)ceil_div(d.M, BM), (unsigned)ceil_div(d.N, BN), (unsigned)d.nsplit);
  constexpr int NT = (BM / TM) * (BN / TN);
  constexpr bool kQuadA = sizeof(T) == 4 && (BM * BK / NT) % 4 == 0;
  constexpr bool kQuadB = sizeof(T) == 4 && (BN * BK / NT) % 4 == 0;
  const bool a16 = (reinterpret_cast<uintptr_t>(d.a) & 15) == 0, b16 = (reinterpret_cast<uintptr_t>(d.b) & 15) == 0;
  if constexpr (kQuadA) {
    if ((d.a_kfast & 3) == 3 && a16) {
      contract2_kernel<T, BM, BN, BK, TM, TN, 1><<<grid, NT, 0, st>>>(d);
      return;
    }
    if constexpr (kQuadB) {
      if ((d.a_kfast & 3) == 2 && (d.b_nfast & 3) == 3 && a16 && b16) {
        contract2_kernel<T, BM, BN, BK, TM, TN, 2><<<grid, NT, 0, st>>>(d);
        return;
      }
    }
  }
  contract2_kernel<T, BM, BN, BK, TM, TN, 0><<<grid, NT, 0, st>>>(d);
}

template <typename T>
static void launch_contract_t(const gfb_contract_desc &d, cudaStream_t st) {
  // variant choice mirrored by lowering.contract_tile
  static const bool v1 = getenv("GFB_CONTRACT_V1") != nullptr;
  constexpr bool f32 = sizeof(T) == 4;
  if (v1) {
    if (d.M <= 48 * 4 && d.N <= 32)
      launch_contract<T, 48, 32, 3, 2>(d, st);
    else if (d.N <= 16)
      launch_contract<T, 128, 16, 4, 2>(d, st);
    else if (d.N <= 32)
      launch_contract<T, 128, 32, 4, 4>(d, st);
    else
      launch_contract<T, 64, 64, 4, 4>(d, st);
  } else if (f32 && d.M > 48 && d.M <= 144 && d.N <= 32) {
    launch_contract2<T, 144, 32, 9, 8>(d, st);  // few outputs, long k: whole output per CTA (weight adjoints)
  } else if (d.M <= 48 * 4 && d.N <= 32) {
    launch_contract2<T, 48, 32, 3, 2>(d, st);  // few outputs, long k (weight adjoints)
  } else if constexpr (f32) {
    if (d.N <= 16)
      launch_contract2<T, 256, 16, 8, 2>(d, st);
    else if (d.N <= 32)
      launch_contract2<T, 256, 32, 8, 4>(d, st);
    else
      launch_contract2<T, 128, 64, 8, 4>(d, st);
  } else {
    if (d.N <= 16)
      launch_contract2<T, 128, 16, 4, 2>(d, st);
    else if (d.N <= 32)
      launch_contract2<T, 128, 32, 4, 4>(d, st);
    else
      launch_contract2<T, 64, 64, 4, 4>(d, st);
  }
  if (d.nsplit > 1) contract_finish_kernel<T><<<(unsigned)ceil_div(d.M * d.N, 32), 1024, 0, st>>>(d);
}

}  // namespace gfb

using namespace gfb;

extern "C" int gfb_contract_launch(const gfb_contract_desc *d, void *stream) {
  if (!d || !d->a || !d->b || !d->d || !d->mtab || !d->ntab || !d->ktab || d->M <= 0 || d->N <= 0 || d->K <= 0 ||
      d->nsplit < 1 || d->ncm < 0 || d->ncm > 2 || d->ncn < 0 || d->ncn > 2 || d->mstride < 3 + d->ncm ||
      d->nstride < 3 + d->ncn || d->kstride < 2 + d->ncm + d->ncn)
    return set_error(GFB_EINVAL, "gfb_contract_launch: bad descriptor");
  if (d->nsplit > 1 && !d->workspace) return set_error(GFB_EINVAL, "gfb_contract_launch: split-k needs a workspace");
  if (d->M > ((int64_t)1 << 40) || d->N > 65535 * 64 || d->nsplit > 65535)
    return set_error(GFB_EINVAL, "gfb_contract_launch: extents out of range");
  cudaStream_t st = (cudaStream_t)stream;
  if (d->dtype == GFB_F64)
    launch_contract_t<double>(*d, st);
  else
    launch_contract_t<float>(*d, st);
  return check_launch("contract");
}
