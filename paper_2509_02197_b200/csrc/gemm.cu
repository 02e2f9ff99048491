// matmul library node: C (= | +=) op(A) @ op(B), row-major operands.
//
// Reference: Executor._exec_library "matmul" (interpreter.py:433-446) and the
// adjoint jobs gA += g op(B)^T, gB += op(A)^T g (autodiff.py:780-802).
// Shape classes (dispatch in gfb_matmul):
//   K == 1            rank-1 update (outer-product adjoints of matvecs), HBM
//   N == 1 / M == 1   matrix-vector products (atax / bicg), HBM-bound
//   otherwise         tiled GEMM: fp64 on the DMMA tensor path
//                     (mma.sync.m8n8k4.f64 -> DMMA), fp32 on FFMA (split-K
//                     when the tile grid does not cover the SMs)
#include <algorithm>
#include <cstdlib>

#include "gfb_common.cuh"
#include "gfb_internal.h"

namespace gfb {

// ---------------------------------------------------------------------------
// fp32 FFMA GEMM: 64 x 128 CTA tile, BK = 16, 256 threads each owning a
// 4 x 8 register block (a: one 16-byte shared load, b: two), next tile
// prefetched into registers while the current one is consumed. Skinny
// problems (the mlp layers: M = batch = 64) split K over blockIdx.z so the
// grid covers the SMs; fp32 partials are reduced in a fixed order.

constexpr int kSM = 64, kSN = 128, kSK = 16;
constexpr int kSAP = kSM + 4, kSBP = kSN + 4;

template <bool TA, bool TB>
__global__ void __launch_bounds__(256, 2) sgemm_kernel(int64_t M, int64_t N, int64_t K, const float *__restrict__ A,
                                                    int64_t lda, const float *__restrict__ B, int64_t ldb,
                                                    float *C, int64_t ldc, int accumulate, float *partial,
                                                    int64_t kchunk) {
  __shared__ __align__(16) float As[kSK][kSAP];
  __shared__ __align__(16) float Bs[kSK][kSBP];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int64_t m0 = (int64_t)blockIdx.y * kSM, n0 = (int64_t)blockIdx.x * kSN;
  const int64_t kb = (int64_t)blockIdx.z * kchunk, ke = min(kb + kchunk, K);
  // element (mm, kk) / (kk, nn) owned by this thread in the load of a tile
  auto a_at = [&](int r, int &mm, int &kk) {
    const int e = tid + r * 256;
    if (TA) {
      mm = e % kSM;
      kk = e / kSM;
    } else {
      kk = e % kSK;
      mm = e / kSK;
    }
  };
  auto b_at = [&](int r, int &kk, int &nn) {
    const int e = tid + r * 256;
    if (TB) {
      kk = e % kSK;
      nn = e / kSK;
    } else {
      nn = e % kSN;
      kk = e / kSN;
    }
  };
  float ra[kSM * kSK / 256], rb[kSN * kSK / 256];
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int r = 0; r < kSM * kSK / 256; ++r) {
      int mm, kk;
      a_at(r, mm, kk);
      const int64_t gm = m0 + mm, gk = k0 + kk;
      ra[r] = (gm < M && gk < ke) ? (TA ? A[gk * lda + gm] : A[gm * lda + gk]) : 0.f;
    }
#pragma unroll
    for (int r = 0; r < kSN * kSK / 256; ++r) {
      int kk, nn;
      b_at(r, kk, nn);
      const int64_t gn = n0 + nn, gk = k0 + kk;
      rb[r] = (gn < N && gk < ke) ? (TB ? B[gn * ldb + gk] : B[gk * ldb + gn]) : 0.f;
    }
  };
  auto stash = [&]() {
#pragma unroll
    for (int r = 0; r < kSM * kSK / 256; ++r) {
      int mm, kk;
      a_at(r, mm, kk);
      As[kk][mm] = ra[r];
    }
#pragma unroll
    for (int r = 0; r < kSN * kSK / 256; ++r) {
      int kk, nn;
      b_at(r, kk, nn);
      Bs[kk][nn] = rb[r];
    }
  };
  float acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  if (kb < ke) load(kb);
  for (int64_t k0 = kb; k0 < ke; k0 += kSK) {
    __syncthreads();
    stash();
    __syncthreads();
    if (k0 + kSK < ke) load(k0 + kSK);
#pragma unroll
    for (int kk = 0; kk < kSK; ++kk) {
      const float4 a = *reinterpret_cast<const float4 *>(&As[kk][ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4 *>(&Bs[kk][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4 *>(&Bs[kk][64 + tx * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w};
      const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t gn = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
      if (gn >= N) continue;
      if (partial) {
        partial[((int64_t)blockIdx.z * M + gm) * N + gn] = acc[i][j];
      } else {
        float *c = C + gm * ldc + gn;
        *c = accumulate ? *c + acc[i][j] : acc[i][j];
      }
    }
  }
}

__global__ void sgemm_splits_finish(int64_t M, int64_t N, int64_t ns, const float *__restrict__ partial, float *C,
                                    int64_t ldc, int accumulate) {
  const int64_t MN = M * N;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < MN; e += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int64_t q = 0; q < ns; ++q) s += partial[q * MN + e];
    const int64_t m = e / N, n = e - m * N;
    float *c = C + m * ldc + n;
    *c = accumulate ? *c + s : s;
  }
}

static int64_t sgemm_splits(int64_t M, int64_t N, int64_t K) {
  const int64_t tiles = ceil_div(M, kSM) * ceil_div(N, kSN);
  const int64_t target = 2 * (int64_t)sm_count();
  if (tiles >= target) return 1;
  int64_t ns = ceil_div(target, tiles);
  const int64_t maxs = K / (4 * kSK);
  if (ns > maxs) ns = maxs;
  return ns < 1 ? 1 : ns;
}

static int sgemm(int ta, int tb, int64_t M, int64_t N, int64_t K, const float *A, int64_t lda, const float *B,
                 int64_t ldb, float *C, int64_t ldc, int accumulate, void *ws, cudaStream_t st) {
  const int64_t ns = sgemm_splits(M, N, K);
  const int64_t chunk = ceil_div(ceil_div(K, ns), kSK) * kSK;
  const int64_t nz = ceil_div(K, chunk);
  float *partial = nz > 1 ? (float *)ws : nullptr;
  dim3 grid((unsigned)ceil_div(N, kSN), (unsigned)ceil_div(M, kSM), (unsigned)nz);
  if (ta && tb)
    sgemm_kernel<true, true><<<grid, 256, 0, st>>>(M, N, K, A, lda, B, ldb, C, ldc, accumulate, partial, chunk);
  else if (ta)
    sgemm_kernel<true, false><<<grid, 256, 0, st>>>(M, N, K, A, lda, B, ldb, C, ldc, accumulate, partial, chunk);
  else if (tb)
    sgemm_kernel<false, true><<<grid, 256, 0, st>>>(M, N, K, A, lda, B, ldb, C, ldc, accumulate, partial, chunk);
  else
    sgemm_kernel<false, false><<<grid, 256, 0, st>>>(M, N, K, A, lda, B, ldb, C, ldc, accumulate, partial, chunk);
  if (nz > 1) {
    const unsigned blocks = (unsigned)min(ceil_div(M * N, 256), (int64_t)sm_count() * 8);
    sgemm_splits_finish<<<blocks, 256, 0, st>>>(M, N, nz, partial, C, ldc, accumulate);
  }
  return check_launch("sgemm");
}

// ---------------------------------------------------------------------------
// fp64 DMMA GEMM: 64x64 CTA tile, BK = 16, 4 warps each owning 32x32 (4x4
// m8n8 tiles), mma.sync.aligned.m8n8k4.row.col.f64 (-> DMMA.8x8x4 on
// sm_100a; the larger f64 shapes decompose into the same instruction).
// Operands stream through a 3-stage cp.async ring in their stored
// orientation: A as [m][k] (no ta) or [k][m] (ta), B as [k][n] (no tb) or
// [n][k] (tb). Row pitches of 4 (mod 16) doubles keep every fragment load
// conflict-free in either orientation. Small tiles with 3 CTAs (12 warps) per
// SM hide the DMMA latency better than one 128x128 CTA per SM
// (tools/lab/dgemm_lab.cu: 32.2 vs 26.7 TF/s at 4000^3; cuBLAS 34.5).

static bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

constexpr int kDM = 64, kDN = 64, kDK = 16, kDS = 3;

__device__ __forceinline__ void dmma884(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int V>
__device__ __forceinline__ void cp_async_f64(double *s, const double *g, bool ok) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  if constexpr (V == 2)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(g), "r"(ok ? 16 : 0));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(g), "r"(ok ? 8 : 0));
}

// one operand tile (rows x cols of the STORED matrix, contiguous along cols)
template <int V, int ROWS, int COLS>
__device__ __forceinline__ void dmma_stage(double *s, const double *g, int64_t ld, int64_t r0, int64_t c0,
                                           int64_t R, int64_t Cn, int tid) {
  constexpr int P = COLS + 4, CH = COLS / V;
#pragma unroll
  for (int c = tid; c < ROWS * CH; c += 128) {
    const int r = c / CH, cc = (c % CH) * V;
    const int64_t gr = r0 + r, gc = c0 + cc;
    const bool ok = gr < R && gc < Cn;  // V == 2: Cn even, so a chunk is all in or all out
    cp_async_f64<V>(s + r * P + cc, ok ? g + gr * ld + gc : g, ok);
  }
}

template <int TA, int TB, int V>
__global__ void __launch_bounds__(128, 3) dgemm_dmma_kernel(int64_t M, int64_t N, int64_t K,
                                                            const double *__restrict__ A, int64_t lda,
                                                            const double *__restrict__ B, int64_t ldb, double *C,
                                                            int64_t ldc, int accumulate) {
  constexpr int SA = TA ? kDK * (kDM + 4) : kDM * (kDK + 4);
  constexpr int SB = TB ? kDN * (kDK + 4) : kDK * (kDN + 4);
  extern __shared__ __align__(16) double dsm[];
  double *As = dsm, *Bs = dsm + kDS * SA;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int64_t m0 = (int64_t)blockIdx.y * kDM, n0 = (int64_t)blockIdx.x * kDN;
  const int64_t ktiles = (K + kDK - 1) / kDK;
  auto load = [&](int64_t kt, int slot) {
    const int64_t k0 = kt * kDK;
    if constexpr (TA) dmma_stage<V, kDK, kDM>(As + slot * SA, A, lda, k0, m0, K, M, tid);
    else dmma_stage<V, kDM, kDK>(As + slot * SA, A, lda, m0, k0, M, K, tid);
    if constexpr (TB) dmma_stage<V, kDN, kDK>(Bs + slot * SB, B, ldb, n0, k0, N, K, tid);
    else dmma_stage<V, kDK, kDN>(Bs + slot * SB, B, ldb, k0, n0, K, N, tid);
  };
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll
  for (int s = 0; s < kDS - 1; ++s) {
    if (s < ktiles) load(s, s);
    asm volatile("cp.async.commit_group;\n");
  }
  // m8n8k4 fragments: A(row) lane -> A[lane/4][lane%4]; B(col) lane ->
  // B[lane%4][lane/4]; D lane -> D[lane/4][2*(lane%4) + {0,1}]
  const int fr = lane >> 2, fc = lane & 3;
  for (int64_t kt = 0; kt < ktiles; ++kt) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(kDS - 2));
    __syncthreads();  // tile kt visible to all; slot (kt-1)%S free for reuse
    if (kt + kDS - 1 < ktiles) load(kt + kDS - 1, (int)((kt + kDS - 1) % kDS));
    asm volatile("cp.async.commit_group;\n");
    const double *as = As + (kt % kDS) * SA, *bs = Bs + (kt % kDS) * SB;
#pragma unroll
    for (int ks = 0; ks < kDK; ks += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
        af[a] = TA ? as[(ks + fc) * (kDM + 4) + wm + a * 8 + fr] : as[(wm + a * 8 + fr) * (kDK + 4) + ks + fc];
#pragma unroll
      for (int b = 0; b < 4; ++b)
        bf[b] = TB ? bs[(wn + b * 8 + fr) * (kDK + 4) + ks + fc] : bs[(ks + fc) * (kDN + 4) + wn + b * 8 + fr];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma884(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
  }
  asm volatile("cp.async.wait_group 0;\n");
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int64_t gm = m0 + wm + a * 8 + fr;
    if (gm >= M) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t gn = n0 + wn + b * 8 + 2 * fc + h;
        if (gn >= N) continue;
        double *c = C + gm * ldc + gn;
        *c = accumulate ? *c + acc[a][b][h] : acc[a][b][h];
      }
  }
}

template <int TA, int TB, int V>
static int dgemm_dmma_t(int64_t M, int64_t N, int64_t K, const double *A, int64_t lda, const double *B, int64_t ldb,
                        double *C, int64_t ldc, int accumulate, cudaStream_t st) {
  constexpr int SA = TA ? kDK * (kDM + 4) : kDM * (kDK + 4);
  constexpr int SB = TB ? kDN * (kDK + 4) : kDK * (kDN + 4);
  constexpr int smem = kDS * (SA + SB) * 8;
  ensure_smem(dgemm_dmma_kernel<TA, TB, V>, smem);
  dim3 grid((unsigned)ceil_div(N, kDN), (unsigned)ceil_div(M, kDM));
  dgemm_dmma_kernel<TA, TB, V><<<grid, 128, smem, st>>>(M, N, K, A, lda, B, ldb, C, ldc, accumulate);
  return check_launch("dgemm_dmma");
}

static int dgemm_dmma(int ta, int tb, int64_t M, int64_t N, int64_t K, const double *A, int64_t lda, const double *B,
                      int64_t ldb, double *C, int64_t ldc, int accumulate, cudaStream_t st) {
  // 16-byte chunks need both operands 16-byte aligned with even leading
  // dimensions and even extents along the contiguous axis
  const int64_t ca = ta ? M : K, cb = tb ? K : N;
  const bool v2 = aligned16(A) && aligned16(B) && lda % 2 == 0 && ldb % 2 == 0 && ca % 2 == 0 && cb % 2 == 0;
#define GFB_DMMA(TA, TB)                                                                                      \
  if (ta == TA && tb == TB)                                                                                   \
    return v2 ? dgemm_dmma_t<TA, TB, 2>(M, N, K, A, lda, B, ldb, C, ldc, accumulate, st)                      \
              : dgemm_dmma_t<TA, TB, 1>(M, N, K, A, lda, B, ldb, C, ldc, accumulate, st);
  GFB_DMMA(0, 0)
  GFB_DMMA(0, 1)
  GFB_DMMA(1, 0)
  GFB_DMMA(1, 1)
#undef GFB_DMMA
  return set_error(GFB_EINVAL, "gfb_matmul: bad transpose flags");
}

// ---------------------------------------------------------------------------
// matrix-vector: y[i] = sum_k op(A)(i,k) x[k]

// op(A)(i,k) contiguous in k: one warp per output row
template <typename T>
__global__ void __launch_bounds__(256) gemv_rowdot_kernel(int64_t M, int64_t K, const T *__restrict__ A,
                                                          int64_t lda, const T *__restrict__ x, int64_t incx,
                                                          T *y, int64_t incy, int accumulate) {
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= M) return;
  const T *a = A + row * lda;
  // eight independent partial sums keep eight loads per lane in flight
  T part[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) part[u] = T(0);
  int64_t k = lane;
  for (; k + 7 * 32 < K; k += 8 * 32) {
#pragma unroll
    for (int u = 0; u < 8; ++u) part[u] = fma(a[k + u * 32], x[(k + u * 32) * incx], part[u]);
  }
  for (; k < K; k += 32) part[0] = fma(a[k], x[k * incx], part[0]);
  T acc = ((part[0] + part[1]) + (part[2] + part[3])) + ((part[4] + part[5]) + (part[6] + part[7]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if (lane == 0) {
    T *o = y + row * incy;
    *o = accumulate ? (T)(*o + acc) : acc;
  }
}

// op(A)(i,k) = S[k*lds + i] (contiguous in i): split-K column sums.
// partial[s][i] over k-chunk s; a second pass reduces the splits in order.
template <typename T>
__global__ void __launch_bounds__(256) gemv_colsum_kernel(int64_t M, int64_t K, const T *__restrict__ S,
                                                          int64_t lds, const T *__restrict__ x, int64_t incx,
                                                          T *partial, int64_t kchunk) {
  __shared__ T red[8][33];
  const int64_t i = (int64_t)blockIdx.x * 32 + (threadIdx.x & 31);
  const int g = threadIdx.x >> 5;
  const int64_t kb = (int64_t)blockIdx.y * kchunk;
  const int64_t ke = min(kb + kchunk, K);
  T part[4] = {T(0), T(0), T(0), T(0)};
  if (i < M) {
    int64_t k = kb + g;
    for (; k + 24 < ke; k += 32) {
#pragma unroll
      for (int u = 0; u < 4; ++u) part[u] = fma(S[(k + 8 * u) * lds + i], x[(k + 8 * u) * incx], part[u]);
    }
    for (; k < ke; k += 8) part[0] = fma(S[k * lds + i], x[k * incx], part[0]);
  }
  red[g][threadIdx.x & 31] = (part[0] + part[1]) + (part[2] + part[3]);
  __syncthreads();
  if (g == 0 && i < M) {
    T s = T(0);
#pragma unroll
    for (int q = 0; q < 8; ++q) s += red[q][threadIdx.x];
    partial[(int64_t)blockIdx.y * M + i] = s;
  }
}

template <typename T>
__global__ void splits_finish_kernel(int64_t M, int64_t nsplit, const T *__restrict__ partial, T *y, int64_t incy,
                                     int accumulate) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M) return;
  T s = T(0);
  for (int64_t q = 0; q < nsplit; ++q) s += partial[q * M + i];
  T *o = y + i * incy;
  *o = accumulate ? (T)(*o + s) : s;
}

// rank-1: C[i,j] (+)= u[i*incu] * v[j*incv]
template <typename T>
__global__ void __launch_bounds__(256) rank1_kernel(int64_t M, int64_t N, const T *__restrict__ u, int64_t incu,
                                                    const T *__restrict__ v, int64_t incv, T *C, int64_t ldc,
                                                    int accumulate) {
  for (int64_t i = blockIdx.y; i < M; i += gridDim.y) {
    const T ui = u[i * incu];
    T *row = C + i * ldc;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x) {
      const T r = ui * v[j * incv];
      row[j] = accumulate ? (T)(row[j] + r) : r;
    }
  }
}

// 16-byte vector variants (aligned operands, unit-stride vectors): half /
// a quarter of the load instructions, four independent 16-byte partial sums
// in flight per lane.
template <typename T>
struct Vec16;
template <>
struct Vec16<double> {
  using type = double2;
  static constexpr int W = 2;
  __device__ static double dot(double2 a, double2 b) { return fma(a.x, b.x, a.y * b.y); }
  __device__ static double2 fmav(double2 a, double2 b, double2 c) {
    return make_double2(fma(a.x, b.x, c.x), fma(a.y, b.y, c.y));
  }
  __device__ static double2 zero() { return make_double2(0.0, 0.0); }
  __device__ static double2 splat(double s) { return make_double2(s, s); }
  __device__ static double get(double2 v, int i) { return i == 0 ? v.x : v.y; }
};
template <>
struct Vec16<float> {
  using type = float4;
  static constexpr int W = 4;
  __device__ static float dot(float4 a, float4 b) { return fmaf(a.x, b.x, fmaf(a.y, b.y, fmaf(a.z, b.z, a.w * b.w))); }
  __device__ static float4 fmav(float4 a, float4 b, float4 c) {
    return make_float4(fmaf(a.x, b.x, c.x), fmaf(a.y, b.y, c.y), fmaf(a.z, b.z, c.z), fmaf(a.w, b.w, c.w));
  }
  __device__ static float4 zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
  __device__ static float4 splat(float s) { return make_float4(s, s, s, s); }
  __device__ static float get(float4 v, int i) { return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w; }
};

// column sums with W adjacent columns per lane (32*W per CTA)
template <typename T>
__global__ void __launch_bounds__(256) gemv_colsum_vec_kernel(int64_t M, int64_t K, const T *__restrict__ S,
                                                              int64_t lds, const T *__restrict__ x, int64_t incx,
                                                              T *partial, int64_t kchunk) {
  using VT = Vec16<T>;
  using V = typename VT::type;
  constexpr int W = VT::W;
  __shared__ V red[8][32];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t i = ((int64_t)blockIdx.x * 32 + lane) * W;  // first of this lane's W columns (M % W == 0)
  const int64_t kb = (int64_t)blockIdx.y * kchunk, ke = min(kb + kchunk, K);
  V p[4] = {VT::zero(), VT::zero(), VT::zero(), VT::zero()};
  if (i < M) {
    int64_t k = kb + g;
    for (; k + 24 < ke; k += 32) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t kk = k + 8 * u;
        p[u] = VT::fmav(*reinterpret_cast<const V *>(S + kk * lds + i), VT::splat(x[kk * incx]), p[u]);
      }
    }
    for (; k < ke; k += 8) p[0] = VT::fmav(*reinterpret_cast<const V *>(S + k * lds + i), VT::splat(x[k * incx]), p[0]);
  }
  V t;
  if constexpr (W == 2) {
    t = make_double2((p[0].x + p[1].x) + (p[2].x + p[3].x), (p[0].y + p[1].y) + (p[2].y + p[3].y));
  } else {
    t = make_float4((p[0].x + p[1].x) + (p[2].x + p[3].x), (p[0].y + p[1].y) + (p[2].y + p[3].y),
                    (p[0].z + p[1].z) + (p[2].z + p[3].z), (p[0].w + p[1].w) + (p[2].w + p[3].w));
  }
  red[g][lane] = t;
  __syncthreads();
  if (g == 0 && i < M) {
    T sum[W];
#pragma unroll
    for (int c = 0; c < W; ++c) sum[c] = T(0);
#pragma unroll
    for (int q = 0; q < 8; ++q)
#pragma unroll
      for (int c = 0; c < W; ++c) sum[c] += VT::get(red[q][lane], c);
#pragma unroll
    for (int c = 0; c < W; ++c) partial[(int64_t)blockIdx.y * M + i + c] = sum[c];
  }
}

// rank-1 with 16-byte row stores (C rows aligned, v contiguous)
template <typename T>
__global__ void __launch_bounds__(256) rank1_vec_kernel(int64_t M, int64_t N, const T *__restrict__ u, int64_t incu,
                                                        const T *__restrict__ v, T *C, int64_t ldc,
                                                        int accumulate) {
  using VT = Vec16<T>;
  using V = typename VT::type;
  constexpr int W = VT::W;
  const int64_t nv = N / W;
  const V *vv = reinterpret_cast<const V *>(v);
  for (int64_t i = blockIdx.y; i < M; i += gridDim.y) {
    const T ui = u[i * incu];
    V *row = reinterpret_cast<V *>(C + i * ldc);
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nv; j += (int64_t)gridDim.x * blockDim.x) {
      const V r = VT::fmav(VT::splat(ui), vv[j], accumulate ? row[j] : VT::zero());
      row[j] = r;
    }
    if (blockIdx.x == 0)
      for (int64_t j = nv * W + threadIdx.x; j < N; j += blockDim.x) {
        const T r = ui * v[j];
        C[i * ldc + j] = accumulate ? (T)(C[i * ldc + j] + r) : r;
      }
  }
}


// Row dots with a whole CTA per row (grid-stride over rows): the row's
// 16-byte vectors are spread over 256 threads, so one row is a single round
// of loads in flight instead of a warp's long sequential walk.
template <typename T>
__global__ void __launch_bounds__(256) gemv_rowdot_cta_kernel(int64_t M, int64_t K, const T *__restrict__ A,
                                                              int64_t lda, const T *__restrict__ x, T *y,
                                                              int64_t incy, int accumulate) {
  using VT = Vec16<T>;
  using V = typename VT::type;
  constexpr int W = VT::W;
  __shared__ T red[8];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t nv = K / W;
  const V *xv = reinterpret_cast<const V *>(x);
  for (int64_t row = blockIdx.x; row < M; row += gridDim.x) {
    const V *a = reinterpret_cast<const V *>(A + row * lda);
    T p[4] = {T(0), T(0), T(0), T(0)};
    int64_t j = t;
    for (; j + 768 < nv; j += 1024) {
#pragma unroll
      for (int u = 0; u < 4; ++u) p[u] += VT::dot(a[j + 256 * u], xv[j + 256 * u]);
    }
    for (; j < nv; j += 256) p[0] += VT::dot(a[j], xv[j]);
    for (int64_t k = nv * W + t; k < K; k += 256) p[1] = fma(A[row * lda + k], x[k], p[1]);
    T acc = (p[0] + p[1]) + (p[2] + p[3]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (t == 0) {
      T s = T(0);
#pragma unroll
      for (int w = 0; w < 8; ++w) s += red[w];
      T *o = y + row * incy;
      *o = accumulate ? (T)(*o + s) : s;
    }
    __syncthreads();
  }
}

static int64_t colsum_splits(int64_t M, int64_t K) {
  int64_t cols_blocks = ceil_div(M, 32);
  int64_t want = ceil_div((int64_t)sm_count() * 4, cols_blocks);
  int64_t maxs = ceil_div(K, 64);
  if (want > maxs) want = maxs;
  return want < 1 ? 1 : want;
}

template <typename T>
static int gemv_colsum(int64_t M, int64_t K, const T *S, int64_t lds, const T *x, int64_t incx, T *y, int64_t incy,
                       int accumulate, void *ws, cudaStream_t st) {
  int64_t ns = colsum_splits(M, K);
  int64_t chunk = ceil_div(K, ns);
  T *partial = (T *)ws;
  constexpr int W = Vec16<T>::W;
  if (aligned16(S) && lds % W == 0 && M % W == 0) {
    dim3 grid((unsigned)ceil_div(M, 32 * W), (unsigned)ns);
    gemv_colsum_vec_kernel<T><<<grid, 256, 0, st>>>(M, K, S, lds, x, incx, partial, chunk);
  } else {
    dim3 grid((unsigned)ceil_div(M, 32), (unsigned)ns);
    gemv_colsum_kernel<T><<<grid, 256, 0, st>>>(M, K, S, lds, x, incx, partial, chunk);
  }
  splits_finish_kernel<T><<<(unsigned)ceil_div(M, 256), 256, 0, st>>>(M, ns, partial, y, incy, accumulate);
  return check_launch("gemv_colsum");
}

template <typename T>
static int matmul_t(int ta, int tb, int64_t M, int64_t N, int64_t K, const T *A, int64_t lda, const T *B, int64_t ldb,
                    T *C, int64_t ldc, int accumulate, void *ws, cudaStream_t st) {
  if (M <= 0 || N <= 0) return GFB_OK;
  if (K == 0) {
    if (!accumulate) {
      for (int64_t i = 0; i < M; ++i) cudaMemsetAsync(C + i * ldc, 0, (size_t)N * sizeof(T), st);
    }
    return check_launch("matmul_k0");
  }
  if (K == 1) {
    // op(A) column 0: element i at A[i*lda] (no ta) or A[i] (ta: A stored [1, M])
    int64_t incu = ta ? 1 : lda;
    int64_t incv = tb ? ldb : 1;  // op(B) row 0: B[j] (no tb) or B[j*ldb] (tb: stored [N,1])
    constexpr int W = Vec16<T>::W;
    if (incv == 1 && aligned16(B) && aligned16(C) && ldc % W == 0) {
      dim3 grid((unsigned)min(ceil_div(N / W, 256 * 8), (int64_t)8),
                (unsigned)min(M, (int64_t)sm_count() * 8));
      rank1_vec_kernel<T><<<grid, 256, 0, st>>>(M, N, A, incu, B, C, ldc, accumulate);
    } else {
      dim3 grid((unsigned)min(ceil_div(N, 256), (int64_t)8), (unsigned)min(M, (int64_t)65535));
      rank1_kernel<T><<<grid, 256, 0, st>>>(M, N, A, incu, B, incv, C, ldc, accumulate);
    }
    return check_launch("rank1");
  }
  constexpr int32_t kDt = sizeof(T) == 8 ? GFB_F64 : GFB_F32;
  if (N == 1) {
    // x = op(B)(:,0): B[k*ldb] (no tb) or B[k] (tb)
    int64_t incx = tb ? 1 : ldb;
    // one-pass streaming kernel (matvec.cu) over A as stored
    if (incx == 1 && ldc == 1) {
      if (!ta && gfb_matvec_pair_usable(kDt, M, K, lda, A, B))
        return gfb_matvec_pair(kDt, M, K, A, lda, B, C, accumulate, nullptr, nullptr, 0, 0, ws, st);
      if (ta && gfb_matvec_pair_usable(kDt, K, M, lda, A, nullptr))
        return gfb_matvec_pair(kDt, K, M, A, lda, nullptr, nullptr, 0, B, C, accumulate, 0, ws, st);
    }
    if (!ta) {
      constexpr int W = Vec16<T>::W;
      if (incx == 1 && aligned16(A) && aligned16(B) && lda % W == 0) {
        const unsigned blocks = (unsigned)min(M, (int64_t)sm_count() * 8);
        gemv_rowdot_cta_kernel<T><<<blocks, 256, 0, st>>>(M, K, A, lda, B, C, ldc, accumulate);
      } else {
        gemv_rowdot_kernel<T><<<(unsigned)ceil_div(M, 8), 256, 0, st>>>(M, K, A, lda, B, incx, C, ldc, accumulate);
      }
      return check_launch("gemv_rowdot");
    }
    return gemv_colsum<T>(M, K, A, lda, B, incx, C, ldc, accumulate, ws, st);
  }
  if (M == 1) {
    // y[j] = sum_k op(A)(0,k) op(B)(k,j); op(A) row 0: A[k] (no ta) or A[k*lda] (ta)
    int64_t incx = ta ? lda : 1;
    if (incx == 1) {
      if (tb && gfb_matvec_pair_usable(kDt, N, K, ldb, B, A))
        return gfb_matvec_pair(kDt, N, K, B, ldb, A, C, accumulate, nullptr, nullptr, 0, 0, ws, st);
      if (!tb && gfb_matvec_pair_usable(kDt, K, N, ldb, B, nullptr))
        return gfb_matvec_pair(kDt, K, N, B, ldb, nullptr, nullptr, 0, A, C, accumulate, 0, ws, st);
    }
    if (tb) {  // op(B)(k,j) = B[j*ldb + k]: row dots
      constexpr int W = Vec16<T>::W;
      if (incx == 1 && aligned16(A) && aligned16(B) && ldb % W == 0) {
        const unsigned blocks = (unsigned)min(N, (int64_t)sm_count() * 8);
        gemv_rowdot_cta_kernel<T><<<blocks, 256, 0, st>>>(N, K, B, ldb, A, C, 1, accumulate);
      } else {
        gemv_rowdot_kernel<T><<<(unsigned)ceil_div(N, 8), 256, 0, st>>>(N, K, B, ldb, A, incx, C, 1, accumulate);
      }
      return check_launch("gemv_rowdot");
    }
    return gemv_colsum<T>(N, K, B, ldb, A, incx, C, 1, accumulate, ws, st);
  }
  return -1;  // general GEMM handled by the caller
}

}  // namespace gfb

using namespace gfb;

extern "C" int64_t gfb_matmul_workspace_bytes(int32_t dtype, int32_t ta, int32_t tb, int64_t M, int64_t N,
                                              int64_t K) {
  int64_t es = dtype == GFB_F64 ? 8 : 4;
  if (K > 1 && N == 1 && ta)
    return std::max(colsum_splits(M, K) * M * es, gfb_matvec_pair_workspace_bytes(dtype, K, M, 1));
  if (K > 1 && M == 1 && !tb && N > 1)
    return std::max(colsum_splits(N, K) * N * es, gfb_matvec_pair_workspace_bytes(dtype, K, N, 1));
  if (dtype != GFB_F64 && K > 1 && M > 1 && N > 1 && sgemm_tc_usable(M, N, K)) return sgemm_tc_workspace(M, N, K);
  if (dtype != GFB_F64 && K > 1 && M > 1 && N > 1) {
    const int64_t ns = sgemm_splits(M, N, K);
    if (ns > 1) {
      const int64_t chunk = ceil_div(ceil_div(K, ns), kSK) * kSK;
      const int64_t nz = ceil_div(K, chunk);
      if (nz > 1) return nz * M * N * 4;
    }
  }
  return 0;
}

extern "C" int gfb_matmul(int32_t dtype, int32_t ta, int32_t tb, int64_t M, int64_t N, int64_t K, const void *A,
                          int64_t lda, const void *B, int64_t ldb, void *C, int64_t ldc, int32_t accumulate,
                          void *workspace, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (gfb_matmul_workspace_bytes(dtype, ta, tb, M, N, K) > 0 && !workspace)
    return set_error(GFB_EINVAL, "gfb_matmul: workspace required");
  int rc;
  if (dtype == GFB_F64) {
    rc = matmul_t<double>(ta, tb, M, N, K, (const double *)A, lda, (const double *)B, ldb, (double *)C, ldc,
                          accumulate, workspace, st);
    if (rc >= 0) return rc;
    return dgemm_dmma(ta, tb, M, N, K, (const double *)A, lda, (const double *)B, ldb, (double *)C, ldc, accumulate,
                      st);
  }
  rc = matmul_t<float>(ta, tb, M, N, K, (const float *)A, lda, (const float *)B, ldb, (float *)C, ldc, accumulate,
                       workspace, st);
  if (rc >= 0) return rc;
  if (sgemm_tc_usable(M, N, K))
    return sgemm_tc(ta, tb, M, N, K, (const float *)A, lda, (const float *)B, ldb, (float *)C, ldc, accumulate,
                    workspace, st);
  return sgemm(ta, tb, M, N, K, (const float *)A, lda, (const float *)B, ldb, (float *)C, ldc, accumulate, workspace,
               st);
}
