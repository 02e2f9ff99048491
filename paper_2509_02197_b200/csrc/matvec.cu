// Matrix-vector adjoint family (atax / bicg): one pass over
// a row-major matrix A[R, C] computes
//     r[i] (+)= sum_j A[i,j] u[j]          (row dots,   A @ u)
//     c[j] (+)= sum_i A[i,j] v[i]          (column sums, A^T @ v)
// together. v is either its own vector or, in chain mode, the freshly
// computed r itself (atax: t = A x; y = A^T t), which one pass can do because
// row i of A is on chip when t[i] is complete. The reference runs these as
// separate matmul library nodes (interpreter.py:433-446; adjoint jobs
// autodiff.py:780-802); the lowering pairs two nodes over the same matrix.
//
// HBM-bound: the matrix is streamed once. One persistent CTA per SM owns a
// contiguous band of rows. Whole rows arrive by 1-D bulk copies
// (cp.async.bulk, one elected thread, mbarrier transaction counts) into a
// ring of shared-memory stages, several rows ahead. Thread t owns the 16-byte
// column vectors t + 256 q of every row: u and the column-sum partials stay
// in registers for the whole band, so a row costs a handful of shared-memory
// loads and FMAs plus one block reduction for its dot. Column partials of the
// bands are summed by a second kernel in a fixed order (deterministic).
//
// Also here: the fused rank-2 update C (= | +=) u1 v1^T + u2 v2^T, which
// merges the two outer-product adjoint jobs that write one matrix gradient
// into a single write pass.
#include <cstdint>
#include <cstdlib>

#include "gfb_common.cuh"
#include "gfb_internal.h"

namespace gfb {
namespace {

constexpr int kThreads = 256;
constexpr int kStageBudget = 200 * 1024;  // shared-memory ring bytes

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

// 1-D bulk global -> shared copy completing on an mbarrier
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <typename T>
struct V16;
template <>
struct V16<double> {
  using type = double2;
  static constexpr int W = 2;
  __device__ static double dot(double2 a, double2 b, double acc) { return fma(a.x, b.x, fma(a.y, b.y, acc)); }
  __device__ static void axpy(double2 &y, double2 a, double s) {
    y.x = fma(a.x, s, y.x);
    y.y = fma(a.y, s, y.y);
  }
  __device__ static double2 zero() { return make_double2(0.0, 0.0); }
  __device__ static double2 add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
};
template <>
struct V16<float> {
  using type = float4;
  static constexpr int W = 4;
  __device__ static float dot(float4 a, float4 b, float acc) {
    return fmaf(a.x, b.x, fmaf(a.y, b.y, fmaf(a.z, b.z, fmaf(a.w, b.w, acc))));
  }
  __device__ static void axpy(float4 &y, float4 a, float s) {
    y.x = fmaf(a.x, s, y.x);
    y.y = fmaf(a.y, s, y.y);
    y.z = fmaf(a.z, s, y.z);
    y.w = fmaf(a.w, s, y.w);
  }
  __device__ static float4 zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
  __device__ static float4 add(float4 a, float4 b) { return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }
};

struct MvArgs {
  int64_t R, C, lda;     // rows, columns (elements), row pitch (elements)
  const void *A;
  const void *u;         // row-dot vector (C), or null
  void *r;               // row-dot output (R), or null
  const void *v;         // column-sum vector (R), or null (chain: v = new r)
  void *partial;         // [gridDim.x][C] column-sum partials, or null
  int32_t r_acc, chain, stages;
};

// Q = 16-byte column vectors per thread (C <= 256 * Q * W, Q <= 8: two CTAs
// per SM fit the register file)
// KIND fixes the halves at compile time: 1 rows only, 2 columns only,
// 3 both with an independent v, 4 both in chain mode; 0 reads the descriptor
template <typename T, int Q, int KIND>
__global__ void __launch_bounds__(kThreads, 512 / kThreads) matvec_pair_kernel(MvArgs p) {
  using VT = V16<T>;
  using V = typename VT::type;
  constexpr int W = VT::W;
  extern __shared__ __align__(128) unsigned char smem[];
  const int S = p.stages;
  const int64_t cv = p.C / W;  // vectors per row
  const size_t row_bytes = (size_t)p.C * sizeof(T);
  const size_t stage_bytes = (row_bytes + 127) & ~(size_t)127;
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + (size_t)S * stage_bytes);
  T(*red)[kThreads / 32] = reinterpret_cast<T(*)[kThreads / 32]>(bar + S);

  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t i0 = (int64_t)blockIdx.x * p.R / gridDim.x;
  const int64_t i1 = (int64_t)(blockIdx.x + 1) * p.R / gridDim.x;
  const int n = (int)(i1 - i0);
  const int cv32 = (int)cv;
  const T *A = static_cast<const T *>(p.A);
  const bool has_row = KIND == 0 ? p.u != nullptr : (KIND != 2);
  const bool has_col = KIND == 0 ? p.partial != nullptr : (KIND != 1);
  const bool chain = KIND == 0 ? p.chain != 0 : (KIND == 4);

  if (t == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (t == 0) {
    for (int s = 0; s < S && s < n; ++s) {
      mbar_expect_tx(&bar[s], (uint32_t)row_bytes);
      bulk_load(smem + (size_t)s * stage_bytes, A + (i0 + s) * p.lda, (uint32_t)row_bytes, &bar[s]);
    }
  }

  V uq[Q], cq[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int64_t j = t + (int64_t)kThreads * q;
    uq[q] = (has_row && j < cv) ? reinterpret_cast<const V *>(p.u)[j] : VT::zero();
    cq[q] = VT::zero();
  }
  // per-row scalar operands, fetched one row ahead (off the critical path)
  const T *vsrc = chain ? (p.r_acc ? static_cast<const T *>(p.r) : nullptr) : static_cast<const T *>(p.v);
  T vnext = (has_col && vsrc && n > 0) ? vsrc[i0] : T(0);

  int s = 0;
  uint32_t phase = 0;
  for (int k = 0; k < n; ++k) {
    const T vcur = vnext;
    if (has_col && vsrc && k + 1 < n) vnext = vsrc[i0 + k + 1];
    mbar_wait(&bar[s], phase);
    const V *row = reinterpret_cast<const V *>(smem + (size_t)s * stage_bytes);
    V a[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int j = t + kThreads * q;
      a[q] = j < cv32 ? row[j] : VT::zero();
    }
    T dot = T(0);
    if (has_row) {
      T d2[2] = {T(0), T(0)};
#pragma unroll
      for (int q = 0; q < Q; ++q) d2[q & 1] = VT::dot(a[q], uq[q], d2[q & 1]);
      dot = d2[0] + d2[1];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
      if (lane == 0) red[k & 1][warp] = dot;
    }
    __syncthreads();  // stage s fully read; row dot partials visible
    if (t == 0 && k + S < n) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&bar[s], (uint32_t)row_bytes);
      bulk_load(smem + (size_t)s * stage_bytes, A + (i0 + k + S) * p.lda, (uint32_t)row_bytes, &bar[s]);
    }
    T tval = T(0);
    if (has_row) {
#pragma unroll
      for (int w = 0; w < kThreads / 32; ++w) tval += red[k & 1][w];
    }
    T vi = vcur;
    if (has_row && t == 0) {
      T *ro = static_cast<T *>(p.r) + i0 + k;
      // chain + r_acc: vcur is the old r[i] (read a row ahead by every thread)
      *ro = p.r_acc ? (T)((chain ? vcur : *ro) + tval) : tval;
    }
    if (chain) vi = p.r_acc ? (T)(vcur + tval) : tval;
    if (has_col) {
#pragma unroll
      for (int q = 0; q < Q; ++q) VT::axpy(cq[q], a[q], vi);
    }
    if (++s == S) {
      s = 0;
      phase ^= 1u;
    }
  }
  if (!has_col) return;
  V *out = reinterpret_cast<V *>(static_cast<T *>(p.partial) + (int64_t)blockIdx.x * p.C);
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int j = t + kThreads * q;
    if (j < cv32) out[j] = cq[q];
  }
}

// c[j] (+)= sum_b partial[b][j], b in a fixed order: 32 columns x 32 split
// groups per CTA (a few L2 latency rounds per thread)
template <typename T>
__global__ void __launch_bounds__(1024) colsum_finish_kernel(int64_t C, int64_t nb, const T *__restrict__ partial,
                                                             T *c, int32_t c_acc) {
  __shared__ T red[32][33];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + lane;
  T s[4] = {T(0), T(0), T(0), T(0)};
  if (j < C) {
    int64_t b = g;
    for (; b + 96 < nb; b += 128) {
#pragma unroll
      for (int u = 0; u < 4; ++u) s[u] += partial[(b + 32 * u) * C + j];
    }
    for (; b < nb; b += 32) s[0] += partial[b * C + j];
  }
  red[g][lane] = (s[0] + s[1]) + (s[2] + s[3]);
  __syncthreads();
  if (g == 0 && j < C) {
    T tot = T(0);
#pragma unroll
    for (int q = 0; q < 32; ++q) tot += red[q][lane];
    c[j] = c_acc ? (T)(c[j] + tot) : tot;
  }
}

// C[i, j] (= | +=) u1[i] v1[j] (+ u2[i] v2[j]); rows band per CTA row, the
// v vectors of this thread's columns held in registers across the band
template <typename T, bool TWO, bool ACC>
__global__ void __launch_bounds__(256) rank2_kernel(int64_t M, int64_t N, const T *__restrict__ u1,
                                                    const T *__restrict__ v1, const T *__restrict__ u2,
                                                    const T *__restrict__ v2, T *__restrict__ C, int64_t ldc,
                                                    int64_t rows) {
  using VT = V16<T>;
  using V = typename VT::type;
  constexpr int W = VT::W;
  const int64_t nv = N / W;
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nv) return;
  const V a1 = reinterpret_cast<const V *>(v1)[j];
  const V a2 = TWO ? reinterpret_cast<const V *>(v2)[j] : VT::zero();
  const int64_t i0 = (int64_t)blockIdx.y * rows, i1 = min(i0 + rows, M);
#pragma unroll 4
  for (int64_t i = i0; i < i1; ++i) {
    V *row = reinterpret_cast<V *>(C + i * ldc);
    V o = ACC ? row[j] : VT::zero();
    VT::axpy(o, a1, u1[i]);
    if (TWO) VT::axpy(o, a2, u2[i]);
    row[j] = o;
  }
}

// resident CTAs per SM (a single 8-warp CTA per SM streams at only ~3.2 TB/s
// on B200; tools/lab/mv_lab.cu)
int pair_ctas_per_sm() {
  static int v = 0;
  if (!v) {
    const char *e = getenv("GFB_MV_CTAS");
    v = e ? atoi(e) : 512 / kThreads;
    if (v < 1) v = 1;
    if (v > 4) v = 4;
  }
  return v;
}

int64_t pair_blocks(int64_t R) {
  int64_t b = (int64_t)sm_count() * pair_ctas_per_sm();
  return b > R ? R : b;
}

template <typename T>
int launch_pair(const MvArgs &a0, int64_t nblocks, cudaStream_t st) {
  using VT = V16<T>;
  constexpr int W = VT::W;
  MvArgs a = a0;
  const int64_t cv = a.C / W;
  const size_t row_bytes = (size_t)a.C * sizeof(T);
  const size_t stage_bytes = (row_bytes + 127) & ~(size_t)127;
  int S = (int)(kStageBudget / pair_ctas_per_sm() / stage_bytes);
  if (S > 8) S = 8;
  if (S < 2) S = 2;
  a.stages = S;
  const size_t smem = (size_t)S * stage_bytes + (size_t)S * 8 + 2 * (kThreads / 32) * sizeof(T);
  const dim3 grid((unsigned)nblocks);
  const int kind = (a.u && a.partial) ? (a.chain ? 4 : 3) : (a.u ? 1 : 2);
#define GFB_MV_CASE(QQ)                                                                                  \
  if (cv <= (int64_t)kThreads * QQ) {                                                                    \
    auto k = kind == 4   ? matvec_pair_kernel<T, QQ, 4>                                                  \
             : kind == 3 ? matvec_pair_kernel<T, QQ, 3>                                                  \
             : kind == 1 ? matvec_pair_kernel<T, QQ, 1>                                                  \
                         : matvec_pair_kernel<T, QQ, 2>;                                                 \
    ensure_smem(k, smem);                                                                                \
    k<<<grid, kThreads, smem, st>>>(a);                                                                  \
    return check_launch("matvec_pair");                                                                  \
  }
  GFB_MV_CASE(1)
  GFB_MV_CASE(2)
  GFB_MV_CASE(4)
  GFB_MV_CASE(8)
#undef GFB_MV_CASE
  return set_error(GFB_EUNSUPPORTED, "matvec_pair: row too long");
}

bool al16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

// Shapes the one-pass kernel takes: 16-byte aligned rows, whole vectors,
// at least two ring stages, at least one row per band.
static bool pair_usable(int32_t dtype, int64_t R, int64_t C, int64_t lda, const void *A, const void *u,
                        const void *v, const void *r) {
  const int64_t es = dtype == GFB_F64 ? 8 : 4, W = 16 / es;
  if (R < 1 || C < W || C % W || lda % W) return false;
  if (C > (int64_t)kThreads * 8 * W) return false;
  const size_t stage = ((size_t)C * es + 127) & ~(size_t)127;
  if (kStageBudget / pair_ctas_per_sm() / stage < 2) return false;
  if (!al16(A) || (u && !al16(u))) return false;
  (void)v;
  (void)r;
  return true;
}

}  // namespace gfb

using namespace gfb;

extern "C" int64_t gfb_matvec_pair_workspace_bytes(int32_t dtype, int64_t R, int64_t C, int32_t has_col) {
  if (!has_col) return 0;
  const int64_t es = dtype == GFB_F64 ? 8 : 4;
  return pair_blocks(R) * C * es;
}

extern "C" int gfb_matvec_pair(int32_t dtype, int64_t R, int64_t C, const void *A, int64_t lda, const void *u,
                               void *r, int32_t r_acc, const void *v, void *c, int32_t c_acc, int32_t chain,
                               void *workspace, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (R <= 0 || C <= 0) return GFB_OK;
  if ((u == nullptr) != (r == nullptr)) return set_error(GFB_EINVAL, "gfb_matvec_pair: u and r go together");
  if (chain && (r == nullptr || c == nullptr)) return set_error(GFB_EINVAL, "gfb_matvec_pair: chain needs r and c");
  if (c && !chain && !v) return set_error(GFB_EINVAL, "gfb_matvec_pair: column sums need v");
  if (!pair_usable(dtype, R, C, lda, A, u, v, r)) return set_error(GFB_EUNSUPPORTED, "gfb_matvec_pair: shape");
  if (c && !workspace) return set_error(GFB_EINVAL, "gfb_matvec_pair: workspace required");
  MvArgs a;
  a.R = R;
  a.C = C;
  a.lda = lda;
  a.A = A;
  a.u = u;
  a.r = r;
  a.v = v;
  a.partial = c ? workspace : nullptr;
  a.r_acc = r_acc;
  a.chain = chain;
  a.stages = 0;
  const int64_t nb = pair_blocks(R);
  int rc = dtype == GFB_F64 ? launch_pair<double>(a, nb, st) : launch_pair<float>(a, nb, st);
  if (rc || !c) return rc;
  const unsigned fb = (unsigned)ceil_div(C, 32);
  if (dtype == GFB_F64)
    colsum_finish_kernel<double><<<fb, 1024, 0, st>>>(C, nb, (const double *)workspace, (double *)c, c_acc);
  else
    colsum_finish_kernel<float><<<fb, 1024, 0, st>>>(C, nb, (const float *)workspace, (float *)c, c_acc);
  return check_launch("matvec_pair_finish");
}

extern "C" int gfb_matvec_pair_usable(int32_t dtype, int64_t R, int64_t C, int64_t lda, const void *A,
                                      const void *u) {
  return pair_usable(dtype, R, C, lda, A, u, nullptr, nullptr) ? 1 : 0;
}

extern "C" int gfb_rank2(int32_t dtype, int64_t M, int64_t N, const void *u1, const void *v1, const void *u2,
                         const void *v2, void *C, int64_t ldc, int32_t accumulate, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (M <= 0 || N <= 0) return GFB_OK;
  const int64_t es = dtype == GFB_F64 ? 8 : 4, W = 16 / es;
  if (N % W || ldc % W || !al16(C) || !al16(v1) || (v2 && !al16(v2)))
    return set_error(GFB_EUNSUPPORTED, "gfb_rank2: shape");
  const int64_t nv = N / W;
  const int64_t xb = ceil_div(nv, 256);
  // about eight CTAs per SM in total, bands of rows
  int64_t yb = ceil_div((int64_t)sm_count() * 8, xb);
  if (yb > M) yb = M;
  const int64_t rows = ceil_div(M, yb);
  yb = ceil_div(M, rows);
  const dim3 grid((unsigned)xb, (unsigned)yb);
  const bool two = u2 != nullptr;
#define GFB_R2(T, TW, AC)                                                                                        \
  rank2_kernel<T, TW, AC><<<grid, 256, 0, st>>>(M, N, (const T *)u1, (const T *)v1, (const T *)u2, (const T *)v2, \
                                                (T *)C, ldc, rows)
  if (dtype == GFB_F64) {
    if (two) {
      if (accumulate) GFB_R2(double, true, true); else GFB_R2(double, true, false);
    } else {
      if (accumulate) GFB_R2(double, false, true); else GFB_R2(double, false, false);
    }
  } else {
    if (two) {
      if (accumulate) GFB_R2(float, true, true); else GFB_R2(float, true, false);
    } else {
      if (accumulate) GFB_R2(float, false, true); else GFB_R2(float, false, false);
    }
  }
#undef GFB_R2
  return check_launch("rank2");
}
