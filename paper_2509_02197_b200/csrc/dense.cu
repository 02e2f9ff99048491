// Whole-array library nodes: reduce_sum, elementwise, broadcast, box fill.
//
// Reference semantics: Executor._exec_library (interpreter.py:428-476),
// _apply_unary / _BINARY_LIB (interpreter.py:553-597), the reduce_sum adjoint
// broadcast map (autodiff.py:940-960) and zero-init on first touch
// (interpreter.py:171-189). All kernels are HBM-bound streaming passes:
// grid-stride, coalesced, 16-byte vector accesses where alignment allows.
#include "gfb_common.cuh"
#include "gfb_internal.h"

namespace gfb {

constexpr int kThreads = 256;

static int64_t stream_blocks(int64_t n, int64_t per_thread) {
  int64_t b = ceil_div(n, (int64_t)kThreads * per_thread);
  int64_t cap = (int64_t)sm_count() * 8;
  if (b > cap) b = cap;
  return b < 1 ? 1 : b;
}

// ---------------------------------------------------------------------------
// reduce_sum: deterministic two-pass tree (fixed grid for a given n)

static int64_t reduce_blocks(int64_t n) {
  int64_t b = ceil_div(n, (int64_t)kThreads * 16);
  int64_t cap = 148 * 8;  // independent of the device so the order is stable
  if (b > cap) b = cap;
  return b < 1 ? 1 : b;
}

template <typename TI>
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double warp_part[kThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) warp_part[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < 32) {
    s = threadIdx.x < kThreads / 32 ? warp_part[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  }
  return s;  // valid in thread 0
}

template <typename TI>
__global__ void __launch_bounds__(kThreads) reduce_pass1(const TI *__restrict__ x, int64_t n,
                                                         double *__restrict__ part) {
  pdl_wait();  // programmatic dependent launch: global memory after the wait
  PdlRelease pdl_release_;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  const int64_t t0 = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if ((reinterpret_cast<uintptr_t>(x) & 15) == 0) {
    // 16-byte vectors, four independent fp64 partial sums per thread
    constexpr int W = 16 / sizeof(TI);
    const int64_t nv = n / W;
    for (int64_t i = t0; i < nv; i += stride) {
      const TI *v = x + i * W;
      if constexpr (W == 4) {
        const float4 q = *reinterpret_cast<const float4 *>(v);
        acc[0] += q.x, acc[1] += q.y, acc[2] += q.z, acc[3] += q.w;
      } else {
        const double2 q = *reinterpret_cast<const double2 *>(v);
        acc[0] += q.x, acc[1] += q.y;
      }
    }
    for (int64_t i = nv * W + t0; i < n; i += stride) acc[2] += (double)x[i];
  } else {
    for (int64_t i = t0; i < n; i += stride) acc[0] += (double)x[i];
  }
  double s = block_sum<TI>((acc[0] + acc[1]) + (acc[2] + acc[3]));
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// n small enough for one block (nb == 1): one launch instead of two (a
// fixed-order strided sum and block sum, deterministic)
template <typename TI, typename TO>
__global__ void __launch_bounds__(kThreads) reduce_single(const TI *__restrict__ x, int64_t n, TO *out,
                                                          int accumulate) {
  pdl_wait();  // programmatic dependent launch: global memory after the wait
  PdlRelease pdl_release_;
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += kThreads) acc += (double)x[i];
  double s = block_sum<TI>(acc);
  if (threadIdx.x == 0) {
    TO r = (TO)s;
    *out = accumulate ? (TO)(*out + r) : r;
  }
}

template <typename TO>
__global__ void __launch_bounds__(kThreads) reduce_pass2(const double *__restrict__ part, int64_t nb, TO *out,
                                                         int accumulate) {
  pdl_wait();  // programmatic dependent launch: global memory after the wait
  PdlRelease pdl_release_;
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < nb; i += kThreads) acc += part[i];
  double s = block_sum<TO>(acc);
  if (threadIdx.x == 0) {
    TO r = (TO)s;
    *out = accumulate ? (TO)(*out + r) : r;
  }
}

// ---------------------------------------------------------------------------
// elementwise

template <typename T>
__global__ void __launch_bounds__(kThreads) ew_kernel(int op, T c, const T *__restrict__ a, int64_t n_a,
                                                      const T *__restrict__ b, int64_t n_b, T *out, int64_t n,
                                                      int accumulate, uint32_t *err) {
  pdl_wait();  // programmatic dependent launch: global memory after the wait
  PdlRelease pdl_release_;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
    T x = a[n_a == 1 ? 0 : i];
    T r;
    if (b == nullptr) {
      if (op == GFB_OP_IN)
        r = x;
      else if (op == GFB_OP_MUL)
        r = x * c;
      else
        r = apply_unary<T>(op, x, err);
    } else {
      r = apply_binary<T>(op, x, b[n_b == 1 ? 0 : i], err);
    }
    if (accumulate) r = out[i] + r;
    out[i] = r;
  }
}

// Vectorised elementwise for the common operators on full-length,
// 16-byte-aligned operands: the operator is a template parameter (no
// per-element dispatch) and every access is a 16-byte vector.
template <typename T>
struct EwVec;
template <>
struct EwVec<float> {
  using V = float4;
  static constexpr int W = 4;
};
template <>
struct EwVec<double> {
  using V = double2;
  static constexpr int W = 2;
};

template <typename T, int OP>
__device__ __forceinline__ T ew_apply(T x, T y, T c, uint32_t &bad) {
  if constexpr (OP == GFB_OP_IN) return x;
  if constexpr (OP == -1) return x * c;  // scale by a constant
  if constexpr (OP == GFB_OP_ADD) return x + y;
  if constexpr (OP == GFB_OP_SUB) return x - y;
  if constexpr (OP == GFB_OP_MUL) return x * y;
  if constexpr (OP == GFB_OP_DIV) {
    if (y == T(0)) bad |= GFB_EBIT_DIV0;
    return x / y;
  }
  if constexpr (OP == GFB_OP_EXP) return t_exp(x);
  return x;
}

template <typename T, int OP, bool HASB>
__global__ void __launch_bounds__(kThreads) ew_vec_kernel(T c, const T *__restrict__ a, const T *__restrict__ b,
                                                          T *out, int64_t nv, int accumulate, uint32_t *err) {
  pdl_wait();  // programmatic dependent launch: global memory after the wait
  PdlRelease pdl_release_;
  using V = typename EwVec<T>::V;
  constexpr int W = EwVec<T>::W;
  const V *av = reinterpret_cast<const V *>(a);
  const V *bv = reinterpret_cast<const V *>(b);
  V *ov = reinterpret_cast<V *>(out);
  uint32_t bad = 0;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < nv; i += stride) {
    const V x = av[i];
    V y = x;
    if (HASB) y = bv[i];
    V o = accumulate ? ov[i] : V{};
    const T *xs = reinterpret_cast<const T *>(&x);
    const T *ys = reinterpret_cast<const T *>(&y);
    T *os = reinterpret_cast<T *>(&o);
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const T r = ew_apply<T, OP>(xs[w], ys[w], c, bad);
      os[w] = accumulate ? os[w] + r : r;
    }
    ov[i] = o;
  }
  if (bad) raise_bits(err, bad);
}

template <typename T>
static bool ew_vec_launch(int op, T c, const T *a, int64_t n_a, const T *b, int64_t n_b, T *out, int64_t n,
                          int accumulate, uint32_t *err, cudaStream_t st) {
  constexpr int W = EwVec<T>::W;
  auto al = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (n % W || n_a != n || !al(a) || !al(out) || (b && (n_b != n || !al(b)))) return false;
  const int64_t nv = n / W;
  const unsigned blocks = (unsigned)stream_blocks(nv, 2);
#define GFB_EW(OPC, HB) launch_pdl(ew_vec_kernel<T, OPC, HB>, blocks, kThreads, 0, st, c, a, b, out, nv, accumulate, err)
  if (!b) {
    if (op == GFB_OP_IN) GFB_EW(GFB_OP_IN, false);
    else if (op == GFB_OP_MUL) GFB_EW(-1, false);
    else if (op == GFB_OP_EXP) GFB_EW(GFB_OP_EXP, false);
    else return false;
  } else {
    if (op == GFB_OP_ADD) GFB_EW(GFB_OP_ADD, true);
    else if (op == GFB_OP_SUB) GFB_EW(GFB_OP_SUB, true);
    else if (op == GFB_OP_MUL) GFB_EW(GFB_OP_MUL, true);
    else if (op == GFB_OP_DIV) GFB_EW(GFB_OP_DIV, true);
    else return false;
  }
#undef GFB_EW
  return true;
}

template <typename T>
__global__ void __launch_bounds__(kThreads) broadcast_kernel(const void *src, int32_t src_dtype, double scale,
                                                             T *out, int64_t n, int accumulate) {
  pdl_wait();  // programmatic dependent launch: global memory after the wait
  PdlRelease pdl_release_;
  double v = scale;
  if (src) v *= (src_dtype == GFB_F64 ? *(const double *)src : (double)*(const float *)src);
  const T tv = (T)v;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  const int64_t t0 = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  int64_t done = 0;
  if ((reinterpret_cast<uintptr_t>(out) & 15) == 0) {  // 16-byte stores
    using V = typename EwVec<T>::V;
    constexpr int W = EwVec<T>::W;
    const int64_t nv = n / W;
    V *ov = reinterpret_cast<V *>(out);
    for (int64_t i = t0; i < nv; i += stride) {
      V o = accumulate ? ov[i] : V{};
      T *os = reinterpret_cast<T *>(&o);
#pragma unroll
      for (int w = 0; w < W; ++w) os[w] = accumulate ? (T)(os[w] + tv) : tv;
      ov[i] = o;
    }
    done = nv * W;
  }
  for (int64_t i = done + t0; i < n; i += stride) out[i] = accumulate ? (T)(out[i] + tv) : tv;
}

template <typename T>
__global__ void __launch_bounds__(kThreads) fill_box_kernel(T *dst, int64_t d1, int64_t d2, int64_t lo0,
                                                            int64_t lo1, int64_t lo2, int64_t e0, int64_t e1,
                                                            int64_t e2, T value) {
  pdl_wait();  // programmatic dependent launch: global memory after the wait
  PdlRelease pdl_release_;
  const int64_t total = e0 * e1 * e2;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  for (int64_t f = (int64_t)blockIdx.x * kThreads + threadIdx.x; f < total; f += stride) {
    int64_t k = f % e2, r = f / e2;
    int64_t j = r % e1, i = r / e1;
    dst[((lo0 + i) * d1 + (lo1 + j)) * d2 + (lo2 + k)] = value;
  }
}

}  // namespace gfb

using namespace gfb;

extern "C" int64_t gfb_reduce_workspace_bytes(int64_t n) { return reduce_blocks(n) * 8; }

extern "C" int gfb_reduce_sum(const void *x, int32_t xdtype, int64_t n, void *out, int32_t odtype,
                              int32_t accumulate, void *workspace, void *stream) {
  if (!out || (!x && n > 0) || !workspace) return set_error(GFB_EINVAL, "gfb_reduce_sum: null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  int64_t nb = reduce_blocks(n);
  double *part = (double *)workspace;
  if (n > 0 && nb == 1) {
#define GFB_RS(TI, TO) launch_pdl(reduce_single<TI, TO>, 1, kThreads, 0, st, (const TI *)x, n, (TO *)out, accumulate)
    if (xdtype == GFB_F64) {
      if (odtype == GFB_F64) GFB_RS(double, double); else GFB_RS(double, float);
    } else {
      if (odtype == GFB_F64) GFB_RS(float, double); else GFB_RS(float, float);
    }
#undef GFB_RS
    return check_launch("reduce_sum");
  }
  if (n <= 0) {
    nb = 1;
    cudaMemsetAsync(part, 0, 8, st);
  } else if (xdtype == GFB_F64) {
    launch_pdl(reduce_pass1<double>, (unsigned)nb, kThreads, 0, st, (const double *)x, n, part);
  } else {
    launch_pdl(reduce_pass1<float>, (unsigned)nb, kThreads, 0, st, (const float *)x, n, part);
  }
  if (odtype == GFB_F64)
    launch_pdl(reduce_pass2<double>, 1, kThreads, 0, st, part, nb, (double *)out, accumulate);
  else
    launch_pdl(reduce_pass2<float>, 1, kThreads, 0, st, part, nb, (float *)out, accumulate);
  return check_launch("reduce_sum");
}

extern "C" int gfb_elementwise(int32_t op, double c, const void *a, int64_t n_a, const void *b, int64_t n_b,
                               void *out, int64_t n, int32_t dtype, int32_t accumulate, uint32_t *err,
                               void *stream) {
  if (n <= 0) return GFB_OK;
  if (!a || !out) return set_error(GFB_EINVAL, "gfb_elementwise: null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == GFB_F64 ? ew_vec_launch<double>(op, c, (const double *)a, n_a, (const double *)b, n_b,
                                               (double *)out, n, accumulate, err, st)
                       : ew_vec_launch<float>(op, (float)c, (const float *)a, n_a, (const float *)b, n_b,
                                              (float *)out, n, accumulate, err, st))
    return check_launch("elementwise");
  unsigned blocks = (unsigned)stream_blocks(n, 4);
  if (dtype == GFB_F64)
    launch_pdl(ew_kernel<double>, blocks, kThreads, 0, st, op, c, (const double *)a, n_a, (const double *)b, n_b,
                                                   (double *)out, n, accumulate, err);
  else
    launch_pdl(ew_kernel<float>, blocks, kThreads, 0, st, op, (float)c, (const float *)a, n_a, (const float *)b, n_b,
                                                  (float *)out, n, accumulate, err);
  return check_launch("elementwise");
}

extern "C" int gfb_broadcast(const void *src, int32_t src_dtype, double scale, void *out, int64_t n,
                             int32_t dtype, int32_t accumulate, void *stream) {
  if (n <= 0) return GFB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned blocks = (unsigned)stream_blocks(n, 4);
  if (dtype == GFB_F64)
    launch_pdl(broadcast_kernel<double>, blocks, kThreads, 0, st, src, src_dtype, scale, (double *)out, n, accumulate);
  else
    launch_pdl(broadcast_kernel<float>, blocks, kThreads, 0, st, src, src_dtype, scale, (float *)out, n, accumulate);
  return check_launch("broadcast");
}

extern "C" int gfb_fill_box(void *dst, int32_t dtype, int32_t rank, const int64_t *dims, const int64_t *lo,
                            const int64_t *hi, double value, void *stream) {
  if (rank < 0 || rank > 3) return set_error(GFB_EUNSUPPORTED, "gfb_fill_box: rank > 3");
  int64_t D[3] = {1, 1, 1}, L[3] = {0, 0, 0}, E[3] = {1, 1, 1};
  for (int r = 0; r < rank; ++r) {
    int k = 3 - rank + r;
    D[k] = dims[r];
    L[k] = lo[r];
    E[k] = hi[r] - lo[r];
    if (E[k] <= 0) return GFB_OK;
  }
  int64_t total = E[0] * E[1] * E[2];
  cudaStream_t st = (cudaStream_t)stream;
  unsigned blocks = (unsigned)stream_blocks(total, 4);
  if (dtype == GFB_F64)
    launch_pdl(fill_box_kernel<double>, blocks, kThreads, 0, st, (double *)dst, D[1], D[2], L[0], L[1], L[2], E[0], E[1],
                                                         E[2], value);
  else
    launch_pdl(fill_box_kernel<float>, blocks, kThreads, 0, st, (float *)dst, D[1], D[2], L[0], L[1], L[2], E[0], E[1],
                                                        E[2], (float)value);
  return check_launch("fill_box");
}
