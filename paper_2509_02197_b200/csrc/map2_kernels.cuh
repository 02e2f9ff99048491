// Vectorised map kernels (gfb.h, gfb_map2_desc): device templates shared by
// the bytecode instantiation (map2.cu) and the ahead-of-time compiled tasklet
// bodies (gen_tasklets.cu).
//
// Replaces the per-point interpretation of MapNode bodies (Executor.
// _exec_map / _exec_tasklet, interpreter.py:478-507, :405-426) for
// rectangular spaces:
//  * the host folds the box into loop dimensions and merges adjacent ones,
//    so a warp decomposes its row index once and walks the innermost
//    dimension with plain int32 strides;
//  * the bytecode carries its static stack depth, so the evaluation stack
//    lives in registers: every instruction is one uniform two-level switch
//    (depth, opcode) whose cases touch compile-time register slots, applied
//    to V points per lane; generated bodies skip the dispatch entirely;
//  * warp-coalesced operands: lane l of a warp owns points l + 32 v.
#pragma once

#include <algorithm>
#include <type_traits>

#include "gfb_common.cuh"
#include "gfb_internal.h"

namespace gfb {

constexpr int kM2Depth = GFB_M2_DEPTH;
constexpr int kM2Warps = 8;  // 256-thread CTAs
constexpr int kM2Bases = GFB_MAX_INPUTS + GFB_M2_OUTS;

template <typename T, int V>
__device__ __forceinline__ void m2_unary(int op, T (&x)[V], uint32_t vm, uint32_t &bad) {
  switch (op) {
    case GFB_OP_NEG:
#pragma unroll
      for (int v = 0; v < V; ++v) x[v] = -x[v];
      break;
    case GFB_OP_SIN:
#pragma unroll
      for (int v = 0; v < V; ++v) x[v] = t_sin(x[v]);
      break;
    case GFB_OP_COS:
#pragma unroll
      for (int v = 0; v < V; ++v) x[v] = t_cos(x[v]);
      break;
    case GFB_OP_EXP:
#pragma unroll
      for (int v = 0; v < V; ++v) x[v] = t_exp(x[v]);
      break;
    case GFB_OP_LOG:
#pragma unroll
      for (int v = 0; v < V; ++v) {
        if (((vm >> v) & 1) && !(x[v] > T(0))) bad |= GFB_EBIT_LOG;
        x[v] = t_log(x[v]);
      }
      break;
    case GFB_OP_SQRT:
#pragma unroll
      for (int v = 0; v < V; ++v) {
        if (((vm >> v) & 1) && x[v] < T(0)) bad |= GFB_EBIT_SQRT;
        x[v] = sqrt(x[v]);
      }
      break;
    case GFB_OP_TANH:
#pragma unroll
      for (int v = 0; v < V; ++v) x[v] = t_tanh(x[v]);
      break;
    case GFB_OP_ABS:
#pragma unroll
      for (int v = 0; v < V; ++v) x[v] = fabs(x[v]);
      break;
    case GFB_OP_SIGN:
#pragma unroll
      for (int v = 0; v < V; ++v)
        x[v] = x[v] > T(0) ? T(1) : (x[v] < T(0) ? T(-1) : (x[v] == T(0) ? T(0) : x[v]));
      break;
    default:
      break;
  }
}

template <typename T, int V>
__device__ __forceinline__ void m2_binary(int op, T (&a)[V], const T (&b)[V], uint32_t vm, uint32_t &bad) {
  switch (op) {
    case GFB_OP_ADD:
#pragma unroll
      for (int v = 0; v < V; ++v) a[v] = a[v] + b[v];
      break;
    case GFB_OP_SUB:
#pragma unroll
      for (int v = 0; v < V; ++v) a[v] = a[v] - b[v];
      break;
    case GFB_OP_MUL:
#pragma unroll
      for (int v = 0; v < V; ++v) a[v] = a[v] * b[v];
      break;
    case GFB_OP_DIV:
#pragma unroll
      for (int v = 0; v < V; ++v) {
        if (((vm >> v) & 1) && b[v] == T(0)) bad |= GFB_EBIT_DIV0;
        a[v] = a[v] / b[v];
      }
      break;
    case GFB_OP_IDIV:
#pragma unroll
      for (int v = 0; v < V; ++v) {
        if (((vm >> v) & 1) && b[v] == T(0)) bad |= GFB_EBIT_IDIV0;
        a[v] = np_floordiv(a[v], b[v]);
      }
      break;
    case GFB_OP_MOD:
#pragma unroll
      for (int v = 0; v < V; ++v) {
        if (((vm >> v) & 1) && b[v] == T(0)) bad |= GFB_EBIT_MOD0;
        a[v] = np_mod(a[v], b[v]);
      }
      break;
    case GFB_OP_MIN:
#pragma unroll
      for (int v = 0; v < V; ++v) a[v] = b[v] < a[v] ? b[v] : a[v];
      break;
    case GFB_OP_MAX:
#pragma unroll
      for (int v = 0; v < V; ++v) a[v] = b[v] > a[v] ? b[v] : a[v];
      break;
    case GFB_OP_POW:
#pragma unroll
      for (int v = 0; v < V; ++v) {
        if ((vm >> v) & 1) {
          if (a[v] == T(0) && b[v] < T(0)) bad |= GFB_EBIT_POW;
          if (a[v] < T(0) && b[v] != floor(b[v])) bad |= GFB_EBIT_POW;
        }
        a[v] = t_pow(a[v], b[v]);
      }
      break;
    default:
      break;
  }
}

// error bits are collected for valid points only (masked-off lanes evaluate
// on placeholder values) and raised once per evaluation

template <typename T, int V, int D, typename F>
__device__ __forceinline__ void m2_step(int op, int arg, T (&s)[kM2Depth][V], const double *consts, F &fetch,
                                        uint32_t vm, uint32_t &bad) {
  if (op == GFB_OP_IN) {
    if constexpr (D < kM2Depth) fetch(arg, s[D]);
  } else if (op == GFB_OP_CONST) {
    if constexpr (D < kM2Depth) {
      const T c = (T)consts[arg];
#pragma unroll
      for (int v = 0; v < V; ++v) s[D][v] = c;
    }
  } else if (op >= GFB_OP_NEG) {
    if constexpr (D >= 1 && D <= kM2Depth) m2_unary<T, V>(op, s[D - 1], vm, bad);
  } else {
    if constexpr (D >= 2 && D <= kM2Depth) m2_binary<T, V>(op, s[D - 2], s[D - 1], vm, bad);
  }
}

template <typename T, int V, typename F>
__device__ __forceinline__ void m2_eval(const gfb_map2_desc &d, int start, int len, F &fetch, uint32_t vm,
                                        T (&res)[V]) {
  T s[kM2Depth][V];
  uint32_t bad = 0;
  for (int pc = start; pc < start + len; ++pc) {
    const uint32_t ins = d.code[pc];
    const int op = (int)(ins & 63u), dep = (int)((ins >> 6) & 15u), arg = (int)(ins >> 10);
    switch (dep) {
      case 0: m2_step<T, V, 0>(op, arg, s, d.consts, fetch, vm, bad); break;
      case 1: m2_step<T, V, 1>(op, arg, s, d.consts, fetch, vm, bad); break;
      case 2: m2_step<T, V, 2>(op, arg, s, d.consts, fetch, vm, bad); break;
      case 3: m2_step<T, V, 3>(op, arg, s, d.consts, fetch, vm, bad); break;
      case 4: m2_step<T, V, 4>(op, arg, s, d.consts, fetch, vm, bad); break;
      case 5: m2_step<T, V, 5>(op, arg, s, d.consts, fetch, vm, bad); break;
      default: m2_step<T, V, 6>(op, arg, s, d.consts, fetch, vm, bad); break;
    }
  }
  if (bad) raise_bits(d.err, bad);
#pragma unroll
  for (int v = 0; v < V; ++v) res[v] = s[0][v];
}

// Loads of input k at the item's points on demand (the body's IN); masked-
// off points read 1. at(k, v): int32 element offset of operand k at point v
// (the host only routes spaces whose offsets fit in int32 here).
template <typename T, int V, typename At>
struct M2Fetch {
  const gfb_map2_desc &d;
  At &at;
  uint32_t vm;
  __device__ __forceinline__ void operator()(int k, T (&dst)[V]) const {
    const gfb_m2_operand &o = d.in[k];
    if (o.dtype == GFB_F64) {
      const double *p = (const double *)o.base;
#pragma unroll
      for (int v = 0; v < V; ++v) dst[v] = ((vm >> v) & 1) ? (T)p[at(k, v)] : T(1);
    } else {
      const float *p = (const float *)o.base;
#pragma unroll
      for (int v = 0; v < V; ++v) dst[v] = ((vm >> v) & 1) ? (T)p[at(k, v)] : T(1);
    }
  }
};

// Per-warp row bases (nd > 2): lane k < n_in + n_out computes operand k's
// offset of the row (all coordinates but the innermost), then the warp syncs.
__device__ __forceinline__ void m2_row_bases(const gfb_map2_desc &d, int32_t row, int lane, int32_t *sb) {
  __syncwarp();
  if (lane < d.n_in + d.n_out) {
    const gfb_m2_operand &o = lane < d.n_in ? d.in[lane] : d.out[lane - d.n_in];
    int32_t rem = row, off = (int32_t)o.c0;
    for (int dd = d.ndim - 2; dd >= 0; --dd) {
      const int32_t e = (int32_t)d.ext[dd];
      const int32_t k = rem % e;
      rem /= e;
      off += (int32_t)o.s[dd] * k;
    }
    sb[lane] = off;
  }
  __syncwarp();
}

__device__ __forceinline__ bool m2_row_in_clear(const gfb_map2_desc &d, int32_t row) {
  int32_t rem = row;
  bool in = true;
  for (int dd = d.ndim - 2; dd >= 0; --dd) {
    const int32_t e = (int32_t)d.ext[dd];
    const int32_t k = rem % e;
    rem /= e;
    in &= k >= d.clear_lo[dd] && k < d.clear_hi[dd];
  }
  return in;
}

template <typename T>
__device__ __forceinline__ T m2_base(const gfb_map2_desc &d, bool inside, int32_t off) {
  if (d.clear_mode == 1 || d.clear_mode == 3 || (d.clear_mode == 2 && inside)) return T(0);
  return load_as<T>(const_cast<void *>(d.out[0].base), d.out[0].dtype, off);
}

__device__ __forceinline__ const gfb_m2_operand &m2_op(const gfb_map2_desc &d, int k) {
  return k < d.n_in ? d.in[k] : d.out[k - d.n_in];
}

// Body policies: VmBody interprets the bytecode; generated bodies
// (gen_tasklets.cu) are the same tasklets compiled ahead of time.
struct VmBody {
  template <typename T, int V, typename F>
  static __device__ __forceinline__ void eval(const gfb_map2_desc &d, int o, F &fetch, uint32_t vm, T (&r)[V]) {
    m2_eval<T, V>(d, d.code_start[o], d.code_len[o], fetch, vm, r);
  }
};

// evaluate every output at the item's points and store them
template <typename T, int V, typename Body, typename At>
__device__ __forceinline__ void m2_points(const gfb_map2_desc &d, At &at, uint32_t vm) {
  M2Fetch<T, V, At> fetch{d, at, vm};
  for (int o = 0; o < d.n_out; ++o) {
    T r[V];
    Body::template eval<T, V>(d, o, fetch, vm, r);
    const gfb_m2_operand &wo = d.out[o];
    const int k = d.n_in + o;
    if (wo.dtype == GFB_F64) {
      double *p = (double *)wo.base;
#pragma unroll
      for (int v = 0; v < V; ++v)
        if ((vm >> v) & 1) p[at(k, v)] = d.wcr[o] ? p[at(k, v)] + (double)r[v] : (double)r[v];
    } else {
      float *p = (float *)wo.base;
#pragma unroll
      for (int v = 0; v < V; ++v)
        if ((vm >> v) & 1) p[at(k, v)] = d.wcr[o] ? p[at(k, v)] + (float)r[v] : (float)r[v];
    }
  }
}

// LAYOUT 0: ndim == 2, warp item = (row, 32*V points of the row)
// LAYOUT 1: ndim == 2 with a short row: warp item = 32*V consecutive points
//           of the flattened space, row = point / E by a multiply-shift
// LAYOUT 2: ndim > 2, row bases staged per warp in shared memory
template <typename T, int V, int LAYOUT, typename Body>
__global__ void __launch_bounds__(256) map2_pointwise_kernel(const __grid_constant__ gfb_map2_desc d, int32_t rows,
                                                             int32_t cpr, uint64_t magic) {
  pdl_wait();  // programmatic dependent launch: global memory after the wait
  PdlRelease pdl_release_;
  __shared__ int32_t sbase[kM2Warps][kM2Bases];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nd = d.ndim;
  const int32_t E = (int32_t)d.ext[nd - 1];
  const int32_t total = rows * E;
  const int32_t items = LAYOUT == 1 ? (int32_t)ceil_div(total, 32 * V) : rows * cpr;
  int32_t *sb = sbase[w];
  for (int32_t it = blockIdx.x * kM2Warps + w; it < items; it += gridDim.x * kM2Warps) {
    if (LAYOUT == 1) {
      int32_t rw[V], cl[V];
      uint32_t vm = 0;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int32_t f = it * 32 * V + lane + 32 * v;
        vm |= (uint32_t)(f < total) << v;
        rw[v] = (int32_t)(((uint64_t)(uint32_t)f * magic) >> 40);
        cl[v] = f - rw[v] * E;
      }
      auto at = [&](int k, int v) -> int32_t {
        const gfb_m2_operand &o = m2_op(d, k);
        return (int32_t)o.c0 + (int32_t)o.s[0] * rw[v] + (int32_t)o.s[1] * cl[v];
      };
      m2_points<T, V, Body>(d, at, vm);
    } else {
      const int32_t row = cpr == 1 ? it : it / cpr, chunk = it - row * cpr;
      if (LAYOUT == 2) m2_row_bases(d, row, lane, sb);
      const int32_t i0 = chunk * 32 * V + lane;
      uint32_t vm = 0;
#pragma unroll
      for (int v = 0; v < V; ++v) vm |= (uint32_t)(i0 + 32 * v < E) << v;
      auto at = [&](int k, int v) -> int32_t {
        const gfb_m2_operand &o = m2_op(d, k);
        const int32_t si = (int32_t)o.s[LAYOUT == 0 ? 1 : nd - 1];
        const int32_t rb = LAYOUT == 0 ? (int32_t)o.c0 + (int32_t)o.s[0] * row : sb[k];
        return rb + si * i0 + v * (32 * si);
      };
      m2_points<T, V, Body>(d, at, vm);
    }
  }
}

template <typename T, int V, bool ROW1, typename Body>
__global__ void __launch_bounds__(256) map2_reduce_inner_kernel(const __grid_constant__ gfb_map2_desc d,
                                                                int32_t rows) {
  pdl_wait();  // programmatic dependent launch: global memory after the wait
  PdlRelease pdl_release_;
  __shared__ int32_t sbase[kM2Warps][kM2Bases];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nd = d.ndim;
  const int32_t E = (int32_t)d.ext[nd - 1];
  int32_t *sb = sbase[w];
  for (int32_t row = blockIdx.x * kM2Warps + w; row < rows; row += gridDim.x * kM2Warps) {
    if (!ROW1) m2_row_bases(d, row, lane, sb);
    auto rowbase = [&](int k) -> int32_t {
      const gfb_m2_operand &o = m2_op(d, k);
      return ROW1 ? (int32_t)o.c0 + (int32_t)o.s[0] * row : sb[k];
    };
    T acc = T(0);
    for (int32_t c0 = 0; c0 < E; c0 += 32 * V) {
      const int32_t i0 = c0 + lane;
      uint32_t vm = 0;
#pragma unroll
      for (int v = 0; v < V; ++v) vm |= (uint32_t)(i0 + 32 * v < E) << v;
      auto at = [&](int k, int v) -> int32_t {
        const int32_t si = (int32_t)m2_op(d, k).s[ROW1 ? 1 : nd - 1];
        return rowbase(k) + si * i0 + v * (32 * si);
      };
      M2Fetch<T, V, decltype(at)> fetch{d, at, vm};
      T r[V];
      Body::template eval<T, V>(d, 0, fetch, vm, r);
#pragma unroll
      for (int v = 0; v < V; ++v)
        if ((vm >> v) & 1) acc += r[v];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      const int32_t off = rowbase(d.n_in);
      const bool inside = d.clear_mode == 2 ? m2_row_in_clear(d, row) : true;
      store_as<T>(const_cast<void *>(d.out[0].base), d.out[0].dtype, off, m2_base<T>(d, inside, off) + acc);
    }
  }
}

// column sums: lane = column, V rows per warp iteration (V loads in flight)
template <typename T, int V, typename Body>
__global__ void __launch_bounds__(256) map2_reduce_outer_kernel(const __grid_constant__ gfb_map2_desc d) {
  pdl_wait();  // programmatic dependent launch: global memory after the wait
  PdlRelease pdl_release_;
  __shared__ T red[kM2Warps][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int32_t R = (int32_t)d.ext[0], E = (int32_t)d.ext[1];
  const int s = blockIdx.y, ns = d.nsplit;
  const int32_t rb = (int32_t)((int64_t)R * s / ns), re = (int32_t)((int64_t)R * (s + 1) / ns);
  const int32_t i = blockIdx.x * 32 + lane;
  T acc = T(0);
  for (int32_t r = rb + w * V; r < re; r += kM2Warps * V) {
    uint32_t vm = 0;
#pragma unroll
    for (int v = 0; v < V; ++v) vm |= (uint32_t)(i < E && r + v < re) << v;
    auto at = [&](int k, int v) -> int32_t {
      const gfb_m2_operand &o = m2_op(d, k);
      return (int32_t)o.c0 + (int32_t)o.s[0] * (r + v) + (int32_t)o.s[1] * i;
    };
    M2Fetch<T, V, decltype(at)> fetch{d, at, vm};
    T x[V];
    Body::template eval<T, V>(d, 0, fetch, vm, x);
#pragma unroll
    for (int v = 0; v < V; ++v)
      if ((vm >> v) & 1) acc += x[v];
  }
  red[w][lane] = acc;
  __syncthreads();
  if (w != 0 || i >= E) return;
  T sum = T(0);
  for (int ww = 0; ww < kM2Warps; ++ww) sum += red[ww][lane];
  if (ns > 1) {
    ((double *)d.workspace)[(int64_t)s * E + i] = (double)sum;
  } else {
    const gfb_m2_operand &wo = d.out[0];
    const int32_t off = (int32_t)wo.c0 + (int32_t)wo.s[1] * i;
    const bool inside = i >= d.clear_lo[1] && i < d.clear_hi[1];
    store_as<T>(const_cast<void *>(wo.base), wo.dtype, off, m2_base<T>(d, inside, off) + sum);
  }
}

template <typename T>
__global__ void __launch_bounds__(1024) map2_finish_kernel(const __grid_constant__ gfb_map2_desc d) {
  pdl_wait();  // programmatic dependent launch: global memory after the wait
  PdlRelease pdl_release_;
  // 32 columns x 32 split groups per CTA: group g sums splits g, g + 32, ...
  // (a few L2 round trips per thread instead of nsplit), then the groups are
  // added in order (deterministic)
  __shared__ double red[32][33];
  const int32_t E = (int32_t)d.ext[1];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int32_t i = blockIdx.x * 32 + lane;
  const double *ws = (const double *)d.workspace;
  double s4[4] = {0.0, 0.0, 0.0, 0.0};
  if (i < E) {
    int s = g;
    for (; s + 96 < d.nsplit; s += 128) {
#pragma unroll
      for (int u = 0; u < 4; ++u) s4[u] += ws[(int64_t)(s + 32 * u) * E + i];
    }
    for (; s < d.nsplit; s += 32) s4[0] += ws[(int64_t)s * E + i];
  }
  red[g][lane] = (s4[0] + s4[1]) + (s4[2] + s4[3]);
  __syncthreads();
  if (g != 0 || i >= E) return;
  double sum = 0.0;
#pragma unroll
  for (int q = 0; q < 32; ++q) sum += red[q][lane];
  const gfb_m2_operand &wo = d.out[0];
  const int32_t off = (int32_t)wo.c0 + (int32_t)wo.s[1] * i;
  const bool inside = i >= d.clear_lo[1] && i < d.clear_hi[1];
  store_as<T>(const_cast<void *>(wo.base), wo.dtype, off, m2_base<T>(d, inside, off) + (T)sum);
}

// 16-byte variant (fp32, two loop dimensions, inner strides 0 or 1, host-
// checked alignment): lane l owns the four consecutive points 4l..4l+3 of a
// 128-point chunk, so a stride-1 operand is one float4 load / store and a
// stride-0 operand (broadcast along the row) one scalar load.
struct M2FetchVec4 {
  const gfb_map2_desc &d;
  int32_t row, i0;
  uint32_t vm;
  __device__ __forceinline__ void operator()(int k, float (&dst)[4]) const {
    const gfb_m2_operand &o = d.in[k];
    const float *p = (const float *)o.base + ((int32_t)o.c0 + (int32_t)o.s[0] * row);
    if (!vm) {
      dst[0] = dst[1] = dst[2] = dst[3] = 1.f;
    } else if (o.s[1] == 0) {
      dst[0] = dst[1] = dst[2] = dst[3] = p[0];
    } else {
      const float4 q = *reinterpret_cast<const float4 *>(p + i0);
      dst[0] = q.x, dst[1] = q.y, dst[2] = q.z, dst[3] = q.w;
    }
  }
};

// FLAT: rows shorter than 128 points; a warp item is 128 consecutive points
// of the flattened space and each lane finds its own (row, column)
template <typename Body, bool FLAT>
__global__ void __launch_bounds__(256) map2_pointwise_vec4_kernel(const __grid_constant__ gfb_map2_desc d,
                                                                  int32_t rows, int32_t cpr) {
  pdl_wait();  // programmatic dependent launch: global memory after the wait
  PdlRelease pdl_release_;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int32_t E = (int32_t)d.ext[1];
  const int32_t items = FLAT ? (int32_t)ceil_div((int64_t)rows * E, 128) : rows * cpr;
  for (int32_t it = blockIdx.x * kM2Warps + w; it < items; it += gridDim.x * kM2Warps) {
    int32_t row, i0;
    uint32_t vm;
    if (FLAT) {
      const int32_t f = it * 128 + lane * 4;
      row = f / E;
      i0 = f - row * E;
      vm = row < rows ? 0xFu : 0u;
    } else {
      row = cpr == 1 ? it : it / cpr;
      i0 = (it - row * cpr) * 128 + lane * 4;
      vm = i0 < E ? 0xFu : 0u;
    }
    M2FetchVec4 fetch{d, row, i0, vm};
    for (int o = 0; o < d.n_out; ++o) {
      float r[4];
      Body::template eval<float, 4>(d, o, fetch, vm, r);
      if (!vm) continue;
      const gfb_m2_operand &wo = d.out[o];
      float *p = (float *)wo.base + ((int32_t)wo.c0 + (int32_t)wo.s[0] * row + i0);
      float4 v = make_float4(r[0], r[1], r[2], r[3]);
      if (d.wcr[o]) {
        const float4 a = *reinterpret_cast<const float4 *>(p);
        v.x += a.x, v.y += a.y, v.z += a.z, v.w += a.w;
      }
      *reinterpret_cast<float4 *>(p) = v;
    }
  }
}

template <typename Body>
__global__ void __launch_bounds__(256) map2_reduce_inner_vec4_kernel(const __grid_constant__ gfb_map2_desc d,
                                                                     int32_t rows) {
  pdl_wait();  // programmatic dependent launch: global memory after the wait
  PdlRelease pdl_release_;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int32_t E = (int32_t)d.ext[1];
  for (int32_t row = blockIdx.x * kM2Warps + w; row < rows; row += gridDim.x * kM2Warps) {
    float acc = 0.f;
    for (int32_t c0 = 0; c0 < E; c0 += 128) {
      const int32_t i0 = c0 + lane * 4;
      const uint32_t vm = i0 < E ? 0xFu : 0u;
      M2FetchVec4 fetch{d, row, i0, vm};
      float r[4];
      Body::template eval<float, 4>(d, 0, fetch, vm, r);
      if (vm) acc += (r[0] + r[1]) + (r[2] + r[3]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      const gfb_m2_operand &wo = d.out[0];
      const int32_t off = (int32_t)wo.c0 + (int32_t)wo.s[0] * row;
      const bool inside = d.clear_mode == 2 ? (row >= d.clear_lo[0] && row < d.clear_hi[0]) : true;
      store_as<float>(const_cast<void *>(wo.base), wo.dtype, off, m2_base<float>(d, inside, off) + acc);
    }
  }
}

// Prefetched operands of one vec4 item. Generated bodies fetch with
// constant input indices, so after inlining these are plain registers: the
// ILP kernels below load every input of U items before evaluating any of
// them (a warp has U items of HBM latency in flight instead of one).
constexpr int kM2CacheIn = 4;
struct M2Cached {
  const float (&c)[kM2CacheIn][4];
  __device__ __forceinline__ void operator()(int k, float (&dst)[4]) const {
#pragma unroll
    for (int j = 0; j < 4; ++j) dst[j] = c[k][j];
  }
};

// the inputs of U items for a generated body: input count and which inputs
// are row scalars (stride 0 along the row on the 16-byte paths) are
// compile-time, so the loads of all items of one input issue back to back
template <typename Body, int U>
__device__ __forceinline__ void m2_prefetch_static(const gfb_map2_desc &d, const int32_t (&row)[U],
                                                   const int32_t (&i0)[U], const uint32_t (&vm)[U],
                                                   float (&c)[U][kM2CacheIn][4]) {
  static_assert(Body::kNIn <= kM2CacheIn, "generated ILP bodies take at most four inputs");
#pragma unroll
  for (int k = 0; k < Body::kNIn; ++k) {
    const gfb_m2_operand &o = d.in[k];
    const float *base = (const float *)o.base + (int32_t)o.c0;
    const int32_t s0 = (int32_t)o.s[0];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float *p = base + s0 * row[u];
      if (!vm[u]) {
        c[u][k][0] = c[u][k][1] = c[u][k][2] = c[u][k][3] = 1.f;
      } else if ((Body::kRowScalar >> k) & 1u) {
        c[u][k][0] = c[u][k][1] = c[u][k][2] = c[u][k][3] = p[0];
      } else {
        const float4 q = *reinterpret_cast<const float4 *>(p + i0[u]);
        c[u][k][0] = q.x, c[u][k][1] = q.y, c[u][k][2] = q.z, c[u][k][3] = q.w;
      }
    }
  }
}

// pointwise, U warp items per iteration (generated bodies, n_in <= 4)
template <typename Body, bool FLAT, int U>
__global__ void __launch_bounds__(256) map2_pointwise_ilp_kernel(const __grid_constant__ gfb_map2_desc d,
                                                                 int32_t rows, int32_t cpr, uint64_t magic) {
  pdl_wait();  // programmatic dependent launch: global memory after the wait
  PdlRelease pdl_release_;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int32_t E = (int32_t)d.ext[1];
  const int32_t items = FLAT ? (int32_t)ceil_div((int64_t)rows * E, 128) : rows * cpr;
  for (int32_t it0 = (blockIdx.x * kM2Warps + w) * U; it0 < items; it0 += gridDim.x * kM2Warps * U) {
    int32_t row[U], i0[U];
    uint32_t vm[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int32_t it = it0 + u;
      if (FLAT) {
        const int32_t f = it * 128 + lane * 4;
        // f / E by a precomputed multiplier (exact for f < 2^24, E < 128)
        row[u] = (int32_t)(((uint64_t)(uint32_t)f * magic) >> 40);
        i0[u] = f - row[u] * E;
        vm[u] = (it < items && row[u] < rows) ? 0xFu : 0u;
      } else {
        row[u] = cpr == 1 ? it : it / cpr;
        i0[u] = (it - row[u] * cpr) * 128 + lane * 4;
        vm[u] = (it < items && i0[u] < E) ? 0xFu : 0u;
      }
    }
    float c[U][kM2CacheIn][4];
    m2_prefetch_static<Body, U>(d, row, i0, vm, c);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      M2Cached fetch{c[u]};
#pragma unroll
      for (int o = 0; o < Body::kNOut; ++o) {
        float r[4];
        Body::template eval<float, 4>(d, o, fetch, vm[u], r);
        if (!vm[u]) continue;
        const gfb_m2_operand &wo = d.out[o];
        float *p = (float *)wo.base + ((int32_t)wo.c0 + (int32_t)wo.s[0] * row[u] + i0[u]);
        float4 v = make_float4(r[0], r[1], r[2], r[3]);
        if (d.wcr[o]) {
          const float4 a = *reinterpret_cast<const float4 *>(p);
          v.x += a.x, v.y += a.y, v.z += a.z, v.w += a.w;
        }
        *reinterpret_cast<float4 *>(p) = v;
      }
    }
  }
}

// row sums of rows of at most 128 points, U rows per warp iteration
template <typename Body, int U>
__global__ void __launch_bounds__(256) map2_reduce_row_ilp_kernel(const __grid_constant__ gfb_map2_desc d,
                                                                  int32_t rows) {
  pdl_wait();  // programmatic dependent launch: global memory after the wait
  PdlRelease pdl_release_;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int32_t E = (int32_t)d.ext[1];
  for (int32_t r0 = (blockIdx.x * kM2Warps + w) * U; r0 < rows; r0 += gridDim.x * kM2Warps * U) {
    int32_t row[U], i0[U];
    uint32_t vm[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      row[u] = r0 + u;
      i0[u] = lane * 4;
      vm[u] = (row[u] < rows && i0[u] < E) ? 0xFu : 0u;
    }
    float c[U][kM2CacheIn][4];
    m2_prefetch_static<Body, U>(d, row, i0, vm, c);
    float acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      M2Cached fetch{c[u]};
      float r[4];
      Body::template eval<float, 4>(d, 0, fetch, vm[u], r);
      acc[u] = vm[u] ? (r[0] + r[1]) + (r[2] + r[3]) : 0.f;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int u = 0; u < U; ++u) acc[u] += __shfl_down_sync(0xffffffffu, acc[u], o);
    if (lane == 0) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (row[u] >= rows) continue;
        const gfb_m2_operand &wo = d.out[0];
        const int32_t off = (int32_t)wo.c0 + (int32_t)wo.s[0] * row[u];
        const bool inside = d.clear_mode == 2 ? (row[u] >= d.clear_lo[0] && row[u] < d.clear_hi[0]) : true;
        store_as<float>(const_cast<void *>(wo.base), wo.dtype, off, m2_base<float>(d, inside, off) + acc[u]);
      }
    }
  }
}

// column sums (mode 2) with 16-byte column quads: a warp instruction covers
// 32 / qpr rows x qpr quads (qpr = quads per row slice, a power of two
// <= 32), four row groups in flight per iteration; lanes holding the same
// quad combine by shuffles, warps through shared memory
struct M2FetchVec4Row {
  const gfb_map2_desc &d;
  int32_t row, col;
  uint32_t vm;
  __device__ __forceinline__ void operator()(int k, float (&dst)[4]) const {
    const gfb_m2_operand &o = d.in[k];
    const float *p = (const float *)o.base + ((int32_t)o.c0 + (int32_t)o.s[0] * row);
    if (!vm) {
      dst[0] = dst[1] = dst[2] = dst[3] = 1.f;
    } else if (o.s[1] == 0) {
      dst[0] = dst[1] = dst[2] = dst[3] = p[0];
    } else {
      const float4 q = *reinterpret_cast<const float4 *>(p + col);
      dst[0] = q.x, dst[1] = q.y, dst[2] = q.z, dst[3] = q.w;
    }
  }
};

template <typename Body>
__global__ void __launch_bounds__(256) map2_reduce_outer_vec4_kernel(const __grid_constant__ gfb_map2_desc d,
                                                                     int qpr) {
  pdl_wait();  // programmatic dependent launch: global memory after the wait
  PdlRelease pdl_release_;
  __shared__ float4 red[kM2Warps][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int32_t R = (int32_t)d.ext[0], E = (int32_t)d.ext[1];
  const int s = blockIdx.y, ns = d.nsplit;
  const int32_t rb = (int32_t)((int64_t)R * s / ns), re = (int32_t)((int64_t)R * (s + 1) / ns);
  const int rpi = 32 / qpr, q = lane % qpr, rsub = lane / qpr;
  const int32_t col = blockIdx.x * 128 + 4 * q;
  const bool colok = col < E;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const int32_t step = kM2Warps * rpi;
  for (int32_t r0 = rb + w * rpi + rsub; r0 < re; r0 += 4 * step) {
    float v[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int32_t r = r0 + u * step;
      const uint32_t vm = (colok && r < re) ? 0xFu : 0u;
      M2FetchVec4Row fetch{d, r, col, vm};
      Body::template eval<float, 4>(d, 0, fetch, vm, v[u]);
      if (!vm) v[u][0] = v[u][1] = v[u][2] = v[u][3] = 0.f;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      acc.x += v[u][0];
      acc.y += v[u][1];
      acc.z += v[u][2];
      acc.w += v[u][3];
    }
  }
  for (int o = qpr; o < 32; o <<= 1) {
    acc.x += __shfl_down_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_down_sync(0xffffffffu, acc.y, o);
    acc.z += __shfl_down_sync(0xffffffffu, acc.z, o);
    acc.w += __shfl_down_sync(0xffffffffu, acc.w, o);
  }
  red[w][lane] = acc;
  __syncthreads();
  if (w != 0 || lane >= qpr || !colok) return;
  float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int ww = 0; ww < kM2Warps; ++ww) {
    t.x += red[ww][lane].x;
    t.y += red[ww][lane].y;
    t.z += red[ww][lane].z;
    t.w += red[ww][lane].w;
  }
  const float tv[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int32_t i = col + j;
    if (ns > 1) {
      ((double *)d.workspace)[(int64_t)s * E + i] = (double)tv[j];
    } else {
      const gfb_m2_operand &wo = d.out[0];
      const int32_t off = (int32_t)wo.c0 + (int32_t)wo.s[1] * i;
      const bool inside = i >= d.clear_lo[1] && i < d.clear_hi[1];
      store_as<float>(const_cast<void *>(wo.base), wo.dtype, off, m2_base<float>(d, inside, off) + tv[j]);
    }
  }
}

// host: may the fp32 two-dimensional launch use the 16-byte variant?
inline bool m2_vec4_ok(const gfb_map2_desc &d) {
  if (d.compute_f64 || d.ndim != 2 || d.ext[1] % 4 != 0) return false;
  if (d.mode == 2) {  // column quads: 128-column blocks, or one power-of-two slice
    const int64_t E = d.ext[1];
    if (E % 128 != 0 && !(E < 128 && ((E / 4) & (E / 4 - 1)) == 0)) return false;
  }
  for (int k = 0; k < d.n_in + d.n_out; ++k) {
    const gfb_m2_operand &o = k < d.n_in ? d.in[k] : d.out[k - d.n_in];
    if (o.dtype != GFB_F32) return false;
    if (d.mode != 0 && k >= d.n_in) continue;  // reduction targets are written by single lanes
    if (o.s[1] == 0) continue;
    if (o.s[1] != 1 || o.c0 % 4 || o.s[0] % 4 || (reinterpret_cast<uintptr_t>(o.base) & 15)) return false;
  }
  return true;
}

// MODE: the one mode a generated body is used with, or -1 (every mode)
template <typename T, int V, typename Body, int MODE = -1, bool UNIFORM = false>
inline int launch_map2(const gfb_map2_desc &d, cudaStream_t st) {
  // bodies that evaluate row-scalar inputs once per lane assume a lane's
  // points share a row: the 16-byte (vec4) paths; anything else runs the
  // evaluator
  if constexpr (UNIFORM) {
    if (!(std::is_same<T, float>::value && V == 4 && m2_vec4_ok(d))) return launch_map2<T, V, VmBody, MODE>(d, st);
  }
  const int nd = d.ndim;
  const int64_t E = d.ext[nd - 1];
  int64_t rows = 1;
  for (int dd = 0; dd < nd - 1; ++dd) rows *= d.ext[dd];
  const int64_t cap = (int64_t)sm_count() * 8;  // resident CTAs of 256 threads
  if (d.mode != MODE && MODE != -1) return set_error(GFB_EINVAL, "gfb_map2_launch: generated body used in another mode");
  if constexpr (std::is_same<T, float>::value && V == 4) {
    if (m2_vec4_ok(d)) {
      if constexpr (MODE == -1 || MODE == 0) {
        if (d.mode == 0) {
          const int64_t cpr = ceil_div(E, 128);
          if constexpr (!std::is_same<Body, VmBody>::value) {
            if (d.n_in <= kM2CacheIn) {
              constexpr int U = 2;
              const int64_t items = E < 128 ? ceil_div(rows * E, 128) : rows * cpr;
              const int64_t blocks = std::max<int64_t>(std::min<int64_t>(ceil_div(items, kM2Warps * U), cap * 4), 1);
              if (E < 128)
                launch_pdl(map2_pointwise_ilp_kernel<Body, true, U>, (unsigned)blocks, 256, 0, st, d, (int32_t)rows, 1,
                           (((uint64_t)1 << 40) + (uint64_t)E - 1) / (uint64_t)E);
              else
                launch_pdl(map2_pointwise_ilp_kernel<Body, false, U>, (unsigned)blocks, 256, 0, st, d, (int32_t)rows,
                           (int32_t)cpr, (uint64_t)0);
              return check_launch("map2");
            }
          }
          if (E < 128) {
            const int64_t blocks =
                std::max<int64_t>(std::min<int64_t>(ceil_div(rows * E, 128 * kM2Warps), cap * 4), 1);
            launch_pdl(map2_pointwise_vec4_kernel<Body, true>, (unsigned)blocks, 256, 0, st, d, (int32_t)rows, 1);
          } else {
            const int64_t blocks =
                std::max<int64_t>(std::min<int64_t>(ceil_div(rows * cpr, kM2Warps), cap * 4), 1);
            launch_pdl(map2_pointwise_vec4_kernel<Body, false>, (unsigned)blocks, 256, 0, st, d, (int32_t)rows,
                                                                                       (int32_t)cpr);
          }
          return check_launch("map2");
        }
      }
      if constexpr (MODE == -1 || MODE == 1) {
        if (d.mode == 1) {
          if constexpr (!std::is_same<Body, VmBody>::value) {
            if (d.n_in <= kM2CacheIn && E <= 128) {
              constexpr int U = 4;
              const int64_t blocks =
                  std::max<int64_t>(std::min<int64_t>(ceil_div(rows, kM2Warps * U), cap * 4), 1);
              launch_pdl(map2_reduce_row_ilp_kernel<Body, U>, (unsigned)blocks, 256, 0, st, d, (int32_t)rows);
              return check_launch("map2");
            }
          }
          const int64_t blocks = std::max<int64_t>(std::min<int64_t>(ceil_div(rows, kM2Warps), cap * 4), 1);
          launch_pdl(map2_reduce_inner_vec4_kernel<Body>, (unsigned)blocks, 256, 0, st, d, (int32_t)rows);
          return check_launch("map2");
        }
      }
      if constexpr (MODE == -1 || MODE == 2) {
        if (d.mode == 2) {
          const int qpr = (int)std::min<int64_t>(E, 128) / 4;
          dim3 grid((unsigned)ceil_div(E, 128), (unsigned)d.nsplit);
          launch_pdl(map2_reduce_outer_vec4_kernel<Body>, grid, 256, 0, st, d, qpr);
          if (d.nsplit > 1) {
            launch_pdl(map2_finish_kernel<T>, (unsigned)ceil_div(E, 32), 1024, 0, st, d);
          }
          return check_launch("map2");
        }
      }
    }
  }
  if constexpr (MODE == -1 || MODE == 0) {
    if (d.mode == 0) {
      const int64_t cpr = ceil_div(E, 32 * V);
      if (nd == 2 && E < 32 * V && E < 512) {
        const uint64_t magic = (((uint64_t)1 << 40) + (uint64_t)E - 1) / (uint64_t)E;
        const int64_t blocks =
            std::max<int64_t>(std::min<int64_t>(ceil_div(rows * E, 32 * V * kM2Warps), cap * 4), 1);
        launch_pdl(map2_pointwise_kernel<T, V, 1, Body>, (unsigned)blocks, 256, 0, st, d, (int32_t)rows, (int32_t)cpr, magic);
      } else {
        const int64_t blocks = std::max<int64_t>(std::min<int64_t>(ceil_div(rows * cpr, kM2Warps), cap * 4), 1);
        if (nd == 2)
          launch_pdl(map2_pointwise_kernel<T, V, 0, Body>, (unsigned)blocks, 256, 0, st, d, (int32_t)rows, (int32_t)cpr, 0);
        else
          launch_pdl(map2_pointwise_kernel<T, V, 2, Body>, (unsigned)blocks, 256, 0, st, d, (int32_t)rows, (int32_t)cpr, 0);
      }
    }
  }
  if constexpr (MODE == -1 || MODE == 1) {
    if (d.mode == 1) {
      const int64_t blocks = std::max<int64_t>(std::min<int64_t>(ceil_div(rows, kM2Warps), cap * 4), 1);
      if (nd == 2)
        launch_pdl(map2_reduce_inner_kernel<T, V, true, Body>, (unsigned)blocks, 256, 0, st, d, (int32_t)rows);
      else
        launch_pdl(map2_reduce_inner_kernel<T, V, false, Body>, (unsigned)blocks, 256, 0, st, d, (int32_t)rows);
    }
  }
  if constexpr (MODE == -1 || MODE == 2) {
    if (d.mode == 2) {
      dim3 grid((unsigned)ceil_div(E, 32), (unsigned)d.nsplit);
      launch_pdl(map2_reduce_outer_kernel<T, V, Body>, grid, 256, 0, st, d);
      if (d.nsplit > 1) {
        launch_pdl(map2_finish_kernel<T>, (unsigned)ceil_div(E, 32), 1024, 0, st, d);
      }
    }
  }
  return check_launch("map2");
}

}  // namespace gfb
