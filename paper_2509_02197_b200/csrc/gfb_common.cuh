// Shared device helpers: element access, the tasklet bytecode VM, error word.
//
// Tasklet bodies are the reference's symbolic expressions (symexpr.py:29-31)
// compiled by the host lowering to a postfix bytecode. Semantics follow the
// reference evaluator (symexpr.py:75-209): eager domain errors instead of NaN,
// floor-style idiv/mod (numpy divmod), sign(0) = 0.
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/gfb.h"

namespace gfb {

template <typename T>
__device__ __forceinline__ T load_as(const void *base, int32_t dtype, int64_t off) {
  return dtype == GFB_F64 ? (T)(((const double *)base)[off])
                          : (T)(((const float *)base)[off]);
}

template <typename T>
__device__ __forceinline__ void store_as(void *base, int32_t dtype, int64_t off, T v) {
  if (dtype == GFB_F64)
    ((double *)base)[off] = (double)v;
  else
    ((float *)base)[off] = (float)v;
}

template <typename T>
__device__ __forceinline__ void add_as(void *base, int32_t dtype, int64_t off, T v) {
  if (dtype == GFB_F64)
    ((double *)base)[off] += (double)v;
  else
    ((float *)base)[off] += (float)v;
}

template <typename T>
__device__ __forceinline__ void atomic_add_as(void *base, int32_t dtype, int64_t off, T v) {
  if (dtype == GFB_F64)
    atomicAdd(((double *)base) + off, (double)v);
  else
    atomicAdd(((float *)base) + off, (float)v);
}

__device__ __forceinline__ void raise_bits(uint32_t *err, uint32_t bits) {
  if (err) atomicOr(err, bits);
}

// numpy-compatible float floor division / remainder (npy_divmod)
template <typename T>
__device__ __forceinline__ T np_mod(T a, T b) {
  T m = fmod(a, b);
  if (m != T(0)) {
    if ((b < T(0)) != (m < T(0))) m += b;
  } else {
    m = copysign(T(0), b);
  }
  return m;
}

template <typename T>
__device__ __forceinline__ T np_floordiv(T a, T b) {
  T m = fmod(a, b);
  T div = (a - m) / b;
  if (m != T(0) && ((b < T(0)) != (m < T(0)))) div -= T(1);
  T fl;
  if (div != T(0)) {
    fl = floor(div);
    if (div - fl > T(0.5)) fl += T(1);
  } else {
    fl = copysign(T(0), a / b);
  }
  return fl;
}

template <typename T>
__device__ __forceinline__ T t_sin(T x) { return sin(x); }
template <>
__device__ __forceinline__ float t_sin<float>(float x) { return sinf(x); }
template <typename T>
__device__ __forceinline__ T t_cos(T x) { return cos(x); }
template <>
__device__ __forceinline__ float t_cos<float>(float x) { return cosf(x); }
template <typename T>
__device__ __forceinline__ T t_exp(T x) { return exp(x); }
template <>
__device__ __forceinline__ float t_exp<float>(float x) { return expf(x); }
template <typename T>
__device__ __forceinline__ T t_log(T x) { return log(x); }
template <>
__device__ __forceinline__ float t_log<float>(float x) { return logf(x); }
template <typename T>
__device__ __forceinline__ T t_tanh(T x) { return tanh(x); }
template <>
__device__ __forceinline__ float t_tanh<float>(float x) { return tanhf(x); }
template <typename T>
__device__ __forceinline__ T t_pow(T x, T y) { return pow(x, y); }
template <>
__device__ __forceinline__ float t_pow<float>(float x, float y) { return powf(x, y); }

template <typename T>
__device__ __forceinline__ T apply_unary(int op, T x, uint32_t *err) {
  switch (op) {
    case GFB_OP_NEG: return -x;
    case GFB_OP_SIN: return t_sin(x);
    case GFB_OP_COS: return t_cos(x);
    case GFB_OP_EXP: return t_exp(x);
    case GFB_OP_LOG:
      if (!(x > T(0))) raise_bits(err, GFB_EBIT_LOG);
      return t_log(x);
    case GFB_OP_SQRT:
      if (x < T(0)) raise_bits(err, GFB_EBIT_SQRT);
      return sqrt(x);
    case GFB_OP_TANH: return t_tanh(x);
    case GFB_OP_ABS: return fabs(x);
    case GFB_OP_SIGN: return x > T(0) ? T(1) : (x < T(0) ? T(-1) : (x == T(0) ? T(0) : x));
    default: return x;
  }
}

template <typename T>
__device__ __forceinline__ T apply_binary(int op, T a, T b, uint32_t *err) {
  switch (op) {
    case GFB_OP_ADD: return a + b;
    case GFB_OP_SUB: return a - b;
    case GFB_OP_MUL: return a * b;
    case GFB_OP_DIV:
      if (b == T(0)) raise_bits(err, GFB_EBIT_DIV0);
      return a / b;
    case GFB_OP_IDIV:
      if (b == T(0)) raise_bits(err, GFB_EBIT_IDIV0);
      return np_floordiv(a, b);
    case GFB_OP_MOD:
      if (b == T(0)) raise_bits(err, GFB_EBIT_MOD0);
      return np_mod(a, b);
    // Python min/max on scalars (symexpr.py:107-116): keep `a` unless `b` wins
    case GFB_OP_MIN: return b < a ? b : a;
    case GFB_OP_MAX: return b > a ? b : a;
    case GFB_OP_POW: {
      if (a == T(0) && b < T(0)) raise_bits(err, GFB_EBIT_POW);
      if (a < T(0) && b != floor(b)) raise_bits(err, GFB_EBIT_POW);
      return t_pow(a, b);
    }
    default: return a;
  }
}

constexpr int kVmStack = 12;

// Evaluate one bytecode segment. `fetch(k)` returns input operand k at the
// current point (loads are issued on demand and hit L1 when repeated).
template <typename T, typename Fetch>
__device__ __forceinline__ T vm_eval(const uint8_t *code, const uint8_t *arg, int start, int len,
                                     const double *consts, Fetch fetch, uint32_t *err) {
  T st[kVmStack];
  int sp = 0;
  for (int pc = start; pc < start + len; ++pc) {
    int op = code[pc];
    if (op == GFB_OP_IN) {
      st[sp++] = fetch(arg[pc]);
    } else if (op == GFB_OP_CONST) {
      st[sp++] = (T)consts[arg[pc]];
    } else if (op >= GFB_OP_NEG) {
      st[sp - 1] = apply_unary<T>(op, st[sp - 1], err);
    } else {
      T b = st[--sp];
      st[sp - 1] = apply_binary<T>(op, st[sp - 1], b, err);
    }
  }
  return st[0];
}

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Programmatic dependent launch: a kernel launched with the programmatic
// stream-serialization attribute may start (prologue from its descriptor)
// while its predecessor drains; pdl_wait() blocks until the predecessor's
// memory is visible and must precede every global access. No-ops for a
// plain launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// releases the successor launch when the thread leaves the kernel (any
// return path): its CTAs then start only as this grid drains, instead of
// holding slots the grid's later waves need
struct PdlRelease {
  __device__ __forceinline__ ~PdlRelease() { pdl_trigger(); }
};

}  // namespace gfb
