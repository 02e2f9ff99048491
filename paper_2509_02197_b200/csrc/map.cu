// Generic map kernels: pointwise maps and atomic-free gather passes.
//
// Replaces the reference's per-point interpretation of MapNode bodies
// (Executor._exec_map / _exec_tasklet, interpreter.py:478-507, :405-426).
// The tasklet body runs as bytecode (gfb_common.cuh); subsets arrive as
// affine element offsets precomputed by the host lowering, which has already
// bounds-checked every subset over the whole iteration space.
#include <cooperative_groups.h>

#include <cstdio>

#include "gfb_common.cuh"
#include "gfb_internal.h"

namespace gfb {

// Membership test for a point (box coordinates already placed into x).
__device__ __forceinline__ bool in_space(const gfb_space &s, const int64_t *x) {
  for (int p = 0; p < s.nparams; ++p) {
    int64_t lo = s.lo0[p], hi = s.hi0[p];
    if (s.triangular) {
      for (int q = 0; q < p; ++q) {
        lo += s.loc[p][q] * x[q];
        hi += s.hic[p][q] * x[q];
      }
    }
    if (x[p] < lo || x[p] >= hi) return false;
    if (s.step[p] != 1 && ((x[p] - lo) % s.step[p]) != 0) return false;
  }
  return true;
}

// Box coordinate k along parameter p -> parameter value.
__device__ __forceinline__ int64_t box_coord(const gfb_space &s, int p, int64_t k) {
  return s.triangular ? s.box_lo[p] + k : s.box_lo[p] + k * s.step[p];
}

__device__ __forceinline__ int64_t operand_offset(const gfb_operand &o, const int64_t *x, int np) {
  int64_t off = o.c0;
#pragma unroll
  for (int p = 0; p < GFB_MAX_PARAMS; ++p)
    if (p < np) off += o.s[p] * x[p];
  return off;
}

template <typename T>
__global__ void __launch_bounds__(256) map_pointwise_kernel(const __grid_constant__ gfb_map_desc d,
                                                            int64_t total) {
  const int np = d.space.nparams;
  for (int64_t flat = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; flat < total;
       flat += (int64_t)gridDim.x * blockDim.x) {
    int64_t x[GFB_MAX_PARAMS];
    int64_t rem = flat;
    for (int p = np - 1; p >= 0; --p) {
      int64_t e = d.space.box_ext[p];
      x[p] = box_coord(d.space, p, rem % e);
      rem /= e;
    }
    if (d.space.triangular && !in_space(d.space, x)) continue;
    auto fetch = [&](int k) -> T {
      return load_as<T>(d.in[k].base, d.in[k].dtype, operand_offset(d.in[k], x, np));
    };
    // read-all-then-write: every output value is formed before any store
    T vals[GFB_MAX_OUTPUTS];
#pragma unroll
    for (int o = 0; o < GFB_MAX_OUTPUTS; ++o)
      if (o < d.n_out)
        vals[o] = vm_eval<T>(d.code, d.arg, d.code_start[o], d.code_len[o], d.consts, fetch, d.err);
#pragma unroll
    for (int o = 0; o < GFB_MAX_OUTPUTS; ++o) {
      if (o >= d.n_out) break;
      const gfb_operand &w = d.out[o];
      int64_t off = operand_offset(w, x, np);
      if (d.wcr[o] == 0)
        store_as<T>(w.base, w.dtype, off, vals[o]);
      else if (d.wcr[o] == 1)
        add_as<T>(w.base, w.dtype, off, vals[o]);
      else
        atomic_add_as<T>(w.base, w.dtype, off, vals[o]);
    }
  }
}

// ---------------------------------------------------------------------------
// sequential loop nests by hyperplanes (gfb_wave_desc)

template <typename T>
__global__ void __launch_bounds__(256) wavefront_kernel(const __grid_constant__ gfb_wave_desc w) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const gfb_map_desc &d = w.map;
  const int np = d.space.nparams, sv = w.solve;
  const int64_t cs = w.c[sv], ns = d.space.box_ext[sv];
  int64_t cand = 1;
  for (int p = 0; p < np; ++p)
    if (p != sv) cand *= d.space.box_ext[p];
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  const int64_t g0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t h = 0; h <= w.hmax; ++h) {
    for (int64_t flat = g0; flat < cand; flat += gstride) {
      int64_t k[GFB_MAX_PARAMS];
      int64_t rem = flat, part = 0;
      for (int p = np - 1; p >= 0; --p) {
        if (p == sv) continue;
        const int64_t e = d.space.box_ext[p];
        k[p] = rem % e;
        rem /= e;
        part += w.c[p] * k[p];
      }
      const int64_t r = h - part;
      if (r < 0 || r % cs != 0 || r / cs >= ns) continue;
      k[sv] = r / cs;
      int64_t x[GFB_MAX_PARAMS];
      for (int p = 0; p < np; ++p) x[p] = d.space.box_lo[p] + k[p] * d.space.step[p];
      auto fetch = [&](int q) -> T {
        return load_as<T>(d.in[q].base, d.in[q].dtype, operand_offset(d.in[q], x, np));
      };
      // read-all-then-write per point, outputs in declaration order
      T vals[GFB_MAX_OUTPUTS];
#pragma unroll
      for (int o = 0; o < GFB_MAX_OUTPUTS; ++o)
        if (o < d.n_out) vals[o] = vm_eval<T>(d.code, d.arg, d.code_start[o], d.code_len[o], d.consts, fetch, d.err);
      for (int o = 0; o < d.n_out; ++o) {
        const gfb_operand &q = d.out[o];
        const int64_t off = operand_offset(q, x, np);
        if (d.wcr[o] == 0)
          store_as<T>(q.base, q.dtype, off, vals[o]);
        else
          add_as<T>(q.base, q.dtype, off, vals[o]);
      }
    }
    if (h < w.hmax) {
      __threadfence();
      grid.sync();
    }
  }
}

// ---------------------------------------------------------------------------
// gather pass

__device__ __forceinline__ void unravel(int64_t flat, int rank, const int64_t *lo, const int64_t *ext,
                                        int64_t *y) {
  for (int r = rank - 1; r >= 0; --r) {
    y[r] = lo[r] + flat % ext[r];
    flat /= ext[r];
  }
}

// Sum of the contributions of term t to target y over free-loop indices
// f = f0, f0+fstride, ... < f1.
template <typename T>
__device__ T gather_term(const gfb_gather_desc &d, const gfb_term &t, const int64_t *y, int64_t f0,
                         int64_t f1, int64_t fstride) {
  const int np = d.space.nparams;
  T acc = T(0);
  for (int64_t f = f0; f < f1; f += fstride) {
    int64_t x[GFB_MAX_PARAMS];
    int64_t rem = f;
    for (int p = np - 1; p >= 0; --p) {
      if (t.row_of[p] >= 0) continue;
      int64_t e = d.space.box_ext[p];
      x[p] = box_coord(d.space, p, rem % e);
      rem /= e;
    }
    bool ok = true;
    for (int k = 0; k < t.npiv; ++k) {
      int p = t.order[k];
      int r = t.row_of[p];
      int64_t v = y[r] - t.off[r];
      for (int q = 0; q < np; ++q)
        if (q != p) v -= t.C[r][q] * x[q];
      x[p] = v * t.C[r][p];  // C in {-1, +1}
    }
    // consistency of every row (pivot rows hold by construction)
    for (int r = 0; r < d.rank && ok; ++r) {
      int64_t v = t.off[r];
      for (int q = 0; q < np; ++q) v += t.C[r][q] * x[q];
      ok = (v == y[r]);
    }
    if (!ok || !in_space(d.space, x)) continue;
    auto fetch = [&](int k) -> T {
      return load_as<T>(d.in[k].base, d.in[k].dtype, operand_offset(d.in[k], x, np));
    };
    acc += vm_eval<T>(d.code, d.arg, t.code_start, t.code_len, d.consts, fetch, d.err);
  }
  return acc;
}

__device__ __forceinline__ int64_t term_free_total(const gfb_gather_desc &d, const gfb_term &t) {
  int64_t n = 1;
  for (int p = 0; p < d.space.nparams; ++p)
    if (t.row_of[p] < 0) n *= d.space.box_ext[p];
  return n;
}

template <typename T>
__device__ __forceinline__ T gather_base(const gfb_gather_desc &d, const int64_t *y, int64_t off) {
  if (d.clear_mode == 1 || d.clear_mode == 3) return T(0);
  if (d.clear_mode == 2) {
    bool inside = true;
    for (int r = 0; r < d.rank; ++r) inside &= (y[r] >= d.clear_lo[r] && y[r] < d.clear_hi[r]);
    if (inside) return T(0);
  }
  return load_as<T>(d.dst, d.dtype, off);
}

template <typename T>
__global__ void __launch_bounds__(256) gather_kernel(const __grid_constant__ gfb_gather_desc d, int64_t ny) {
  const int lanes = d.lanes_on_free ? 32 : 1;
  const int64_t per_block = 256 / lanes;
  const int64_t yflat = (int64_t)blockIdx.x * per_block + threadIdx.x / lanes;
  const int lane = threadIdx.x % lanes;
  const int s = blockIdx.y, ns = d.nsplit;
  if (yflat >= ny) return;
  int64_t y[GFB_MAX_RANK];
  unravel(yflat, d.rank, d.ybox_lo, d.ybox_ext, y);
  T acc = T(0);
  for (int k = 0; k < d.n_terms; ++k) {
    const gfb_term &t = d.terms[k];
    int64_t F = term_free_total(d, t);
    int64_t f0 = F * s / ns, f1 = F * (s + 1) / ns;
    acc += gather_term<T>(d, t, y, f0 + lane, f1, lanes);
  }
  if (lanes > 1) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if (lane != 0) return;
  }
  if (ns > 1) {
    ((T *)d.workspace)[(int64_t)s * ny + yflat] = acc;
    return;
  }
  int64_t off = 0;
  for (int r = 0; r < d.rank; ++r) off += y[r] * d.dst_strides[r];
  store_as<T>(d.dst, d.dtype, off, gather_base<T>(d, y, off) + acc);
}

template <typename T>
__global__ void gather_finish_kernel(const __grid_constant__ gfb_gather_desc d, int64_t ny) {
  int64_t yflat = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (yflat >= ny) return;
  T acc = T(0);
  for (int s = 0; s < d.nsplit; ++s) acc += ((const T *)d.workspace)[(int64_t)s * ny + yflat];
  int64_t y[GFB_MAX_RANK];
  unravel(yflat, d.rank, d.ybox_lo, d.ybox_ext, y);
  int64_t off = 0;
  for (int r = 0; r < d.rank; ++r) off += y[r] * d.dst_strides[r];
  store_as<T>(d.dst, d.dtype, off, gather_base<T>(d, y, off) + acc);
}

static int64_t ybox_count(const gfb_gather_desc *d) {
  int64_t n = 1;
  for (int r = 0; r < d->rank; ++r) n *= d->ybox_ext[r];
  return n;
}

}  // namespace gfb

using namespace gfb;

extern "C" int gfb_map_launch(const gfb_map_desc *d, void *stream) {
  if (!d || d->space.nparams < 0 || d->space.nparams > GFB_MAX_PARAMS || d->n_in > GFB_MAX_INPUTS ||
      d->n_out > GFB_MAX_OUTPUTS || d->n_out < 0)
    return set_error(GFB_EINVAL, "gfb_map_launch: bad descriptor");
  int64_t total = 1;
  for (int p = 0; p < d->space.nparams; ++p) total *= d->space.box_ext[p];
  if (total <= 0) return GFB_OK;
  int64_t blocks = ceil_div(total, 256);
  int64_t cap = (int64_t)sm_count() * 16;
  if (blocks > cap) blocks = cap;
  cudaStream_t st = (cudaStream_t)stream;
  if (d->compute_f64)
    map_pointwise_kernel<double><<<(unsigned)blocks, 256, 0, st>>>(*d, total);
  else
    map_pointwise_kernel<float><<<(unsigned)blocks, 256, 0, st>>>(*d, total);
  return check_launch("map_pointwise");
}

extern "C" int64_t gfb_gather_workspace_bytes(const gfb_gather_desc *d) {
  if (!d || d->nsplit <= 1) return 0;
  return (int64_t)d->nsplit * ybox_count(d) * (d->compute_f64 ? 8 : 4);
}

extern "C" int gfb_gather_launch(const gfb_gather_desc *d, void *stream) {
  if (!d || d->rank < 0 || d->rank > GFB_MAX_RANK || d->n_terms < 1 || d->n_terms > 4 || d->nsplit < 1 ||
      d->nsplit > 65535)
    return set_error(GFB_EINVAL, "gfb_gather_launch: bad descriptor");
  if (d->nsplit > 1 && !d->workspace) return set_error(GFB_EINVAL, "gfb_gather_launch: workspace missing");
  int64_t ny = ybox_count(d);
  if (ny <= 0) return GFB_OK;
  int64_t per_block = d->lanes_on_free ? 8 : 256;
  dim3 grid((unsigned)ceil_div(ny, per_block), (unsigned)d->nsplit);
  cudaStream_t st = (cudaStream_t)stream;
  if (d->compute_f64)
    gather_kernel<double><<<grid, 256, 0, st>>>(*d, ny);
  else
    gather_kernel<float><<<grid, 256, 0, st>>>(*d, ny);
  int rc = check_launch("gather");
  if (rc || d->nsplit == 1) return rc;
  unsigned fb = (unsigned)ceil_div(ny, 256);
  if (d->compute_f64)
    gather_finish_kernel<double><<<fb, 256, 0, st>>>(*d, ny);
  else
    gather_finish_kernel<float><<<fb, 256, 0, st>>>(*d, ny);
  return check_launch("gather_finish");
}

extern "C" int gfb_wave_launch(const gfb_wave_desc *w, void *stream) {
  const gfb_map_desc *d = w ? &w->map : nullptr;
  if (!d || d->space.nparams < 1 || d->space.nparams > GFB_MAX_PARAMS || d->n_in > GFB_MAX_INPUTS ||
      d->n_out > GFB_MAX_OUTPUTS || d->n_out < 1 || w->solve < 0 || w->solve >= d->space.nparams ||
      w->c[w->solve] <= 0 || w->hmax < 0)
    return set_error(GFB_EINVAL, "gfb_wave_launch: bad descriptor");
  int64_t cand = 1;
  for (int p = 0; p < d->space.nparams; ++p)
    if (p != w->solve) cand *= d->space.box_ext[p];
  // one cooperative grid: every resident CTA (the grid barrier needs them all)
  int per_sm = 0;
  const void *fn = d->compute_f64 ? (const void *)wavefront_kernel<double> : (const void *)wavefront_kernel<float>;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0) != cudaSuccess || per_sm < 1) per_sm = 1;
  int64_t blocks = ceil_div(cand, 256);
  const int64_t cap = (int64_t)sm_count() * per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  void *args[] = {const_cast<gfb_wave_desc *>(w)};
  cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3((unsigned)blocks), dim3(256), args, 0, (cudaStream_t)stream);
  if (e != cudaSuccess) return set_error(GFB_ECUDA, cudaGetErrorString(e));
  return check_launch("wavefront");
}
