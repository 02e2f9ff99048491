// gfb_map2_launch: dispatch to an ahead-of-time compiled tasklet body
// (gen_tasklets.cu) when one matches the descriptor's bytecode, else the
// register-stack bytecode evaluator. See map2_kernels.cuh.
#include <cstdlib>

#include "map2_kernels.cuh"

namespace gfb {

struct M2Special {
  uint64_t key;
  int (*launch)(const gfb_map2_desc &, cudaStream_t);
};
extern const M2Special kM2Specials[];
extern const int kM2NumSpecials;

// FNV-1a over the fields that determine the generated code; mirrored by
// tools/gen_tasklets.py (m2_key)
uint32_t m2_uniform_mask(const gfb_map2_desc &d) {
  if (d.compute_f64 || d.ndim < 1) return 0;
  uint32_t m = 0;
  for (int k = 0; k < d.n_in && k < 32; ++k)
    if (d.in[k].s[d.ndim - 1] == 0) m |= 1u << k;
  return m;
}

uint64_t m2_key(const gfb_map2_desc &d) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](uint32_t x) {
    for (int b = 0; b < 4; ++b) {
      h ^= (x >> (8 * b)) & 0xffu;
      h *= 1099511628211ull;
    }
  };
  mix((uint32_t)d.mode);
  mix((uint32_t)d.compute_f64);
  mix((uint32_t)d.n_in);
  mix((uint32_t)d.n_out);
  for (int o = 0; o < d.n_out; ++o) {
    mix((uint32_t)d.code_start[o]);
    mix((uint32_t)d.code_len[o]);
    for (int pc = d.code_start[o]; pc < d.code_start[o] + d.code_len[o]; ++pc) mix(d.code[pc]);
  }
  // fp32 inputs constant along the innermost loop dimension (row scalars):
  // bodies generated for this pattern evaluate them once per lane
  const uint32_t um = m2_uniform_mask(d);
  if (um) mix(0x55000000u | um);
  return h;
}

}  // namespace gfb

using namespace gfb;

extern "C" int64_t gfb_map2_workspace_bytes(const gfb_map2_desc *d) {
  if (!d || d->mode != 2 || d->nsplit <= 1) return 0;
  return (int64_t)d->nsplit * d->ext[1] * 8;
}

extern "C" int gfb_map2_launch(const gfb_map2_desc *d, void *stream) {
  if (!d || d->ndim < 1 || d->ndim > GFB_M2_DIMS || d->n_in < 0 || d->n_in > GFB_MAX_INPUTS || d->n_out < 1 ||
      d->n_out > GFB_M2_OUTS || d->mode < 0 || d->mode > 2)
    return set_error(GFB_EINVAL, "gfb_map2_launch: bad descriptor");
  if (d->mode != 0 && d->n_out != 1) return set_error(GFB_EINVAL, "gfb_map2_launch: reductions have one output");
  if (d->mode == 2 && (d->ndim != 2 || d->nsplit < 1 || d->nsplit > 65535 || (d->nsplit > 1 && !d->workspace)))
    return set_error(GFB_EINVAL, "gfb_map2_launch: bad column reduction");
  int64_t points = 1;
  for (int dd = 0; dd < d->ndim; ++dd) {
    if (d->ext[dd] <= 0) return GFB_OK;  // empty space
    points *= d->ext[dd];
  }
  // int32 index arithmetic: every point count and operand offset must fit
  if (points >= ((int64_t)1 << 31) - 4096) return set_error(GFB_EINVAL, "gfb_map2_launch: space too large for int32");
  for (int k = 0; k < d->n_in + d->n_out; ++k) {
    const gfb_m2_operand &o = k < d->n_in ? d->in[k] : d->out[k - d->n_in];
    int64_t lo = o.c0, hi = o.c0;
    for (int dd = 0; dd < d->ndim; ++dd) {
      const int64_t a = o.s[dd] * (d->ext[dd] - 1);
      lo += a < 0 ? a : 0;
      hi += a > 0 ? a : 0;
    }
    if (lo < 0 || hi >= ((int64_t)1 << 31)) return set_error(GFB_EINVAL, "gfb_map2_launch: offsets exceed int32");
  }
  for (int o = 0; o < d->n_out; ++o)
    if (d->code_start[o] < 0 || d->code_len[o] < 1 || d->code_start[o] + d->code_len[o] > GFB_MAX_CODE)
      return set_error(GFB_EINVAL, "gfb_map2_launch: bad code segment");
  cudaStream_t st = (cudaStream_t)stream;
  if (getenv("GFB_NO_GEN") == nullptr) {
    const uint64_t key = m2_key(*d);
    for (int i = 0; i < kM2NumSpecials; ++i)
      if (kM2Specials[i].key == key) return kM2Specials[i].launch(*d, st);
  }
  // points per lane: 4 (fp32) / 2 (fp64) keep several loads in flight per
  // operand without pushing the register stack out of registers
  if (d->compute_f64) return launch_map2<double, 2, VmBody>(*d, st);
  return launch_map2<float, 4, VmBody>(*d, st);
}
