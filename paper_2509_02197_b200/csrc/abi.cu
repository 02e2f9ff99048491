// C-ABI plumbing: status strings, device queries, plain copies.
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <map>
#include <utility>

#include "gfb_common.cuh"
#include "gfb_internal.h"

namespace gfb {

static thread_local char g_last_error[512] = "";

int set_error(int code, const char *msg) {
  std::snprintf(g_last_error, sizeof(g_last_error), "%s", msg);
  return code;
}

int check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    std::snprintf(g_last_error, sizeof(g_last_error), "%s: %s", what, cudaGetErrorString(e));
    return GFB_ECUDA;
  }
  return GFB_OK;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char *e = getenv("GFB_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

void ensure_smem_attr(const void *kernel, int bytes) {
  // the largest size set so far per (kernel, device): launches of one
  // kernel may use different dynamic sizes (matvec ring stages)
  static std::mutex mu;
  static std::map<std::pair<const void *, int>, int> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  int &have = done[{kernel, dev}];
  if (bytes > have) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    have = bytes;
  }
}

int sm_count() {
  static int cached = 0;
  if (!cached) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || cached <= 0)
      cached = 148;
  }
  return cached;
}

}  // namespace gfb

using namespace gfb;

extern "C" int gfb_abi_version(void) { return GFB_ABI_VERSION; }

extern "C" const char *gfb_last_error(void) { return g_last_error; }

extern "C" int gfb_device_sm_count(void) { return sm_count(); }

extern "C" int gfb_copy(void *dst, const void *src, int64_t bytes, void *stream) {
  if (bytes <= 0) return GFB_OK;
  cudaError_t e = cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream);
  if (e != cudaSuccess) return set_error(GFB_ECUDA, cudaGetErrorString(e));
  return GFB_OK;
}

extern "C" int gfb_plane_copy(void *dst, const void *src, int64_t plane_elems, int32_t dtype, int64_t nplanes,
                              void *stream) {
  int64_t bytes = plane_elems * nplanes * (dtype == GFB_F64 ? 8 : 4);
  return gfb_copy(dst, src, bytes, stream);
}

// Layout self-check for foreign bindings (ctypes in _lib.py): sizes of the
// descriptor structs in declaration order.
extern "C" int gfb_struct_sizes(int64_t *out, int32_t cap) {
  const int64_t s[12] = {(int64_t)sizeof(gfb_space),       (int64_t)sizeof(gfb_operand),
                        (int64_t)sizeof(gfb_map_desc),    (int64_t)sizeof(gfb_term),
                        (int64_t)sizeof(gfb_gather_desc), (int64_t)sizeof(gfb_stencil_desc),
                        (int64_t)sizeof(gfb_star_op),     (int64_t)sizeof(gfb_star_pair_desc),
                        (int64_t)sizeof(gfb_contract_desc), (int64_t)sizeof(gfb_map2_desc),
                        (int64_t)sizeof(gfb_wave_desc),   (int64_t)sizeof(gfb_halo_desc)};
  int n = cap < 12 ? cap : 12;
  for (int i = 0; i < n; ++i) out[i] = s[i];
  return n;
}
