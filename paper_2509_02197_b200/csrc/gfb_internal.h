// Host-side helpers shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include "../../include/gfb.h"

namespace gfb {

int set_error(int code, const char *msg);
bool pdl_enabled();

// launch with the programmatic stream-serialization attribute (the kernel
// calls pdl_wait() before touching global memory; GFB_PDL=0 disables)
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<Args &&>(args)...);
}
int check_launch(const char *what);
int sm_count();

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) per (kernel, device)
// whenever a launch needs more than was set: the attribute is per device, so
// a process driving engines on two GPUs must set it on each (abi.cu;
// thread-safe)
void ensure_smem_attr(const void *kernel, int bytes);
template <typename... KArgs>
inline void ensure_smem(void (*kernel)(KArgs...), size_t bytes) {
  ensure_smem_attr(reinterpret_cast<const void *>(kernel), (int)bytes);
}

// fp32 GEMM on tcgen05 (3xTF32, sgemm_tc.cu)
bool sgemm_tc_usable(int64_t M, int64_t N, int64_t K);
int64_t sgemm_tc_workspace(int64_t M, int64_t N, int64_t K);
int sgemm_tc(int ta, int tb, int64_t M, int64_t N, int64_t K, const float *A, int64_t lda, const float *B,
             int64_t ldb, float *C, int64_t ldc, int accumulate, void *ws, cudaStream_t st);

}  // namespace gfb
