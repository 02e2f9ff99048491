// Host-side helpers shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include "../../include/gfb.h"

namespace gfb {

int set_error(int code, const char *msg);
int check_launch(const char *what);
int sm_count();

// fp32 GEMM on tcgen05 (3xTF32, sgemm_tc.cu)
bool sgemm_tc_usable(int64_t M, int64_t N, int64_t K);
int64_t sgemm_tc_workspace(int64_t M, int64_t N, int64_t K);
int sgemm_tc(int ta, int tb, int64_t M, int64_t N, int64_t K, const float *A, int64_t lda, const float *B,
             int64_t ldb, float *C, int64_t ldc, int accumulate, void *ws, cudaStream_t st);

}  // namespace gfb
