// Pure 1-D bulk-copy (cp.async.bulk) streaming throughput: one thread per CTA
// keeps S chunks of CH bytes in flight through an mbarrier ring and re-issues
// as soon as a chunk lands (no consumers). fp64 4000^2 = 128 MB, alternating.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)
__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(bar)), "r"(c) : "memory"); }
__device__ __forceinline__ void mbar_tx(uint64_t *bar, uint32_t b) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(bar)), "r"(b) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su(bar)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void *d, const void *s, uint32_t n, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(d)), "l"(s), "r"(n), "r"(su(bar)) : "memory");
}
__global__ void tma_stream(const char *src, int64_t total, int ch, int S, double *out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t *bar = (uint64_t *)(sm + (size_t)S * ch);
  const int64_t nch = total / ch;
  const int64_t c0 = (int64_t)blockIdx.x * nch / gridDim.x, c1 = (int64_t)(blockIdx.x + 1) * nch / gridDim.x;
  if (threadIdx.x != 0) return;
  for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int64_t n = c1 - c0;
  for (int s = 0; s < S && s < n; ++s) { mbar_tx(&bar[s], ch); bulk(sm + (size_t)s * ch, src + (c0 + s) * ch, ch, &bar[s]); }
  double acc = 0;
  for (int64_t k = 0; k < n; ++k) {
    const int s = (int)(k % S);
    mbar_wait(&bar[s], (uint32_t)((k / S) & 1));
    acc += *(volatile double *)(sm + (size_t)s * ch);
    if (k + S < n) { mbar_tx(&bar[s], ch); bulk(sm + (size_t)s * ch, src + (c0 + k + S) * ch, ch, &bar[s]); }
  }
  if (acc == 1234.5) out[0] = acc;
}
int main() {
  const int64_t total = 4000LL * 4000 * 8;
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  char *A[2]; double *o;
  for (int k = 0; k < 2; ++k) { CK(cudaMalloc(&A[k], total)); CK(cudaMemset(A[k], 0, total)); }
  CK(cudaMalloc(&o, 8));
  CK(cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int per : {1, 2, 4}) for (int ch : {4096, 16384, 32768}) for (int S : {2, 4, 6}) {
    size_t smem = (size_t)S * ch + 64;
    if (smem * per > 220 * 1024) continue;
    int grid = sms * per;
    auto launch = [&](const char *a) { tma_stream<<<grid, 32, smem>>>(a, total, ch, S, o); };
    for (int w = 0; w < 3; ++w) launch(A[w & 1]);
    CK(cudaDeviceSynchronize());
    std::vector<float> ts;
    for (int i = 0; i < 21; ++i) { cudaEventRecord(e0); launch(A[i & 1]); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); ts.push_back(ms); }
    CK(cudaGetLastError());
    std::sort(ts.begin(), ts.end());
    printf("ctas/sm %d chunk %6d stages %d inflight/SM %4zu KB  median %7.2f us  %6.0f GB/s\n", per, ch, S, (size_t)per * S * ch / 1024, ts[10] * 1e3, total / (ts[10] * 1e-3) / 1e9);
  }
  return 0;
}
