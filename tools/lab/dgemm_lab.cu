// Standalone DGEMM variant lab (not part of the product): times DMMA kernel
// variants against cuBLAS on C = A(MxK) B(KxN), row-major, and checks them.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o dgemm_lab dgemm_lab.cu -lcublas
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <cublas_v2.h>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma884(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp16(void *s, const void *g, bool ok) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(g), "r"(ok ? 16 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N> __device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---- v0: the engine's current kernel (register staged, single buffer)
constexpr int kDM = 128, kDN = 128, kDK = 16;
__global__ void __launch_bounds__(256) v0(int64_t M, int64_t N, int64_t K, const double *__restrict__ A, int64_t lda,
                                          const double *__restrict__ B, int64_t ldb, double *C, int64_t ldc) {
  __shared__ double As[kDK][kDM + 4];
  __shared__ double Bs[kDK][kDN + 4];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp >> 2) * 64, wn = (warp & 3) * 32;
  const int64_t m0 = (int64_t)blockIdx.y * kDM, n0 = (int64_t)blockIdx.x * kDN;
  double acc[8][4][2] = {};
  double ra[8], rb[8];
  auto fetch = [&](int64_t k0) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      int e = tid + r * 256;
      int mm = e / kDK, kk = e % kDK;
      int64_t gm = m0 + mm, gk = k0 + kk;
      ra[r] = (gm < M && gk < K) ? A[gm * lda + gk] : 0.0;
      int nn = e % kDN, kb = e / kDN;
      int64_t gn = n0 + nn, gkb = k0 + kb;
      rb[r] = (gn < N && gkb < K) ? B[gkb * ldb + gn] : 0.0;
    }
  };
  auto stash = [&]() {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      int e = tid + r * 256;
      As[e % kDK][e / kDK] = ra[r];
      Bs[e / kDN][e % kDN] = rb[r];
    }
  };
  const int fr = lane >> 2, fc = lane & 3;
  fetch(0);
  for (int64_t k0 = 0; k0 < K; k0 += kDK) {
    stash();
    __syncthreads();
    if (k0 + kDK < K) fetch(k0 + kDK);
#pragma unroll
    for (int ks = 0; ks < kDK; ks += 4) {
      double af[8], bf[4];
#pragma unroll
      for (int a = 0; a < 8; ++a) af[a] = As[ks + fc][wm + a * 8 + fr];
#pragma unroll
      for (int b = 0; b < 4; ++b) bf[b] = Bs[ks + fc][wn + b * 8 + fr];
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma884(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    int64_t gm = m0 + wm + a * 8 + fr;
    if (gm >= M) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        int64_t gn = n0 + wn + b * 8 + 2 * fc + h;
        if (gn < N) C[gm * ldc + gn] = acc[a][b][h];
      }
  }
}

// ---- v1: cp.async multistage, natural layouts As[m][k] (pitch BK+4), Bs[k][n] (pitch BN+4)
template <int BM, int BN, int BK, int WM, int WN, int S, int MINB>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * 32, MINB)
    v1(int64_t M, int64_t N, int64_t K, const double *__restrict__ A, int64_t lda, const double *__restrict__ B,
       int64_t ldb, double *C, int64_t ldc) {
  constexpr int NT = (BM / WM) * (BN / WN) * 32;
  constexpr int PA = BK + 4, PB = BN + 4;
  constexpr int MT = WM / 8, NTL = WN / 8;
  extern __shared__ __align__(16) double sm[];
  double *As = sm, *Bs = sm + S * BM * PA;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp / (BN / WN)) * WM, wn = (warp % (BN / WN)) * WN;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const int64_t ktiles = (K + BK - 1) / BK;
  auto load = [&](int64_t kt, int slot) {
    const int64_t k0 = kt * BK;
    double *as = As + slot * BM * PA, *bs = Bs + slot * BK * PB;
#pragma unroll
    for (int c = tid; c < BM * BK / 2; c += NT) {
      int mm = c / (BK / 2), kk = (c % (BK / 2)) * 2;
      int64_t gm = m0 + mm, gk = k0 + kk;
      bool ok = gm < M && gk < K;
      cp16(as + mm * PA + kk, ok ? A + gm * lda + gk : A, ok);
    }
#pragma unroll
    for (int c = tid; c < BK * BN / 2; c += NT) {
      int kk = c / (BN / 2), nn = (c % (BN / 2)) * 2;
      int64_t gn = n0 + nn, gk = k0 + kk;
      bool ok = gn < N && gk < K;
      cp16(bs + kk * PB + nn, ok ? B + gk * ldb + gn : B, ok);
    }
  };
  double acc[MT][NTL][2];
#pragma unroll
  for (int a = 0; a < MT; ++a)
#pragma unroll
    for (int b = 0; b < NTL; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll
  for (int s = 0; s < S - 1; ++s) {
    if (s < ktiles) load(s, s);
    cp_commit();
  }
  const int fr = lane >> 2, fc = lane & 3;
  for (int64_t kt = 0; kt < ktiles; ++kt) {
    cp_wait<S - 2>();
    __syncthreads();
    {
      int64_t nk = kt + S - 1;
      if (nk < ktiles) load(nk, (int)(nk % S));
      cp_commit();
    }
    const int slot = (int)(kt % S);
    const double *as = As + slot * BM * PA, *bs = Bs + slot * BK * PB;
#pragma unroll
    for (int ks = 0; ks < BK; ks += 4) {
      double af[MT], bf[NTL];
#pragma unroll
      for (int a = 0; a < MT; ++a) af[a] = as[(wm + a * 8 + fr) * PA + ks + fc];
#pragma unroll
      for (int b = 0; b < NTL; ++b) bf[b] = bs[(ks + fc) * PB + wn + b * 8 + fr];
#pragma unroll
      for (int a = 0; a < MT; ++a)
#pragma unroll
        for (int b = 0; b < NTL; ++b) dmma884(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
  }
#pragma unroll
  for (int a = 0; a < MT; ++a) {
    int64_t gm = m0 + wm + a * 8 + fr;
    if (gm >= M) continue;
#pragma unroll
    for (int b = 0; b < NTL; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        int64_t gn = n0 + wn + b * 8 + 2 * fc + h;
        if (gn < N) C[gm * ldc + gn] = acc[a][b][h];
      }
  }
}

template <int BM, int BN, int BK, int WM, int WN, int S, int MINB>
float run_v1(int64_t M, int64_t N, int64_t K, const double *A, const double *B, double *C, int reps) {
  constexpr int NT = (BM / WM) * (BN / WN) * 32;
  size_t smem = (size_t)S * (BM * (BK + 4) + BK * (BN + 4)) * 8;
  auto k = v1<BM, BN, BK, WM, WN, S, MINB>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM));
  k<<<grid, NT, smem>>>(M, N, K, A, K, B, N, C, N);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) k<<<grid, NT, smem>>>(M, N, K, A, K, B, N, C, N);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  if (err) printf("err %s\n", cudaGetErrorString(err));
  return ms / reps;
}

static double check(const std::vector<double> &ref, double *dC, size_t n) {
  std::vector<double> h(n);
  cudaMemcpy(h.data(), dC, n * 8, cudaMemcpyDeviceToHost);
  double e = 0;
  for (size_t i = 0; i < n; ++i) e = fmax(e, fabs(h[i] - ref[i]) / fmax(1.0, fabs(ref[i])));
  return e;
}

int main(int argc, char **argv) {
  int64_t M = argc > 1 ? atoll(argv[1]) : 4000, N = M, K = M;
  int reps = 10;
  size_t na = M * K, nb = K * N, nc = M * N;
  std::vector<double> h(na > nb ? na : nb);
  double *A, *B, *C;
  cudaMalloc(&A, na * 8); cudaMalloc(&B, nb * 8); cudaMalloc(&C, nc * 8);
  srand(1);
  for (size_t i = 0; i < na; ++i) h[i] = rand() / (double)RAND_MAX - 0.5;
  cudaMemcpy(A, h.data(), na * 8, cudaMemcpyHostToDevice);
  for (size_t i = 0; i < nb; ++i) h[i] = rand() / (double)RAND_MAX - 0.5;
  cudaMemcpy(B, h.data(), nb * 8, cudaMemcpyHostToDevice);
  double flops = 2.0 * M * N * K;
  cublasHandle_t hd; cublasCreate(&hd);
  double one = 1, zero = 0;
  // row-major C = A B  <=>  col-major C^T = B^T A^T
  cublasDgemm(hd, CUBLAS_OP_N, CUBLAS_OP_N, N, M, K, &one, B, N, A, K, &zero, C, N);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) cublasDgemm(hd, CUBLAS_OP_N, CUBLAS_OP_N, N, M, K, &one, B, N, A, K, &zero, C, N);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
  printf("cublas           %8.3f ms %6.2f TF\n", ms, flops / ms / 1e9);
  std::vector<double> ref(nc);
  cudaMemcpy(ref.data(), C, nc * 8, cudaMemcpyDeviceToHost);
  {
    dim3 grid((N + 127) / 128, (M + 127) / 128);
    v0<<<grid, 256>>>(M, N, K, A, K, B, N, C, N);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) v0<<<grid, 256>>>(M, N, K, A, K, B, N, C, N);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
    printf("v0               %8.3f ms %6.2f TF err %.2e\n", ms, flops / ms / 1e9, check(ref, C, nc));
  }
#define RUN(BM, BN, BK, WM, WN, S, MB)                                                                           \
  {                                                                                                              \
    cudaMemset(C, 0, nc * 8);                                                                                    \
    float t = run_v1<BM, BN, BK, WM, WN, S, MB>(M, N, K, A, B, C, reps);                                         \
    printf("v1 %3d %3d %2d %3d %3d S%d B%d %8.3f ms %6.2f TF err %.2e\n", BM, BN, BK, WM, WN, S, MB, t,          \
           flops / t / 1e9, check(ref, C, nc));                                                                  \
  }
  RUN(64, 64, 16, 32, 32, 4, 3)
  RUN(64, 64, 16, 32, 32, 3, 3)
  RUN(64, 64, 8, 32, 32, 4, 4)
  RUN(64, 64, 8, 32, 32, 5, 4)
  RUN(64, 64, 32, 32, 32, 2, 3)
  RUN(64, 64, 16, 32, 32, 2, 4)
  RUN(64, 64, 16, 32, 16, 4, 2)
  RUN(64, 64, 16, 16, 32, 4, 2)
  RUN(64, 32, 16, 32, 32, 4, 5)
  RUN(32, 64, 16, 32, 32, 4, 5)
  RUN(128, 64, 8, 32, 32, 4, 2)
  RUN(128, 128, 8, 32, 32, 4, 1)
  return 0;
}
