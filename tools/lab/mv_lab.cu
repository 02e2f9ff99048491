// Variants of the one-pass row-dot + column-sum (chain) kernel, fp64 4000^2.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mv_lab mv_lab.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cmath>
#include <algorithm>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

// floor: streaming read-sum, U x 16B loads in flight per thread
template <int U>
__global__ void __launch_bounds__(256) readsum(int64_t n2, const double2 *__restrict__ a, double *out) {
  double s = 0;
  int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * 256;
  for (; i + (U - 1) * stride < n2; i += U * stride) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(a + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) s += v[u].x + v[u].y;
  }
  for (; i < n2; i += stride) { double2 v = a[i]; s += v.x + v.y; }
  if (s == 12345.678) out[0] = s;
}

template <int U>
__global__ void __launch_bounds__(256) readband(int64_t n2, const double2 *__restrict__ a, double *out) {
  double s = 0;
  const int64_t b0 = (int64_t)blockIdx.x * n2 / gridDim.x, b1 = (int64_t)(blockIdx.x + 1) * n2 / gridDim.x;
  int64_t i = b0 + threadIdx.x;
  for (; i + (U - 1) * 256 < b1; i += U * 256) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(a + i + u * 256);
#pragma unroll
    for (int u = 0; u < U; ++u) s += v[u].x + v[u].y;
  }
  for (; i < b1; i += 256) { double2 v = a[i]; s += v.x + v.y; }
  if (s == 12345.678) out[0] = s;
}

// register-prefetched rows: CTA band of rows, thread owns vectors t + 256 q, P rows in flight
template <int NT, int Q, int P>
__global__ void __launch_bounds__(NT) pair_reg(int64_t R, int64_t C, const double *__restrict__ A, const double *__restrict__ u,
                                               double *__restrict__ r, double *__restrict__ partial) {
  __shared__ double red[2][NT / 32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t i0 = (int64_t)blockIdx.x * R / gridDim.x, i1 = (int64_t)(blockIdx.x + 1) * R / gridDim.x;
  const int64_t n = i1 - i0, cv = C / 2;
  double2 uq[Q], cq[Q], buf[P][Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    int64_t j = t + NT * q;
    uq[q] = j < cv ? reinterpret_cast<const double2 *>(u)[j] : make_double2(0, 0);
    cq[q] = make_double2(0, 0);
  }
#pragma unroll
  for (int p = 0; p < P; ++p)
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      int64_t j = t + NT * q;
      buf[p][q] = (p < n && j < cv) ? __ldcs(reinterpret_cast<const double2 *>(A + (i0 + p) * C) + j) : make_double2(0, 0);
    }
  for (int64_t k = 0; k < n; k += P) {
#pragma unroll
    for (int p = 0; p < P; ++p) {
      if (k + p >= n) break;
      double2 a[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) a[q] = buf[p][q];
      // refill this slot with row k + p + P
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        int64_t j = t + NT * q;
        if (k + p + P < n && j < cv) buf[p][q] = __ldcs(reinterpret_cast<const double2 *>(A + (i0 + k + p + P) * C) + j);
      }
      double d0 = 0, d1 = 0;
#pragma unroll
      for (int q = 0; q < Q; ++q) { if (q & 1) d1 = fma(a[q].x, uq[q].x, fma(a[q].y, uq[q].y, d1)); else d0 = fma(a[q].x, uq[q].x, fma(a[q].y, uq[q].y, d0)); }
      double d = d0 + d1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
      const int par = (int)((k + p) & 1);
      if (lane == 0) red[par][warp] = d;
      __syncthreads();
      double tv = 0;
#pragma unroll
      for (int w = 0; w < NT / 32; ++w) tv += red[par][w];
      if (t == 0) r[i0 + k + p] = tv;
#pragma unroll
      for (int q = 0; q < Q; ++q) { cq[q].x = fma(a[q].x, tv, cq[q].x); cq[q].y = fma(a[q].y, tv, cq[q].y); }
    }
  }
  double2 *out = reinterpret_cast<double2 *>(partial + (int64_t)blockIdx.x * C);
#pragma unroll
  for (int q = 0; q < Q; ++q) { int64_t j = t + NT * q; if (j < cv) out[j] = cq[q]; }
}

__global__ void finish(int64_t C, int64_t nb, const double *__restrict__ partial, double *c) {
  __shared__ double red[8][33];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + lane;
  double s[4] = {0, 0, 0, 0};
  if (j < C) {
    int64_t b = g;
    for (; b + 24 < nb; b += 32) {
#pragma unroll
      for (int u = 0; u < 4; ++u) s[u] += partial[(b + 8 * u) * C + j];
    }
    for (; b < nb; b += 8) s[0] += partial[b * C + j];
  }
  red[g][lane] = (s[0] + s[1]) + (s[2] + s[3]);
  __syncthreads();
  if (g == 0 && j < C) { double tot = 0; for (int q = 0; q < 8; ++q) tot += red[q][lane]; c[j] = tot; }
}

int main() {
  const int64_t R = 4000, C = 4000;
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  std::vector<double> hA(R * C), hu(C);
  srand(1);
  for (auto &v : hA) v = rand() / (double)RAND_MAX - 0.5;
  for (auto &v : hu) v = rand() / (double)RAND_MAX - 0.5;
  std::vector<double> rr(R), cc(C, 0.0);
  for (int64_t i = 0; i < R; ++i) { double s = 0; for (int64_t j = 0; j < C; ++j) s += hA[i * C + j] * hu[j]; rr[i] = s; }
  for (int64_t i = 0; i < R; ++i) for (int64_t j = 0; j < C; ++j) cc[j] += hA[i * C + j] * rr[i];
  double *A[2], *u, *r, *c, *part, *o;
  for (int k = 0; k < 2; ++k) { CK(cudaMalloc(&A[k], R * C * 8)); CK(cudaMemcpy(A[k], hA.data(), R * C * 8, cudaMemcpyHostToDevice)); }
  CK(cudaMalloc(&u, C * 8)); CK(cudaMalloc(&r, R * 8)); CK(cudaMalloc(&c, C * 8)); CK(cudaMalloc(&o, 8));
  CK(cudaMalloc(&part, (int64_t)1024 * C * 8));
  CK(cudaMemcpy(u, hu.data(), C * 8, cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char *name, bool chk, auto launch) {
    for (int w = 0; w < 3; ++w) launch(A[w & 1]);
    CK(cudaDeviceSynchronize());
    std::vector<float> ts;
    for (int i = 0; i < 21; ++i) {
      cudaEventRecord(e0); launch(A[i & 1]); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); ts.push_back(ms);
    }
    CK(cudaGetLastError());
    std::sort(ts.begin(), ts.end());
    double err = 0;
    if (chk) {
      std::vector<double> hc(C), hr(R);
      CK(cudaMemcpy(hc.data(), c, C * 8, cudaMemcpyDeviceToHost)); CK(cudaMemcpy(hr.data(), r, R * 8, cudaMemcpyDeviceToHost));
      for (int64_t j = 0; j < C; ++j) err = fmax(err, fabs(hc[j] - cc[j]) / fmax(1.0, fabs(cc[j])));
      for (int64_t j = 0; j < R; ++j) err = fmax(err, fabs(hr[j] - rr[j]) / fmax(1.0, fabs(rr[j])));
    }
    float med = ts[10];
    printf("%-30s median %7.2f us  %6.0f GB/s  err %.1e\n", name, med * 1e3, R * C * 8 / (med * 1e-3) / 1e9, err);
  };
  for (int mult : {4, 8, 16}) {
    char nm[64];
    snprintf(nm, 64, "readsum U4 x%d", mult);
    run(nm, false, [&](double *a) { readsum<4><<<sms * mult, 256>>>(R * C / 2, (const double2 *)a, o); });
    snprintf(nm, 64, "readsum U8 x%d", mult);
    run(nm, false, [&](double *a) { readsum<8><<<sms * mult, 256>>>(R * C / 2, (const double2 *)a, o); });
  }
  for (int mult : {1, 2, 8}) {
    char nm[64];
    snprintf(nm, 64, "readband U8 x%d", mult);
    run(nm, false, [&](double *a) { readband<8><<<sms * mult, 256>>>(R * C / 2, (const double2 *)a, o); });
    snprintf(nm, 64, "readband U16 x%d", mult);
    run(nm, false, [&](double *a) { readband<16><<<sms * mult, 256>>>(R * C / 2, (const double2 *)a, o); });
    snprintf(nm, 64, "readsum U8 grid x%d", mult);
    run(nm, false, [&](double *a) { readsum<8><<<sms * mult, 256>>>(R * C / 2, (const double2 *)a, o); });
  }
  {
    char nm[64];
    int nb = sms;
#define PR(NT, Q, P) snprintf(nm, 64, "pair_reg NT%d Q%d P%d", NT, Q, P); \
    run(nm, true, [&](double *a) { pair_reg<NT, Q, P><<<nb, NT>>>(R, C, a, u, r, part); finish<<<(C + 31) / 32, 256>>>(C, nb, part, c); });
    PR(256, 8, 2) PR(512, 4, 1) PR(512, 4, 2) PR(512, 4, 3) PR(1024, 2, 1) PR(1024, 2, 2) PR(1024, 2, 4)
  }
  return 0;
}
