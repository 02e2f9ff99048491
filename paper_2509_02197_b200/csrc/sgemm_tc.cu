// fp32 GEMM on the 5th-generation tensor cores: 3xTF32 split precision with
// tcgen05.mma (kind::tf32), accumulators in TMEM.
//
// The mlp matmuls and their adjoints (reference matmul library node,
// interpreter.py:433-446; adjoint jobs autodiff.py:780-802) are fp32 with a
// 1e-5 relative tolerance, which plain TF32 (10-bit mantissa) cannot meet.
// Each operand is split as x = hi + lo with hi = tf32(x), lo = tf32(x - hi),
// and C = A_hi B_hi + A_hi B_lo + A_lo B_hi is accumulated in fp32 TMEM
// (the dropped A_lo B_lo term is ~2^-22 relative).
//
// CTA: 256 threads, tile 128 (M) x BN (N) x 32 (K) per stage, two smem
// stages. All threads stage a k-slab as 16-byte chunks (row, 4 k): the
// global loads of slab t are issued before waiting for its smem slot, then
// hi/lo split and stored into the K-major SWIZZLE_128B canonical layout the
// UMMA smem descriptors describe (row = 32 fp32 = 128 B; 8-row atoms of
// 1 KiB). One elected thread issues 4 k-steps x 3 MMAs per slab and commits
// them to the slab's mbarrier, which the stagers wait on before refilling
// it. Epilogue: tcgen05.ld of the warp's TMEM lane quarter (rows), 8 columns
// at a time. Skinny problems split K over blockIdx.z with fp32 partials
// reduced in order.
#include <algorithm>

#include "gfb_common.cuh"
#include "gfb_internal.h"

namespace gfb {

constexpr int kTcM = 128, kTcK = 32, kTcThreads = 256;

__device__ __forceinline__ uint32_t tc_smem(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ float tf32_round(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// K-major SWIZZLE_128B canonical layout: element (row r, k) of a 32-wide
// k-slab lives at byte r*128 + ((k/4) ^ (r%8))*16 + (k%4)*4
__device__ __forceinline__ uint32_t sw128(int r, int k) {
  return (uint32_t)(r * 128 + ((((k >> 2) ^ (r & 7)) << 4) | ((k & 3) << 2)));
}

__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);        // start address
  d |= (uint64_t)1 << 16;                         // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;               // stride byte offset: 8-row atom
  d |= (uint64_t)1 << 46;                         // descriptor version (sm100)
  d |= (uint64_t)2 << 61;                         // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void tc_mbar_init(uint64_t *bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc_smem(bar)) : "memory");
}

__device__ __forceinline__ void tc_mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(tc_smem(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, int acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void tc_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(tc_smem(bar))
               : "memory");
}

template <int BN>
struct TcSmem {
  // [stage][hi/lo] slabs; 1 KiB aligned (swizzle atoms)
  alignas(1024) float a[2][2][kTcM * kTcK];
  alignas(1024) float b[2][2][BN * kTcK];
  uint64_t mbar[2];
  uint64_t done;
  uint32_t tmem;
};

template <int BN, bool TA, bool TB>
__global__ void __launch_bounds__(kTcThreads, 1)
    sgemm_tc_kernel(int M, int N, int K, const float *__restrict__ A, int64_t lda, const float *__restrict__ B,
                    int64_t ldb, float *C, int64_t ldc, int accumulate, float *partial, int kchunk) {
  extern __shared__ __align__(1024) unsigned char tc_raw[];
  // align the dynamic region to 1 KiB by hand (the runtime guarantees 16 B)
  TcSmem<BN> &S = *reinterpret_cast<TcSmem<BN> *>((reinterpret_cast<uintptr_t>(tc_raw) + 1023) & ~(uintptr_t)1023);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.y * kTcM, n0 = blockIdx.x * BN;
  const int kb = blockIdx.z * kchunk, ke = min(kb + kchunk, K);
  const int nslab = (ke - kb + kTcK - 1) / kTcK;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc_smem(&S.tmem)),
                 "r"(BN < 32 ? 32 : BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    tc_mbar_init(&S.mbar[0]);
    tc_mbar_init(&S.mbar[1]);
    tc_mbar_init(&S.done);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = S.tmem;

  // instruction descriptor: D f32, A/B tf32, both K-major, N, M
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                         ((uint32_t)(kTcM >> 4) << 24);

  // A k-slab is staged as 16-byte chunks: (row, 4 consecutive k). Chunk c
  // of a thread: rows of op(A) first (kTcM * 8 chunks), then op(B)^T.
  constexpr int kChA = kTcM * (kTcK / 4), kChB = BN * (kTcK / 4);
  constexpr int kPer = (kChA + kChB) / kTcThreads;
  static_assert((kChA + kChB) % kTcThreads == 0, "chunks / threads");
  const bool avec = !TA && (lda % 4 == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
  const bool bvec = TB && (ldb % 4 == 0) && ((reinterpret_cast<uintptr_t>(B) & 15) == 0);
  // chunk -> (operand, row, k-chunk). Consecutive lanes walk the contiguous
  // direction of the source so the global loads coalesce.
  auto chunk_of = [&](int c, bool &isb, int &r, int &kc) {
    isb = c >= kChA;
    const int e = isb ? c - kChA : c;
    const int rows = isb ? BN : kTcM;
    const bool kfast = isb ? TB : !TA;
    if (kfast) {  // lanes along k: 8 chunks of one row, then the next row
      kc = e % 8;
      r = e / 8;
    } else {  // lanes along the row index
      r = e % rows;
      kc = e / rows;
    }
  };
  auto load = [&](float4(&reg)[kPer], int k0) {
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      bool isb;
      int r, kc;
      chunk_of(tid + i * kTcThreads, isb, r, kc);
      const int gk = k0 + kc * 4;
      float v[4] = {0.f, 0.f, 0.f, 0.f};
      if (!isb) {
        const int gm = m0 + r;
        if (gm < M) {
          if (avec && gk + 3 < ke) {
            const float4 q = *reinterpret_cast<const float4 *>(A + (int64_t)gm * lda + gk);
            v[0] = q.x, v[1] = q.y, v[2] = q.z, v[3] = q.w;
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (gk + j < ke) v[j] = TA ? A[(int64_t)(gk + j) * lda + gm] : A[(int64_t)gm * lda + gk + j];
          }
        }
      } else {
        const int gn = n0 + r;
        if (gn < N) {
          if (bvec && gk + 3 < ke) {
            const float4 q = *reinterpret_cast<const float4 *>(B + (int64_t)gn * ldb + gk);
            v[0] = q.x, v[1] = q.y, v[2] = q.z, v[3] = q.w;
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (gk + j < ke) v[j] = TB ? B[(int64_t)gn * ldb + gk + j] : B[(int64_t)(gk + j) * ldb + gn];
          }
        }
      }
      reg[i] = make_float4(v[0], v[1], v[2], v[3]);
    }
  };
  auto store = [&](const float4(&reg)[kPer], int s) {
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      bool isb;
      int r, kc;
      chunk_of(tid + i * kTcThreads, isb, r, kc);
      unsigned char *hi = reinterpret_cast<unsigned char *>(isb ? S.b[s][0] : S.a[s][0]);
      unsigned char *lo = reinterpret_cast<unsigned char *>(isb ? S.b[s][1] : S.a[s][1]);
      const float4 x = reg[i];
      const float4 h = make_float4(tf32_round(x.x), tf32_round(x.y), tf32_round(x.z), tf32_round(x.w));
      const float4 l = make_float4(tf32_round(x.x - h.x), tf32_round(x.y - h.y), tf32_round(x.z - h.z),
                                   tf32_round(x.w - h.w));
      const uint32_t o = sw128(r, kc * 4);
      *reinterpret_cast<float4 *>(hi + o) = h;
      *reinterpret_cast<float4 *>(lo + o) = l;
    }
    // make the generic-proxy stores visible to the tensor core's async proxy
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  };

  // one slab: its registers were loaded two slabs ago; the loads of slab
  // t + 2 go out first so two slabs of global latency overlap the staging
  // and the MMAs
  auto slab = [&](int t, float4(&cur)[kPer], float4(&ahead)[kPer]) {
    const int s = t & 1;
    if (t + 2 < nslab) load(ahead, kb + (t + 2) * kTcK);
    if (t >= 2) tc_mbar_wait(&S.mbar[s], (uint32_t)(((t - 2) >> 1) & 1));
    store(cur, s);
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t ah = tc_smem(S.a[s][0]), al = tc_smem(S.a[s][1]);
      const uint32_t bh = tc_smem(S.b[s][0]), bl = tc_smem(S.b[s][1]);
#pragma unroll
      for (int ks = 0; ks < kTcK / 8; ++ks) {  // 8 tf32 = 32 B per MMA k-step
        const uint32_t off = ks * 32;
        const int acc = (t > 0 || ks > 0) ? 1 : 0;
        tc_mma(tmem, umma_desc_sw128(ah + off), umma_desc_sw128(bh + off), idesc, acc);
        tc_mma(tmem, umma_desc_sw128(ah + off), umma_desc_sw128(bl + off), idesc, 1);
        tc_mma(tmem, umma_desc_sw128(al + off), umma_desc_sw128(bh + off), idesc, 1);
      }
      tc_commit(&S.mbar[s]);
      if (t == nslab - 1) tc_commit(&S.done);
    }
  };
  float4 r0[kPer], r1[kPer], r2[kPer];
  if (nslab > 0) load(r0, kb);
  if (nslab > 1) load(r1, kb + kTcK);
  for (int t = 0; t < nslab; t += 3) {
    slab(t, r0, r2);
    if (t + 1 >= nslab) break;
    slab(t + 1, r1, r0);
    if (t + 2 >= nslab) break;
    slab(t + 2, r2, r1);
  }
  if (nslab > 0) tc_mbar_wait(&S.done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  // epilogue: warp w reads TMEM lane quarter w % 4 (tile rows) and column
  // half w / 4; thread = one row
  const int quarter = warp & 3, half = warp >> 2;
  const int row = quarter * 32 + lane, gm = m0 + row;
#pragma unroll 1
  for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); c += 8) {
    uint32_t v[8];
    const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)c;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int gn = n0 + c + j;
      if (gn >= N) continue;
      const float x = nslab > 0 ? __uint_as_float(v[j]) : 0.f;
      if (partial) {
        partial[((int64_t)blockIdx.z * M + gm) * N + gn] = x;
      } else {
        float *o = C + (int64_t)gm * ldc + gn;
        *o = accumulate ? *o + x : x;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN < 32 ? 32 : BN));
}

__global__ void tc_splits_finish(int64_t M, int64_t N, int64_t ns, const float *__restrict__ partial, float *C,
                                 int64_t ldc, int accumulate) {
  const int64_t MN = M * N;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < MN; e += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int64_t q = 0; q < ns; ++q) s += partial[q * MN + e];
    const int64_t m = e / N, n = e - m * N;
    float *c = C + m * ldc + n;
    *c = accumulate ? *c + s : s;
  }
}

static int tc_bn(int64_t N) { return N <= 64 ? 64 : 128; }

int64_t sgemm_tc_splits(int64_t M, int64_t N, int64_t K) {
  const int64_t tiles = ceil_div(M, kTcM) * ceil_div(N, tc_bn(N));
  const int64_t target = (int64_t)sm_count();
  if (tiles >= target) return 1;
  int64_t ns = ceil_div(target, tiles);
  const int64_t maxs = K / (4 * kTcK);
  if (ns > maxs) ns = maxs;
  return ns < 1 ? 1 : ns;
}

bool sgemm_tc_usable(int64_t M, int64_t N, int64_t K) {
  static const bool off = getenv("GFB_NO_TC") != nullptr;
  return !off && M < (1ll << 31) && N < (1ll << 31) && K < (1ll << 31) && M > 1 && N > 1 && K > 1;
}

template <int BN, bool TA, bool TB>
static void launch_tc(dim3 grid, int M, int N, int K, const float *A, int64_t lda, const float *B, int64_t ldb,
                      float *C, int64_t ldc, int accumulate, float *partial, int kchunk, cudaStream_t st) {
  const size_t smem = sizeof(TcSmem<BN>) + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(sgemm_tc_kernel<BN, TA, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  sgemm_tc_kernel<BN, TA, TB><<<grid, kTcThreads, smem, st>>>(M, N, K, A, lda, B, ldb, C, ldc, accumulate, partial,
                                                               kchunk);
}

template <int BN>
static void launch_tc_t(int ta, int tb, dim3 grid, int M, int N, int K, const float *A, int64_t lda,
                        const float *B, int64_t ldb, float *C, int64_t ldc, int accumulate, float *partial,
                        int kchunk, cudaStream_t st) {
  if (ta && tb)
    launch_tc<BN, true, true>(grid, M, N, K, A, lda, B, ldb, C, ldc, accumulate, partial, kchunk, st);
  else if (ta)
    launch_tc<BN, true, false>(grid, M, N, K, A, lda, B, ldb, C, ldc, accumulate, partial, kchunk, st);
  else if (tb)
    launch_tc<BN, false, true>(grid, M, N, K, A, lda, B, ldb, C, ldc, accumulate, partial, kchunk, st);
  else
    launch_tc<BN, false, false>(grid, M, N, K, A, lda, B, ldb, C, ldc, accumulate, partial, kchunk, st);
}

int sgemm_tc(int ta, int tb, int64_t M, int64_t N, int64_t K, const float *A, int64_t lda, const float *B,
             int64_t ldb, float *C, int64_t ldc, int accumulate, void *ws, cudaStream_t st) {
  const int BN = tc_bn(N);
  const int64_t ns = sgemm_tc_splits(M, N, K);
  const int64_t chunk = ceil_div(ceil_div(K, ns), kTcK) * kTcK;
  const int64_t nz = ceil_div(K, chunk);
  float *partial = nz > 1 ? (float *)ws : nullptr;
  dim3 grid((unsigned)ceil_div(N, BN), (unsigned)ceil_div(M, kTcM), (unsigned)nz);
  if (BN == 64)
    launch_tc_t<64>(ta, tb, grid, (int)M, (int)N, (int)K, A, lda, B, ldb, C, ldc, accumulate, partial, (int)chunk, st);
  else
    launch_tc_t<128>(ta, tb, grid, (int)M, (int)N, (int)K, A, lda, B, ldb, C, ldc, accumulate, partial, (int)chunk,
                     st);
  if (nz > 1) {
    const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(M * N, 256), (int64_t)sm_count() * 8);
    tc_splits_finish<<<blocks, 256, 0, st>>>(M, N, nz, partial, C, ldc, accumulate);
  }
  return check_launch("sgemm_tc");
}

int64_t sgemm_tc_workspace(int64_t M, int64_t N, int64_t K) {
  const int64_t ns = sgemm_tc_splits(M, N, K);
  const int64_t chunk = ceil_div(ceil_div(K, ns), kTcK) * kTcK;
  const int64_t nz = ceil_div(K, chunk);
  return nz > 1 ? nz * M * N * 4 : 0;
}

}  // namespace gfb
