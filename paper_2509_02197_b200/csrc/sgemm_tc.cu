// fp32 GEMM on the 5th-generation tensor cores: 3xTF32 split precision with
// tcgen05.mma (kind::tf32), accumulators in TMEM.
//
// The mlp matmuls and their adjoints (reference matmul library node,
// interpreter.py:433-446; adjoint jobs autodiff.py:780-802) are fp32 with a
// 1e-5 relative tolerance, which plain TF32 (10-bit mantissa) cannot meet.
// Each operand is split as x = hi + lo with hi = x truncated to TF32 and
// lo = x - hi (exact; the tensor core keeps its top bits),
// and C = A_hi B_hi + A_hi B_lo + A_lo B_hi is accumulated in fp32 TMEM
// (the dropped A_lo B_lo term is ~2^-22 relative).
//
// CTA: 256 threads, tile 128 (M) x BN (N, 32..128) x 32 (K) per stage,
// three smem stages; skinny problems run transposed (C^T = B^T A^T) so the
// large dimension fills the MMA's 128 rows. All threads stage a k-slab as 16-byte chunks (row, 4 k): the
// global loads of slab t are issued before waiting for its smem slot, then
// hi/lo split and stored into the K-major SWIZZLE_128B canonical layout the
// UMMA smem descriptors describe (row = 32 fp32 = 128 B; 8-row atoms of
// 1 KiB). One elected thread issues 4 k-steps x 3 MMAs per slab and commits
// them to the slab's mbarrier, which the stagers wait on before refilling
// it. Epilogue: tcgen05.ld of the warp's TMEM lane quarter (rows), 8 columns
// at a time. Skinny problems split K over blockIdx.z with fp32 partials
// reduced in order.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <type_traits>

#include "gfb_common.cuh"
#include "gfb_internal.h"
#include "tc_common.cuh"

namespace gfb {

constexpr int kTcStages = 3;

template <int BN>
struct TcSmem {
  // [stage][hi/lo] slabs; 1 KiB aligned (swizzle atoms)
  alignas(1024) float a[kTcStages][2][kTcM * kTcK];
  alignas(1024) float b[kTcStages][2][BN * kTcK];
  uint64_t mbar[kTcStages];
  uint64_t done;
  uint32_t tmem;
};

// C[m * csm + n * csn] (+)= sum_k op(A)(m, k) op(B)(k, n); the host maps the
// transposed orientation (C^T = op(B)^T op(A)^T) onto this with csm = 1
template <int BN, bool TA, bool TB>
__global__ void __launch_bounds__(kTcThreads, 1)
    sgemm_tc_kernel(int M, int N, int K, const float *__restrict__ A, int64_t lda, const float *__restrict__ B,
                    int64_t ldb, float *C, int64_t csm, int64_t csn, int accumulate, float *partial, int kchunk) {
  pdl_wait();  // programmatic dependent launch: global memory after the wait
  PdlRelease pdl_release_;
  extern __shared__ __align__(1024) unsigned char tc_raw[];
  // align the dynamic region to 1 KiB by hand (the runtime guarantees 16 B)
  TcSmem<BN> &S = *reinterpret_cast<TcSmem<BN> *>((reinterpret_cast<uintptr_t>(tc_raw) + 1023) & ~(uintptr_t)1023);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.y * kTcM, n0 = blockIdx.x * BN;
  const int kb = blockIdx.z * kchunk, ke = min(kb + kchunk, K);
  const int nslab = (ke - kb + kTcK - 1) / kTcK;
  constexpr int kCols = BN < 32 ? 32 : BN;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc_smem(&S.tmem)),
                 "r"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < kTcStages; ++i) tc_mbar_init(&S.mbar[i]);
    tc_mbar_init(&S.done);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = S.tmem;
  uint32_t sa_hi[kTcStages], sa_lo[kTcStages], sb_hi[kTcStages], sb_lo[kTcStages];
#pragma unroll
  for (int i = 0; i < kTcStages; ++i) {
    sa_hi[i] = tc_smem(S.a[i][0]);
    sa_lo[i] = tc_smem(S.a[i][1]);
    sb_hi[i] = tc_smem(S.b[i][0]);
    sb_lo[i] = tc_smem(S.b[i][1]);
  }

  // instruction descriptor: D f32, A/B tf32, both K-major, N, M
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                         ((uint32_t)(kTcM >> 4) << 24);

  // A k-slab is staged as 16-byte chunks: (row, 4 consecutive k). Chunk c
  // of a thread: rows of op(A) first (kTcM * 8 chunks), then op(B)^T.
  constexpr int kChA = kTcM * (kTcK / 4), kChB = BN * (kTcK / 4);
  constexpr int kPer = (kChA + kChB + kTcThreads - 1) / kTcThreads;
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
      kc = e & 7;
      r = e >> 3;
    } else {  // lanes along the row index
      r = e % rows;
      kc = e / rows;
    }
  };
  auto load = [&](float4(&reg)[kPer], int k0) {
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int c = tid + i * kTcThreads;
      if ((kChA + kChB) % kTcThreads != 0 && c >= kChA + kChB) break;
      bool isb;
      int r, kc;
      chunk_of(c, isb, r, kc);
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
      const int c = tid + i * kTcThreads;
      if ((kChA + kChB) % kTcThreads != 0 && c >= kChA + kChB) break;
      bool isb;
      int r, kc;
      chunk_of(c, isb, r, kc);
      // 32-bit shared addresses keep these st.shared (not generic stores)
      const uint32_t hi = isb ? sb_hi[s] : sa_hi[s], lo = isb ? sb_lo[s] : sa_lo[s];
      const float4 x = reg[i];
      const float4 h = make_float4(tf32_hi(x.x), tf32_hi(x.y), tf32_hi(x.z), tf32_hi(x.w));
      const float4 l = make_float4(x.x - h.x, x.y - h.y, x.z - h.z, x.w - h.w);
      const uint32_t o = sw128(r, kc * 4);
      sts128(hi + o, h);
      sts128(lo + o, l);
    }
    // make the generic-proxy stores visible to the tensor core's async proxy
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  };

  // one slab: its registers were loaded two slabs ago; the loads of slab
  // t + 2 go out first so two slabs of global latency overlap the staging
  // and the MMAs; the smem ring has kTcStages slots
  auto slab = [&](int t, float4(&cur)[kPer], float4(&ahead)[kPer]) {
    const int s = t % kTcStages;
    if (t + 2 < nslab) load(ahead, kb + (t + 2) * kTcK);
    if (t >= kTcStages) tc_mbar_wait(&S.mbar[s], (uint32_t)(((t - kTcStages) / kTcStages) & 1));
    store(cur, s);
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t ah = sa_hi[s], al = sa_lo[s], bh = sb_hi[s], bl = sb_lo[s];
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
  constexpr int kHalf = BN / 2 < 8 ? 8 : BN / 2;
  constexpr int kGrp = kHalf < 32 ? kHalf : 32;  // columns per round: all loads of a round in flight
#pragma unroll 1
  for (int c0 = half * kHalf; c0 < (half + 1) * kHalf && c0 < BN; c0 += kGrp) {
    uint32_t v[kGrp];
#pragma unroll
    for (int g = 0; g < kGrp; g += 8) {
      const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(c0 + g);
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                   : "=r"(v[g]), "=r"(v[g + 1]), "=r"(v[g + 2]), "=r"(v[g + 3]), "=r"(v[g + 4]), "=r"(v[g + 5]),
                     "=r"(v[g + 6]), "=r"(v[g + 7])
                   : "r"(taddr));
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (csn == 1) {
      // row-major C: transpose the warp's 32 rows x kGrp columns through
      // (now idle) stage memory so lanes walk consecutive columns of a row
      float *scr = S.a[0][0] + warp * (32 * (kGrp + 1));
#pragma unroll
      for (int j = 0; j < kGrp; ++j) scr[lane * (kGrp + 1) + j] = nslab > 0 ? __uint_as_float(v[j]) : 0.f;
      __syncwarp();
      if (lane < kGrp) {
        const int gn = n0 + c0 + lane;
        for (int r = 0; r < 32; ++r) {
          const int rm = m0 + quarter * 32 + r;
          if (rm >= M || gn >= N) continue;
          const float x = scr[r * (kGrp + 1) + lane];
          // split-K partials are laid out like C ([z][m][n] here)
          float *o = partial ? partial + ((int64_t)blockIdx.z * M + rm) * N + gn : C + (int64_t)rm * csm + gn;
          *o = accumulate && !partial ? *o + x : x;
        }
      }
      __syncwarp();
      continue;
    }
    if (gm >= M) continue;
    float old[kGrp];
    if (!partial && accumulate) {
#pragma unroll
      for (int j = 0; j < kGrp; ++j) {
        const int gn = n0 + c0 + j;
        old[j] = gn < N ? C[(int64_t)gm * csm + (int64_t)gn * csn] : 0.f;
      }
    }
#pragma unroll
    for (int j = 0; j < kGrp; ++j) {
      const int gn = n0 + c0 + j;
      if (gn >= N) continue;
      const float x = nslab > 0 ? __uint_as_float(v[j]) : 0.f;
      if (partial)
        partial[((int64_t)blockIdx.z * N + gn) * M + gm] = x;  // column-major C: [z][n][m], lanes coalesced
      else
        C[(int64_t)gm * csm + (int64_t)gn * csn] = accumulate ? old[j] + x : x;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols));
}

// ---------------------------------------------------------------------------
// TMA-fed variant (16-byte aligned operands): one elected producer thread
// streams raw fp32 k-slabs by cp.async.bulk.tensor into a ring in the
// SWIZZLE_128B canonical layout of either major (K-major: one box of 32 k x
// rows; MN-major: one 32 (MN) x 32 (k) box per 128-byte atom, described to
// the MMA as MN-major); the tensor core truncates fp32 operands to TF32
// itself (checked bit for bit against an explicit hi copy), so the raw slab
// IS the hi operand and six splitter warps only write lo = x - trunc(x),
// elementwise at the same offsets; one elected thread issues the MMAs.
// Global loads no longer wait on the staging threads, so a CTA keeps several
// slabs of HBM traffic in flight (the skinny, weight-streaming mlp shapes are
// HBM-bound).
constexpr int kTmaSplitWarps = 6;

template <int BN, bool AKM, bool BKM, bool SK = false>
struct TmaCfg {
  static constexpr int kRawA = kTcM * kTcK * 4, kRawB = BN * kTcK * 4;  // bytes
  // per stage: raw A (= hi A), lo A, raw B (= hi B), lo B
  static constexpr int kStage = 2 * (kRawA + kRawB);
  // SK (short k: at most two slabs per CTA): one stage, so several CTAs
  // share an SM and one CTA's epilogue overlaps another's loads
  static constexpr int kStages = SK ? 1 : ((200 * 1024) / kStage > 4 ? 4 : (200 * 1024) / kStage);
  static constexpr int kSmem = kStages * kStage + 1024 /* align */ + 256 /* barriers */;
};

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

// one raw slab: K-major = a (32 k) x rows box at (k0, mn0); MN-major = one
// 32 (MN) x 32 (k) box per atom at (mn0 + 32 a, k0)
template <int ROWS, bool KM>
__device__ __forceinline__ void load_slab(uint32_t dst, const CUtensorMap *map, uint32_t bar, int k0, int mn0) {
  if constexpr (KM) {
    tma_load_2d(dst, map, bar, k0, mn0);
  } else {
#pragma unroll
    for (int a = 0; a < ROWS / 32; ++a) tma_load_2d(dst + a * (kTcK * 128), map, bar, mn0 + 32 * a, k0);
  }
}

__device__ __forceinline__ void tc_mbar_init_n(uint64_t *bar, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tc_smem(bar)), "r"(n) : "memory");
}

__device__ __forceinline__ void tc_mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc_smem(bar)) : "memory");
}

__device__ __forceinline__ void tc_mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc_smem(bar)), "r"(bytes)
               : "memory");
}

// lo operand of one raw slab of `rows` rows (either major: elementwise, the
// same canonical offsets as the raw slab)
template <int ROWS>
__device__ __forceinline__ void split_slab(uint32_t raw, uint32_t lo, int st) {
  constexpr int kNSt = kTmaSplitWarps * 32;
#pragma unroll 2
  for (int c = st; c < ROWS * 8; c += kNSt) {
    float4 x;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w)
                 : "r"(raw + c * 16));
    sts128(lo + c * 16, make_float4(x.x - tf32_hi(x.x), x.y - tf32_hi(x.y), x.z - tf32_hi(x.z), x.w - tf32_hi(x.w)));
  }
}

// UMMA descriptor of an MN-major tf32 operand. The only MN-major layout the
// tensor core takes for 32-bit types is "128B swizzle with 32-byte atoms"
// (layout type 1; TMA's SWIZZLE_128B_ATOM_32B writes it): 128-byte MN rows
// whose 32-byte granules are XOR-ed with the row index mod 4. Here: 32-element
// MN atoms of 32 k rows (4 KiB apart: leading byte offset), 4-row k groups
// 512 B apart (stride byte offset)
__device__ __forceinline__ uint64_t umma_desc_sw128_mn(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((kTcK * 128) >> 4) << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)1 << 61;
  return d;
}

template <int BN, bool AKM, bool BKM, bool SK>
__global__ void __launch_bounds__(kTcThreads, 2)  // <= 128 registers: two short-k CTAs per SM
    sgemm_tma_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap,
                     const __grid_constant__ CUtensorMap cmap, int M, int N, int K, float *C, int64_t csm,
                     int64_t csn, int accumulate, float *partial, int kchunk, int cmode) {
  PdlRelease pdl_release_;
  using Cfg = TmaCfg<BN, AKM, BKM, SK>;
  constexpr int S = Cfg::kStages;
  extern __shared__ __align__(1024) unsigned char tm_raw[];
  unsigned char *base = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(tm_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t *full = reinterpret_cast<uint64_t *>(base + S * Cfg::kStage);
  uint64_t *split = full + S, *empty = split + S, *done = empty + S;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(done + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.y * kTcM, n0 = blockIdx.x * BN;
  const int kb = blockIdx.z * kchunk, ke = min(kb + kchunk, K);
  const int nslab = ke > kb ? (ke - kb + kTcK - 1) / kTcK : 0;
  // TMEM: columns [0, BN) accumulate A_hi B_hi + A_lo B_hi, [BN, 2 BN) A_hi B_lo
  // (one N = 2 BN MMA over the adjacent hi | lo rows of B): two MMAs per
  // k-step instead of three, a third less shared-memory operand traffic
  constexpr int kCols = 2 * BN < 32 ? 32 : 2 * BN;
  // stage layout (byte offsets): rawA | loA | rawB | loB (lo right after hi
  // along the operand's rows: one MMA reads B's hi | lo as 2 BN rows)
  constexpr int oRawA = 0, oLoA = Cfg::kRawA, oRawB = 2 * Cfg::kRawA, oLoB = oRawB + Cfg::kRawB;
  const uint32_t sbase = tc_smem(base);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc_smem(tmem_slot)),
                 "r"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    for (int i = 0; i < S; ++i) {
      tc_mbar_init_n(&full[i], 1);
      tc_mbar_init_n(&split[i], kTmaSplitWarps);
      tc_mbar_init_n(&empty[i], 1);
    }
    tc_mbar_init_n(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  // programmatic dependent launch: the TMEM allocation and barrier set-up
  // above overlap the previous launch's drain; global memory after the wait
  pdl_wait();

  if (warp == 0) {
    if (lane == 0) {  // producer
      for (int t = 0; t < nslab; ++t) {
        const int s = t % S;
        if (t >= S) tc_mbar_wait(&empty[s], (uint32_t)(((t / S) - 1) & 1));
        const uint32_t st = sbase + s * Cfg::kStage;
        const int k0 = kb + t * kTcK;
        tc_mbar_expect_tx(&full[s], Cfg::kRawA + Cfg::kRawB);
        load_slab<kTcM, AKM>(st + oRawA, &amap, tc_smem(&full[s]), k0, m0);
        load_slab<BN, BKM>(st + oRawB, &bmap, tc_smem(&full[s]), k0, n0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      // operand majors: bit 15 (A) / 16 (B) set = MN-major
      constexpr uint32_t kMaj = (AKM ? 0u : 1u << 15) | (BKM ? 0u : 1u << 16);
      const uint32_t idesc2 = (1u << 4) | (2u << 7) | (2u << 10) | kMaj | ((uint32_t)((2 * BN) >> 3) << 17) |
                              ((uint32_t)(kTcM >> 4) << 24);
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | kMaj | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(kTcM >> 4) << 24);
      // one MMA k-step (8 tf32): 32 B along a K-major row, one 8-row k group
      // (1 KiB) of an MN-major atom
      auto desc = [](uint32_t a, int ks, auto km) {
        return decltype(km)::value ? umma_desc_sw128(a + ks * 32) : umma_desc_sw128_mn(a + ks * 1024);
      };
      for (int t = 0; t < nslab; ++t) {
        const int s = t % S;
        tc_mbar_wait(&split[s], (uint32_t)((t / S) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t st = sbase + s * Cfg::kStage;
        const uint32_t ah = st + oRawA, al = st + oLoA, bh = st + oRawB;
        using AK = std::integral_constant<bool, AKM>;
        using BK = std::integral_constant<bool, BKM>;
#pragma unroll
        for (int ks = 0; ks < kTcK / 8; ++ks) {
          const int acc = (t > 0 || ks > 0) ? 1 : 0;
          tc_mma(tmem, desc(ah, ks, AK{}), desc(bh, ks, BK{}), idesc2, acc);  // [B_hi | B_lo]
          tc_mma(tmem, desc(al, ks, AK{}), desc(bh, ks, BK{}), idesc, 1);
        }
        tc_commit(&empty[s]);
      }
      if (nslab > 0) tc_commit(done);
    }
  } else {  // splitters
    const int st_id = tid - 64;
    for (int t = 0; t < nslab; ++t) {
      const int s = t % S;
      tc_mbar_wait(&full[s], (uint32_t)((t / S) & 1));
      const uint32_t st = sbase + s * Cfg::kStage;
      split_slab<kTcM>(st + oRawA, st + oLoA, st_id);
      split_slab<BN>(st + oRawB, st + oLoB, st_id);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) tc_mbar_arrive(&split[s]);
    }
  }
  __syncwarp();
  if (nslab > 0) tc_mbar_wait(done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  // epilogue: warp w reads TMEM lane quarter w % 4 and column half w / 4;
  // the ring is idle now and stages the TMA stores (or serves as transpose
  // scratch for the split-K partials)
  const int quarter = warp & 3, half = warp >> 2;
  const int row = quarter * 32 + lane, gm = m0 + row;
  constexpr int kHalf = BN / 2 < 8 ? 8 : BN / 2;
  constexpr int kGrp = kHalf < 32 ? kHalf : 32;
#pragma unroll 1
  for (int c0 = half * kHalf; c0 < (half + 1) * kHalf && c0 < BN; c0 += kGrp) {
    uint32_t v[kGrp], v2[kGrp];
#pragma unroll
    for (int g = 0; g < kGrp; g += 8) {
      const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(c0 + g);
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                   : "=r"(v[g]), "=r"(v[g + 1]), "=r"(v[g + 2]), "=r"(v[g + 3]), "=r"(v[g + 4]), "=r"(v[g + 5]),
                     "=r"(v[g + 6]), "=r"(v[g + 7])
                   : "r"(taddr));
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                   : "=r"(v2[g]), "=r"(v2[g + 1]), "=r"(v2[g + 2]), "=r"(v2[g + 3]), "=r"(v2[g + 4]),
                     "=r"(v2[g + 5]), "=r"(v2[g + 6]), "=r"(v2[g + 7])
                   : "r"(taddr + (uint32_t)BN));
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < kGrp; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) + __uint_as_float(v2[j]));
    if constexpr (kGrp == 32) {
      if (cmode) {
        // stage the warp's 32 x 32 block (4 KiB slot per warp and column
        // group) and write it with one TMA store (a TMA add-reduction when
        // accumulating); the tensor map clips rows / columns past M / N
        const uint32_t stg = sbase + (uint32_t)(warp * (kHalf / 32) + (c0 - half * kHalf) / 32) * 4096u;
        if (nslab == 0) {
#pragma unroll
          for (int j = 0; j < kGrp; ++j) v[j] = 0u;
        }
        if (cmode == 1) {  // row-major C: row = lane, SWIZZLE_128B rows of 32 columns
#pragma unroll
          for (int c = 0; c < 8; ++c)
            sts128(stg + lane * 128 + ((c ^ (lane & 7)) << 4),
                   make_float4(__uint_as_float(v[4 * c]), __uint_as_float(v[4 * c + 1]),
                               __uint_as_float(v[4 * c + 2]), __uint_as_float(v[4 * c + 3])));
        } else {  // column-major C: row = column j, lanes along m
#pragma unroll
          for (int j = 0; j < kGrp; ++j)
            asm volatile("st.shared.f32 [%0], %1;" ::"r"(stg + j * 128 + lane * 4), "f"(__uint_as_float(v[j]))
                         : "memory");
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          const int x0 = cmode == 1 ? n0 + c0 : m0 + quarter * 32, x1 = cmode == 1 ? m0 + quarter * 32 : n0 + c0;
          if (accumulate)
            asm volatile(
                "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                    reinterpret_cast<uint64_t>(&cmap)),
                "r"(x0), "r"(x1), "r"(stg)
                : "memory");
          else
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                             reinterpret_cast<uint64_t>(&cmap)),
                         "r"(x0), "r"(x1), "r"(stg)
                         : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        continue;
      }
    }
    if (csn == 1) {
      float *scr = reinterpret_cast<float *>(base) + warp * (32 * (kGrp + 1));
#pragma unroll
      for (int j = 0; j < kGrp; ++j) scr[lane * (kGrp + 1) + j] = nslab > 0 ? __uint_as_float(v[j]) : 0.f;
      __syncwarp();
      if (lane < kGrp) {
        const int gn = n0 + c0 + lane;
        for (int r = 0; r < 32; ++r) {
          const int rm = m0 + quarter * 32 + r;
          if (rm >= M || gn >= N) continue;
          const float x = scr[r * (kGrp + 1) + lane];
          // split-K partials are laid out like C ([z][m][n] here)
          float *o = partial ? partial + ((int64_t)blockIdx.z * M + rm) * N + gn : C + (int64_t)rm * csm + gn;
          *o = accumulate && !partial ? *o + x : x;
        }
      }
      __syncwarp();
      continue;
    }
    if (gm >= M) continue;
    float old[kGrp];
    if (!partial && accumulate) {
#pragma unroll
      for (int j = 0; j < kGrp; ++j) {
        const int gn = n0 + c0 + j;
        old[j] = gn < N ? C[(int64_t)gm * csm + (int64_t)gn * csn] : 0.f;
      }
    }
#pragma unroll
    for (int j = 0; j < kGrp; ++j) {
      const int gn = n0 + c0 + j;
      if (gn >= N) continue;
      const float x = nslab > 0 ? __uint_as_float(v[j]) : 0.f;
      if (partial)
        partial[((int64_t)blockIdx.z * N + gn) * M + gm] = x;  // column-major C: [z][n][m], lanes coalesced
      else
        C[(int64_t)gm * csm + (int64_t)gn * csn] = accumulate ? old[j] + x : x;
    }
  }
  // the staged blocks must stay in shared memory until the stores read them
  if (cmode && lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols));
}

static PFN_cuTensorMapEncodeTiled_v12000 tc_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

// 2-D fp32 tensor map: inner extent `inner` (contiguous), `outer` rows of
// `ld` elements, box (bi, bo)
static bool tc_map(CUtensorMap *map, const float *p, int64_t inner, int64_t outer, int64_t ld, int bi, int bo,
                   CUtensorMapSwizzle swz) {
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
  cuuint32_t box[2] = {(cuuint32_t)bi, (cuuint32_t)bo};
  cuuint32_t estr[2] = {1, 1};
  return tc_encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(p), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swz,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, bool AKM, bool BKM, bool SK>
static int launch_tma_k(dim3 grid, int M, int N, int K, const float *A, int64_t lda, const float *B, int64_t ldb,
                      float *C, int64_t csm, int64_t csn, int accumulate, float *partial, int kchunk,
                      cudaStream_t st) {
  CUtensorMap am, bm;
  constexpr CUtensorMapSwizzle kK = CU_TENSOR_MAP_SWIZZLE_128B, kMN = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
  const bool ok = (AKM ? tc_map(&am, A, K, M, lda, kTcK, kTcM, kK) : tc_map(&am, A, M, K, lda, 32, kTcK, kMN)) &&
                  (BKM ? tc_map(&bm, B, K, N, ldb, kTcK, BN, kK) : tc_map(&bm, B, N, K, ldb, 32, kTcK, kMN));
  if (!ok) return -1;
  // TMA-store epilogue: whole C (not split-K partials), 16-byte aligned rows,
  // 32-column groups (BN >= 64)
  CUtensorMap cm{};
  int cmode = 0;
  static const bool no_cstore = getenv("GFB_TC_NO_TMA_STORE") != nullptr;
  if (!no_cstore && BN >= 64 && !partial && (reinterpret_cast<uintptr_t>(C) & 15) == 0) {
    if (csn == 1 && csm % 4 == 0 && tc_map(&cm, C, N, M, csm, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B))
      cmode = 1;
    else if (csm == 1 && csn % 4 == 0 && tc_map(&cm, C, M, N, csn, 32, 32, CU_TENSOR_MAP_SWIZZLE_NONE))
      cmode = 2;
  }
  constexpr int smem = TmaCfg<BN, AKM, BKM, SK>::kSmem;
  static_assert(BN < 64 || TmaCfg<BN, AKM, BKM, SK>::kStages * TmaCfg<BN, AKM, BKM, SK>::kStage >= 8 * (BN / 64) * 4096,
                "epilogue staging exceeds the ring");
  ensure_smem(sgemm_tma_kernel<BN, AKM, BKM, SK>, smem);
  launch_pdl(sgemm_tma_kernel<BN, AKM, BKM, SK>, grid, kTcThreads, smem, st, am, bm, cm, M, N, K, C, csm, csn, accumulate,
                                                                     partial, kchunk, cmode);
  return 0;
}

template <int BN, bool AKM, bool BKM>
static int launch_tma(dim3 grid, int M, int N, int K, const float *A, int64_t lda, const float *B, int64_t ldb,
                      float *C, int64_t csm, int64_t csn, int accumulate, float *partial, int kchunk,
                      cudaStream_t st) {
  static const bool no_sk = getenv("GFB_TMA_NO_SK") != nullptr;
  // short k and more tiles than SMs (one-stage CTAs then share SMs)
  if (!no_sk && kchunk <= 2 * kTcK && (int64_t)grid.x * grid.y * grid.z > (int64_t)sm_count())
    return launch_tma_k<BN, AKM, BKM, true>(grid, M, N, K, A, lda, B, ldb, C, csm, csn, accumulate, partial, kchunk,
                                            st);
  return launch_tma_k<BN, AKM, BKM, false>(grid, M, N, K, A, lda, B, ldb, C, csm, csn, accumulate, partial, kchunk,
                                           st);
}

template <int BN>
static int launch_tma_t(int ta, int tb, dim3 grid, int M, int N, int K, const float *A, int64_t lda,
                        const float *B, int64_t ldb, float *C, int64_t csm, int64_t csn, int accumulate,
                        float *partial, int kchunk, cudaStream_t st) {
  // op(A) K-major <=> not transposed; op(B) K-major <=> transposed
  if (!ta && tb) return launch_tma<BN, true, true>(grid, M, N, K, A, lda, B, ldb, C, csm, csn, accumulate, partial, kchunk, st);
  if (!ta) return launch_tma<BN, true, false>(grid, M, N, K, A, lda, B, ldb, C, csm, csn, accumulate, partial, kchunk, st);
  if (tb) return launch_tma<BN, false, true>(grid, M, N, K, A, lda, B, ldb, C, csm, csn, accumulate, partial, kchunk, st);
  return launch_tma<BN, false, false>(grid, M, N, K, A, lda, B, ldb, C, csm, csn, accumulate, partial, kchunk, st);
}

static bool tma_ok(const float *A, int64_t lda, const float *B, int64_t ldb) {
  static const bool off = getenv("GFB_NO_TMA_GEMM") != nullptr;
  return !off && tc_encode_fn() != nullptr && lda % 4 == 0 && ldb % 4 == 0 &&
         (reinterpret_cast<uintptr_t>(A) & 15) == 0 && (reinterpret_cast<uintptr_t>(B) & 15) == 0;
}

// C (+)= the fixed-order sum of the ns split-K partials, which are laid out
// like C (row-major [z][m][n] when csn == 1, else column-major [z][n][m]) so
// both the partial stores and this pass are coalesced
__global__ void tc_splits_finish(int64_t M, int64_t N, int64_t ns, const float *__restrict__ partial, float *C,
                                 int64_t csm, int64_t csn, int accumulate) {
  pdl_wait();  // programmatic dependent launch: global memory after the wait
  PdlRelease pdl_release_;
  const int64_t MN = M * N;
  const bool rows = csn == 1;
  const int64_t inner = rows ? N : M;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < MN; e += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
#pragma unroll 4
    for (int64_t q = 0; q < ns; ++q) s += __ldg(partial + q * MN + e);
    const int64_t o = e / inner, i = e - o * inner;
    float *c = rows ? C + o * csm + i : C + i * csm + o * csn;
    *c = accumulate ? *c + s : s;
  }
}

static int tc_bn(int64_t N) { return N <= 32 ? 32 : (N <= 64 ? 64 : 128); }

// Orientation: the MMA's M side is fixed at 128 rows, its N side is 32..128;
// put the larger output dimension on the M side (skinny problems such as
// the mlp's batch-64 layers then waste no rows)
static bool tc_swap(int64_t M, int64_t N) { return M < N && M <= 128; }

int64_t sgemm_tc_splits(int64_t M, int64_t N, int64_t K) {
  if (tc_swap(M, N)) std::swap(M, N);
  const int64_t tiles = ceil_div(M, kTcM) * ceil_div(N, tc_bn(N));
  const int64_t target = (int64_t)sm_count();
  if (tiles >= target) return 1;
  // one CTA per SM (the ring fills shared memory): stay within one wave
  int64_t ns = target / tiles;
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
                      float *C, int64_t csm, int64_t csn, int accumulate, float *partial, int kchunk,
                      cudaStream_t st) {
  const size_t smem = sizeof(TcSmem<BN>) + 1024;
  ensure_smem(sgemm_tc_kernel<BN, TA, TB>, (int)smem);
  launch_pdl(sgemm_tc_kernel<BN, TA, TB>, grid, kTcThreads, smem, st, M, N, K, A, lda, B, ldb, C, csm, csn, accumulate,
                                                               partial, kchunk);
}

template <int BN>
static void launch_tc_t(int ta, int tb, dim3 grid, int M, int N, int K, const float *A, int64_t lda,
                        const float *B, int64_t ldb, float *C, int64_t csm, int64_t csn, int accumulate,
                        float *partial, int kchunk, cudaStream_t st) {
  if (ta && tb)
    launch_tc<BN, true, true>(grid, M, N, K, A, lda, B, ldb, C, csm, csn, accumulate, partial, kchunk, st);
  else if (ta)
    launch_tc<BN, true, false>(grid, M, N, K, A, lda, B, ldb, C, csm, csn, accumulate, partial, kchunk, st);
  else if (tb)
    launch_tc<BN, false, true>(grid, M, N, K, A, lda, B, ldb, C, csm, csn, accumulate, partial, kchunk, st);
  else
    launch_tc<BN, false, false>(grid, M, N, K, A, lda, B, ldb, C, csm, csn, accumulate, partial, kchunk, st);
}

int sgemm_tc(int ta, int tb, int64_t M, int64_t N, int64_t K, const float *A, int64_t lda, const float *B,
             int64_t ldb, float *C, int64_t ldc, int accumulate, void *ws, cudaStream_t st) {
  const int64_t ns = sgemm_tc_splits(M, N, K);
  int64_t csm = ldc, csn = 1;
  if (tc_swap(M, N)) {
    // C^T = op(B)^T op(A)^T: op'(A') = op(B)^T is "transposed" exactly when
    // op(B) is not, and likewise for B'
    std::swap(M, N);
    std::swap(A, B);
    std::swap(lda, ldb);
    const int nta = tb ? 0 : 1, ntb = ta ? 0 : 1;
    ta = nta;
    tb = ntb;
    csm = 1;
    csn = ldc;
  }
  const int BN = tc_bn(N);
  const int64_t chunk = ceil_div(ceil_div(K, ns), kTcK) * kTcK;
  const int64_t nz = ceil_div(K, chunk);
  float *partial = nz > 1 ? (float *)ws : nullptr;
  dim3 grid((unsigned)ceil_div(N, BN), (unsigned)ceil_div(M, kTcM), (unsigned)nz);
  int rc = -1;
  if (tma_ok(A, lda, B, ldb)) {
    if (BN == 32)
      rc = launch_tma_t<32>(ta, tb, grid, (int)M, (int)N, (int)K, A, lda, B, ldb, C, csm, csn, accumulate, partial,
                            (int)chunk, st);
    else if (BN == 64)
      rc = launch_tma_t<64>(ta, tb, grid, (int)M, (int)N, (int)K, A, lda, B, ldb, C, csm, csn, accumulate, partial,
                            (int)chunk, st);
    else
      rc = launch_tma_t<128>(ta, tb, grid, (int)M, (int)N, (int)K, A, lda, B, ldb, C, csm, csn, accumulate,
                             partial, (int)chunk, st);
  }
  if (rc == 0) {
    // TMA-fed kernel launched
  } else if (BN == 32)
    launch_tc_t<32>(ta, tb, grid, (int)M, (int)N, (int)K, A, lda, B, ldb, C, csm, csn, accumulate, partial,
                    (int)chunk, st);
  else if (BN == 64)
    launch_tc_t<64>(ta, tb, grid, (int)M, (int)N, (int)K, A, lda, B, ldb, C, csm, csn, accumulate, partial,
                    (int)chunk, st);
  else
    launch_tc_t<128>(ta, tb, grid, (int)M, (int)N, (int)K, A, lda, B, ldb, C, csm, csn, accumulate, partial,
                     (int)chunk, st);
  if (nz > 1) {
    const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(M * N, 256), (int64_t)sm_count() * 8);
    launch_pdl(tc_splits_finish, blocks, 256, 0, st, M, N, nz, partial, C, csm, csn, accumulate);
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
