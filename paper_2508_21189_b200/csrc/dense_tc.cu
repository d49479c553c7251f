// K-TC — dense tensor-core apply  Y[n,k] = scale * A[n,d] * B[d,k]  with float32 A, on tcgen05.
//
// Shared engine for every test matrix whose dense form is cheap to feed the tensor cores:
//   * sparse sign Omega (densified once to exact +-1 bf16; scale = 1/sqrt(zeta))  — config 3
//   * Khatri-Rao Omega (columns f0[:,j] (x) f1[:,j], exact +-1 bf16; scale = 1/sqrt(k)) — config 5
//   * Gaussian Omega (bf16 hi + lo split of the float64 draws)                       — reference
//
// Precision.  float32 A is split in-kernel into bf16 hi + lo (x = hi + lo + O(2^-18 |x|)):
//   Y = A_hi B_hi + A_lo B_hi (+ A_hi B_lo when B is split).
// The tcgen05 fp32 accumulator loses ~1e-9 * K relative accuracy over a K-long chain (measured,
// tools/tc_precision.py: 8e-5 at K = 65536), so TMEM only ever holds CHUNK_KB k-blocks (1024 of K)
// of a sum: the MMA warp alternates two TMEM accumulators and dedicated reducer warps fold each
// finished chunk into fp32 register sums (round-to-nearest adds).  Result: ~3e-6 at any K.
//
// CTA = 512 threads (one per SM, persistent over (M-tile, N-block, K-split) work units):
//   WG0  warp 0: TMA producer of A (fp32) and B^T tiles (bf16, K-major, SWIZZLE_128B) | warp 1: MMA
//        warp 2: TMEM allocator                                           (regs trimmed to 32)
//   WG1  warps 4..7 : A converters — the fp32 A tile lands by TMA in the stage; converters read it,
//        meet at a named barrier, and overwrite it in place with bf16 hi/lo in the UMMA K-major
//        SW128 layout                                                                 (128 regs)
//   WG2+WG3 warps 8..15 : reducers — tcgen05.ld of finished chunks, fp32 sums in registers
//        (warp w: TMEM lane group w%4, column half (w-8)/4), final scale + store         (168 regs)
// smem ring of `stages` x {A 32 KB (fp32 -> bf16 hi/lo in place), B_hi BN*128 B (, B_lo)}; mbarriers
// tma_full/full/empty per stage and acc_full/acc_empty per TMEM accumulator.
// With an exact B (NB = 1) and more than 128 rows the CTA-pair form below runs instead
// (dense_tc_pair_kernel, tcgen05 cta_group::2): config 5 1.71 -> 1.59 ms, config 3 1.71 -> 1.55 ms.
#include <cuda.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "sm100.cuh"

namespace skb {
namespace {

using namespace sm100;

constexpr int BM = 128;
constexpr int BK = 64;               // bf16 elements per 128-byte swizzle row
constexpr int CHUNK_KB = 16;         // k-blocks accumulated in TMEM before a register fold
constexpr int kThreads = 512;
constexpr uint32_t kAStageBytes = BM * BK * 4;  // fp32 A staging tile (TMA, no swizzle): 32 KB
constexpr int kMaxBNH = 128;
constexpr int kKrLag = 8;             // KR lockstep: k-blocks a producer may run ahead of its partner         // columns per reducer thread (BN <= 256)

struct TcParams {
  const float* A;
  int64_t M, K, lda;
  int N, BN, nblocks, ksplit, kb_per_split, stages, astages;
  uint32_t tmem_cols;
  float scale;
  float* Y;        // final output (ksplit == 1) ...
  int64_t ldy;
  float* part;     // ... or partial sums [ksplit][M][N] (ksplit > 1)
  int num_units;
  int mtiles;
  // Khatri-Rao mode (dense_tc_pair_kernel<.., KR = 1>): K = (P, q) with q < dl fastest, A read
  // through a 3-D map (q >= dl of a 64-wide k-block is zero-filled).
  // KR = 1: F^T (k x dl bf16) resident in shared memory, chunk = one P (kr_qb k-blocks), a finished
  //         chunk folded with the column weights W[P][col] (the product of the other factors' rows).
  const float* kr_w;
  int64_t kr_ldw;
  // +-1 column weights (every W[P][col] = +-wabs, wabs folded into scale): bit col % 32 of
  // kr_wbits[P * kr_ldwb + col / 32] set when negative; NULL = the float32 weights above.  The
  // reducers load a chunk's 128 bits per warp (four words, issued before the accumulator wait)
  // instead of waiting on a float load per group of 16 columns.
  const uint32_t* kr_wbits;
  int64_t kr_ldwb;
  // KR with N-block groups: per-CTA count of A k-blocks its producer has issued (zeroed per launch);
  // a producer stays within kKrLag k-blocks of the same-rank CTA of the next group's pair, which
  // reads the same A tiles, so the second read of each tile is an L2 hit.  NULL: no lockstep.
  int* kr_progress;
  int kr_qb;       // k-blocks per P (ceil(dl / 64))
  int kr_ngroups;  // N blocks, one per group of pairs (each pair keeps one N block)
  int out_t;       // result transposed: element (row, col) -> Y[col * ldy + row] (through the reduce)
  int kr_a2d;      // dl % 64 == 0: A through the 2-D map (k-block kb = columns 64 kb ..), else 3-D
};


template <int N>
__device__ __forceinline__ void setmaxnreg_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}
template <int N>
__device__ __forceinline__ void setmaxnreg_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}

__device__ __forceinline__ float lds32f(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts128u(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

__device__ __forceinline__ uint32_t ldg_nc_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
// the sign words of columns col .. col + 127 of one weight row (words past the slab's n columns: 0)
__device__ __forceinline__ uint4 ldg_wbits(const uint32_t* row, int col, int n) {
  uint4 v = make_uint4(0u, 0u, 0u, 0u);
  const uint32_t* q = row + (col >> 5);
  if (col < n) v.x = ldg_nc_u32(q);
  if (col + 32 < n) v.y = ldg_nc_u32(q + 1);
  if (col + 64 < n) v.z = ldg_nc_u32(q + 2);
  if (col + 96 < n) v.w = ldg_nc_u32(q + 3);
  return v;
}
__device__ __forceinline__ float4 ldg_nc_v4(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}

struct Unit {
  int mt, nb, ks;
};
__device__ __forceinline__ Unit unit_of(const TcParams& p, int u) {
  Unit r;
  r.nb = u % p.nblocks;
  const int t = u / p.nblocks;
  r.ks = t % p.ksplit;
  r.mt = t / p.ksplit;
  return r;
}

// TA = false: Y[M,N] = A[M,K] * B  (A row-major, the M x K operand read as stored).
// TA = true : Y[M,N] = A^T * B with A stored [K rows][M cols] (the "TN" product Q^T A of rsvd):
//             the TMA lands a 64 (K) x 128 (M) fp32 box and the converters transpose while they
//             split, writing the same K-major SW128 bf16 tiles the MMA reads in the TA = false case.
template <int NB, bool TA>
__global__ void __launch_bounds__(kThreads, 1)
    dense_tc_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_bhi,
                    const __grid_constant__ CUtensorMap tm_blo, const TcParams p) {
  extern __shared__ uint8_t smem_dyn[];
  // keep the pointer derived from the __shared__ array (integer offset) so accesses stay LDS/STS
  uint8_t* smem = smem_dyn + ((1024u - (sm100::smem_u32(smem_dyn) & 1023u)) & 1023u);
  // stage = { A: fp32 tile by TMA, converted in place to bf16 hi [0,16K) + lo [16K,32K) ; B^T tile(s) }
  const uint32_t a_bytes = BM * 128;
  const uint32_t b_bytes = (uint32_t)p.BN * 128;
  const uint32_t stage_bytes = kAStageBytes + NB * b_bytes;
  const int S = p.stages;
  uint64_t* tma_full = reinterpret_cast<uint64_t*>(smem + (size_t)S * stage_bytes);
  uint64_t* full = tma_full + S;       // converted (count: 4 converter warps)
  uint64_t* empty = full + S;          // consumed by the MMA (tcgen05.commit)
  uint64_t* acc_full = empty + S;      // [2]
  uint64_t* acc_empty = acc_full + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&tma_full[s], 1);
      mbar_init(&full[s], 4);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 8);
    }
    fence_mbar_init();
    tma_prefetch_desc(&tm_a);
    tma_prefetch_desc(&tm_bhi);
    if (NB == 2) tma_prefetch_desc(&tm_blo);
  }
  if (warp == 2) tmem_alloc(tmem_slot, p.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int nk = (int)((p.K + BK - 1) / BK);

  if (warp < 4) {
    setmaxnreg_dec<32>();
    if (warp == 0 && lane == 0) {
      // ---------------------------------------------------------------- producer (TMA: A fp32 + B^T bf16)
      int s = 0;
      uint32_t ph = 0;
      for (int u = blockIdx.x; u < p.num_units; u += gridDim.x) {
        const Unit w = unit_of(p, u);
        const int kb0 = w.ks * p.kb_per_split, kb1 = min(nk, kb0 + p.kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* st = smem + (size_t)s * stage_bytes;
          mbar_arrive_expect_tx(&tma_full[s], kAStageBytes + NB * b_bytes);
          if (TA) tma_load_2d(st, &tm_a, &tma_full[s], w.mt * BM, kb * BK);
          else tma_load_2d(st, &tm_a, &tma_full[s], kb * BK, w.mt * BM);
          tma_load_2d(st + kAStageBytes, &tm_bhi, &tma_full[s], kb * BK, w.nb * p.BN);
          if (NB == 2) tma_load_2d(st + kAStageBytes + b_bytes, &tm_blo, &tma_full[s], kb * BK, w.nb * p.BN);
          if (++s == S) { s = 0; ph ^= 1; }
        }
      }
    } else if (warp == 1 && lane == 0) {
      // ---------------------------------------------------------------- MMA issuer
      const uint32_t idesc = idesc_bf16_f32(BM, p.BN);
      int s = 0;
      uint32_t ph = 0;
      uint32_t chunk_seq = 0;  // global chunk counter -> accumulator buffer and phase
      for (int u = blockIdx.x; u < p.num_units; u += gridDim.x) {
        const Unit w = unit_of(p, u);
        const int kb0 = w.ks * p.kb_per_split, kb1 = min(nk, kb0 + p.kb_per_split);
        for (int c0 = kb0; c0 < kb1; c0 += CHUNK_KB, ++chunk_seq) {
          const uint32_t buf = chunk_seq & 1, use = chunk_seq >> 1;
          mbar_wait(&acc_empty[buf], (use & 1) ^ 1);
          tc_fence_after();
          const uint32_t d = tmem + buf * (uint32_t)p.BN;
          const int c1 = min(kb1, c0 + CHUNK_KB);
          for (int kb = c0; kb < c1; ++kb) {
            mbar_wait(&full[s], ph);
            tc_fence_after();
            const uint32_t st = smem_u32(smem + (size_t)s * stage_bytes);
            const uint32_t a_hi = st, a_lo = st + a_bytes, b_hi = st + kAStageBytes, b_lo = b_hi + b_bytes;
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint64_t dah = sdesc_kmajor_sw128(a_hi + kk * 32);
              const uint64_t dal = sdesc_kmajor_sw128(a_lo + kk * 32);
              const uint64_t dbh = sdesc_kmajor_sw128(b_hi + kk * 32);
              umma_bf16(d, dah, dbh, idesc, (kb > c0 || kk > 0) ? 1u : 0u);
              umma_bf16(d, dal, dbh, idesc, 1u);
              if (NB == 2) umma_bf16(d, dah, sdesc_kmajor_sw128(b_lo + kk * 32), idesc, 1u);
            }
            umma_commit(&empty[s]);
            if (++s == S) { s = 0; ph ^= 1; }
          }
          umma_commit(&acc_full[buf]);
        }
      }
    }
  } else if (warp < 8) {
    setmaxnreg_dec<128>();
    // ---------------------------------------------------------------- A converters
    const int ct = threadIdx.x - 128;      // 0..127
    const int c4 = ct & 15;                // float4 column within the 64-wide K block
    const int rsub = ct >> 4;              // 0..7
    int s = 0;
    uint32_t ph = 0;
    for (int u = blockIdx.x; u < p.num_units; u += gridDim.x) {
      const Unit w = unit_of(p, u);
      const int kb0 = w.ks * p.kb_per_split, kb1 = min(nk, kb0 + p.kb_per_split);
      for (int kb = kb0; kb < kb1; ++kb) {
        if constexpr (TA) {
          // staging tile [64 k][128 m] fp32; thread ct = m reads its column (one 128-byte line per
          // warp load) and writes row m of the K-major tiles as eight 16-byte chunks (k / 8)
          mbar_wait(&tma_full[s], ph);
          const uint32_t st = smem_u32(smem + (size_t)s * stage_bytes);
          float col[BK];
#pragma unroll
          for (int i = 0; i < BK; ++i) col[i] = lds32f(st + (uint32_t)(i * BM + ct) * 4u);
          asm volatile("bar.sync 1, 128;" ::: "memory");
#pragma unroll
          for (int g = 0; g < BK / 8; ++g) {
            uint32_t h[4], l[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float x0 = col[8 * g + 2 * q], x1 = col[8 * g + 2 * q + 1];
              h[q] = cvt_bf16x2(x1, x0);
              l[q] = cvt_bf16x2(x1 - __uint_as_float(h[q] & 0xffff0000u), x0 - __uint_as_float(h[q] << 16));
            }
            const uint32_t off = (uint32_t)ct * 128u + ((((uint32_t)g) ^ ((uint32_t)ct & 7u)) << 4);
            sts128u(st + off, h[0], h[1], h[2], h[3]);
            sts128u(st + a_bytes + off, l[0], l[1], l[2], l[3]);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&full[s]);
          if (++s == S) { s = 0; ph ^= 1; }
          continue;
        }
        float4 cur[16];
        mbar_wait(&tma_full[s], ph);
        const uint32_t st = smem_u32(smem + (size_t)s * stage_bytes);
        const uint32_t at = st + (rsub * BK + c4 * 4) * 4;
#pragma unroll
        for (int i = 0; i < 16; ++i) cur[i] = lds128(at + i * 8 * BK * 4);
        // every converter thread has read its fp32 values before any bf16 write lands in place
        asm volatile("bar.sync 1, 128;" ::: "memory");
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int r = rsub + 8 * i;
          const float4 v = cur[i];
          const uint32_t h01 = cvt_bf16x2(v.y, v.x), h23 = cvt_bf16x2(v.w, v.z);
          const float l0 = v.x - __uint_as_float(h01 << 16), l1 = v.y - __uint_as_float(h01 & 0xffff0000u);
          const float l2 = v.z - __uint_as_float(h23 << 16), l3 = v.w - __uint_as_float(h23 & 0xffff0000u);
          const uint32_t lo01 = cvt_bf16x2(l1, l0), lo23 = cvt_bf16x2(l3, l2);
          const uint32_t off = r * 128 + (((c4 >> 1) ^ (r & 7)) << 4) + ((c4 & 1) << 3);
          sts64(st + off, h01, h23);
          sts64(st + a_bytes + off, lo01, lo23);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[s]);
        if (++s == S) { s = 0; ph ^= 1; }
      }
    }
  } else {
    setmaxnreg_inc<168>();
    // ---------------------------------------------------------------- reducers + output
    const int lg = warp & 3;                 // TMEM lane group
    const int half = (warp - 8) >> 2;        // column half: [0, bh0) and [bh0, BN), bh0 = 16-aligned
    const int bh0 = ((p.BN >> 1) + 15) & ~15;
    const int hoff = half * bh0;
    const int bnh = half == 0 ? bh0 : p.BN - bh0;  // columns of this half (BN % 16 == 0)
    uint32_t chunk_seq = 0;
    for (int u = blockIdx.x; u < p.num_units; u += gridDim.x) {
      const Unit w = unit_of(p, u);
      const int kb0 = w.ks * p.kb_per_split, kb1 = min(nk, kb0 + p.kb_per_split);
      float sum[kMaxBNH];
#pragma unroll
      for (int j = 0; j < kMaxBNH; ++j) sum[j] = 0.f;
      for (int c0 = kb0; c0 < kb1; c0 += CHUNK_KB, ++chunk_seq) {
        const uint32_t buf = chunk_seq & 1, use = chunk_seq >> 1;
        mbar_wait(&acc_full[buf], use & 1);
        tc_fence_after();
        const uint32_t base = tmem + ((uint32_t)(32 * lg) << 16) + buf * (uint32_t)p.BN + hoff;
#pragma unroll
        for (int g = 0; g < kMaxBNH / 16; ++g) {
          if (g * 16 < bnh) {
            uint32_t r[16];
            tmem_ld16(base + g * 16, r);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j) sum[g * 16 + j] += __uint_as_float(r[j]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[buf]);
      }
      const int64_t row = (int64_t)w.mt * BM + 32 * lg + lane;
      if (row < p.M) {
        const int col0 = w.nb * p.BN + hoff;
        float* out;
        float sc;
        if (p.ksplit == 1) {
          out = p.Y + row * p.ldy + col0;
          sc = p.scale;
        } else {
          out = p.part + ((int64_t)w.ks * p.M + row) * p.N + col0;
          sc = 1.0f;
        }
#pragma unroll
        for (int g = 0; g < kMaxBNH / 16; ++g) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int c = g * 16 + j;
            if (c < bnh && col0 + c < p.N) out[c] = sum[c] * sc;
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, p.tmem_cols);
  }
}

// ------------------------------------------------------------------------------------ CTA pairs
// The same engine on a CTA pair (cluster of 2 on one TPC, tcgen05 cta_group::2): one MMA of
// M = 256 (128 rows of A from each CTA's shared memory) x N = BN, with B^T split by N — each CTA
// stages only BN/2 rows of the B tile, and the pair's tensor cores share them. Per k-block of 64
// and SM the shared-memory traffic drops from 224 KB (A fp32 32 + convert 64 + B 32 + MMA reads
// 96) to 176 KB, the B-tile half also buys a fourth ring stage. The leader (rank 0) issues the
// MMAs; both CTAs convert their own A rows and arrive on the leader's `full` barrier; commits
// multicast to both CTAs' `empty` / `acc_full`; reducers of both CTAs release the leader's
// `acc_empty`. Each CTA's TMEM holds its own 128 rows x BN of the pair's accumulator.
// Cross-CTA arrives use the default (.cta) release, as CUTLASS's ClusterBarrier: a .release.cluster
// arrive per stage from the converters cost 2.77 ms at config 5 (vs 1.59 ms).
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of `bar` in CTA `cta` of this cluster
__device__ __forceinline__ uint32_t mapa_u32(const void* p, uint32_t cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(sm100::smem_u32(p)), "r"(cta));
  return r;
}
// remote arrive with the default (.release, .cta) semantics, as CUTLASS's ClusterBarrier::arrive: the
// data it publishes is this CTA's own shared memory, read by this SM's half of the pair MMA
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive once on `bar` (same offset) in both CTAs of the pair when this thread's MMAs complete
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          sm100::smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

// Persistent schedule of a pair. Dense: units u = pair, pair + npairs, ... decoded by unit_of. KR:
// the pairs form kr_ngroups groups, group g keeps N block g (its B source) and walks t = (mt, ks)
// with the pairs of its group (pairs p and p + 1 work on the same A rows at the same time, so the
// second N block's read of A is an L2 hit).
struct PairSched {
  int first, step, count, nb;
};
template <int KR>
__device__ __forceinline__ PairSched pair_sched(const TcParams& p, int pair, int npairs) {
  PairSched s;
  if constexpr (KR != 0) {
    s.nb = pair % p.kr_ngroups;
    s.first = pair / p.kr_ngroups;
    s.step = npairs / p.kr_ngroups;
    s.count = p.mtiles * p.ksplit;
  } else {
    s.nb = 0;
    s.first = pair;
    s.step = npairs;
    s.count = p.num_units;
  }
  return s;
}
template <int KR>
__device__ __forceinline__ Unit pair_unit(const TcParams& p, const PairSched& s, int t) {
  if constexpr (KR != 0) {
    Unit r;
    r.mt = t / p.ksplit;
    r.ks = t % p.ksplit;
    r.nb = s.nb;
    return r;
  } else {
    return unit_of(p, t);
  }
}

// KR = 0: dense B^T streamed by TMA with A.
// KR = 1: Khatri-Rao: F^T resident in shared memory (qb tiles per CTA half), one P per TMEM chunk,
//         reducers fold each chunk scaled by W[P, :].  Omega is never formed.
template <int NB, bool TA, int KR>
__global__ void __launch_bounds__(kThreads, 1)
    dense_tc_pair_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                         const __grid_constant__ CUtensorMap tm_blo, const TcParams p) {
  // KR = 1: Khatri-Rao with float32 weights; KR = 3: the same with +-1 weights as sign bits
  constexpr bool KR1 = KR == 1 || KR == 3;
  extern __shared__ uint8_t smem_dyn[];
  uint8_t* smem = smem_dyn + ((1024u - (sm100::smem_u32(smem_dyn) & 1023u)) & 1023u);
  const uint32_t a_bytes = BM * 128;
  const int bnh2 = p.BN >> 1;                      // B^T rows staged by each CTA
  const uint32_t bh_bytes = (uint32_t)bnh2 * 128;
  // stage = {A, B half (, B_lo half)}; KR = 1: stage = {A}, the B halves of all q blocks resident
  const uint32_t stage_bytes = KR1 ? kAStageBytes : kAStageBytes + NB * bh_bytes;
  const int S = p.stages;
  const int qb = KR ? p.kr_qb : 1;
  uint8_t* resident = smem + (size_t)S * stage_bytes;  // KR = 1: [NB][qb] F^T tiles of bh_bytes
  const uint32_t res_bytes = KR1 ? (uint32_t)NB * (uint32_t)qb * bh_bytes : 0u;
  uint64_t* tma_full = reinterpret_cast<uint64_t*>(resident + res_bytes);
  uint64_t* full = tma_full + S;       // leader: converted (and, KR = 2, synthesised) in both CTAs
  uint64_t* empty = full + S;          // consumed by the pair MMA (multicast commit)
  uint64_t* acc_full = empty + S;      // [2] (multicast commit)
  uint64_t* acc_empty = acc_full + 2;  // [2] leader: drained by both CTAs (16 reducer warps)
  uint64_t* res_full = acc_empty + 2;  // KR = 1: this CTA's resident B half has landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(res_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const PairSched sc = pair_sched<KR>(p, pair, npairs);
  const int cqb = KR1 ? qb : CHUNK_KB;  // k-blocks per TMEM chunk
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&tma_full[s], 1);
      mbar_init(&full[s], 8);  // leader: the converter warps of both CTAs
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 16);
    }
    mbar_init(res_full, 1);
    fence_mbar_init();
    tma_prefetch_desc(&tm_a);
    tma_prefetch_desc(&tm_b);
    if (NB == 2) tma_prefetch_desc(&tm_blo);
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sm100::smem_u32(tmem_slot)),
                 "r"(p.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();  // barriers initialised and TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int nk = (int)((p.K + BK - 1) / BK);  // KR: p.K = P * qb * 64 (q padded to whole k-blocks)
  const uint32_t full_leader = mapa_u32(full, 0);       // full[0] in the leader; + 8 s
  const uint32_t acc_empty_leader = mapa_u32(acc_empty, 0);

  if (warp < 4) {
    setmaxnreg_dec<48>();  // 128 x 48 + 128 x 128 + 256 x 168 = 64K registers
    if (warp == 0 && lane == 0) {
      // -------------------------------------------------------------- producer (this CTA's rows + B half)
      if constexpr (KR1) {  // resident F^T half of N block sc.nb: qb tiles of 64 (q) x bnh2 (columns)
        const int brow0 = sc.nb * p.BN + (int)rank * bnh2;
        mbar_arrive_expect_tx(res_full, res_bytes);
        for (int q = 0; q < qb; ++q) {
          tma_load_2d(resident + (size_t)q * bh_bytes, &tm_b, res_full, q * BK, brow0);
          if (NB == 2) tma_load_2d(resident + (size_t)(qb + q) * bh_bytes, &tm_blo, res_full, q * BK, brow0);
        }
      }
      const uint32_t tx_bytes = KR1 ? kAStageBytes : stage_bytes;
      int s = 0;
      uint32_t ph = 0;
      // KR lockstep with the partner pair (same A rows, next N block)
      int* my_prog = nullptr;
      const volatile int* partner_prog = nullptr;
      if (KR != 0 && p.kr_progress != nullptr && p.kr_ngroups > 1) {
        const int partner = sc.first * p.kr_ngroups + (sc.nb + 1) % p.kr_ngroups;
        if (partner < npairs && partner != pair) {
          my_prog = p.kr_progress + blockIdx.x;
          partner_prog = p.kr_progress + 2 * partner + (int)rank;
        }
      }
      int issued = 0, partner_seen = 0;
      for (int t = sc.first; t < sc.count; t += sc.step) {
        const Unit w = pair_unit<KR>(p, sc, t);
        const int kb0 = w.ks * p.kb_per_split, kb1 = min(nk, kb0 + p.kb_per_split);
        const int row0 = (2 * w.mt + (int)rank) * BM;
        const int brow0 = w.nb * p.BN + (int)rank * bnh2;
        for (int kb = kb0; kb < kb1; ++kb) {
          if (my_prog != nullptr) {
            if ((issued & 3) == 0) *reinterpret_cast<volatile int*>(my_prog) = issued;
            if (issued > partner_seen + kKrLag) {
              // bounded wait: a partner that is not resident (another kernel holds its SM) must not
              // hold this CTA, so after ~50 us without progress the lockstep is dropped
              const long long t0 = clock64();
              while (issued > (partner_seen = *partner_prog) + kKrLag) {
                if (clock64() - t0 > 100000) {
                  *reinterpret_cast<volatile int*>(my_prog) = 1 << 30;
                  my_prog = nullptr;
                  break;
                }
                __nanosleep(128);
              }
            }
            ++issued;
          }
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* st = smem + (size_t)s * stage_bytes;
          mbar_arrive_expect_tx(&tma_full[s], tx_bytes);
          if (KR != 0 && !p.kr_a2d) {  // A as (q, P, row) [TA: (col, q, P)]; box 64 q x 1 P x 128, q >= dl zero
            const int P = kb / qb, q0 = (kb - P * qb) * BK;
            if (TA) tma_load_3d(st, &tm_a, &tma_full[s], row0, q0, P);
            else tma_load_3d(st, &tm_a, &tma_full[s], q0, P, row0);
          } else if (KR != 0) {  // dl % 64 == 0: the plain 2-D map (measured faster than the 3-D box)
            if (TA) tma_load_2d(st, &tm_a, &tma_full[s], row0, kb * BK);
            else tma_load_2d(st, &tm_a, &tma_full[s], kb * BK, row0);
          } else {
            if (TA) tma_load_2d(st, &tm_a, &tma_full[s], row0, kb * BK);
            else tma_load_2d(st, &tm_a, &tma_full[s], kb * BK, row0);
            tma_load_2d(st + kAStageBytes, &tm_b, &tma_full[s], kb * BK, brow0);
            if (NB == 2) tma_load_2d(st + kAStageBytes + bh_bytes, &tm_blo, &tma_full[s], kb * BK, brow0);
          }
          if (++s == S) { s = 0; ph ^= 1; }
        }
      }
      if (KR != 0 && p.kr_progress != nullptr)  // done (or lockstep dropped): never hold the partner
        *reinterpret_cast<volatile int*>(p.kr_progress + blockIdx.x) = 1 << 30;
    } else if (warp == 1 && lane == 0 && rank == 0) {
      // -------------------------------------------------------------- MMA issuer (leader only)
      const uint32_t idesc = idesc_bf16_f32(2 * BM, p.BN);
      int s = 0;
      uint32_t ph = 0;
      uint32_t chunk_seq = 0;
      for (int t = sc.first; t < sc.count; t += sc.step) {
        const Unit w = pair_unit<KR>(p, sc, t);
        const int kb0 = w.ks * p.kb_per_split, kb1 = min(nk, kb0 + p.kb_per_split);
        for (int c0 = kb0; c0 < kb1; c0 += cqb, ++chunk_seq) {
          const uint32_t buf = chunk_seq & 1, use = chunk_seq >> 1;
          mbar_wait(&acc_empty[buf], (use & 1) ^ 1);
          tc_fence_after();
          const uint32_t d = tmem + buf * (uint32_t)p.BN;
          const int c1 = min(kb1, c0 + cqb);
          for (int kb = c0; kb < c1; ++kb) {
            mbar_wait(&full[s], ph);
            tc_fence_after();
            const uint32_t st = sm100::smem_u32(smem + (size_t)s * stage_bytes);
            const uint32_t a_hi = st, a_lo = st + a_bytes;
            const uint32_t b = KR1 ? sm100::smem_u32(resident) + (uint32_t)(kb - c0) * bh_bytes : st + kAStageBytes;
            const uint32_t blo = KR1 ? b + (uint32_t)qb * bh_bytes : b + bh_bytes;
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint64_t db = sdesc_kmajor_sw128(b + kk * 32);
              umma_bf16_pair(d, sdesc_kmajor_sw128(a_hi + kk * 32), db, idesc, (kb > c0 || kk > 0) ? 1u : 0u);
              umma_bf16_pair(d, sdesc_kmajor_sw128(a_lo + kk * 32), db, idesc, 1u);
              if (NB == 2)
                umma_bf16_pair(d, sdesc_kmajor_sw128(a_hi + kk * 32), sdesc_kmajor_sw128(blo + kk * 32), idesc, 1u);
            }
            umma_commit_pair(&empty[s]);
            if (++s == S) { s = 0; ph ^= 1; }
          }
          umma_commit_pair(&acc_full[buf]);
        }
      }
    }
  } else if (warp < 8) {
    setmaxnreg_dec<128>();
    // -------------------------------------------------------------- A converters (as dense_tc_kernel)
    const int ct = threadIdx.x - 128;
    const int c4 = ct & 15;
    const int rsub = ct >> 4;
    // KR = 1: the leader's first MMA reads both CTAs' resident B halves; it waits for every converter
    // warp of both CTAs, so each CTA's converters first wait for their own CTA's resident half
    if constexpr (KR1) mbar_wait(res_full, 0);
    int s = 0;
    uint32_t ph = 0;
    for (int t = sc.first; t < sc.count; t += sc.step) {
      const Unit w = pair_unit<KR>(p, sc, t);
      const int kb0 = w.ks * p.kb_per_split, kb1 = min(nk, kb0 + p.kb_per_split);
      for (int kb = kb0; kb < kb1; ++kb) {
        if constexpr (TA) {  // transpose while splitting (as dense_tc_kernel<NB, true>)
          mbar_wait(&tma_full[s], ph);
          const uint32_t st = sm100::smem_u32(smem + (size_t)s * stage_bytes);
          float col[BK];
#pragma unroll
          for (int i = 0; i < BK; ++i) col[i] = lds32f(st + (uint32_t)(i * BM + ct) * 4u);
          asm volatile("bar.sync 1, 128;" ::: "memory");
#pragma unroll
          for (int g = 0; g < BK / 8; ++g) {
            uint32_t h[4], l[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float x0 = col[8 * g + 2 * q], x1 = col[8 * g + 2 * q + 1];
              h[q] = cvt_bf16x2(x1, x0);
              l[q] = cvt_bf16x2(x1 - __uint_as_float(h[q] & 0xffff0000u), x0 - __uint_as_float(h[q] << 16));
            }
            const uint32_t off = (uint32_t)ct * 128u + ((((uint32_t)g) ^ ((uint32_t)ct & 7u)) << 4);
            sts128u(st + off, h[0], h[1], h[2], h[3]);
            sts128u(st + a_bytes + off, l[0], l[1], l[2], l[3]);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive_remote(full_leader + 8u * (uint32_t)s);
          if (++s == S) { s = 0; ph ^= 1; }
          continue;
        }
        float4 cur[16];
        mbar_wait(&tma_full[s], ph);
        const uint32_t st = sm100::smem_u32(smem + (size_t)s * stage_bytes);
        const uint32_t at = st + (rsub * BK + c4 * 4) * 4;
#pragma unroll
        for (int i = 0; i < 16; ++i) cur[i] = lds128(at + i * 8 * BK * 4);
        asm volatile("bar.sync 1, 128;" ::: "memory");
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int r = rsub + 8 * i;
          const float4 v = cur[i];
          const uint32_t h01 = cvt_bf16x2(v.y, v.x), h23 = cvt_bf16x2(v.w, v.z);
          const float l0 = v.x - __uint_as_float(h01 << 16), l1 = v.y - __uint_as_float(h01 & 0xffff0000u);
          const float l2 = v.z - __uint_as_float(h23 << 16), l3 = v.w - __uint_as_float(h23 & 0xffff0000u);
          const uint32_t lo01 = cvt_bf16x2(l1, l0), lo23 = cvt_bf16x2(l3, l2);
          const uint32_t off = r * 128 + (((c4 >> 1) ^ (r & 7)) << 4) + ((c4 & 1) << 3);
          sts64(st + off, h01, h23);
          sts64(st + a_bytes + off, lo01, lo23);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(full_leader + 8u * (uint32_t)s);
        if (++s == S) { s = 0; ph ^= 1; }
      }
    }
  } else {
    setmaxnreg_inc<168>();
    // -------------------------------------------------------------- reducers + output (own 128 rows)
    const int lg = warp & 3;
    const int half = (warp - 8) >> 2;
    const int bh0 = ((p.BN >> 1) + 15) & ~15;
    const int hoff = half * bh0;
    const int bnh = half == 0 ? bh0 : p.BN - bh0;
    uint32_t chunk_seq = 0;
    for (int t = sc.first; t < sc.count; t += sc.step) {
      const Unit w = pair_unit<KR>(p, sc, t);
      const int kb0 = w.ks * p.kb_per_split, kb1 = min(nk, kb0 + p.kb_per_split);
      const int col0 = w.nb * p.BN + hoff;
      float sum[kMaxBNH];
#pragma unroll
      for (int j = 0; j < kMaxBNH; ++j) sum[j] = 0.f;
      // KR = 1 with +-1 weights: the chunk's sign words for columns col0 .. col0 + 127 (col0 is a
      // multiple of 32 whenever kr_wbits is set), loaded before the wait for the chunk's accumulator
      constexpr bool wsign = KR == 3;
      for (int c0 = kb0; c0 < kb1; c0 += cqb, ++chunk_seq) {
        const uint32_t buf = chunk_seq & 1, use = chunk_seq >> 1;
        uint4 wb = make_uint4(0u, 0u, 0u, 0u);
        if (wsign) wb = ldg_wbits(p.kr_wbits + (int64_t)(c0 / qb) * p.kr_ldwb, col0, p.N);
        mbar_wait(&acc_full[buf], use & 1);
        tc_fence_after();
        const uint32_t base = tmem + ((uint32_t)(32 * lg) << 16) + buf * (uint32_t)p.BN + hoff;
        if constexpr (wsign) {
#pragma unroll
          for (int g = 0; g < kMaxBNH / 16; ++g) {
            if (g * 16 < bnh) {
              uint32_t r[16];
              tmem_ld16(base + g * 16, r);
              const uint32_t word = (g >> 1) == 0 ? wb.x : (g >> 1) == 1 ? wb.y : (g >> 1) == 2 ? wb.z : wb.w;
              tmem_ld_wait();
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const int bit = (g & 1) * 16 + j;
                sum[g * 16 + j] += __uint_as_float(r[j] ^ ((word << (31 - bit)) & 0x80000000u));
              }
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_remote(acc_empty_leader + 8u * buf);
          continue;
        }
        // KR = 1: the chunk's column weights W[P][col0 ...] (the same address in every lane: broadcast)
        const float4* wrow = nullptr;
        if constexpr (KR == 1) wrow = reinterpret_cast<const float4*>(p.kr_w + (int64_t)(c0 / qb) * p.kr_ldw + col0);
#pragma unroll
        for (int g = 0; g < kMaxBNH / 16; ++g) {
          if (g * 16 < bnh) {
            uint32_t r[16];
            tmem_ld16(base + g * 16, r);
            if constexpr (KR == 1) {
              float wv[16];
#pragma unroll
              for (int j = 0; j < 4; ++j) {  // issued with the TMEM load, consumed after its wait
                const float4 x = ldg_nc_v4(wrow + 4 * g + j);
                wv[4 * j] = x.x;
                wv[4 * j + 1] = x.y;
                wv[4 * j + 2] = x.z;
                wv[4 * j + 3] = x.w;
              }
              tmem_ld_wait();
#pragma unroll
              for (int j = 0; j < 16; ++j) sum[g * 16 + j] = fmaf(wv[j], __uint_as_float(r[j]), sum[g * 16 + j]);
            } else {
              tmem_ld_wait();
#pragma unroll
              for (int j = 0; j < 16; ++j) sum[g * 16 + j] += __uint_as_float(r[j]);
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(acc_empty_leader + 8u * buf);
      }
      const int64_t row = (int64_t)(2 * w.mt + (int)rank) * BM + 32 * lg + lane;
      if constexpr (KR == 0) {
        const bool direct = p.ksplit == 1 && !p.out_t;
        // partial sums (or a transposed result): tc_splitk_reduce forms Y
        float* const obase = direct ? p.Y : p.part + (int64_t)w.ks * p.M * p.N;
        const int64_t ld = direct ? p.ldy : (int64_t)p.N;
        const float sc2 = direct ? p.scale : 1.0f;
        // (dense engine only: the Khatri-Rao reducers' register budget, 128 sums + the fold, would spill)
        if ((bnh & 7) == 0 && (col0 & 7) == 0 && (ld & 7) == 0 && col0 + bnh <= p.N &&
            (reinterpret_cast<uintptr_t>(obase) & 31) == 0) {
          // lane pairs complete 32-byte sectors (each lane holds one row: a lane's own 16-byte store
          // would cover half a sector): the even lane writes columns [b, b+4) and the odd lane
          // [b+4, b+8) of the same row, one row per instruction, after a shfl.xor exchange of 4 values
          const bool odd = lane & 1;
          const int64_t row_e = row - (odd ? 1 : 0), row_o = row_e + 1;
#pragma unroll
          for (int b = 0; b < kMaxBNH; b += 8) {
            if (b < bnh) {
              float mine[4], got[4];
#pragma unroll
              for (int q = 0; q < 4; ++q) {  // static register indices (a runtime index would spill sum[])
                const float lo = sum[b + q], hi = sum[b + 4 + q];
                got[q] = __shfl_xor_sync(0xffffffffu, odd ? lo : hi, 1);
                mine[q] = odd ? hi : lo;
              }
              const float* v1 = odd ? got : mine;  // row_e's part
              const float* v2 = odd ? mine : got;  // row_o's part
              const int c = col0 + b + (odd ? 4 : 0);
              if (row_e < p.M)
                *reinterpret_cast<float4*>(obase + row_e * ld + c) =
                    make_float4(v1[0] * sc2, v1[1] * sc2, v1[2] * sc2, v1[3] * sc2);
              if (row_o < p.M)
                *reinterpret_cast<float4*>(obase + row_o * ld + c) =
                    make_float4(v2[0] * sc2, v2[1] * sc2, v2[2] * sc2, v2[3] * sc2);
            }
          }
          continue;
        }
      } else {
        // Khatri-Rao reducers: 16-byte stores of the row's columns (no exchange: 168 registers hold
        // the 128 sums), a quarter of the scalar stores' instructions
        const bool direct = p.ksplit == 1 && !p.out_t;
        float* const obase = direct ? p.Y : p.part + (int64_t)w.ks * p.M * p.N;
        const int64_t ld = direct ? p.ldy : (int64_t)p.N;
        const float sc2 = direct ? p.scale : 1.0f;
        if ((bnh & 3) == 0 && (col0 & 3) == 0 && (ld & 3) == 0 && col0 + bnh <= p.N &&
            (reinterpret_cast<uintptr_t>(obase) & 15) == 0) {
          if (row < p.M) {
            float* out = obase + row * ld + col0;
#pragma unroll
            for (int c = 0; c < kMaxBNH; c += 4)
              if (c < bnh)
                *reinterpret_cast<float4*>(out + c) =
                    make_float4(sum[c] * sc2, sum[c + 1] * sc2, sum[c + 2] * sc2, sum[c + 3] * sc2);
          }
          continue;
        }
      }
      if (row < p.M) {
        float* out;
        float sc2;
        if (p.ksplit == 1 && !p.out_t) {
          out = p.Y + row * p.ldy + col0;
          sc2 = p.scale;
        } else {  // partial sums (or a transposed result): tc_splitk_reduce forms Y
          out = p.part + ((int64_t)w.ks * p.M + row) * p.N + col0;
          sc2 = 1.0f;
        }
#pragma unroll
        for (int g = 0; g < kMaxBNH / 16; ++g) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int c = g * 16 + j;
            if (c < bnh && col0 + c < p.N) out[c] = sum[c] * sc2;
          }
        }
      }
    }
  }
  tc_fence_before();
  cluster_sync_all();  // both CTAs done with the pair's TMEM
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(p.tmem_cols) : "memory");
  }
}

// Y = scale * sum_s part[s] (fixed order); out_t: element (r, c) -> Y[c * ldy + r]
__global__ void tc_splitk_reduce(const float* __restrict__ part, int ksplit, int64_t M, int N, float scale,
                                 float* __restrict__ Y, int64_t ldy, int out_t = 0) {
  if (!out_t && (N & 3) == 0 && (ldy & 3) == 0 && ((reinterpret_cast<uintptr_t>(part) | reinterpret_cast<uintptr_t>(Y)) & 15) == 0) {
    // float4 elements; the (row, column) position advances by the grid stride without a division per
    // element (the 64-bit divide / modulo of the generic loop dominated this memory-bound kernel)
    const int64_t n4 = N >> 2, total4 = M * n4;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i0 >= total4) return;
    int64_t r = i0 / n4, c = i0 - r * n4;
    const int64_t dr = stride / n4, dc = stride - dr * n4;
    const float4* p4 = reinterpret_cast<const float4*>(part);
    for (int64_t i = i0; i < total4; i += stride) {
      float4 acc = p4[r * n4 + c];
      for (int q = 1; q < ksplit; ++q) {
        const float4 v = p4[(q * M + r) * n4 + c];
        acc.x += v.x;
        acc.y += v.y;
        acc.z += v.z;
        acc.w += v.w;
      }
      *reinterpret_cast<float4*>(Y + r * ldy + 4 * c) =
          make_float4(acc.x * scale, acc.y * scale, acc.z * scale, acc.w * scale);
      r += dr;
      c += dc;
      if (c >= n4) {
        c -= n4;
        ++r;
      }
    }
    return;
  }
  const int64_t total = M * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r, c;
    if (out_t) {  // consecutive threads -> consecutive r (coalesced Y^T writes)
      c = i / M;
      r = i % M;
    } else {
      r = i / N;
      c = i % N;
    }
    float s = 0.f;
    for (int q = 0; q < ksplit; ++q) s += part[(q * M + r) * N + c];
    if (out_t) Y[c * ldy + r] = s * scale;
    else Y[r * ldy + c] = s * scale;
  }
}

// ------------------------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  // resolved once (thread-safe static initialisation: trials may run on a host thread pool)
  static const EncodeTiledFn fn = [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<EncodeTiledFn>(ptr);
    return static_cast<EncodeTiledFn>(nullptr);
  }();
  ensure_context();
  return fn;
}

// B^T: [N rows][K cols] bf16, row stride ldb elements; box 64 (K) x box_rows (N), SWIZZLE_128B.
int make_bt_map(CUtensorMap* m, const void* bt, int64_t N, int64_t K, int64_t ldb, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(SK_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)N};
  cuuint64_t strides[1] = {(cuuint64_t)ldb * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(bt), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SK_EINVAL, "cuTensorMapEncodeTiled failed (alignment of B^T / ldb?)");
  return SK_OK;
}

// A: [M rows][K cols] fp32, box 64 (K) x 128 (M), no swizzle (staging tile read by the converters).
int make_a_map(CUtensorMap* m, const float* a, int64_t M, int64_t K, int64_t lda) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(SK_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)M};
  cuuint64_t strides[1] = {(cuuint64_t)lda * 4};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)BM};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(a), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(SK_EINVAL, "cuTensorMapEncodeTiled(A) failed with CUresult " + std::to_string((int)r) +
                               " (alignment of A / lda?)");
  return SK_OK;
}

// A stored [K rows][M cols] fp32 (the TN product): box 128 (M, contiguous) x 64 (K), no swizzle.
int make_at_map(CUtensorMap* m, const float* a, int64_t M, int64_t K, int64_t lda) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(SK_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)M, (cuuint64_t)K};
  cuuint64_t strides[1] = {(cuuint64_t)lda * 4};
  cuuint32_t box[2] = {(cuuint32_t)BM, (cuuint32_t)BK};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(a), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(SK_EINVAL, "cuTensorMapEncodeTiled(A^T) failed with CUresult " + std::to_string((int)r) +
                               " (alignment of A / lda?)");
  return SK_OK;
}

struct Plan {
  int BN, nblocks, ksplit, kb_per_split, mtiles, units, stages, astages;
  size_t smem, ws_bytes;
};

Plan make_plan(int64_t n, int64_t d, int64_t k, int NB, bool wide_b = false) {
  Plan pl{};
  // N blocks of at most 256 columns (two TMEM accumulators of BN columns each), BN % 16 == 0; a
  // split B doubles the B tile, so it keeps 128 columns unless re-reading A per N block would cost
  // more than the shallower ring (wide_b: the TN product, whose A strip is the big operand)
  const int64_t bn_max = (NB == 2 && !wide_b) ? 128 : 256;
  pl.nblocks = (int)((k + bn_max - 1) / bn_max);
  const int64_t per = (k + pl.nblocks - 1) / pl.nblocks;
  pl.BN = (int)((per + 15) / 16 * 16);  // UMMA N (M = 128) is any multiple of 16
  pl.mtiles = (int)((n + BM - 1) / BM);
  const int nk = (int)((d + BK - 1) / BK);
  const int tiles = pl.mtiles * pl.nblocks;
  const int sms = sm_count();
  // split K when there are too few tiles to keep every SM busy (each split >= 4 chunks)
  int ks = 1;
  while (tiles * ks < 4 * sms && (nk + 2 * ks - 1) / (2 * ks) >= 4 * CHUNK_KB) ks *= 2;
  pl.kb_per_split = (nk + ks - 1) / ks;
  pl.kb_per_split = (pl.kb_per_split + CHUNK_KB - 1) / CHUNK_KB * CHUNK_KB;
  pl.ksplit = (nk + pl.kb_per_split - 1) / pl.kb_per_split;
  pl.units = tiles * pl.ksplit;
  const size_t stage_bytes = kAStageBytes + (size_t)NB * pl.BN * 128;
  const size_t budget = 227 * 1024 - 1024 - 512;
  int stages = (int)(budget / stage_bytes);
  if (stages > 6) stages = 6;
  pl.stages = stages;
  pl.astages = 0;
  pl.smem = 1024 + stages * stage_bytes + (3 * stages + 4) * 8 + 16;
  pl.ws_bytes = pl.ksplit > 1 ? (size_t)pl.ksplit * n * k * sizeof(float) : 0;
  return pl;
}

// CTA-pair plan: units = (pair of M tiles, N block, K split), BN <= 256 (TMEM: two
// accumulators of BN columns in each CTA), each CTA stages BN/2 rows of B^T per stage.
Plan make_plan_pair(int64_t n, int64_t d, int64_t k, int NB) {
  Plan pl{};
  pl.nblocks = (int)((k + 255) / 256);
  const int64_t per = (k + pl.nblocks - 1) / pl.nblocks;
  pl.BN = (int)((per + 15) / 16 * 16);  // cta_group::2: N % 16 == 0, so each half is a multiple of 8 rows
  pl.mtiles = (int)((n + 2 * BM - 1) / (2 * BM));  // M-tile pairs
  const int nk = (int)((d + BK - 1) / BK);
  const int tiles = pl.mtiles * pl.nblocks;
  const int pairs = sm_count() / 2;
  int ks = 1;
  while (tiles * ks < 4 * pairs && (nk + 2 * ks - 1) / (2 * ks) >= 4 * CHUNK_KB) ks *= 2;
  pl.kb_per_split = (nk + ks - 1) / ks;
  pl.kb_per_split = (pl.kb_per_split + CHUNK_KB - 1) / CHUNK_KB * CHUNK_KB;
  pl.ksplit = (nk + pl.kb_per_split - 1) / pl.kb_per_split;
  pl.units = tiles * pl.ksplit;
  const size_t stage_bytes = kAStageBytes + (size_t)NB * (pl.BN / 2) * 128;
  const size_t budget = 227 * 1024 - 1024 - 512;
  int stages = (int)(budget / stage_bytes);
  if (stages > 6) stages = 6;
  pl.stages = stages;
  pl.astages = 0;
  pl.smem = 1024 + stages * stage_bytes + (3 * stages + 5) * 8 + 16;
  pl.ws_bytes = pl.ksplit > 1 ? (size_t)pl.ksplit * n * k * sizeof(float) : 0;
  return pl;
}

bool use_pair(int64_t n) {
  if (n <= BM) return false;
  const char* e = getenv("SKETCH_B200_TC_PAIR");
  return !(e && e[0] == '0');
}

// launch the CTA-pair engine: a persistent grid of the co-resident 2-CTA clusters
int launch_pair(int NB, bool TA, const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mbl, TcParams& p,
                size_t smem, cudaStream_t s) {
  using KernT = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const TcParams);
  KernT kern = TA ? (NB == 2 ? dense_tc_pair_kernel<2, true, 0> : dense_tc_pair_kernel<1, true, 0>)
                  : (NB == 2 ? dense_tc_pair_kernel<2, false, 0> : dense_tc_pair_kernel<1, false, 0>);
  allow_smem(kern, smem);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(2 * (sm_count() / 2)));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // persistent grid = the clusters that can be co-resident (GPCs with an odd SM count leave an
  // SM without a partner, so this can be below sm_count() / 2)
  static std::atomic<int> max_clusters_v[4] = {};
  int max_clusters = max_clusters_v[(NB - 1) + 2 * (TA ? 1 : 0)].load(std::memory_order_relaxed);
  if (max_clusters == 0) {
    int mc = 0;
    if (cudaOccupancyMaxActiveClusters(&mc, kern, &cfg) != cudaSuccess || mc < 1) {
      cudaGetLastError();
      mc = sm_count() / 2;
    }
    max_clusters = mc;
    max_clusters_v[(NB - 1) + 2 * (TA ? 1 : 0)].store(mc, std::memory_order_relaxed);
    if (getenv("SKETCH_B200_TC_PAIR_VERBOSE")) fprintf(stderr, "dense_tc pair: %d co-resident clusters\n", mc);
  }
  const int npairs = p.num_units < max_clusters ? p.num_units : max_clusters;
  cfg.gridDim = dim3((unsigned)(2 * npairs));
  return cudaLaunchKernelEx(&cfg, kern, ma, mb, mbl, p) == cudaSuccess ? SK_OK : SK_ECUDA;
}

// ------------------------------------------------------------------------------------ Khatri-Rao
// Y = scale * sum_P (A[:, P, :] F) * W[P, :] on the CTA-pair engine with F resident (KR = true).
// A viewed as 3-D (q < dl, P, row) [TA: (col, q, P)], box 64 x 1 x 128: q >= dl is zero-filled,
// so dl need not be a multiple of 64 (dl % 4 == 0 for the TMA strides).
int make_a3_map(CUtensorMap* m, const float* a, int64_t rows, int64_t P, int64_t dl, int64_t lda, bool ta) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(SK_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3], strides[2];
  cuuint32_t box[3];
  if (!ta) {  // A [rows][P * dl]: (q, P, row)
    dims[0] = (cuuint64_t)dl; dims[1] = (cuuint64_t)P; dims[2] = (cuuint64_t)rows;
    strides[0] = (cuuint64_t)dl * 4; strides[1] = (cuuint64_t)lda * 4;
    box[0] = BK; box[1] = 1; box[2] = BM;
  } else {    // B [P * dl][rows]: (col, q, P)
    dims[0] = (cuuint64_t)rows; dims[1] = (cuuint64_t)dl; dims[2] = (cuuint64_t)P;
    strides[0] = (cuuint64_t)lda * 4; strides[1] = (cuuint64_t)dl * lda * 4;
    box[0] = BM; box[1] = BK; box[2] = 1;
  }
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(a), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SK_EINVAL, "cuTensorMapEncodeTiled(KR A) failed (alignment of A / lda / dl?)");
  return SK_OK;
}

constexpr int kKrMaxCols = 2048;  // columns per launch (N blocks <= 8, one group of pairs per block)

struct KrPlan {
  int BN, nblocks, qb, ksplit, kb_per_split, mtiles, stages, npairs;
  size_t smem, ws_bytes;
};

using KernT = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const TcParams);
KernT kr_kernel(int NB, bool TA, bool wsign = false) {
  if (wsign)
    return TA ? (NB == 2 ? dense_tc_pair_kernel<2, true, 3> : dense_tc_pair_kernel<1, true, 3>)
              : (NB == 2 ? dense_tc_pair_kernel<2, false, 3> : dense_tc_pair_kernel<1, false, 3>);
  return TA ? (NB == 2 ? dense_tc_pair_kernel<2, true, 1> : dense_tc_pair_kernel<1, true, 1>)
            : (NB == 2 ? dense_tc_pair_kernel<2, false, 1> : dense_tc_pair_kernel<1, false, 1>);
}

// co-resident 2-CTA clusters of a KR kernel at this shared-memory size
int kr_max_clusters(KernT kern, size_t smem) {
  allow_smem(kern, smem);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(2 * (sm_count() / 2)));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int mc = 0;
  if (cudaOccupancyMaxActiveClusters(&mc, kern, &cfg) != cudaSuccess || mc < 1) {
    cudaGetLastError();
    mc = sm_count() / 2;
  }
  return mc;
}

// kslab = columns of this launch (<= kKrMaxCols); maxc <= 0: no device query (workspace sizing)
bool make_plan_kr(KrPlan& pl, int64_t n, int64_t P, int64_t dl, int64_t kslab, int NB, int maxc, bool ta) {
  pl = KrPlan{};
  pl.qb = (int)((dl + BK - 1) / BK);
  pl.nblocks = (int)((kslab + 255) / 256);
  const size_t budget = 227 * 1024 - 1024 - 512;
  size_t res = 0;
  for (;;) {  // resident F^T halves: shrink the N block until they fit next to >= 2 A stages
    const int64_t per = (kslab + pl.nblocks - 1) / pl.nblocks;
    pl.BN = (int)((per + 15) / 16 * 16);
    res = (size_t)NB * pl.qb * (pl.BN / 2) * 128;
    if (res <= 160 * 1024) break;
    if (pl.BN <= 32) return false;
    pl.nblocks *= 2;
  }
  int stages = (int)((budget - res) / kAStageBytes);
  if (stages > 6) stages = 6;  // config 5: 5 stages (measured 1.77 ms; 4: 1.95, 3: 1.83, 2: 2.30)
  pl.stages = stages;
  pl.smem = 1024 + (size_t)stages * kAStageBytes + res + (3 * stages + 5) * 8 + 16;
  pl.mtiles = (int)((n + 2 * BM - 1) / (2 * BM));
  const int mc = maxc > 0 ? maxc : sm_count() / 2;
  const int gp = mc / pl.nblocks > 0 ? mc / pl.nblocks : 1;  // pairs per N-block group
  int ks = 1;
  while ((int64_t)pl.mtiles * ks < 4 * gp && P / (2 * ks) >= 2) ks *= 2;
  const int64_t p_per = (P + ks - 1) / ks;
  pl.kb_per_split = (int)(p_per * pl.qb);
  pl.ksplit = (int)((P + p_per - 1) / p_per);
  const int64_t work = (int64_t)pl.mtiles * pl.ksplit;
  pl.npairs = (int)((work < gp ? work : gp) * pl.nblocks);
  pl.ws_bytes = (pl.ksplit > 1 || ta) ? (size_t)pl.ksplit * n * kslab * sizeof(float) : 0;
  return true;
}

constexpr size_t kKrProgressBytes = 2048;  // one int per CTA (<= 512 CTAs)
size_t kr_workspace(int64_t n, int64_t P, int64_t dl, int64_t k, int NB, bool ta) {
  size_t ws = 0;
  for (int64_t c0 = 0; c0 < k; c0 += kKrMaxCols) {
    const int64_t ks = k - c0 < kKrMaxCols ? k - c0 : kKrMaxCols;
    KrPlan pl, pl1;
    if (!make_plan_kr(pl, n, P, dl, ks, NB, -1, ta)) return 0;
    // the real grid may hold fewer pairs per group (more K splits): size for 2 pairs per group too
    make_plan_kr(pl1, n, P, dl, ks, NB, 2 * pl.nblocks, ta);
    const size_t w = pl.ws_bytes > pl1.ws_bytes ? pl.ws_bytes : pl1.ws_bytes;
    if (w > ws) ws = w;
  }
  return ((ws + 255) & ~(size_t)255) + kKrProgressBytes;  // + the lockstep counters
}

// rows: output rows (A rows, or B columns when TA); out: Y [rows][k] (ldy) or, when TA, X [k][rows]
int kr_run(bool TA, const float* A, int64_t rows, int64_t P, int64_t dl, int64_t lda, const uint16_t* ft_hi,
           const uint16_t* ft_lo, int64_t ldf, const float* W, int64_t ldw, int64_t k, double scale, float* Y,
           int64_t ldy, void* ws, size_t ws_bytes, cudaStream_t s, const char* what,
           const uint32_t* wbits = nullptr, int64_t ldwb = 0, double wabs = 1.0) {
  const int NB = ft_lo ? 2 : 1;
  CUtensorMap ma;
  // dl % 64 == 0: the plain 2-D map (measured faster than the 3-D box: config 5 2.14 -> 1.87 ms)
  const bool a2d = dl % BK == 0;
  int st = a2d ? (TA ? make_at_map(&ma, A, rows, P * dl, lda) : make_a_map(&ma, A, rows, P * dl, lda))
               : make_a3_map(&ma, A, rows, P, dl, lda, TA);
  if (st != SK_OK) return st;
  for (int64_t c0 = 0; c0 < k; c0 += kKrMaxCols) {
    const int64_t kslab = k - c0 < kKrMaxCols ? k - c0 : kKrMaxCols;
    KrPlan pl;
    if (!make_plan_kr(pl, rows, P, dl, kslab, NB, -1, TA))
      return fail(SK_EUNSUPPORTED, std::string(what) + ": resident factor does not fit shared memory");
    // sign-bit weights when every reducer half starts on a 32-column boundary (the BN of the first plan
    // is the one launched: the second plan only changes the pair count and K split)
    const bool use_bits = wbits != nullptr && pl.BN % 64 == 0 && c0 % 32 == 0;
    KernT kern = kr_kernel(NB, TA, use_bits);
    // co-resident pairs per (kernel, smem) — a small cache guarded for concurrent host threads
    static std::mutex maxc_mu;
    static KernT maxc_kern[8] = {};
    static size_t maxc_smem[8] = {};
    static int maxc_val[8] = {};
    int maxc = 0;
    {
      std::lock_guard<std::mutex> lk(maxc_mu);
      int slot = 0;
      while (slot < 7 && maxc_kern[slot] && !(maxc_kern[slot] == kern && maxc_smem[slot] == pl.smem)) ++slot;
      if (maxc_kern[slot] != kern || maxc_smem[slot] != pl.smem) {
        maxc_kern[slot] = kern;
        maxc_smem[slot] = pl.smem;
        maxc_val[slot] = kr_max_clusters(kern, pl.smem);
      }
      maxc = maxc_val[slot];
    }
    if (maxc < pl.nblocks) return fail(SK_EUNSUPPORTED, std::string(what) + ": too few co-resident pairs");
    make_plan_kr(pl, rows, P, dl, kslab, NB, maxc, TA);
    if (pl.ws_bytes > 0 && (ws == nullptr || ws_bytes < pl.ws_bytes))
      return fail(SK_EINVAL, std::string(what) + ": workspace too small (sk_kr_workspace_bytes)");
    // lockstep counters after the partials when the caller's workspace has room (sk_kr_workspace_bytes)
    int* progress = nullptr;
    const size_t prog_off = (pl.ws_bytes + 255) & ~(size_t)255;
    if (ws != nullptr && pl.nblocks > 1 && 2 * pl.npairs * sizeof(int) <= kKrProgressBytes &&
        ws_bytes >= prog_off + kKrProgressBytes && std::getenv("SKETCH_B200_KR_LOCKSTEP") == nullptr) {
      progress = reinterpret_cast<int*>(static_cast<uint8_t*>(ws) + prog_off);
      if (cudaMemsetAsync(progress, 0, 2 * pl.npairs * sizeof(int), s) != cudaSuccess) return check_launch(what);
    }
    CUtensorMap mb, mbl;
    st = make_bt_map(&mb, ft_hi + c0 * ldf, kslab, dl, ldf, pl.BN / 2);
    if (st != SK_OK) return st;
    if (NB == 2) {
      st = make_bt_map(&mbl, ft_lo + c0 * ldf, kslab, dl, ldf, pl.BN / 2);
      if (st != SK_OK) return st;
    } else {
      mbl = mb;
    }
    TcParams p{};
    p.A = A;
    p.M = rows;
    p.K = P * (int64_t)pl.qb * BK;
    p.lda = lda;
    p.N = (int)kslab;
    p.BN = pl.BN;
    p.nblocks = pl.nblocks;
    p.ksplit = pl.ksplit;
    p.kb_per_split = pl.kb_per_split;
    p.stages = pl.stages;
    p.scale = (float)scale;
    p.Y = TA ? Y + c0 * ldy : Y + c0;
    p.ldy = ldy;
    p.part = static_cast<float*>(ws);
    p.num_units = pl.mtiles * pl.ksplit * pl.nblocks;
    p.mtiles = pl.mtiles;
    p.kr_w = W + c0;
    p.kr_ldw = ldw;
    p.kr_progress = progress;
    if (use_bits) {
      p.kr_wbits = wbits + c0 / 32;
      p.kr_ldwb = ldwb;
      p.scale = (float)(scale * wabs);
    }
    p.kr_qb = pl.qb;
    p.kr_ngroups = pl.nblocks;
    p.out_t = TA ? 1 : 0;
    p.kr_a2d = a2d ? 1 : 0;
    uint32_t cols = 32;
    while (cols < (uint32_t)(2 * pl.BN)) cols <<= 1;
    p.tmem_cols = cols;
    allow_smem(kern, pl.smem);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(2 * pl.npairs));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (getenv("SKETCH_B200_TC_PAIR_VERBOSE"))
      fprintf(stderr, "%s: BN %d nblocks %d ksplit %d kb/split %d stages %d pairs %d (max %d) smem %zu\n", what, pl.BN,
              pl.nblocks, pl.ksplit, pl.kb_per_split, pl.stages, pl.npairs, maxc, pl.smem);
    if (cudaLaunchKernelEx(&cfg, kern, ma, mb, mbl, p) != cudaSuccess) return check_launch(what);
    st = check_launch(what);
    if (st != SK_OK) return st;
    if (pl.ksplit > 1 || TA) {
      const int64_t total = rows * kslab;
      int64_t blocks = (total + 255) / 256;
      if (blocks > 8 * (int64_t)sm_count()) blocks = 8 * (int64_t)sm_count();
      tc_splitk_reduce<<<(unsigned)blocks, 256, 0, s>>>(p.part, pl.ksplit, rows, (int)kslab, (float)scale, p.Y, ldy,
                                                       p.out_t);
      st = check_launch(what);
      if (st != SK_OK) return st;
    }
  }
  return SK_OK;
}

int kr_check(const float* A, int64_t rows, int64_t P, int64_t dl, int64_t lda, int64_t minlda, int64_t k,
             const float* Y, int64_t ldy, int64_t minldy, const char* what) {
  if (rows < 0 || P < 1 || dl < 1 || k < 1 || lda < minlda || ldy < minldy)
    return fail(SK_EINVAL, std::string(what) + ": bad shape");
  if (!A || !Y) return fail(SK_EINVAL, std::string(what) + ": null pointer");
  if ((reinterpret_cast<uintptr_t>(A) & 15) || (lda & 3) || (dl & 3))
    return fail(SK_EINVAL, std::string(what) + ": A must be 16-byte aligned with lda, dl multiples of 4");
  return SK_OK;
}

int kr_check_f(const uint16_t* Ft_hi, const uint16_t* Ft_lo, int64_t ldf, int64_t dl, const float* W, int64_t ldw,
               int64_t k, const char* what) {
  if (!Ft_hi || !W || ldf < dl || ldw < k) return fail(SK_EINVAL, std::string(what) + ": bad factor operands");
  if ((reinterpret_cast<uintptr_t>(Ft_hi) & 15) || (ldf & 7) || (Ft_lo && (reinterpret_cast<uintptr_t>(Ft_lo) & 15)))
    return fail(SK_EINVAL, std::string(what) + ": F^T must be 16-byte aligned with ldf a multiple of 8");
  if ((reinterpret_cast<uintptr_t>(W) & 15) || (ldw & 3))
    return fail(SK_EINVAL, std::string(what) + ": W must be 16-byte aligned with ldw a multiple of 4");
  return SK_OK;
}

}  // namespace
}  // namespace skb

extern "C" int sk_dense_tc_supported(int64_t k) { return k >= 1 ? 1 : 0; }

extern "C" size_t sk_dense_tc_workspace_bytes(int64_t n, int64_t d, int64_t k, int split_b) {
  if (n < 1 || d < 1 || k < 1) return 0;
  const size_t a = skb::make_plan(n, d, k, split_b ? 2 : 1).ws_bytes;
  const size_t b = skb::use_pair(n) ? skb::make_plan_pair(n, d, k, split_b ? 2 : 1).ws_bytes : 0;
  return a > b ? a : b;
}

extern "C" int sk_dense_right_tc(const float* A, int64_t n, int64_t d, int64_t lda, const uint16_t* Bt_hi,
                                 const uint16_t* Bt_lo, int64_t ldb, int64_t k, double scale, float* Y, int64_t ldy,
                                 void* ws, size_t ws_bytes, void* stream) {
  using namespace skb;
  if (n < 0 || d < 1 || k < 1 || lda < d || ldb < d || ldy < k)
    return fail(SK_EINVAL, "sk_dense_right_tc: bad shape");
  if (n == 0) return SK_OK;
  if (!A || !Bt_hi || !Y) return fail(SK_EINVAL, "sk_dense_right_tc: null pointer");
  if ((reinterpret_cast<uintptr_t>(A) & 15) || (lda & 3) || (d & 3))
    return fail(SK_EINVAL, "sk_dense_right_tc: A must be 16-byte aligned with lda, d multiples of 4");
  if ((reinterpret_cast<uintptr_t>(Bt_hi) & 15) || (ldb & 7) || (Bt_lo && (reinterpret_cast<uintptr_t>(Bt_lo) & 15)))
    return fail(SK_EINVAL, "sk_dense_right_tc: B^T must be 16-byte aligned with ldb a multiple of 8");
  const int NB = Bt_lo ? 2 : 1;
  if (use_pair(n)) {
    const Plan pl = make_plan_pair(n, d, k, NB);
    if (pl.stages < 2) return fail(SK_EUNSUPPORTED, "sk_dense_right_tc: tile does not fit shared memory");
    if (pl.ksplit > 1 && (ws == nullptr || ws_bytes < pl.ws_bytes))
      return fail(SK_EINVAL, "sk_dense_right_tc: workspace too small (sk_dense_tc_workspace_bytes)");
    CUtensorMap ma, mb, mbl;
    int st = make_a_map(&ma, A, n, d, lda);
    if (st != SK_OK) return st;
    st = make_bt_map(&mb, Bt_hi, k, d, ldb, pl.BN / 2);
    if (st != SK_OK) return st;
    if (NB == 2) {
      st = make_bt_map(&mbl, Bt_lo, k, d, ldb, pl.BN / 2);
      if (st != SK_OK) return st;
    } else {
      mbl = mb;
    }
    TcParams p{};
    p.A = A;
    p.M = n;
    p.K = d;
    p.lda = lda;
    p.N = (int)k;
    p.BN = pl.BN;
    p.nblocks = pl.nblocks;
    p.ksplit = pl.ksplit;
    p.kb_per_split = pl.kb_per_split;
    p.stages = pl.stages;
    p.astages = 0;
    p.scale = (float)scale;
    p.Y = Y;
    p.ldy = ldy;
    p.part = static_cast<float*>(ws);
    p.num_units = pl.units;
    p.mtiles = pl.mtiles;
    uint32_t cols = 32;
    while (cols < (uint32_t)(2 * pl.BN)) cols <<= 1;
    p.tmem_cols = cols;
    cudaStream_t s = as_stream(stream);
    if (launch_pair(NB, false, ma, mb, mbl, p, pl.smem, s) != SK_OK) return check_launch("sk_dense_right_tc(pair)");
    st = check_launch("sk_dense_right_tc(pair)");
    if (st != SK_OK || pl.ksplit == 1) return st;
    const int64_t total = n * k;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 8 * (int64_t)sm_count()) blocks = 8 * (int64_t)sm_count();
    tc_splitk_reduce<<<(unsigned)blocks, 256, 0, s>>>(p.part, pl.ksplit, n, (int)k, (float)scale, Y, ldy);
    return check_launch("sk_dense_right_tc(reduce)");
  }
  const Plan pl = make_plan(n, d, k, NB);
  if (pl.stages < 2) return fail(SK_EUNSUPPORTED, "sk_dense_right_tc: tile does not fit shared memory");
  if (pl.ksplit > 1 && (ws == nullptr || ws_bytes < pl.ws_bytes))
    return fail(SK_EINVAL, "sk_dense_right_tc: workspace too small (sk_dense_tc_workspace_bytes)");
  CUtensorMap ma, mh, ml;
  int st = make_a_map(&ma, A, n, d, lda);
  if (st != SK_OK) return st;
  st = make_bt_map(&mh, Bt_hi, k, d, ldb, pl.BN);
  if (st != SK_OK) return st;
  if (NB == 2) {
    st = make_bt_map(&ml, Bt_lo, k, d, ldb, pl.BN);
    if (st != SK_OK) return st;
  } else {
    ml = mh;
  }
  TcParams p{};
  p.A = A;
  p.M = n;
  p.K = d;
  p.lda = lda;
  p.N = (int)k;
  p.BN = pl.BN;
  p.nblocks = pl.nblocks;
  p.ksplit = pl.ksplit;
  p.kb_per_split = pl.kb_per_split;
  p.stages = pl.stages;
  p.astages = pl.astages;
  p.scale = (float)scale;
  p.Y = Y;
  p.ldy = ldy;
  p.part = static_cast<float*>(ws);
  p.num_units = pl.units;
  p.mtiles = pl.mtiles;
  uint32_t cols = 32;
  while (cols < (uint32_t)(2 * pl.BN)) cols <<= 1;
  p.tmem_cols = cols;
  cudaStream_t s = as_stream(stream);
  const int grid = pl.units < sm_count() ? pl.units : sm_count();
  if (NB == 1) {
    allow_smem(dense_tc_kernel<1, false>, pl.smem);
    dense_tc_kernel<1, false><<<grid, kThreads, pl.smem, s>>>(ma, mh, ml, p);
  } else {
    allow_smem(dense_tc_kernel<2, false>, pl.smem);
    dense_tc_kernel<2, false><<<grid, kThreads, pl.smem, s>>>(ma, mh, ml, p);
  }
  st = check_launch("sk_dense_right_tc");
  if (st != SK_OK || pl.ksplit == 1) return st;
  const int64_t total = n * k;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 8 * (int64_t)sm_count()) blocks = 8 * (int64_t)sm_count();
  tc_splitk_reduce<<<(unsigned)blocks, 256, 0, s>>>(p.part, pl.ksplit, n, (int)k, (float)scale, Y, ldy);
  return check_launch("sk_dense_right_tc(reduce)");
}

extern "C" size_t sk_dense_tn_tc_workspace_bytes(int64_t n, int64_t d, int64_t k) {
  if (n < 1 || d < 1 || k < 1) return 0;
  const size_t a = skb::make_plan(d, n, k, 2, true).ws_bytes;
  const size_t b = skb::use_pair(d) ? skb::make_plan_pair(d, n, k, 2).ws_bytes : 0;
  return a > b ? a : b;
}

// Y[d, k] = scale * A^T W  for A [n rows][d cols] fp32 and W [n][k] given as W^T = Wt (k rows of n,
// bf16 hi + lo, row stride ldw): the rsvd product B^T = A^T Q (reference rand_nla.py:104) on the
// tensor cores with BF16x3 (A hi/lo x W hi, A hi x W lo).
extern "C" int sk_dense_tn_tc(const float* A, int64_t n, int64_t d, int64_t lda, const uint16_t* Wt_hi,
                              const uint16_t* Wt_lo, int64_t ldw, int64_t k, double scale, float* Y, int64_t ldy,
                              void* ws, size_t ws_bytes, void* stream) {
  using namespace skb;
  if (n < 1 || d < 1 || k < 1 || lda < d || ldw < n || ldy < k) return fail(SK_EINVAL, "sk_dense_tn_tc: bad shape");
  if (!A || !Wt_hi || !Wt_lo || !Y) return fail(SK_EINVAL, "sk_dense_tn_tc: null pointer");
  if ((reinterpret_cast<uintptr_t>(A) & 15) || (lda & 3) || (d & 3))
    return fail(SK_EINVAL, "sk_dense_tn_tc: A must be 16-byte aligned with lda, d multiples of 4");
  if ((reinterpret_cast<uintptr_t>(Wt_hi) & 15) || (reinterpret_cast<uintptr_t>(Wt_lo) & 15) || (ldw & 7))
    return fail(SK_EINVAL, "sk_dense_tn_tc: W^T must be 16-byte aligned with ldw a multiple of 8");
  if (use_pair(d)) {  // CTA pairs (cta_group::2), B^T split by N between the pair
    const Plan pl = make_plan_pair(d, n, k, 2);
    if (pl.stages < 2) return fail(SK_EUNSUPPORTED, "sk_dense_tn_tc: tile does not fit shared memory");
    if (pl.ksplit > 1 && (ws == nullptr || ws_bytes < pl.ws_bytes))
      return fail(SK_EINVAL, "sk_dense_tn_tc: workspace too small (sk_dense_tn_tc_workspace_bytes)");
    CUtensorMap ma, mh, ml;
    int st = make_at_map(&ma, A, d, n, lda);
    if (st != SK_OK) return st;
    st = make_bt_map(&mh, Wt_hi, k, n, ldw, pl.BN / 2);
    if (st != SK_OK) return st;
    st = make_bt_map(&ml, Wt_lo, k, n, ldw, pl.BN / 2);
    if (st != SK_OK) return st;
    TcParams p{};
    p.A = A;
    p.M = d;
    p.K = n;
    p.lda = lda;
    p.N = (int)k;
    p.BN = pl.BN;
    p.nblocks = pl.nblocks;
    p.ksplit = pl.ksplit;
    p.kb_per_split = pl.kb_per_split;
    p.stages = pl.stages;
    p.astages = 0;
    p.scale = (float)scale;
    p.Y = Y;
    p.ldy = ldy;
    p.part = static_cast<float*>(ws);
    p.num_units = pl.units;
    p.mtiles = pl.mtiles;
    uint32_t cols = 32;
    while (cols < (uint32_t)(2 * pl.BN)) cols <<= 1;
    p.tmem_cols = cols;
    cudaStream_t s = as_stream(stream);
    if (launch_pair(2, true, ma, mh, ml, p, pl.smem, s) != SK_OK) return check_launch("sk_dense_tn_tc(pair)");
    st = check_launch("sk_dense_tn_tc(pair)");
    if (st != SK_OK || pl.ksplit == 1) return st;
    const int64_t total = d * k;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 8 * (int64_t)sm_count()) blocks = 8 * (int64_t)sm_count();
    tc_splitk_reduce<<<(unsigned)blocks, 256, 0, s>>>(p.part, pl.ksplit, d, (int)k, (float)scale, Y, ldy);
    return check_launch("sk_dense_tn_tc(reduce)");
  }
  const Plan pl = make_plan(d, n, k, 2, true);
  if (pl.stages < 2) return fail(SK_EUNSUPPORTED, "sk_dense_tn_tc: tile does not fit shared memory");
  if (pl.ksplit > 1 && (ws == nullptr || ws_bytes < pl.ws_bytes))
    return fail(SK_EINVAL, "sk_dense_tn_tc: workspace too small (sk_dense_tn_tc_workspace_bytes)");
  CUtensorMap ma, mh, ml;
  int st = make_at_map(&ma, A, d, n, lda);
  if (st != SK_OK) return st;
  st = make_bt_map(&mh, Wt_hi, k, n, ldw, pl.BN);
  if (st != SK_OK) return st;
  st = make_bt_map(&ml, Wt_lo, k, n, ldw, pl.BN);
  if (st != SK_OK) return st;
  TcParams p{};
  p.A = A;
  p.M = d;
  p.K = n;
  p.lda = lda;
  p.N = (int)k;
  p.BN = pl.BN;
  p.nblocks = pl.nblocks;
  p.ksplit = pl.ksplit;
  p.kb_per_split = pl.kb_per_split;
  p.stages = pl.stages;
  p.astages = pl.astages;
  p.scale = (float)scale;
  p.Y = Y;
  p.ldy = ldy;
  p.part = static_cast<float*>(ws);
  p.num_units = pl.units;
  p.mtiles = pl.mtiles;
  uint32_t cols = 32;
  while (cols < (uint32_t)(2 * pl.BN)) cols <<= 1;
  p.tmem_cols = cols;
  cudaStream_t s = as_stream(stream);
  const int grid = pl.units < sm_count() ? pl.units : sm_count();
  allow_smem(dense_tc_kernel<2, true>, pl.smem);
  dense_tc_kernel<2, true><<<grid, kThreads, pl.smem, s>>>(ma, mh, ml, p);
  st = check_launch("sk_dense_tn_tc");
  if (st != SK_OK || pl.ksplit == 1) return st;
  const int64_t total = d * k;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 8 * (int64_t)sm_count()) blocks = 8 * (int64_t)sm_count();
  tc_splitk_reduce<<<(unsigned)blocks, 256, 0, s>>>(p.part, pl.ksplit, d, (int)k, (float)scale, Y, ldy);
  return check_launch("sk_dense_tn_tc(reduce)");
}

// ------------------------------------------------------------------------------------ Khatri-Rao C ABI
// trans = 0: sk_kr_right with n rows; trans = 1: sk_kr_adjoint with n = m columns of B
extern "C" size_t sk_kr_workspace_bytes(int64_t n, int64_t P, int64_t dl, int64_t k, int split_f, int trans) {
  if (n < 1 || P < 1 || dl < 1 || k < 1) return 0;
  return skb::kr_workspace(n, P, dl, k, split_f ? 2 : 1, trans != 0);
}

// Y[n, k] = scale * sum_{P, q} A[i, P * dl + q] * W[P, j] * F[q, j]   (Khatri-Rao, Omega never formed)
extern "C" int sk_kr_right(const float* A, int64_t n, int64_t P, int64_t dl, int64_t lda, const uint16_t* Ft_hi,
                           const uint16_t* Ft_lo, int64_t ldf, const float* W, int64_t ldw, int64_t k, double scale,
                           float* Y, int64_t ldy, void* ws, size_t ws_bytes, void* stream) {
  using namespace skb;
  int st = kr_check(A, n, P, dl, lda, P * dl, k, Y, ldy, k, "sk_kr_right");
  if (st == SK_OK) st = kr_check_f(Ft_hi, Ft_lo, ldf, dl, W, ldw, k, "sk_kr_right");
  if (st != SK_OK || n == 0) return st;
  return kr_run(false, A, n, P, dl, lda, Ft_hi, Ft_lo, ldf, W, ldw, k, scale, Y, ldy, ws, ws_bytes, as_stream(stream),
                "sk_kr_right");
}

// sk_kr_right with +-1 column weights given as sign bits (W[P, j] = wabs * (1 - 2 * bit)), e.g. the
// Rademacher factors of BASELINE config 5; W (float32, the same values) serves N blocks that do not
// start on 32-column boundaries.
extern "C" int sk_kr_right_signs(const float* A, int64_t n, int64_t P, int64_t dl, int64_t lda, const uint16_t* Ft_hi,
                                 const uint16_t* Ft_lo, int64_t ldf, const float* W, int64_t ldw, const uint32_t* Wbits,
                                 int64_t ldwb, double wabs, int64_t k, double scale, float* Y, int64_t ldy, void* ws,
                                 size_t ws_bytes, void* stream) {
  using namespace skb;
  int st = kr_check(A, n, P, dl, lda, P * dl, k, Y, ldy, k, "sk_kr_right_signs");
  if (st == SK_OK && (!Wbits || ldwb < (k + 31) / 32)) st = fail(SK_EINVAL, "sk_kr_right_signs: bad sign words");
  if (st == SK_OK) st = kr_check_f(Ft_hi, Ft_lo, ldf, dl, W, ldw, k, "sk_kr_right_signs");
  if (st != SK_OK || n == 0) return st;
  return kr_run(false, A, n, P, dl, lda, Ft_hi, Ft_lo, ldf, W, ldw, k, scale, Y, ldy, ws, ws_bytes, as_stream(stream),
                "sk_kr_right_signs", Wbits, ldwb, wabs);
}

// X[k, m] = scale * Omega^T B for B [P * dl rows][m] (row stride ldb), read in place (no transposed copy)
extern "C" int sk_kr_adjoint(const float* B, int64_t m, int64_t P, int64_t dl, int64_t ldb, const uint16_t* Ft_hi,
                             const uint16_t* Ft_lo, int64_t ldf, const float* W, int64_t ldw, int64_t k,
                             double scale, float* X, int64_t ldx, void* ws, size_t ws_bytes, void* stream) {
  using namespace skb;
  int st = kr_check(B, m, P, dl, ldb, m, k, X, ldx, m, "sk_kr_adjoint");
  if (st == SK_OK) st = kr_check_f(Ft_hi, Ft_lo, ldf, dl, W, ldw, k, "sk_kr_adjoint");
  if (st != SK_OK || m == 0) return st;
  return kr_run(true, B, m, P, dl, ldb, Ft_hi, Ft_lo, ldf, W, ldw, k, scale, X, ldx, ws, ws_bytes, as_stream(stream),
                "sk_kr_adjoint");
}
