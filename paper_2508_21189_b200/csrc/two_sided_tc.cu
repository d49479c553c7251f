// K6 — fused two-sided sketch on tcgen05:  Y = sy * A Omega  and  X^T = sx * Psi^T A  from ONE read of A.
//
// The generalized-Nystrom drivers need both sketches of the same A (reference rand_nla.py:191-202,
// 230-245: `_sketch_right(a, omega)` and `_sketch_left_adjoint(a, psi)`); run separately they
// stream A twice, and the sparse adjoint re-reads every row of A once per target from L2.  Here each
// 128 x 64 fp32 tile of A lands once in shared memory (TMA), is split into bf16 hi + lo by the
// converter warps, and feeds two tensor-core products:
//
//   MMA1 (right):   Y[buf]   (128 rows x N1 = k)   += A_tile (K-major, M = rows)      x Omega^T tile
//   MMA2 (adjoint): XT[:,kb] (128 targets x 64 col) += PsiT (K-major, K = the 128 rows) x A_tile (as the
//                   MN-major B operand: the same SWIZZLE_128B bytes, read with K = rows, N = columns)
//
// Psi is a sparse sign matrix (zeta targets per row of A, p <= 128 targets): warps 2-3 synthesise the
// exact +-1 bf16 PsiT tile of each 128-row M-tile in shared memory (double-buffered).  A is split hi/lo
// for both products (BF16x2: ~3e-6); Omega^T is bf16 hi (+ lo when it is not exact in bf16).
//
// Columns: a CTA owns a column group of <= 256 columns of A (XT for them stays resident in TMEM across
// its M-tiles); with G > 1 column groups every CTA adds its partial Y with red.global.add into a
// zeroed Y (G = 2: exactly two addends onto zero -> order-independent).  XT is folded from TMEM into
// fp32 registers every kFold M-tiles (bounded tcgen05 accumulation chains, as K-TC) and each CTA writes
// its XT partial; a fixed-order reduction forms X^T.
//
// CTA = 512 threads: warp 0 TMA producer | warp 1 MMA issuer | warps 2-3 PsiT synthesis (warp 2 also
// allocates TMEM) | warps 4-7 A converters | warps 8-15 epilogue (Y tiles, XT folds).
#include <cuda.h>

#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "sm100.cuh"

namespace skb {
namespace {

using namespace sm100;

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kThreads = 512;
constexpr int kColsPerGroup = 256;   // columns of A per CTA column group (4 k-blocks)
constexpr int kFold = 8;             // M-tiles per XT chunk in TMEM (K = 1024 rows)
constexpr uint32_t kAStage = BM * BK * 4;  // fp32 staging, converted in place to bf16 hi [0,16K) + lo [16K,32K)
constexpr uint32_t kPsiBytes = BM * BM * 2;  // PsiT tile: 2 sub-tiles [128 q][64 rows] bf16 (SW128 K-major)

struct TsParams {
  const float* A;
  int64_t n, d, lda;
  int k;                 // columns of Y (<= 128)
  int NY;                // MMA1 N (k rounded up to 16)
  int ncg;               // column groups
  int p;                 // targets (<= 128)
  int zeta;
  const uint8_t* psi;    // [n][zeta]: target q (7 bits) | neg << 7
  float sy, sx;
  float* Y;              // [n][k] (zeroed beforehand when ncg > 1)
  int64_t ldy;
  float* xpart;          // [grid][128][kColsPerGroup] XT partials
  int mtiles;
  int stages;
  int ctas_per_group;
  int nb;                // Omega^T operands: 1 (hi) or 2 (hi + lo)
  int omega_res;         // 1: the column group's Omega^T tiles stay resident in shared memory (loaded once)
  int dbg;               // timing experiments (SKETCH_B200_TS_DBG): 1 no MMA2, 2 no PsiT writes, 4 no Y stores,
                         // 16 per-lane row adds instead of the lane-pair sector adds
};

template <int N>
__device__ __forceinline__ void setmaxnreg_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}
template <int N>
__device__ __forceinline__ void setmaxnreg_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ void sts16(uint32_t addr, uint16_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"(v) : "memory");
}
__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

// MN-major SWIZZLE_128B descriptor (B operand read with N contiguous): 8 K-rows x 64 N-elements per
// 1024-byte atom; K steps between atoms of 1024 B.  N = 64 fits one atom, so both byte offsets are set
// to the atom stride.
__device__ __forceinline__ uint64_t sdesc_mnmajor_sw128(uint32_t saddr, uint32_t n_stride = 1024) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((n_stride >> 4) & 0x3FFF) << 16;  // LBO: the next 64 N-elements (another stage for N = 128)
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// kind::f16 instruction descriptor with B MN-major (transpose B, bit 16)
__host__ __device__ constexpr uint32_t idesc_bf16_f32_bmn(int M, int N) {
  return idesc_bf16_f32(M, N) | (1u << 16);
}

__global__ void __launch_bounds__(kThreads, 1)
    two_sided_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                     const __grid_constant__ CUtensorMap tm_blo, const TsParams p) {
  extern __shared__ uint8_t smem_dyn[];
  uint8_t* smem = smem_dyn + ((1024u - (smem_u32(smem_dyn) & 1023u)) & 1023u);
  const uint32_t b_bytes = (uint32_t)p.NY * 128;        // Omega^T tile: NY rows x 64 (K) bf16
  const uint32_t om_kb = (uint32_t)p.nb * b_bytes;      // one k-block of Omega^T (hi [+ lo])
  const uint32_t stage_bytes = kAStage + (p.omega_res ? 0u : om_kb);
  const int S = p.stages;
  uint8_t* om_buf = smem + (size_t)S * stage_bytes;     // resident Omega^T: [4 k-blocks][hi, lo]
  uint8_t* psi_buf = om_buf + (p.omega_res ? 4 * (size_t)om_kb : 0);  // [2][kPsiBytes]
  uint64_t* bars = reinterpret_cast<uint64_t*>(psi_buf + 2 * kPsiBytes);
  uint64_t* tma_full = bars;           // [S]
  uint64_t* full = tma_full + S;       // [S] converted (4 converter warps)
  uint64_t* empty = full + S;          // [S] consumed (MMA commit)
  uint64_t* psi_full = empty + S;      // [2] synthesised (2 warps)
  uint64_t* psi_empty = psi_full + 2;  // [2] MMA2 done with the tile (commit)
  uint64_t* y_full = psi_empty + 2;    // [2] Y tile complete (commit)
  uint64_t* y_empty = y_full + 2;      // [2] Y tile drained (8 epilogue warps)
  uint64_t* xt_full = y_empty + 2;     // XT chunk complete (commit)
  uint64_t* xt_empty = xt_full + 1;    // XT folded (8 epilogue warps)
  uint64_t* om_full = xt_empty + 1;    // resident Omega^T landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(om_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cg = blockIdx.x % p.ncg;                 // column group
  const int gi = blockIdx.x / p.ncg;                 // CTA index within the group
  const int per = (p.mtiles + p.ctas_per_group - 1) / p.ctas_per_group;
  const int t0 = gi * per, t1 = min(p.mtiles, t0 + per);
  const int c0 = cg * kColsPerGroup;
  const int nkb = (int)min((int64_t)kColsPerGroup / BK, (p.d - c0 + BK - 1) / BK);  // k-blocks of this group
  const int ntiles = t1 > t0 ? t1 - t0 : 0;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&tma_full[s], 1);
      mbar_init(&full[s], 4);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&psi_full[b], 2);
      mbar_init(&psi_empty[b], 1);
      mbar_init(&y_full[b], 1);
      mbar_init(&y_empty[b], 8);
    }
    mbar_init(xt_full, 1);
    mbar_init(xt_empty, 8);
    mbar_init(om_full, 1);
    fence_mbar_init();
    tma_prefetch_desc(&tm_a);
    tma_prefetch_desc(&tm_b);
    if (p.nb == 2) tma_prefetch_desc(&tm_blo);
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tm_xt = tmem;                       // XT: columns [0, 256)
  const uint32_t tm_y = tmem + kColsPerGroup;        // Y: 2 buffers of NY columns

  if (warp < 4) {
    setmaxnreg_dec<48>();
    if (warp == 0 && lane == 0) {
      // ---------------------------------------------------------------- TMA producer
      if (p.omega_res && ntiles > 0) {  // the group's Omega^T k-blocks, once
        mbar_arrive_expect_tx(om_full, (uint32_t)nkb * om_kb);
        for (int kb = 0; kb < nkb; ++kb) {
          tma_load_2d(om_buf + (size_t)kb * om_kb, &tm_b, om_full, c0 + kb * BK, 0);
          if (p.nb == 2) tma_load_2d(om_buf + (size_t)kb * om_kb + b_bytes, &tm_blo, om_full, c0 + kb * BK, 0);
        }
      }
      int s = 0;
      uint32_t ph = 0;
      for (int t = t0; t < t1; ++t)
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* st = smem + (size_t)s * stage_bytes;
          mbar_arrive_expect_tx(&tma_full[s], stage_bytes);
          tma_load_2d(st, &tm_a, &tma_full[s], c0 + kb * BK, t * BM);
          if (!p.omega_res) {
            tma_load_2d(st + kAStage, &tm_b, &tma_full[s], c0 + kb * BK, 0);
            if (p.nb == 2) tma_load_2d(st + kAStage + b_bytes, &tm_blo, &tma_full[s], c0 + kb * BK, 0);
          }
          if (++s == S) { s = 0; ph ^= 1; }
        }
    } else if (warp == 1 && lane == 0) {
      // ---------------------------------------------------------------- MMA issuer
      const uint32_t id1 = idesc_bf16_f32(BM, p.NY);
      const uint32_t id2 = idesc_bf16_f32_bmn(BM, BK);
      const uint32_t id2w = idesc_bf16_f32_bmn(BM, 2 * BK);
      const bool pairing = !(p.dbg & 8);
      if (p.omega_res && ntiles > 0) mbar_wait(om_full, 0);
      int s = 0;
      uint32_t ph = 0;
      for (int i = 0; i < ntiles; ++i) {
        const uint32_t pb = i & 1, pph = (i >> 1) & 1;
        const uint32_t yb = i & 1, yph = (i >> 1) & 1;
        mbar_wait(&psi_full[pb], pph);
        mbar_wait(&y_empty[yb], yph ^ 1);
        const bool fresh = (i % kFold) == 0;  // first M-tile of an XT chunk: overwrite the accumulators
        if (fresh && i > 0) mbar_wait(xt_empty, ((i / kFold) - 1) & 1);
        tc_fence_after();
        const uint64_t dps = sdesc_kmajor_sw128(smem_u32(psi_buf + pb * kPsiBytes));
        const uint32_t dy = tm_y + yb * (uint32_t)p.NY;
        int s_first = -1;  // first stage of a k-block pair held for one N = 128 MMA2
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t st = smem_u32(smem + (size_t)s * stage_bytes);
          // descriptors built once per stage; a K step adds (bytes >> 4) to the 14-bit start address
          const uint64_t dah = sdesc_kmajor_sw128(st), dal = sdesc_kmajor_sw128(st + BM * 128);
          const uint32_t ob = p.omega_res ? smem_u32(om_buf) + (uint32_t)kb * om_kb : st + kAStage;
          const uint64_t dbt = sdesc_kmajor_sw128(ob), dbl = sdesc_kmajor_sw128(ob + b_bytes);
          const uint64_t dmh = sdesc_mnmajor_sw128(st), dml = sdesc_mnmajor_sw128(st + BM * 128);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {  // MMA1: Y += A Omega (K = this k-block's 64 columns)
            const uint64_t o = (uint64_t)(kk * 2);
            umma_bf16(dy, dah + o, dbt + o, id1, (kb > 0 || kk > 0) ? 1u : 0u);
            umma_bf16(dy, dal + o, dbt + o, id1, 1u);
            if (p.nb == 2) umma_bf16(dy, dah + o, dbl + o, id1, 1u);
          }
          // MMA2: XT[:, k-blocks] += PsiT (K = 128 rows) A_tiles.  Two k-blocks in consecutive stages go
          // in one N = 128 MMA (the PsiT operand is read once for both); otherwise N = 64.
          const bool hold = pairing && s_first < 0 && (kb & 1) == 0 && kb + 1 < nkb && s + 1 < S;
          if (hold) {
            s_first = s;
          } else {
            const bool pair = s_first >= 0;
            const uint32_t sb = pair ? smem_u32(smem + (size_t)s_first * stage_bytes) : st;
            const uint64_t bh = pair ? sdesc_mnmajor_sw128(sb, stage_bytes) : dmh;
            const uint64_t bl = pair ? sdesc_mnmajor_sw128(sb + BM * 128, stage_bytes) : dml;
            const uint32_t dx = tm_xt + (uint32_t)(pair ? kb - 1 : kb) * BK;
#pragma unroll
            for (int kr = 0; kr < ((p.dbg & 1) ? 0 : BM / 16); ++kr) {
              const uint64_t da = dps + (uint64_t)((kr >> 2) * ((BM * 128) >> 4) + (kr & 3) * 2);
              const uint64_t ob = (uint64_t)(kr * (2048 >> 4));
              umma_bf16(dx, da, bh + ob, pair ? id2w : id2, (!fresh || kr > 0) ? 1u : 0u);
              umma_bf16(dx, da, bl + ob, pair ? id2w : id2, 1u);
            }
            if (pair) umma_commit(&empty[s_first]);
            umma_commit(&empty[s]);
            s_first = -1;
          }
          if (++s == S) { s = 0; ph ^= 1; }
        }
        umma_commit(&psi_empty[pb]);
        umma_commit(&y_full[yb]);
        if ((i % kFold) == kFold - 1 || i == ntiles - 1) umma_commit(xt_full);
      }
    } else if (warp >= 2) {
      // ---------------------------------------------------------------- PsiT synthesis (warps 2-3)
      // tile [128 q][128 rows] as two SW128 K-major sub-tiles [128 q][64 rows]: element (q, r) at
      // (r / 64) * 16384 + q * 128 + (((r % 64) / 8) ^ (q & 7)) * 16 + (r % 8) * 2
      const int sid = threadIdx.x - 64;  // 0..63
      const int nbytes = BM * p.zeta;    // the tile's entries: contiguous bytes psi[row0 * zeta ..]
      for (int i = 0; i < ntiles; ++i) {
        const uint32_t pb = i & 1, pph = (i >> 1) & 1;
        const int64_t row0 = (int64_t)(t0 + i) * BM;
        const int64_t e0 = row0 * p.zeta, etot = p.n * (int64_t)p.zeta;
        // this thread's 16-byte pieces of the entry block, loaded before the buffer is free
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int b = (sid + 64 * u) * 16;
          v[u] = make_uint4(0u, 0u, 0u, 0u);
          if (b < nbytes) {
            if (e0 + b + 16 <= etot && ((reinterpret_cast<uintptr_t>(p.psi + e0 + b) & 15) == 0)) {
              v[u] = __ldg(reinterpret_cast<const uint4*>(p.psi + e0 + b));
            } else {
              uint32_t w[4] = {0u, 0u, 0u, 0u};
              for (int j = 0; j < 16; ++j)
                if (e0 + b + j < etot) w[j >> 2] |= (uint32_t)__ldg(p.psi + e0 + b + j) << (8 * (j & 3));
              v[u] = make_uint4(w[0], w[1], w[2], w[3]);
            }
          }
        }
        mbar_wait(&psi_empty[pb], pph ^ 1);
        const uint32_t base = smem_u32(psi_buf + pb * kPsiBytes);
        for (int c = sid; c < (int)((p.dbg & 2) ? 0 : kPsiBytes / 16); c += 64) sts128(base + c * 16, 0u, 0u, 0u, 0u);
        asm volatile("bar.sync 2, 64;" ::: "memory");
#pragma unroll
        for (int u = 0; u < ((p.dbg & 2) ? 0 : 4); ++u) {
          const int b = (sid + 64 * u) * 16;
          if (b >= nbytes) continue;
          const uint32_t wv[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int e = b + j;
            const int r = e / p.zeta;
            if (e >= nbytes || row0 + r >= p.n) continue;
            const uint32_t en = (wv[j >> 2] >> (8 * (j & 3))) & 0xffu;
            const uint32_t q = en & 127u;
            const uint32_t off = (uint32_t)(r >> 6) * (BM * 128) + q * 128 +
                                 ((((uint32_t)(r & 63) >> 3) ^ (q & 7u)) << 4) + (uint32_t)(r & 7) * 2;
            sts16(base + off, (en & 128u) ? (uint16_t)0xbf80 : (uint16_t)0x3f80);
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&psi_full[pb]);
      }
    }
  } else if (warp < 8) {
    setmaxnreg_dec<128>();
    // ---------------------------------------------------------------- A converters (fp32 -> bf16 hi/lo)
    const int ct = threadIdx.x - 128;
    const int c4 = ct & 15;
    const int rsub = ct >> 4;
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < ntiles; ++i)
      for (int kb = 0; kb < nkb; ++kb) {
        float4 cur[16];
        mbar_wait(&tma_full[s], ph);
        const uint32_t st = smem_u32(smem + (size_t)s * stage_bytes);
        const uint32_t at = st + (rsub * BK + c4 * 4) * 4;
#pragma unroll
        for (int j = 0; j < 16; ++j) cur[j] = lds128(at + j * 8 * BK * 4);
        asm volatile("bar.sync 1, 128;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int r = rsub + 8 * j;
          const float4 v = cur[j];
          const uint32_t h01 = cvt_bf16x2(v.y, v.x), h23 = cvt_bf16x2(v.w, v.z);
          const float l0 = v.x - __uint_as_float(h01 << 16), l1 = v.y - __uint_as_float(h01 & 0xffff0000u);
          const float l2 = v.z - __uint_as_float(h23 << 16), l3 = v.w - __uint_as_float(h23 & 0xffff0000u);
          const uint32_t lo01 = cvt_bf16x2(l1, l0), lo23 = cvt_bf16x2(l3, l2);
          const uint32_t off = r * 128 + (((c4 >> 1) ^ (r & 7)) << 4) + ((c4 & 1) << 3);
          sts64(st + off, h01, h23);
          sts64(st + BM * 128 + off, lo01, lo23);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[s]);
        if (++s == S) { s = 0; ph ^= 1; }
      }
  } else {
    setmaxnreg_inc<168>();
    // ---------------------------------------------------------------- epilogue: Y tiles and XT folds
    // warp w: TMEM lane group lg = w % 4 (rows / targets 32 lg ..), half h = (w - 8) / 4:
    //   Y columns [h * NY/2, ...), XT columns [h * 128, h * 128 + 128) of this column group
    const int lg = warp & 3, h = (warp - 8) >> 2;
    const int yh = ((p.NY >> 1) + 15) & ~15;          // Y columns of half 0 (16-aligned)
    const int yc0 = h * yh, ycn = h == 0 ? yh : p.NY - yh;
    float xs[128];
#pragma unroll
    for (int j = 0; j < 128; ++j) xs[j] = 0.f;
    for (int i = 0; i < ntiles; ++i) {
      const uint32_t yb = i & 1, yph = (i >> 1) & 1;
      mbar_wait(&y_full[yb], yph);
      tc_fence_after();
      const int64_t row = (int64_t)(t0 + i) * BM + 32 * lg + lane;
      const uint32_t ybase = tm_y + yb * (uint32_t)p.NY + ((uint32_t)(32 * lg) << 16) + (uint32_t)yc0;
      for (int g = 0; g * 16 < ycn; ++g) {
        uint32_t r[16];
        tmem_ld16(ybase + g * 16, r);
        tmem_ld_wait();
        const int col = yc0 + g * 16;
        if (col + 16 <= p.k && (p.ldy & 7) == 0 && !(p.dbg & 4) && !(p.dbg & 16)) {
          // lane pairs complete 32-byte sectors: the even lane of a pair writes / adds columns [b, b+4)
          // and the odd lane [b+4, b+8) of the SAME row, one row per instruction (an exchange of 4
          // values per 8 columns through shfl.xor 1), instead of every lane writing 16 bytes of its
          // own row (section-6 shape: 1.47 -> 1.30 ms)
          const bool odd = lane & 1;
          const int64_t row_e = row - (odd ? 1 : 0), row_o = row_e + 1;
#pragma unroll
          for (int b = 0; b < 16; b += 8) {
            float mine[4], got[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {  // static register indices
              const float lo = __uint_as_float(r[b + q]), hi = __uint_as_float(r[b + 4 + q]);
              got[q] = __shfl_xor_sync(0xffffffffu, odd ? lo : hi, 1);
              mine[q] = odd ? hi : lo;
            }
            // even lane: (row_e, b..b+3) = mine, (row_o, b..b+3) = got
            // odd lane:  (row_e, b+4..b+7) = got, (row_o, b+4..b+7) = mine
            const int c0 = col + b + (odd ? 4 : 0);
            const float* v1 = odd ? got : mine;   // row_e part
            const float* v2 = odd ? mine : got;   // row_o part
            if (p.ncg > 1) {  // two column groups add onto a zeroed Y
              if (row_e < p.n)
                red_add_v4(p.Y + row_e * p.ldy + c0, v1[0] * p.sy, v1[1] * p.sy, v1[2] * p.sy, v1[3] * p.sy);
              if (row_o < p.n)
                red_add_v4(p.Y + row_o * p.ldy + c0, v2[0] * p.sy, v2[1] * p.sy, v2[2] * p.sy, v2[3] * p.sy);
            } else {
              if (row_e < p.n)
                *reinterpret_cast<float4*>(p.Y + row_e * p.ldy + c0) =
                    make_float4(v1[0] * p.sy, v1[1] * p.sy, v1[2] * p.sy, v1[3] * p.sy);
              if (row_o < p.n)
                *reinterpret_cast<float4*>(p.Y + row_o * p.ldy + c0) =
                    make_float4(v2[0] * p.sy, v2[1] * p.sy, v2[2] * p.sy, v2[3] * p.sy);
            }
          }
        } else if (row < p.n && col < p.k && !(p.dbg & 4)) {
          float* out = p.Y + row * p.ldy + col;
          if (p.ncg == 1) {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (col + j < p.k) out[j] = __uint_as_float(r[j]) * p.sy;
          } else if (col + 16 <= p.k && ((p.ldy & 3) == 0)) {
#pragma unroll
            for (int j = 0; j < 16; j += 4)
              red_add_v4(out + j, __uint_as_float(r[j]) * p.sy, __uint_as_float(r[j + 1]) * p.sy,
                         __uint_as_float(r[j + 2]) * p.sy, __uint_as_float(r[j + 3]) * p.sy);
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (col + j < p.k) atomicAdd(out + j, __uint_as_float(r[j]) * p.sy);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&y_empty[yb]);
      if ((i % kFold) == kFold - 1 || i == ntiles - 1) {  // fold the XT chunk into fp32 registers
        mbar_wait(xt_full, (i / kFold) & 1);
        tc_fence_after();
        const uint32_t xbase = tm_xt + ((uint32_t)(32 * lg) << 16) + (uint32_t)(h * 128);
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          if (g * 16 < nkb * BK - h * 128) {
            uint32_t r[16];
            tmem_ld16(xbase + g * 16, r);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j) xs[g * 16 + j] += __uint_as_float(r[j]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(xt_empty);
      }
    }
    // this CTA's XT partial: [128 targets][256 columns of the group]
    float* xp = p.xpart + ((int64_t)blockIdx.x * BM + 32 * lg + lane) * kColsPerGroup + h * 128;
#pragma unroll
    for (int j = 0; j < 128; j += 4)
      *reinterpret_cast<float4*>(xp + j) = make_float4(xs[j], xs[j + 1], xs[j + 2], xs[j + 3]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// X^T[q, c] = sx * sum over the CTAs of column group c / 256 of their partials (fixed order)
__global__ void two_sided_reduce(const float* __restrict__ xpart, int ncg, int ctas_per_group, int p, int64_t d,
                                 float sx, float* __restrict__ XT, int64_t ldx) {
  const int64_t total = (int64_t)p * d;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int q = (int)(i / d);
    const int64_t c = i % d;
    const int cg = (int)(c / kColsPerGroup), cc = (int)(c % kColsPerGroup);
    float s = 0.f;
    for (int g = 0; g < ctas_per_group; ++g) s += xpart[((int64_t)(g * ncg + cg) * BM + q) * kColsPerGroup + cc];
    XT[q * ldx + c] = s * sx;
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int map2d(CUtensorMap* m, CUtensorMapDataType dt, int esz, const void* base, int64_t inner, int64_t outer, int64_t ld,
          int box_in, int box_out, CUtensorMapSwizzle sw) {
  EncodeFn fn = reinterpret_cast<EncodeFn>(sm100::encode_tiled_fn());
  if (!fn) return fail(SK_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * esz)};
  cuuint32_t box[2] = {(cuuint32_t)box_in, (cuuint32_t)box_out};
  cuuint32_t estr[2] = {1, 1};
  if (fn(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return fail(SK_EINVAL, "sk_two_sided_sketch: cuTensorMapEncodeTiled failed (alignment?)");
  return SK_OK;
}

struct TsPlan {
  int ncg, cpg, grid, stages, NY, omega_res;
  size_t smem, ws;
};

TsPlan ts_plan(int64_t n, int64_t d, int64_t k, int nb) {
  TsPlan pl{};
  pl.ncg = (int)((d + kColsPerGroup - 1) / kColsPerGroup);
  pl.NY = (int)((k + 15) / 16 * 16);
  const int mtiles = (int)((n + BM - 1) / BM);
  int cpg = sm_count() / pl.ncg;
  if (cpg < 1) cpg = 1;
  if (cpg > mtiles) cpg = mtiles;
  pl.cpg = cpg;
  pl.grid = cpg * pl.ncg;
  const size_t om_kb = (size_t)nb * pl.NY * 128;
  const size_t fixed = 1024 + 2 * (size_t)kPsiBytes + 64 * 8 + 16;
  // Omega^T resident (loaded once per CTA) when that still leaves as deep an A ring as streaming it
  // with every stage would; otherwise it rides in each stage
  int st_stream = (int)((227 * 1024 - fixed) / (kAStage + om_kb));
  int st_res = (int)((227 * 1024 - fixed - 4 * om_kb) / kAStage);
  if (st_stream > 6) st_stream = 6;
  if (st_res > 6) st_res = 6;
  const bool res = getenv("SKETCH_B200_TS_OMEGA") ? getenv("SKETCH_B200_TS_OMEGA")[0] == 'r' : st_res >= st_stream;
  pl.omega_res = res ? 1 : 0;
  pl.stages = res ? st_res : st_stream;
  pl.smem = res ? fixed + 4 * om_kb + (size_t)st_res * kAStage : fixed + (size_t)st_stream * (kAStage + om_kb);
  pl.ws = (size_t)pl.grid * BM * kColsPerGroup * sizeof(float);
  return pl;
}

}  // namespace
}  // namespace skb

extern "C" size_t sk_two_sided_workspace_bytes(int64_t n, int64_t d, int64_t k, int split_omega) {
  if (n < 1 || d < 1 || k < 1) return 0;
  return skb::ts_plan(n, d, k, split_omega ? 2 : 1).ws;
}

// Y[n,k] = sy * A Omega and XT[p,d] = sx * Psi^T A from one read of A (float32).  Omega given as
// Omega^T bf16 (k x ldb, + residual or NULL); Psi as [n][zeta] uint8 entries q | neg << 7 (p <= 128).
extern "C" int sk_two_sided_sketch(const float* A, int64_t n, int64_t d, int64_t lda, const uint16_t* Bt_hi,
                                   const uint16_t* Bt_lo, int64_t ldb, int64_t k, double sy, const uint8_t* psi,
                                   int32_t zeta, int64_t p, double sx, float* Y, int64_t ldy, float* XT,
                                   int64_t ldx, void* ws, size_t ws_bytes, void* stream) {
  using namespace skb;
  if (n < 0 || d < 1 || k < 1 || k > 128 || p < 1 || p > 128 || zeta < 1 || zeta > 32 || lda < d || ldb < d ||
      ldy < k || ldx < d)
    return fail(SK_EINVAL, "sk_two_sided_sketch: bad shape (k, p <= 128, zeta <= 32)");
  if (!A || !Bt_hi || !psi || !Y || !XT) return fail(SK_EINVAL, "sk_two_sided_sketch: null pointer");
  if ((reinterpret_cast<uintptr_t>(A) & 15) || (lda & 3) || (reinterpret_cast<uintptr_t>(Bt_hi) & 15) || (ldb & 7))
    return fail(SK_EINVAL, "sk_two_sided_sketch: A / Omega^T alignment (16 B, lda % 4, ldb % 8)");
  cudaStream_t s = as_stream(stream);
  const int nb = Bt_lo ? 2 : 1;
  const TsPlan pl = ts_plan(n, d, k, nb);
  if (pl.stages < 2) return fail(SK_EUNSUPPORTED, "sk_two_sided_sketch: tiles do not fit shared memory");
  if (!ws || ws_bytes < pl.ws) return fail(SK_EINVAL, "sk_two_sided_sketch: workspace too small");
  if (n == 0) {
    cudaMemset2DAsync(XT, ldx * 4, 0, d * 4, p, s);
    return check_launch("sk_two_sided_sketch");
  }
  if (pl.ncg > 1 && cudaMemset2DAsync(Y, ldy * 4, 0, k * 4, n, s) != cudaSuccess)
    return check_launch("sk_two_sided_sketch(zero Y)");
  CUtensorMap ma, mb, mbl;
  int st = map2d(&ma, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, A, d, n, lda, BK, BM, CU_TENSOR_MAP_SWIZZLE_NONE);
  if (st != SK_OK) return st;
  st = map2d(&mb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Bt_hi, d, k, ldb, BK, pl.NY, CU_TENSOR_MAP_SWIZZLE_128B);
  if (st != SK_OK) return st;
  if (nb == 2) {
    st = map2d(&mbl, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Bt_lo, d, k, ldb, BK, pl.NY, CU_TENSOR_MAP_SWIZZLE_128B);
    if (st != SK_OK) return st;
  } else {
    mbl = mb;
  }
  TsParams prm{};
  prm.A = A;
  prm.n = n;
  prm.d = d;
  prm.lda = lda;
  prm.k = (int)k;
  prm.NY = pl.NY;
  prm.ncg = pl.ncg;
  prm.p = (int)p;
  prm.zeta = zeta;
  prm.psi = psi;
  prm.sy = (float)sy;
  prm.sx = (float)sx;
  prm.Y = Y;
  prm.ldy = ldy;
  prm.xpart = static_cast<float*>(ws);
  prm.mtiles = (int)((n + BM - 1) / BM);
  prm.stages = pl.stages;
  prm.ctas_per_group = pl.cpg;
  prm.nb = nb;
  prm.omega_res = pl.omega_res;
  {
    const char* e = getenv("SKETCH_B200_TS_DBG");
    prm.dbg = e ? atoi(e) : 0;
  }
  allow_smem(two_sided_kernel, pl.smem);
  two_sided_kernel<<<pl.grid, kThreads, pl.smem, s>>>(ma, mb, mbl, prm);
  st = check_launch("sk_two_sided_sketch");
  if (st != SK_OK) return st;
  int64_t blocks = (p * d + 255) / 256;
  if (blocks > 4 * (int64_t)sm_count()) blocks = 4 * (int64_t)sm_count();
  two_sided_reduce<<<(unsigned)blocks, 256, 0, s>>>(prm.xpart, pl.ncg, pl.cpg, (int)p, d, (float)sx, XT, ldx);
  return check_launch("sk_two_sided_sketch(reduce)");
}
