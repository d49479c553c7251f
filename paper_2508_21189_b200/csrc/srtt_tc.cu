// K3-TC — SRTT (Walsh-Hadamard, d = 8192) with the 128-point half of the transform on tcgen05.
//
// H_8192 = H_64 (x) H_128 in natural order: for a row x (index j = 128 a + b) viewed as X[a][b]
// (64 x 128, row-major = the row as stored),
//     Y = H_64 * X * H_128,   i.e.  Z^T = H_128 * X^T  (tensor cores),  Y^T = Z^T * H_64 (registers).
// Per row of A (one 32 KB slot of a 5-deep ring, one 512-thread CTA per SM):
//   producer  : one 32 KB bulk copy (cp.async.bulk) of the row into its slot
//   converters: (4 warps) sign flip by D, split fp32 -> bf16 hi + lo (exact +-1 H keeps BF16x2 at
//               ~3e-6), each row written in place as its own K-major SWIZZLE_128B B operand
//               (N = 64 rows a, K = 128 columns b as two 64-wide halves, hi then lo)
//   MMA       : (1 thread) per row 16 x tcgen05.mma M=128 (b') N=64 (a) K=16 against the
//               constant H_128 tile (A operand, built once in tensor memory: the tensor cores
//               then read only the 32 KB of converted data per row from shared memory)
//   epilogue  : (2 warpgroups taking alternate rows, thread = TMEM lane = b') tcgen05.ld 64
//               columns (a) per row, 64-point WHT over a in registers (6 FADD2 stages), scatter
//               Y[a'][b'] to the warpgroup's row buffer, then the sampled gather
//               out[c] = scale * sign * Y[row_c] with coalesced stores.
// TMEM: H_128 (64 columns) + four 64-column accumulators.
// Bound: shared-memory bandwidth. Per row the SM moves ~1340 shared wavefronts (TMA write 256,
// converter read 256 + write 256, tensor-core read 256, Y row 256 + gather) against a ~1450-cycle
// HBM budget; measured variants: converters reading global memory directly
// (the L1 data path is the same SRAM), a 4-D TMA that lands rows pre-swizzled (no converter CTA
// barrier), a 6-slot ring with half-row Y buffers — all slower than this layout.
// Replaces SparseRttTM.apply_right (src/sketch/rtt.py:129-140) + wht (rtt.py:28-44) for d = 8192.
#include <cuda.h>

#include "common.cuh"
#include "sm100.cuh"

namespace skb {
namespace {

using namespace sm100;

// Shape of the kernel for d = 2^L (11 <= L <= 13): NA = d / 128 a-rows per row of A.
template <int L>
struct TcCfg {
  static constexpr int D = 1 << L;
  static constexpr int NA = D / 128;                 // N of the per-row MMAs, points of the register WHT
  static constexpr int ROW_BYTES = D * 4;
  static constexpr int TB = NA * 128;                // one hi/lo K-half operand tile (bytes)
  static constexpr int SLOTS = L == 13 ? 5 : (L == 12 ? 10 : 16);  // row ring depth (shared memory)
  static constexpr int NG = D / 512;                 // 4-float groups per converter thread per row
  static_assert(NA >= 16 && NA <= 64, "tile shape");
};
constexpr int TC_ACC = 4;                     // TMEM accumulators of NA columns (after H's 64)
constexpr int TC_TMEM_COLS = 512;             // H_128 (64) + 4 accumulators, power of two
constexpr int TC_SAMP_REGS = 8;               // sampler entries per epilogue thread kept in registers
constexpr int TC_THREADS = 512;               // WG0: producer/MMA/alloc | WG1 converters | WG2,3 epilogue

typedef unsigned long long u64;

__device__ __forceinline__ u64 f2add_(u64 a, u64 b) {
  u64 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 f2sub_(u64 a, u64 b) {
  u64 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

template <int N>
__device__ __forceinline__ void maxnreg_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}
template <int N>
__device__ __forceinline__ void maxnreg_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}

template <int NA>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t (&r)[NA]) {
#pragma unroll
  for (int q = 0; q < NA / 16; ++q) {
    uint32_t (&t)[16] = *reinterpret_cast<uint32_t(*)[16]>(&r[16 * q]);
    tmem_ld16(taddr + 16 * q, t);
  }
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// D[tmem] (+)= A[tmem] * B[smem]^T, bf16 inputs, fp32 accumulate (A read from tensor memory)
__device__ __forceinline__ void umma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
}

// FULL = false: sampled SRTT rows (the sketch). FULL = true: segment mode for rows longer than d:
// the operand is n rows of `period` segments of d floats (segment row r = (r / period, r % period),
// source A + (r / period) * lda + (r % period) * d); the CTA's segments all share r % period (the
// grid is a multiple of `period`), so its D slice is dvals + (blockIdx.x % period) * d; the
// transformed segment is written whole to Y (row r / period, offset (r % period) * d), unscaled.
template <int L, bool FULL>
__global__ void __launch_bounds__(TC_THREADS, 1)
    srtt_wht_tc(const float* __restrict__ A, int64_t n, int64_t lda, const float* __restrict__ dvals,
                const int32_t* __restrict__ samp, int xi, int k, float scale, float* __restrict__ Y, int64_t ldy,
                int period) {
  using C = TcCfg<L>;
  constexpr int TC_SLOTS = C::SLOTS, TC_ROW_BYTES = C::ROW_BYTES, NA = C::NA, TB = C::TB, NG = C::NG;
  extern __shared__ uint8_t smem_dyn[];
  uint8_t* smem = smem_dyn + ((1024u - (smem_u32(smem_dyn) & 1023u)) & 1023u);
  uint8_t* rbuf = smem;                                               // TC_SLOTS row slots x 32 KB
  float* ybufs = reinterpret_cast<float*>(rbuf + TC_SLOTS * TC_ROW_BYTES);  // one Y row per epilogue WG
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(ybufs) + 2 * TC_ROW_BYTES);
  uint64_t* r_tma = bars;                        // [TC_SLOTS] row landed
  uint64_t* r_conv = bars + TC_SLOTS;            // [TC_SLOTS] converted (4 converter warps)
  uint64_t* r_empty = bars + 2 * TC_SLOTS;       // [TC_SLOTS] consumed by the MMA
  uint64_t* t_full = bars + 3 * TC_SLOTS;        // [TC_ACC] accumulator ready
  uint64_t* t_empty = bars + 3 * TC_SLOTS + TC_ACC;  // [TC_ACC] accumulator drained (4 epilogue warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * TC_SLOTS + 2 * TC_ACC);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    for (int s = 0; s < TC_SLOTS; ++s) {
      mbar_init(&r_tma[s], 1);
      mbar_init(&r_conv[s], 4);
      mbar_init(&r_empty[s], 1);
    }
    for (int s = 0; s < TC_ACC; ++s) {
      mbar_init(&t_full[s], 1);
      mbar_init(&t_empty[s], 4);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, TC_TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp >= 8 && warp < 12) {
    // constant H_128 (A operand) into TMEM columns [0, 64): lane b', column c = bf16 pair
    // (H[b'][2c], H[b'][2c+1]) with H[b'][b] = (-1)^popcount(b' & b)
    const int bp = 32 * (warp & 3) + lane;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t hv[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const int b = 2 * (16 * q + c);
        const uint32_t h0 = (__popc(bp & b) & 1) ? 0xBF80u : 0x3F80u;
        const uint32_t h1 = (__popc(bp & (b + 1)) & 1) ? 0xBF80u : 0x3F80u;
        hv[c] = h0 | (h1 << 16);
      }
      tmem_st16(tmem + ((uint32_t)(32 * (warp & 3)) << 16) + 16 * q, hv);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (warp < 4) {
    maxnreg_dec<40>();
    if (warp == 0 && lane == 0) {
      // ------------------------------------------------------------ producer: one row per slot
      int s = 0;
      uint32_t ph = 0;
      for (int64_t row = blockIdx.x; row < n; row += gridDim.x) {
        mbar_wait(&r_empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&r_tma[s], TC_ROW_BYTES);
        const float* src = FULL ? A + (row / period) * lda + (row % period) * C::D : A + row * lda;
        bulk_g2s(rbuf + s * TC_ROW_BYTES, src, TC_ROW_BYTES, &r_tma[s]);
        if (++s == TC_SLOTS) { s = 0; ph ^= 1; }
      }
    } else if (warp == 1 && lane == 0) {
      // ------------------------------------------------------------ MMA issuer
      const uint32_t idesc = idesc_bf16_f32(128, NA);
      int s = 0, buf = 0;
      uint32_t ph = 0, tph = 0;
      for (int64_t row = blockIdx.x; row < n; row += gridDim.x) {
        mbar_wait(&t_empty[buf], tph ^ 1);
        mbar_wait(&r_conv[s], ph);
        tc_fence_after();
        const uint32_t d = tmem + 64 + buf * NA;
        const uint32_t rb = smem_u32(rbuf + s * TC_ROW_BYTES);
#pragma unroll
        for (int kh = 0; kh < 2; ++kh) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint32_t ta = tmem + (uint32_t)(kh * 32 + kk * 8);  // K step of 16 = 8 columns
            const uint64_t dbh = sdesc_kmajor_sw128(rb + kh * TB + kk * 32);
            const uint64_t dbl = sdesc_kmajor_sw128(rb + 2 * TB + kh * TB + kk * 32);
            umma_bf16_ts(d, ta, dbh, idesc, (kh | kk) ? 1u : 0u);
            umma_bf16_ts(d, ta, dbl, idesc, 1u);
          }
        }
        umma_commit(&r_empty[s]);
        umma_commit(&t_full[buf]);
        if (++s == TC_SLOTS) { s = 0; ph ^= 1; }
        if (++buf == TC_ACC) { buf = 0; tph ^= 1; }
      }
    }
  } else if (warp < 8) {
    maxnreg_inc<152>();
    // ------------------------------------------------------------ converters (128 threads)
    // Each row is converted in place into [hi K0 | hi K1 | lo K0 | lo K1], each a K-major
    // SWIZZLE_128B tile of NA rows a x 64 columns b. Thread ct owns NG groups of 4 floats
    // q = ct + 128 i: a = q >> 5, b = 4 (q & 31). Reads are 16-byte contiguous across lanes; writes
    // are 8-byte halves of 16-byte chunks, each half-warp one 128-byte line. D is applied after
    // the split as an XOR on the packed bf16 pairs (round-to-nearest is sign symmetric).
    const int ct = tid - 128;
    if (FULL) dvals += (int64_t)(blockIdx.x % period) * C::D;
    uint32_t dm[2 * NG];
#pragma unroll
    for (int i = 0; i < NG; ++i) {
      const int q = ct + 128 * i;
      const int j0 = (q >> 5) * 128 + 4 * (q & 31);
      const float4 dv = __ldg(reinterpret_cast<const float4*>(dvals + j0));
      dm[2 * i] = (dv.x < 0.f ? 0x8000u : 0u) | (dv.y < 0.f ? 0x80000000u : 0u);
      dm[2 * i + 1] = (dv.z < 0.f ? 0x8000u : 0u) | (dv.w < 0.f ? 0x80000000u : 0u);
    }
    int s = 0;
    uint32_t ph = 0;
    for (int64_t row = blockIdx.x; row < n; row += gridDim.x) {
      mbar_wait(&r_tma[s], ph);
      const uint32_t rsa = smem_u32(rbuf + s * TC_ROW_BYTES);
      float4 v[NG];
#pragma unroll
      for (int i = 0; i < NG; ++i) v[i] = lds128(rsa + (uint32_t)(ct + 128 * i) * 16u);
      asm volatile("bar.sync 1, 128;" ::: "memory");  // all fp32 reads of the row before in-place writes
#pragma unroll
      for (int i = 0; i < NG; ++i) {
        const int q = ct + 128 * i;
        const int a = q >> 5, b4 = q & 31;
        const uint32_t h01 = cvt_bf16x2(v[i].y, v[i].x), h23 = cvt_bf16x2(v[i].w, v[i].z);
        const uint32_t l01 = cvt_bf16x2(v[i].y - __uint_as_float(h01 & 0xffff0000u), v[i].x - __uint_as_float(h01 << 16));
        const uint32_t l23 = cvt_bf16x2(v[i].w - __uint_as_float(h23 & 0xffff0000u), v[i].z - __uint_as_float(h23 << 16));
        const uint32_t off = (uint32_t)(b4 >> 4) * (uint32_t)TB + (uint32_t)a * 128u +
                             (((((uint32_t)b4 & 15u) >> 1) ^ ((uint32_t)a & 7u)) << 4) + (((uint32_t)b4 & 1u) << 3);
        sts64(rsa + off, h01 ^ dm[2 * i], h23 ^ dm[2 * i + 1]);
        sts64(rsa + 2u * TB + off, l01 ^ dm[2 * i], l23 ^ dm[2 * i + 1]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&r_conv[s]);
      if (++s == TC_SLOTS) { s = 0; ph ^= 1; }
    }
  } else {
    maxnreg_inc<152>();
    // ------------------------------------------------------------ epilogue: two warpgroups take
    // alternate rows (accumulators buf = i % TC_ACC, i = local row index), each with its own Y row
    const int ew = (warp >> 2) - 2;  // 0 or 1
    const int lg = warp & 3;
    const int bp = 32 * lg + lane;  // b' = TMEM lane
    const int et = tid & 127;
    float* ybuf = ybufs + ew * (TC_ROW_BYTES / 4);
    const bool fast = !FULL && (xi == 1 && k <= 128 * TC_SAMP_REGS);
    uint32_t se[TC_SAMP_REGS];      // sampler entries c = et + 128 j (xi = 1)
#pragma unroll
    for (int j = 0; j < TC_SAMP_REGS; ++j) {
      const int c = et + 128 * j;
      se[j] = (fast && c < k) ? (uint32_t)__ldg(samp + c) : 0u;
    }
    int buf = ew;
    uint32_t tph = 0;
    for (int64_t row = blockIdx.x + ew * (int64_t)gridDim.x; row < n; row += 2 * (int64_t)gridDim.x) {
      mbar_wait(&t_full[buf], tph);
      tc_fence_after();
      uint32_t z[NA];
      tmem_ld_cols<NA>(tmem + ((uint32_t)(32 * lg) << 16) + 64 + buf * NA, z);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&t_empty[buf]);
      buf += 2;
      if (buf >= TC_ACC) { buf -= TC_ACC; tph ^= 1; }
      // NA-point WHT over a (register index): a-bit 0 inside pairs, the other a-bits on packed pairs
      u64 p[NA / 2];
#pragma unroll
      for (int i = 0; i < NA / 2; ++i) {
        const float x0 = __uint_as_float(z[2 * i]), x1 = __uint_as_float(z[2 * i + 1]);
        const float s0 = x0 + x1, d0 = x0 - x1;
        asm("mov.b64 %0, {%1, %2};" : "=l"(p[i]) : "f"(s0), "f"(d0));
      }
#pragma unroll
      for (int h = 1; h < NA / 2; h <<= 1) {
#pragma unroll
        for (int i = 0; i < NA / 2; ++i) {
          if ((i & h) == 0) {
            const u64 s0 = f2add_(p[i], p[i | h]);
            const u64 d0 = f2sub_(p[i], p[i | h]);
            p[i] = s0;
            p[i | h] = d0;
          }
        }
      }
      if constexpr (FULL) {
        // whole transformed segment: Y[a'][b'] -> y[a' * 128 + b'], 128 consecutive floats per a'
        float* y = Y + (row / period) * ldy + (row % period) * C::D + bp;
#pragma unroll
        for (int i = 0; i < NA / 2; ++i) {
          float lo, hi;
          asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(p[i]));
          y[(2 * i) * 128] = lo;
          y[(2 * i + 1) * 128] = hi;
        }
        continue;
      }
      asm volatile("bar.sync %0, 128;" ::"r"(2 + ew) : "memory");  // previous gather done with ybuf
#pragma unroll
      for (int i = 0; i < NA / 2; ++i) {
        float lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(p[i]));
        ybuf[(2 * i) * 128 + bp] = lo;
        ybuf[(2 * i + 1) * 128 + bp] = hi;
      }
      asm volatile("bar.sync %0, 128;" ::"r"(2 + ew) : "memory");
      float* y = Y + row * ldy;
      if (fast) {
#pragma unroll
        for (int j = 0; j < TC_SAMP_REGS; ++j) {
          const int c = et + 128 * j;
          if (c < k) y[c] = flip_if(ybuf[se[j] & 0x7fffffffu], se[j] >> 31) * scale;
        }
      } else {
        for (int c = et; c < k; c += 128) {
          float acc = 0.f;
          for (int x = 0; x < xi; ++x) {
            const uint32_t e = (uint32_t)__ldg(samp + (int64_t)c * xi + x);
            acc += flip_if(ybuf[e & 0x7fffffffu], e >> 31);
          }
          y[c] = acc * scale;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, TC_TMEM_COLS);
  }
}


template <int L>
int launch_tc_t(const float* A, int64_t n, int64_t lda, const float* dv, const int32_t* samp, int xi, int k,
                double scale, float* Y, int64_t ldy, cudaStream_t s) {
  using C = TcCfg<L>;
  const int grid = (int)(n < sm_count() ? n : sm_count());
  const size_t smem = 1024 + (size_t)(C::SLOTS + 2) * C::ROW_BYTES + 8 * (3 * C::SLOTS + 2 * TC_ACC + 1);
  allow_smem(srtt_wht_tc<L, false>, smem);
  srtt_wht_tc<L, false><<<grid, TC_THREADS, smem, s>>>(A, n, lda, dv, samp, xi, k, (float)scale, Y, ldy, 1);
  return check_launch("sk_srtt_right(tc)");
}

}  // namespace

// Launcher used by sk_srtt_right (srtt.cu) for float32, d = 2^L with 11 <= L <= 13, +-1 diagonal.
int launch_srtt_tc(int L, const float* A, int64_t n, int64_t lda, const float* dv, const int32_t* samp, int xi, int k,
                   double scale, float* Y, int64_t ldy, cudaStream_t s) {
  if (L == 13) return launch_tc_t<13>(A, n, lda, dv, samp, xi, k, scale, Y, ldy, s);
  if (L == 12) return launch_tc_t<12>(A, n, lda, dv, samp, xi, k, scale, Y, ldy, s);
  if (L == 11) return launch_tc_t<11>(A, n, lda, dv, samp, xi, k, scale, Y, ldy, s);
  return fail(SK_EUNSUPPORTED, "sk_srtt_right(tc): no tensor-core variant for this length");
}

}  // namespace skb

// Segment transforms of long rows: Z[r, a*8192 : (a+1)*8192] = H_8192 (D[a*8192 : ...] o A[r, same]),
// unnormalised, for a < d / 8192 (d a multiple of 8192, D exactly +-1).
extern "C" int sk_wht_segments_f32(const float* A, int64_t n, int64_t d, int64_t lda, const float* dvals, float* Z,
                                   int64_t ldz, void* stream) {
  using namespace skb;
  constexpr int L = 13;
  using C = TcCfg<L>;
  if (n < 0 || d < C::D || (d % C::D) || lda < d || ldz < d)
    return fail(SK_EINVAL, "sk_wht_segments_f32: d must be a multiple of 8192 (lda, ldz >= d)");
  if (n == 0) return SK_OK;
  if (!A || !dvals || !Z) return fail(SK_EINVAL, "sk_wht_segments_f32: null pointer");
  if ((reinterpret_cast<uintptr_t>(A) & 15) || (lda & 3) || (reinterpret_cast<uintptr_t>(dvals) & 15))
    return fail(SK_EUNSUPPORTED, "sk_wht_segments_f32: A and D must be 16-byte aligned with lda % 4 == 0");
  const int64_t period = d / C::D, rows = n * period;
  if (period > (1 << 20)) return fail(SK_EINVAL, "sk_wht_segments_f32: too many segments per row");
  // the grid is a multiple of the period so every CTA keeps one D slice
  int64_t grid = sm_count() / period * period;
  if (grid < period) grid = period;
  if (grid > rows) grid = rows;
  const size_t smem = 1024 + (size_t)(C::SLOTS + 2) * C::ROW_BYTES + 8 * (3 * C::SLOTS + 2 * TC_ACC + 1);
  allow_smem(srtt_wht_tc<L, true>, smem);
  srtt_wht_tc<L, true><<<(unsigned)grid, TC_THREADS, smem, as_stream(stream)>>>(A, rows, lda, dvals, nullptr, 1, 1,
                                                                                1.f, Z, ldz, (int)period);
  return check_launch("sk_wht_segments_f32");
}

namespace skb {
namespace {
// Outer transform of long rows, only at the sampled outputs: for sampler entry j = row | neg << 31,
// Y_j = sum_a (-1)^popc((j >> 13) & a) Z[a * 8192 + (j & 8191)], a < period; then
// out[c] = scale * sum_x sign * Y_{j(c, x)}. One thread per (row, c); the Z row is L2-resident.
__global__ void srtt_outer_kernel(const float* __restrict__ Z, int64_t n, int64_t ldz, int period,
                                  const int32_t* __restrict__ samp, int xi, int k, float scale, float* __restrict__ Y,
                                  int64_t ldy) {
  const int64_t total = n * (int64_t)k;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = idx / k;
    const int c = (int)(idx % k);
    const float* z = Z + row * ldz;
    float acc = 0.f;
    for (int x = 0; x < xi; ++x) {
      const uint32_t e = (uint32_t)__ldg(samp + (int64_t)c * xi + x);
      const uint32_t j = e & 0x7fffffffu, hi = j >> 13, lo = j & 8191u;
      float v = 0.f;
      for (int a = 0; a < period; ++a) {
        const float t = __ldg(z + (int64_t)a * 8192 + lo);
        v += (__popc(hi & (uint32_t)a) & 1) ? -t : t;
      }
      acc += flip_if(v, e >> 31);
    }
    Y[row * ldy + c] = acc * scale;
  }
}
}  // namespace
}  // namespace skb

extern "C" int sk_srtt_outer_f32(const float* Z, int64_t n, int64_t d, int64_t ldz, const int32_t* samp, int32_t xi,
                                 int64_t k, double scale, float* Y, int64_t ldy, void* stream) {
  using namespace skb;
  if (n < 0 || d < 8192 || (d % 8192) || ldz < d || k < 1 || xi < 1 || ldy < k)
    return fail(SK_EINVAL, "sk_srtt_outer_f32: bad shape (d a multiple of 8192)");
  if (n == 0) return SK_OK;
  if (!Z || !samp || !Y) return fail(SK_EINVAL, "sk_srtt_outer_f32: null pointer");
  const int64_t total = n * k;
  int64_t grid = (total + 255) / 256;
  if (grid > 64 * (int64_t)sm_count()) grid = 64 * (int64_t)sm_count();
  srtt_outer_kernel<<<(unsigned)grid, 256, 0, as_stream(stream)>>>(Z, n, ldz, (int)(d / 8192), samp, xi, (int)k,
                                                                   (float)scale, Y, ldy);
  return check_launch("sk_srtt_outer_f32");
}
