// K2g — sparse-sign adjoint by row gathers:  SA = scale * Omega^T * A  (S = Omega^T, zeta nonzeros
// per row of Omega = per row of A).
//
// Replaces `_SparseTM.apply_adjoint` = `self.matrix.conj().T @ b` (src/sketch/sparse.py:68-78),
// BASELINE config 4 (S 2048 x 4194304, zeta = 8, A 4194304 x 512 float32).
//
// Omega is given by TARGET rows (CSR of S): for output row q the A rows j it sums, ascending, as
// int32 words j | neg << 31, plus the offsets off[q][p] where row piece p (rows [p*prows,
// (p+1)*prows) of A) starts in q's list. A unit of work is (piece p, output row q, 1 KB column
// block h — 256 float32 / 128 float64 columns):
// one warp walks q's entries inside piece p, fetching the needed A rows with TMA row gathers
// (cp.async.bulk.tensor ... tile::gather4: four arbitrary rows x 1 KB per copy) into a private
// 3-stage ring (entry words staged in a per-warp shared buffer, sign applied by an fma with the
// +-1.0 carried in the word), and sums them in registers — the output row is fixed for the walk, so every
// add has a static register target (no per-entry dispatch). The unit's sum goes to
// part[p][q][h-columns]; the float64 ordered reduction of sparse_adjoint.cu forms SA
// (deterministic: fixed summation order everywhere).
//
// L2: units are handed out piece-major from one global counter, so the warps resident at any time
// all work inside one or two consecutive pieces (~64 MB of A): each A row leaves DRAM about once
// (1.36 x |A| measured at config 4) and is re-served from L2 to its zeta targets x column blocks.
// Config 4: 3.87 ms, bound by the 8 x |A| L2 -> SM gather traffic.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "sm100.cuh"

namespace skb {

int adjoint_reduce_f32(const float* part, int npieces, int64_t k, int64_t m, double scale, float* SA, int64_t ldsa,
                       int accumulate, cudaStream_t s);
int adjoint_reduce_f64(const double* part, int npieces, int64_t k, int64_t m, double scale, double* SA, int64_t ldsa,
                       int accumulate, cudaStream_t s);

namespace {

using namespace sm100;

constexpr int G_WARPS = 16;
constexpr int G_STAGES = 3;
constexpr int G_ROW_BYTES = 1024;                // one gathered row: 256 float32 / 128 float64 columns
constexpr int G_STAGE_BYTES = 4 * G_ROW_BYTES;   // one gather4
typedef unsigned long long u64;

template <typename T>
constexpr int g_cols() {
  return G_ROW_BYTES / (int)sizeof(T);
}

struct GParams {
  int64_t d, m, k, prows;
  int npieces, nhalves;
  int64_t nunits;
  const int32_t* ent;   // CSR of S by target row: j | neg << 31
  const int64_t* off;   // [k][npieces + 1]
  void* part;           // [npieces][k][m]
  int* counter;         // unit counter (zeroed before the launch)
};

__device__ __forceinline__ void gather4(uint32_t dst, const CUtensorMap* tm, uint32_t bar, int col, int r0, int r1,
                                        int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5, %6}], [%7];" ::"r"(dst),
      "l"(tm), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void arrive_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void wait_parity(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void lds128(uint32_t addr, u64& x, u64& y) {
  asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "r"(addr));
}

// acc += v * s on packed pairs: float32 pairs times {s, s} (fma.rn.f32x2) or one float64 times s
template <typename T>
__device__ __forceinline__ void fma_signed(u64& acc, u64 v, uint32_t s32, u64 s64) {
  if constexpr (sizeof(T) == 4) {
    asm("{\n\t.reg .b64 ss;\n\tmov.b64 ss, {%2, %2};\n\tfma.rn.f32x2 %0, %1, ss, %0;\n\t}" : "+l"(acc) : "l"(v), "r"(s32));
  } else {
    asm("fma.rn.f64 %0, %1, %2, %0;" : "+l"(acc) : "l"(v), "l"(s64));
  }
}

constexpr int G_ENT = 512;  // entries of a unit staged in the warp's shared buffer at a time

template <typename T>
__global__ void __launch_bounds__(G_WARPS * 32, 1)
    sparse_adjoint_gather(const __grid_constant__ CUtensorMap tm, const GParams p) {
  constexpr int W = g_cols<T>();
  extern __shared__ __align__(1024) uint8_t smem_dyn[];
  uint8_t* smem = smem_dyn + ((1024u - (smem_u32(smem_dyn) & 1023u)) & 1023u);
  uint32_t* ebuf_all = reinterpret_cast<uint32_t*>(smem + (size_t)G_WARPS * G_STAGES * G_STAGE_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(ebuf_all + G_WARPS * G_ENT);

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0)
    for (int s = 0; s < G_STAGES; ++s) mbar_init(&bars[warp * G_STAGES + s], 1);
  fence_mbar_init();
  if (threadIdx.x == 0) tma_prefetch_desc(&tm);
  __syncwarp();

  const uint32_t ring = smem_u32(smem + (size_t)warp * G_STAGES * G_STAGE_BYTES);
  const uint32_t bar0 = smem_u32(&bars[warp * G_STAGES]);
  uint32_t* ebuf = ebuf_all + warp * G_ENT;
  const uint32_t ebuf_s = smem_u32(ebuf);
  // ring position of the next gather to issue / to consume (stage, phase) — no divisions
  uint32_t is = 0, ip = 0, cs = 0, cp = 0;
  const int64_t kh = p.k * p.nhalves;

  for (;;) {
    int64_t u = 0;
    if (lane == 0) u = atomicAdd(p.counter, 1);
    u = __shfl_sync(0xffffffffu, u, 0);
    if (u >= p.nunits) break;
    const int piece = (int)(u / kh);
    const int64_t rest = u - (int64_t)piece * kh;
    const int64_t q = rest / p.nhalves;
    const int h = (int)(rest - q * p.nhalves);
    const int64_t eb = p.off[q * (p.npieces + 1) + piece], ee = p.off[q * (p.npieces + 1) + piece + 1];
    const int col = h * W;

    u64 a0 = 0ull, a1 = 0ull, b0 = 0ull, b1 = 0ull;
    for (int64_t e0 = eb; e0 < ee; e0 += G_ENT) {
      const int L = (int)min((int64_t)G_ENT, ee - e0);
      // stage the block's entries (coalesced), padded to a multiple of 4 with the last row
      const int Lp = (L + 3) & ~3;
      for (int i = lane; i < Lp; i += 32) ebuf[i] = (uint32_t)p.ent[e0 + min(i, L - 1)];
      __syncwarp();
      const int G = Lp >> 2;
      auto issue = [&](int g) {
        uint32_t w0, w1, w2, w3;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3)
                     : "r"(ebuf_s + 16u * (uint32_t)g));
        arrive_tx(bar0 + 8u * is, G_STAGE_BYTES);
        gather4(ring + is * G_STAGE_BYTES, &tm, bar0 + 8u * is, col, (int)(w0 & 0x7fffffffu), (int)(w1 & 0x7fffffffu),
                (int)(w2 & 0x7fffffffu), (int)(w3 & 0x7fffffffu));
        if (++is == G_STAGES) { is = 0; ip ^= 1u; }
      };
      if (lane == 0)
        for (int g = 0; g < G && g < G_STAGES; ++g) issue(g);
      for (int g = 0; g < G; ++g) {
        wait_parity(bar0 + 8u * cs, cp);
        uint32_t w[4];
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                     : "r"(ebuf_s + 16u * (uint32_t)g));
        const uint32_t base = ring + cs * G_STAGE_BYTES + 16u * lane;
        const int nrow = L - 4 * g;  // >= 4 except in the last group
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          if (t < nrow) {
            const uint32_t s32 = 0x3F800000u | (w[t] & 0x80000000u);                          // +-1.0f
            const u64 s64 = (u64)(0x3FF00000u | (w[t] & 0x80000000u)) << 32;                   // +-1.0
            u64 x0, x1, y0, y1;
            lds128(base + t * G_ROW_BYTES, x0, x1);
            lds128(base + t * G_ROW_BYTES + G_ROW_BYTES / 2, y0, y1);
            fma_signed<T>(a0, x0, s32, s64);
            fma_signed<T>(a1, x1, s32, s64);
            fma_signed<T>(b0, y0, s32, s64);
            fma_signed<T>(b1, y1, s32, s64);
          }
        }
        __syncwarp();  // every lane has read the stage before it is refilled
        if (++cs == G_STAGES) { cs = 0; cp ^= 1u; }
        if (lane == 0 && g + G_STAGES < G) issue(g + G_STAGES);
      }
      __syncwarp();  // the entry buffer is reused by the next block
    }

    // unit partial: part[piece][q][col ...]
    T* out = static_cast<T*>(p.part) + ((int64_t)piece * p.k + q) * p.m;
    constexpr int CPL = 16 / (int)sizeof(T);  // columns per lane per half-row
    T va[CPL], vb[CPL];
    if constexpr (sizeof(T) == 4) {
      va[0] = __uint_as_float((uint32_t)a0);
      va[1] = __uint_as_float((uint32_t)(a0 >> 32));
      va[2] = __uint_as_float((uint32_t)a1);
      va[3] = __uint_as_float((uint32_t)(a1 >> 32));
      vb[0] = __uint_as_float((uint32_t)b0);
      vb[1] = __uint_as_float((uint32_t)(b0 >> 32));
      vb[2] = __uint_as_float((uint32_t)b1);
      vb[3] = __uint_as_float((uint32_t)(b1 >> 32));
    } else {
      va[0] = __longlong_as_double((long long)a0);
      va[1] = __longlong_as_double((long long)a1);
      vb[0] = __longlong_as_double((long long)b0);
      vb[1] = __longlong_as_double((long long)b1);
    }
    const int64_t ca = col + CPL * lane, cb = col + W / 2 + CPL * lane;
    // streaming stores: the partials are read once by the reduction, keep L2 for the A pieces
#pragma unroll
    for (int i = 0; i < CPL; ++i) {
      if (ca + i < p.m) __stcs(out + ca + i, va[i]);
      if (cb + i < p.m) __stcs(out + cb + i, vb[i]);
    }
  }
}

// Narrow operands (m <= 8 columns, any row stride, e.g. the right-hand side b of sketch-and-solve):
// one warp per target row q walks q's whole list (all pieces) with the lanes striding over its
// entries and gathering B[j, 0:m] (B stays L2-resident), float64 sums, a fixed-order warp tree.
template <typename T, int M>
__global__ void __launch_bounds__(256)
    sparse_adjoint_narrow(const T* __restrict__ B, int64_t ldb, int m, const int32_t* __restrict__ ent,
                          const int64_t* __restrict__ off, int npieces, int64_t k, double scale, T* __restrict__ SA,
                          int64_t ldsa) {
  const int lane = threadIdx.x & 31;
  const int64_t q = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (q >= k) return;
  const int64_t e0 = off[q * (npieces + 1)], e1 = off[q * (npieces + 1) + npieces];
  double acc[M];
#pragma unroll
  for (int c = 0; c < M; ++c) acc[c] = 0.0;
  for (int64_t e = e0 + lane; e < e1; e += 32) {
    const uint32_t w = (uint32_t)__ldg(ent + e);
    const T* row = B + (int64_t)(w & 0x7fffffffu) * ldb;
    const double sg = (w >> 31) ? -1.0 : 1.0;
#pragma unroll
    for (int c = 0; c < M; ++c)
      if (c < m) acc[c] = fma(sg, (double)__ldg(row + c), acc[c]);
  }
#pragma unroll
  for (int c = 0; c < M; ++c) {
    double v = acc[c];
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0 && c < m) SA[q * ldsa + c] = (T)(v * scale);
  }
}

struct GPlan {
  int npieces, nhalves;
  int64_t prows, nunits;
  size_t smem, part_bytes;
};

template <typename T>
GPlan gather_plan(int64_t d, int64_t m, int64_t k) {
  GPlan pl{};
  pl.nhalves = (int)((m + g_cols<T>() - 1) / g_cols<T>());
  // pieces of ~64 MB of A: resident warps (148 x 16) work inside one or two pieces at a time
  const int64_t row_bytes = m * (int64_t)sizeof(T);
  int64_t piece_mb = 64;
  if (const char* e = getenv("SKETCH_B200_K2G_PIECE_MB")) piece_mb = std::max(1, atoi(e));
  int64_t prows = std::max<int64_t>(1024, (piece_mb << 20) / std::max<int64_t>(1, row_bytes));
  if (prows > d) prows = d;
  pl.prows = prows;
  pl.npieces = (int)((d + prows - 1) / prows);
  pl.nunits = (int64_t)pl.npieces * k * pl.nhalves;
  pl.smem = 1024 + (size_t)G_WARPS * G_STAGES * G_STAGE_BYTES + (size_t)G_WARPS * G_ENT * 4 + (size_t)G_WARPS * G_STAGES * 8;
  pl.part_bytes = (size_t)pl.npieces * k * m * sizeof(T);
  return pl;
}

template <typename T>
int gather_run(const T* A, int64_t d, int64_t m, int64_t lda, const int32_t* ent, const int64_t* off, int64_t k,
               double scale, T* SA, int64_t ldsa, int accumulate, void* ws, size_t ws_bytes, cudaStream_t s) {
  const GPlan pl = gather_plan<T>(d, m, k);
  const size_t need = pl.part_bytes + 256;
  if (!ws || ws_bytes < need) return fail(SK_EINVAL, "sk_sparse_adjoint_gather: workspace too small");
  sm100::EncodeTiledFnT fn = sm100::encode_tiled_fn();
  if (!fn) return fail(SK_ECUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)m, (cuuint64_t)d};
  cuuint64_t strides[1] = {(cuuint64_t)lda * sizeof(T)};
  cuuint32_t box[2] = {(cuuint32_t)g_cols<T>(), 1};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapDataType dt = sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  if (fn(&tm, dt, 2, const_cast<T*>(A), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return fail(SK_EINVAL, "sk_sparse_adjoint_gather: cannot describe A for TMA");
  GParams p{};
  p.d = d;
  p.m = m;
  p.k = k;
  p.prows = pl.prows;
  p.npieces = pl.npieces;
  p.nhalves = pl.nhalves;
  p.nunits = pl.nunits;
  p.ent = ent;
  p.off = off;
  p.part = ws;
  p.counter = reinterpret_cast<int*>(static_cast<uint8_t*>(ws) + pl.part_bytes);
  cudaMemsetAsync(p.counter, 0, sizeof(int), s);
  allow_smem(sparse_adjoint_gather<T>, pl.smem);
  sparse_adjoint_gather<T><<<(unsigned)sm_count(), G_WARPS * 32, pl.smem, s>>>(tm, p);
  int st = check_launch("sk_sparse_adjoint_gather");
  if (st != SK_OK) return st;
  if constexpr (sizeof(T) == 4)
    return adjoint_reduce_f32(static_cast<const float*>(ws), pl.npieces, k, m, scale, SA, ldsa, accumulate, s);
  else
    return adjoint_reduce_f64(static_cast<const double*>(ws), pl.npieces, k, m, scale, SA, ldsa, accumulate, s);
}

}  // namespace
}  // namespace skb

using namespace skb;

extern "C" int64_t sk_sparse_adjoint_gather_pieces(int dtype, int64_t d, int64_t m, int64_t k, int64_t* piece_rows) {
  if (d < 1 || m < 1 || k < 1) return fail(SK_EINVAL, "sk_sparse_adjoint_gather_pieces: bad shape");
  GPlan pl{};
  if (dtype == SK_F32) pl = gather_plan<float>(d, m, k);
  else if (dtype == SK_F64) pl = gather_plan<double>(d, m, k);
  else return fail(SK_EINVAL, "sk_sparse_adjoint_gather_pieces: bad dtype");
  if (piece_rows) *piece_rows = pl.prows;
  return pl.npieces;
}

extern "C" size_t sk_sparse_adjoint_gather_workspace_bytes(int dtype, int64_t d, int64_t m, int64_t k) {
  if (d < 1 || m < 1 || k < 1) return 0;
  if (dtype == SK_F32) return gather_plan<float>(d, m, k).part_bytes + 256;
  if (dtype == SK_F64) return gather_plan<double>(d, m, k).part_bytes + 256;
  return 0;
}

extern "C" int sk_sparse_adjoint_gather(int dtype, const void* A, int64_t d, int64_t m, int64_t lda,
                                        const int32_t* ent, const int64_t* off, int64_t k, double scale, void* SA,
                                        int64_t ldsa, int accumulate, void* ws, size_t ws_bytes, void* stream) {
  if (d < 1 || m < 0 || k < 1 || lda < m || ldsa < m)
    return fail(SK_EINVAL, "sk_sparse_adjoint_gather: bad shape/leading dimension");
  if (dtype != SK_F32 && dtype != SK_F64) return fail(SK_EINVAL, "sk_sparse_adjoint_gather: bad dtype");
  if (m == 0) return SK_OK;
  if (!A || !SA || !ent || !off) return fail(SK_EINVAL, "sk_sparse_adjoint_gather: null pointer");
  const int64_t q16 = 16 / (dtype == SK_F32 ? 4 : 8);
  if ((reinterpret_cast<uintptr_t>(A) & 15) || (lda % q16))
    return fail(SK_EUNSUPPORTED, "sk_sparse_adjoint_gather: A must be 16-byte aligned with 16-byte rows");
  if (d >= (int64_t)1 << 31) return fail(SK_EUNSUPPORTED, "sk_sparse_adjoint_gather: d must be below 2^31");
  cudaStream_t s = as_stream(stream);
  if (dtype == SK_F32)
    return gather_run<float>(static_cast<const float*>(A), d, m, lda, ent, off, k, scale, static_cast<float*>(SA),
                             ldsa, accumulate, ws, ws_bytes, s);
  return gather_run<double>(static_cast<const double*>(A), d, m, lda, ent, off, k, scale, static_cast<double*>(SA),
                            ldsa, accumulate, ws, ws_bytes, s);
}

extern "C" int sk_sparse_adjoint_narrow(int dtype, const void* B, int64_t d, int64_t m, int64_t ldb, const int32_t* ent,
                                        const int64_t* off, int npieces, int64_t k, double scale, void* SA,
                                        int64_t ldsa, void* stream) {
  if (d < 1 || m < 0 || m > 8 || k < 1 || npieces < 1 || ldb < m || ldsa < m)
    return fail(SK_EINVAL, "sk_sparse_adjoint_narrow: bad shape (m <= 8)/leading dimension");
  if (dtype != SK_F32 && dtype != SK_F64) return fail(SK_EINVAL, "sk_sparse_adjoint_narrow: bad dtype");
  if (m == 0) return SK_OK;
  if (!B || !SA || !ent || !off) return fail(SK_EINVAL, "sk_sparse_adjoint_narrow: null pointer");
  cudaStream_t s = as_stream(stream);
  const unsigned grid = (unsigned)((k + 7) / 8);
  if (dtype == SK_F32) {
    if (m == 1)
      sparse_adjoint_narrow<float, 1><<<grid, 256, 0, s>>>(static_cast<const float*>(B), ldb, 1, ent, off, npieces, k,
                                                            scale, static_cast<float*>(SA), ldsa);
    else
      sparse_adjoint_narrow<float, 8><<<grid, 256, 0, s>>>(static_cast<const float*>(B), ldb, (int)m, ent, off,
                                                            npieces, k, scale, static_cast<float*>(SA), ldsa);
  } else {
    if (m == 1)
      sparse_adjoint_narrow<double, 1><<<grid, 256, 0, s>>>(static_cast<const double*>(B), ldb, 1, ent, off, npieces,
                                                             k, scale, static_cast<double*>(SA), ldsa);
    else
      sparse_adjoint_narrow<double, 8><<<grid, 256, 0, s>>>(static_cast<const double*>(B), ldb, (int)m, ent, off,
                                                             npieces, k, scale, static_cast<double*>(SA), ldsa);
  }
  return check_launch("sk_sparse_adjoint_narrow");
}
