// K2w — float32 sparse-sign adjoint  SA = scale * Omega^T * A  with register accumulators.
//
// Replaces `_SparseTM.apply_adjoint` = `self.matrix.conj().T @ b` (src/sketch/sparse.py:68-78) for
// float32 operands (BASELINE config 4: S = Omega^T, 2048 x 4194304, zeta = 8, A 4194304 x 512).
//
// Work split. A CTA owns a 128-column slice of A (4 columns per lane, 16-byte shared loads) and a
// group of 256 output rows c (16 warps x 16 rows; each lane keeps 16 x 4 accumulators in
// registers), over a contiguous piece of the row chunks (128 rows = one 64 KB tile each, a 3-deep
// TMA ring fed by a producer warp). The 8 groups of a slice read the same tiles at about the same
// time and L2 serves the repeats (DRAM reads stay ~1.04x |A|). Measured alternatives (DESIGN.md
// §K2w): clusters that multicast each tile to the 2/4/8 groups of a slice (the per-chunk
// cross-CTA release costs more than the L2 reads it saves: 11.0 / 13.1 / 23.3 ms vs 9.8 ms),
// 64-column slices (13 ms), 64-row chunks (17.6 ms).
//
// Entries. Host-encoded per (chunk, group) segment (sk_sparse_adjoint_wide_encode): a 17-entry
// uint16 header of warp offsets (multiples of 4) followed by uint16 entries
// (row_in_chunk << 9) | (neg << 4) | (c mod 16), each warp list padded with no-op entries (32).
// A warp reads four entries per uniform 8-byte load; each entry is one 256-byte row read (conflict
// free) added into accumulator c mod 32 through a warp-uniform jump table. Pieces write partial sums; the float64 ordered reduction of
// sparse_adjoint.cu forms SA (deterministic).
#include <cuda.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "sm100.cuh"

namespace skb {

// defined in sparse_adjoint.cu: part[p][k][m] summed over p in order (float64), scaled, stored to SA
int adjoint_reduce_f32(const float* part, int npieces, int64_t k, int64_t m, double scale, float* SA, int64_t ldsa,
                       int accumulate, cudaStream_t s);
int adjoint_reduce_f64(const double* part, int npieces, int64_t k, int64_t m, double scale, double* SA, int64_t ldsa,
                       int accumulate, cudaStream_t s);

namespace {

using namespace sm100;

constexpr int W_R = 128;                 // rows per chunk
constexpr int W_ROW_BYTES = 512;         // bytes of a tile row: 128 float32 or 64 float64 columns (16 per lane)
constexpr int W_WARPS = 16;
constexpr int W_CPW = 16;                // output rows per warp
constexpr int W_CG = W_WARPS * W_CPW;    // output rows per CTA (group)
constexpr int W_HDR = 24;                // header uint16s: 17 warp offsets, padded to 48 bytes
constexpr int W_STAGES = 3;
constexpr uint32_t W_TILE = W_R * W_ROW_BYTES;  // 64 KB
template <typename T>
constexpr int w_cols() {
  return W_ROW_BYTES / (int)sizeof(T);  // columns per CTA slice
}

typedef unsigned long long u64;

__device__ __forceinline__ u64 lds64(uint32_t addr) {
  u64 v;
  asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

struct WParams {
  int64_t d, m, k;
  int nchunks, ngroups, nslices, npieces, chunks_per_piece;
  int64_t chunk_base;  // first encoded chunk of this launch (row block [128 * chunk_base, ...))
  uint32_t stage_bytes;
  const uint16_t* enc;
  const int64_t* seg_off;  // [nchunks * ngroups + 1], uint16 units
  void* part;              // [npieces][k][m] of the element type
};

// Dispatch one entry: index j = (neg << 4) | (c mod 16) selects acc[c mod 16] +=/-= v (four columns
// as two packed pairs) through a warp-uniform indirect branch (brx.idx.uni over a 33-entry jump
// table); j = 32 is a padding no-op.
#define SKB_W_DISPATCH(V0, V1, JJ) \
  asm volatile( \
      "{\n\t" \
      "T_%=: .branchtargets A0_%=, A1_%=, A2_%=, A3_%=, A4_%=, A5_%=, A6_%=, A7_%=, A8_%=, A9_%=, A10_%=, A11_%=, A12_%=, A13_%=, A14_%=, A15_%=, S0_%=, S1_%=, S2_%=, S3_%=, S4_%=, S5_%=, S6_%=, S7_%=, S8_%=, S9_%=, S10_%=, S11_%=, S12_%=, S13_%=, S14_%=, S15_%=, D_%=;\n\t" \
      "brx.idx.uni %34, T_%=;\n\t" \
      "A0_%=: add.rn.f32x2 %0, %0, %32;\n\tadd.rn.f32x2 %1, %1, %33;\n\tbra.uni D_%=;\n\t" \
      "A1_%=: add.rn.f32x2 %2, %2, %32;\n\tadd.rn.f32x2 %3, %3, %33;\n\tbra.uni D_%=;\n\t" \
      "A2_%=: add.rn.f32x2 %4, %4, %32;\n\tadd.rn.f32x2 %5, %5, %33;\n\tbra.uni D_%=;\n\t" \
      "A3_%=: add.rn.f32x2 %6, %6, %32;\n\tadd.rn.f32x2 %7, %7, %33;\n\tbra.uni D_%=;\n\t" \
      "A4_%=: add.rn.f32x2 %8, %8, %32;\n\tadd.rn.f32x2 %9, %9, %33;\n\tbra.uni D_%=;\n\t" \
      "A5_%=: add.rn.f32x2 %10, %10, %32;\n\tadd.rn.f32x2 %11, %11, %33;\n\tbra.uni D_%=;\n\t" \
      "A6_%=: add.rn.f32x2 %12, %12, %32;\n\tadd.rn.f32x2 %13, %13, %33;\n\tbra.uni D_%=;\n\t" \
      "A7_%=: add.rn.f32x2 %14, %14, %32;\n\tadd.rn.f32x2 %15, %15, %33;\n\tbra.uni D_%=;\n\t" \
      "A8_%=: add.rn.f32x2 %16, %16, %32;\n\tadd.rn.f32x2 %17, %17, %33;\n\tbra.uni D_%=;\n\t" \
      "A9_%=: add.rn.f32x2 %18, %18, %32;\n\tadd.rn.f32x2 %19, %19, %33;\n\tbra.uni D_%=;\n\t" \
      "A10_%=: add.rn.f32x2 %20, %20, %32;\n\tadd.rn.f32x2 %21, %21, %33;\n\tbra.uni D_%=;\n\t" \
      "A11_%=: add.rn.f32x2 %22, %22, %32;\n\tadd.rn.f32x2 %23, %23, %33;\n\tbra.uni D_%=;\n\t" \
      "A12_%=: add.rn.f32x2 %24, %24, %32;\n\tadd.rn.f32x2 %25, %25, %33;\n\tbra.uni D_%=;\n\t" \
      "A13_%=: add.rn.f32x2 %26, %26, %32;\n\tadd.rn.f32x2 %27, %27, %33;\n\tbra.uni D_%=;\n\t" \
      "A14_%=: add.rn.f32x2 %28, %28, %32;\n\tadd.rn.f32x2 %29, %29, %33;\n\tbra.uni D_%=;\n\t" \
      "A15_%=: add.rn.f32x2 %30, %30, %32;\n\tadd.rn.f32x2 %31, %31, %33;\n\tbra.uni D_%=;\n\t" \
      "S0_%=: sub.rn.f32x2 %0, %0, %32;\n\tsub.rn.f32x2 %1, %1, %33;\n\tbra.uni D_%=;\n\t" \
      "S1_%=: sub.rn.f32x2 %2, %2, %32;\n\tsub.rn.f32x2 %3, %3, %33;\n\tbra.uni D_%=;\n\t" \
      "S2_%=: sub.rn.f32x2 %4, %4, %32;\n\tsub.rn.f32x2 %5, %5, %33;\n\tbra.uni D_%=;\n\t" \
      "S3_%=: sub.rn.f32x2 %6, %6, %32;\n\tsub.rn.f32x2 %7, %7, %33;\n\tbra.uni D_%=;\n\t" \
      "S4_%=: sub.rn.f32x2 %8, %8, %32;\n\tsub.rn.f32x2 %9, %9, %33;\n\tbra.uni D_%=;\n\t" \
      "S5_%=: sub.rn.f32x2 %10, %10, %32;\n\tsub.rn.f32x2 %11, %11, %33;\n\tbra.uni D_%=;\n\t" \
      "S6_%=: sub.rn.f32x2 %12, %12, %32;\n\tsub.rn.f32x2 %13, %13, %33;\n\tbra.uni D_%=;\n\t" \
      "S7_%=: sub.rn.f32x2 %14, %14, %32;\n\tsub.rn.f32x2 %15, %15, %33;\n\tbra.uni D_%=;\n\t" \
      "S8_%=: sub.rn.f32x2 %16, %16, %32;\n\tsub.rn.f32x2 %17, %17, %33;\n\tbra.uni D_%=;\n\t" \
      "S9_%=: sub.rn.f32x2 %18, %18, %32;\n\tsub.rn.f32x2 %19, %19, %33;\n\tbra.uni D_%=;\n\t" \
      "S10_%=: sub.rn.f32x2 %20, %20, %32;\n\tsub.rn.f32x2 %21, %21, %33;\n\tbra.uni D_%=;\n\t" \
      "S11_%=: sub.rn.f32x2 %22, %22, %32;\n\tsub.rn.f32x2 %23, %23, %33;\n\tbra.uni D_%=;\n\t" \
      "S12_%=: sub.rn.f32x2 %24, %24, %32;\n\tsub.rn.f32x2 %25, %25, %33;\n\tbra.uni D_%=;\n\t" \
      "S13_%=: sub.rn.f32x2 %26, %26, %32;\n\tsub.rn.f32x2 %27, %27, %33;\n\tbra.uni D_%=;\n\t" \
      "S14_%=: sub.rn.f32x2 %28, %28, %32;\n\tsub.rn.f32x2 %29, %29, %33;\n\tbra.uni D_%=;\n\t" \
      "S15_%=: sub.rn.f32x2 %30, %30, %32;\n\tsub.rn.f32x2 %31, %31, %33;\n\tbra.uni D_%=;\n\t" \
      "D_%=:\n\t}" \
      : "+l"(acc[0]), "+l"(acc[1]), "+l"(acc[2]), "+l"(acc[3]), "+l"(acc[4]), "+l"(acc[5]), "+l"(acc[6]), "+l"(acc[7]), "+l"(acc[8]), "+l"(acc[9]), "+l"(acc[10]), "+l"(acc[11]), "+l"(acc[12]), "+l"(acc[13]), "+l"(acc[14]), "+l"(acc[15]), "+l"(acc[16]), "+l"(acc[17]), "+l"(acc[18]), "+l"(acc[19]), "+l"(acc[20]), "+l"(acc[21]), "+l"(acc[22]), "+l"(acc[23]), "+l"(acc[24]), "+l"(acc[25]), "+l"(acc[26]), "+l"(acc[27]), "+l"(acc[28]), "+l"(acc[29]), "+l"(acc[30]), "+l"(acc[31]) \
      : "l"(V0), "l"(V1), "r"(JJ))

// float64 variant: each packed pair register holds one double (two columns per lane)
#define SKB_W_DISPATCH64(V0, V1, JJ) \
  asm volatile( \
      "{\n\t" \
      "T_%=: .branchtargets A0_%=, A1_%=, A2_%=, A3_%=, A4_%=, A5_%=, A6_%=, A7_%=, A8_%=, A9_%=, A10_%=, A11_%=, A12_%=, A13_%=, A14_%=, A15_%=, S0_%=, S1_%=, S2_%=, S3_%=, S4_%=, S5_%=, S6_%=, S7_%=, S8_%=, S9_%=, S10_%=, S11_%=, S12_%=, S13_%=, S14_%=, S15_%=, D_%=;\n\t" \
      "brx.idx.uni %34, T_%=;\n\t" \
      "A0_%=: add.rn.f64 %0, %0, %32;\n\tadd.rn.f64 %1, %1, %33;\n\tbra.uni D_%=;\n\t" \
      "A1_%=: add.rn.f64 %2, %2, %32;\n\tadd.rn.f64 %3, %3, %33;\n\tbra.uni D_%=;\n\t" \
      "A2_%=: add.rn.f64 %4, %4, %32;\n\tadd.rn.f64 %5, %5, %33;\n\tbra.uni D_%=;\n\t" \
      "A3_%=: add.rn.f64 %6, %6, %32;\n\tadd.rn.f64 %7, %7, %33;\n\tbra.uni D_%=;\n\t" \
      "A4_%=: add.rn.f64 %8, %8, %32;\n\tadd.rn.f64 %9, %9, %33;\n\tbra.uni D_%=;\n\t" \
      "A5_%=: add.rn.f64 %10, %10, %32;\n\tadd.rn.f64 %11, %11, %33;\n\tbra.uni D_%=;\n\t" \
      "A6_%=: add.rn.f64 %12, %12, %32;\n\tadd.rn.f64 %13, %13, %33;\n\tbra.uni D_%=;\n\t" \
      "A7_%=: add.rn.f64 %14, %14, %32;\n\tadd.rn.f64 %15, %15, %33;\n\tbra.uni D_%=;\n\t" \
      "A8_%=: add.rn.f64 %16, %16, %32;\n\tadd.rn.f64 %17, %17, %33;\n\tbra.uni D_%=;\n\t" \
      "A9_%=: add.rn.f64 %18, %18, %32;\n\tadd.rn.f64 %19, %19, %33;\n\tbra.uni D_%=;\n\t" \
      "A10_%=: add.rn.f64 %20, %20, %32;\n\tadd.rn.f64 %21, %21, %33;\n\tbra.uni D_%=;\n\t" \
      "A11_%=: add.rn.f64 %22, %22, %32;\n\tadd.rn.f64 %23, %23, %33;\n\tbra.uni D_%=;\n\t" \
      "A12_%=: add.rn.f64 %24, %24, %32;\n\tadd.rn.f64 %25, %25, %33;\n\tbra.uni D_%=;\n\t" \
      "A13_%=: add.rn.f64 %26, %26, %32;\n\tadd.rn.f64 %27, %27, %33;\n\tbra.uni D_%=;\n\t" \
      "A14_%=: add.rn.f64 %28, %28, %32;\n\tadd.rn.f64 %29, %29, %33;\n\tbra.uni D_%=;\n\t" \
      "A15_%=: add.rn.f64 %30, %30, %32;\n\tadd.rn.f64 %31, %31, %33;\n\tbra.uni D_%=;\n\t" \
      "S0_%=: sub.rn.f64 %0, %0, %32;\n\tsub.rn.f64 %1, %1, %33;\n\tbra.uni D_%=;\n\t" \
      "S1_%=: sub.rn.f64 %2, %2, %32;\n\tsub.rn.f64 %3, %3, %33;\n\tbra.uni D_%=;\n\t" \
      "S2_%=: sub.rn.f64 %4, %4, %32;\n\tsub.rn.f64 %5, %5, %33;\n\tbra.uni D_%=;\n\t" \
      "S3_%=: sub.rn.f64 %6, %6, %32;\n\tsub.rn.f64 %7, %7, %33;\n\tbra.uni D_%=;\n\t" \
      "S4_%=: sub.rn.f64 %8, %8, %32;\n\tsub.rn.f64 %9, %9, %33;\n\tbra.uni D_%=;\n\t" \
      "S5_%=: sub.rn.f64 %10, %10, %32;\n\tsub.rn.f64 %11, %11, %33;\n\tbra.uni D_%=;\n\t" \
      "S6_%=: sub.rn.f64 %12, %12, %32;\n\tsub.rn.f64 %13, %13, %33;\n\tbra.uni D_%=;\n\t" \
      "S7_%=: sub.rn.f64 %14, %14, %32;\n\tsub.rn.f64 %15, %15, %33;\n\tbra.uni D_%=;\n\t" \
      "S8_%=: sub.rn.f64 %16, %16, %32;\n\tsub.rn.f64 %17, %17, %33;\n\tbra.uni D_%=;\n\t" \
      "S9_%=: sub.rn.f64 %18, %18, %32;\n\tsub.rn.f64 %19, %19, %33;\n\tbra.uni D_%=;\n\t" \
      "S10_%=: sub.rn.f64 %20, %20, %32;\n\tsub.rn.f64 %21, %21, %33;\n\tbra.uni D_%=;\n\t" \
      "S11_%=: sub.rn.f64 %22, %22, %32;\n\tsub.rn.f64 %23, %23, %33;\n\tbra.uni D_%=;\n\t" \
      "S12_%=: sub.rn.f64 %24, %24, %32;\n\tsub.rn.f64 %25, %25, %33;\n\tbra.uni D_%=;\n\t" \
      "S13_%=: sub.rn.f64 %26, %26, %32;\n\tsub.rn.f64 %27, %27, %33;\n\tbra.uni D_%=;\n\t" \
      "S14_%=: sub.rn.f64 %28, %28, %32;\n\tsub.rn.f64 %29, %29, %33;\n\tbra.uni D_%=;\n\t" \
      "S15_%=: sub.rn.f64 %30, %30, %32;\n\tsub.rn.f64 %31, %31, %33;\n\tbra.uni D_%=;\n\t" \
      "D_%=:\n\t}" \
      : "+l"(acc[0]), "+l"(acc[1]), "+l"(acc[2]), "+l"(acc[3]), "+l"(acc[4]), "+l"(acc[5]), "+l"(acc[6]), "+l"(acc[7]), "+l"(acc[8]), "+l"(acc[9]), "+l"(acc[10]), "+l"(acc[11]), "+l"(acc[12]), "+l"(acc[13]), "+l"(acc[14]), "+l"(acc[15]), "+l"(acc[16]), "+l"(acc[17]), "+l"(acc[18]), "+l"(acc[19]), "+l"(acc[20]), "+l"(acc[21]), "+l"(acc[22]), "+l"(acc[23]), "+l"(acc[24]), "+l"(acc[25]), "+l"(acc[26]), "+l"(acc[27]), "+l"(acc[28]), "+l"(acc[29]), "+l"(acc[30]), "+l"(acc[31]) \
      : "l"(V0), "l"(V1), "r"(JJ))

// Walk entries [a, b) of this warp (a, b multiples of 4): four entries per uniform 8-byte shared
// load; their four row values (16 bytes per lane) are loaded before the four dispatches.
__device__ __forceinline__ void lds128u(uint32_t addr, u64& x, u64& y) {
  asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "r"(addr));
}

template <typename T>
__device__ __forceinline__ void walk(u64 (&acc)[2 * W_CPW], uint32_t tile_lane, uint32_t ent, int a, int b) {
  for (int e = a; e < b; e += 4) {
    const u64 q = lds64(ent + 2u * (uint32_t)e);
    const uint32_t lo = (uint32_t)q, hi = (uint32_t)(q >> 32);
    const uint32_t u0 = lo & 0xffffu, u1 = lo >> 16, u2 = hi & 0xffffu, u3 = hi >> 16;
    u64 a0, b0, a1, b1, a2, b2, a3, b3;
    lds128u(tile_lane + (u0 & 0xfe00u), a0, b0);
    lds128u(tile_lane + (u1 & 0xfe00u), a1, b1);
    lds128u(tile_lane + (u2 & 0xfe00u), a2, b2);
    lds128u(tile_lane + (u3 & 0xfe00u), a3, b3);
    const uint32_t j0 = u0 & 63u, j1 = u1 & 63u, j2 = u2 & 63u, j3 = u3 & 63u;
    if constexpr (sizeof(T) == 4) {
      SKB_W_DISPATCH(a0, b0, j0);
      SKB_W_DISPATCH(a1, b1, j1);
      SKB_W_DISPATCH(a2, b2, j2);
      SKB_W_DISPATCH(a3, b3, j3);
    } else {
      SKB_W_DISPATCH64(a0, b0, j0);
      SKB_W_DISPATCH64(a1, b1, j1);
      SKB_W_DISPATCH64(a2, b2, j2);
      SKB_W_DISPATCH64(a3, b3, j3);
    }
  }
}

template <typename T>
__global__ void __launch_bounds__((W_WARPS + 1) * 32, 1)
    sparse_adjoint_wide(const __grid_constant__ CUtensorMap tm, const WParams p) {
  constexpr int W_COLS = w_cols<T>();
  extern __shared__ uint8_t smem_dyn[];
  uint8_t* smem = smem_dyn + ((1024u - (smem_u32(smem_dyn) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + W_STAGES * p.stage_bytes);
  uint64_t* consumed = full + W_STAGES;  // all 16 consumer warps done with slot s

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = blockIdx.x, slice = blockIdx.y, piece = blockIdx.z;
  const int h0 = piece * p.chunks_per_piece;
  const int nch = (int)min((int64_t)p.chunks_per_piece, (int64_t)p.nchunks - h0);

  if (tid == 0) {
    for (int s = 0; s < W_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&consumed[s], W_WARPS);
    }
    fence_mbar_init();
    tma_prefetch_desc(&tm);
  }
  __syncthreads();

  if (warp == W_WARPS) {
    // ------------------------------------------------------------ producer warp (one thread)
    if (lane == 0) {
      for (int i = 0; i < nch; ++i) {
        const int s = i % W_STAGES;
        if (i >= W_STAGES) mbar_wait(&consumed[s], (uint32_t)(i / W_STAGES - 1) & 1u);
        const int h = h0 + i;
        const int64_t sg = (p.chunk_base + h) * p.ngroups + g;
        const uint32_t seg_bytes = (uint32_t)(p.seg_off[sg + 1] - p.seg_off[sg]) * 2u;
        const uint32_t st = smem_u32(smem + (size_t)s * p.stage_bytes);
        mbar_arrive_expect_tx(&full[s], W_TILE + seg_bytes);
        tma_load_2d(smem + (size_t)s * p.stage_bytes, &tm, &full[s], slice * W_COLS, h * W_R);
        bulk_g2s(st + W_TILE, p.enc + p.seg_off[sg], seg_bytes, smem_u32(&full[s]));
      }
    }
    return;
  }

  u64 acc[2 * W_CPW];
#pragma unroll
  for (int j = 0; j < 2 * W_CPW; ++j) acc[j] = 0ull;

  for (int i = 0; i < nch; ++i) {
    const int s = i % W_STAGES;
    const uint32_t ph = (uint32_t)(i / W_STAGES) & 1u;
    mbar_wait(&full[s], ph);
    const uint32_t st = smem_u32(smem + (size_t)s * p.stage_bytes);
    const uint32_t hdr = st + W_TILE;
    const int a = (int)lds_u16(hdr + 2u * warp), b = (int)lds_u16(hdr + 2u * warp + 2u);
    walk<T>(acc, st + 16u * lane, hdr + 2u * W_HDR, a, b);
    __syncwarp();
    if (lane == 0) mbar_arrive(&consumed[s]);
  }

  {
    constexpr int CPL = 16 / (int)sizeof(T);  // columns per lane
    const int64_t col = (int64_t)slice * W_COLS + CPL * lane;
    T* out = static_cast<T*>(p.part) + (int64_t)piece * p.k * p.m;
#pragma unroll
    for (int j = 0; j < W_CPW; ++j) {
      const int64_t c = (int64_t)g * W_CG + warp * W_CPW + j;
      if (c < p.k) {
        T v[CPL];
        if constexpr (sizeof(T) == 4) {
          v[0] = __uint_as_float((uint32_t)acc[2 * j]);
          v[1] = __uint_as_float((uint32_t)(acc[2 * j] >> 32));
          v[2] = __uint_as_float((uint32_t)acc[2 * j + 1]);
          v[3] = __uint_as_float((uint32_t)(acc[2 * j + 1] >> 32));
        } else {
          v[0] = __longlong_as_double((long long)acc[2 * j]);
          v[1] = __longlong_as_double((long long)acc[2 * j + 1]);
        }
#pragma unroll
        for (int q = 0; q < CPL; ++q)
          if (col + q < p.m) out[c * p.m + col + q] = v[q];
      }
    }
  }
}

struct WPlan {
  int nchunks, ngroups, nslices, npieces, chunks_per_piece;
  uint32_t stage_bytes;
  size_t smem, ws_bytes;
};

WPlan wide_plan(int64_t d, int64_t m, int64_t k, int32_t seg_cap, int cols = 128, int esize = 4) {
  WPlan pl{};
  pl.nchunks = (int)((d + W_R - 1) / W_R);
  pl.ngroups = (int)((k + W_CG - 1) / W_CG);
  pl.nslices = (int)((m + cols - 1) / cols);
  const int64_t roles = (int64_t)pl.ngroups * pl.nslices;
  // one CTA per SM: about 4 waves, with the piece count that fills the last wave best (config 4:
  // 32 roles x 37 pieces = 8 full waves instead of 32 x 19 = 4.1)
  const int64_t sms = sm_count();
  const int64_t pmin = (4 * sms + roles - 1) / roles;
  // at least 8 chunks per piece: the ring must fill, and every piece adds a k x m partial
  const int64_t pcap = std::max<int64_t>(1, (pl.nchunks + 7) / 8);
  int64_t pieces = std::min(pmin, pcap);
  double best = 0.0;
  for (int64_t q = pieces; q <= std::min(2 * pmin, pcap); ++q) {
    const int64_t ctas = roles * q;
    const double fill = (double)ctas / (double)(((ctas + sms - 1) / sms) * sms);
    if (fill > best + 1e-9) {
      best = fill;
      pieces = q;
    }
  }
  pl.chunks_per_piece = (int)((pl.nchunks + pieces - 1) / pieces);
  pl.npieces = (pl.nchunks + pl.chunks_per_piece - 1) / pl.chunks_per_piece;
  pl.stage_bytes = (W_TILE + (uint32_t)seg_cap * 2u + 1023u) & ~1023u;
  pl.smem = 1024 + (size_t)W_STAGES * pl.stage_bytes + 2 * W_STAGES * 8;
  pl.ws_bytes = (size_t)pl.npieces * k * m * esize;
  return pl;
}

}  // namespace
}  // namespace skb

using namespace skb;

extern "C" int64_t sk_sparse_adjoint_wide_encode(int64_t d, int64_t k, int64_t nnz, const int64_t* rows,
                                                 const int64_t* cols, const uint8_t* neg, uint16_t* enc,
                                                 int64_t enc_cap, int64_t* seg_off, int32_t* seg_cap) {
  if (d < 1 || k < 1 || nnz < 0 || !seg_off || !seg_cap || (nnz > 0 && (!rows || !cols || !neg)))
    return fail(SK_EINVAL, "sk_sparse_adjoint_wide_encode: bad arguments");
  const int64_t nchunks = (d + W_R - 1) / W_R, ngroups = (k + W_CG - 1) / W_CG, nseg = nchunks * ngroups;
  // per (segment, warp) entry counts; each warp list is padded to a multiple of 4 with no-op entries
  std::vector<int32_t> cnt((size_t)nseg * W_WARPS, 0);
  for (int64_t e = 0; e < nnz; ++e) {
    const int64_t r = rows[e], c = cols[e];
    if (r < 0 || r >= d || c < 0 || c >= k) return fail(SK_EINVAL, "sk_sparse_adjoint_wide_encode: index out of range");
    ++cnt[(size_t)((r / W_R) * ngroups + c / W_CG) * W_WARPS + (c % W_CG) / W_CPW];
  }
  int64_t total = 0;
  int32_t cap = 0;
  for (int64_t sg = 0; sg < nseg; ++sg) {
    int64_t n = 0;
    for (int w = 0; w < W_WARPS; ++w) n += (cnt[(size_t)sg * W_WARPS + w] + 3) / 4 * 4;
    if (n > 65535) return fail(SK_EUNSUPPORTED, "sk_sparse_adjoint_wide_encode: segment over 65535 entries");
    const int64_t len = W_HDR + (n + 7) / 8 * 8;  // 16-byte multiple (bulk copy granularity)
    seg_off[sg] = total;
    total += len;
    cap = std::max<int32_t>(cap, (int32_t)len);
  }
  seg_off[nseg] = total;
  *seg_cap = cap;
  if (!enc) return total;
  if (enc_cap < total) return fail(SK_EINVAL, "sk_sparse_adjoint_wide_encode: output too small");
  std::fill(enc, enc + total, (uint16_t)32);  // 32 = no-op dispatch index (row 0)
  std::vector<int32_t> pos((size_t)nseg * W_WARPS);
  for (int64_t sg = 0; sg < nseg; ++sg) {
    uint16_t* h = enc + seg_off[sg];
    int32_t run = 0;
    for (int w = 0; w < W_WARPS; ++w) {
      h[w] = (uint16_t)run;
      pos[(size_t)sg * W_WARPS + w] = run;
      run += (cnt[(size_t)sg * W_WARPS + w] + 3) / 4 * 4;
    }
    h[W_WARPS] = (uint16_t)run;
    for (int i = W_WARPS + 1; i < W_HDR; ++i) h[i] = 0;
  }
  for (int64_t e = 0; e < nnz; ++e) {
    const int64_t r = rows[e], c = cols[e];
    const int64_t sg = (r / W_R) * ngroups + c / W_CG;
    int32_t& q = pos[(size_t)sg * W_WARPS + (c % W_CG) / W_CPW];
    enc[seg_off[sg] + W_HDR + q] = (uint16_t)(((r % W_R) << 9) | (neg[e] ? 16 : 0) | (c % W_CPW));
    ++q;
  }
  return total;
}

extern "C" int64_t sk_sparse_adjoint_wide_segments(int64_t d, int64_t k) {
  if (d < 1 || k < 1) return fail(SK_EINVAL, "sk_sparse_adjoint_wide_segments: bad shape");
  return ((d + W_R - 1) / W_R) * ((k + W_CG - 1) / W_CG) + 1;
}

namespace skb {
namespace {

template <typename T>
int wide_rows_t(const T* A, int64_t d, int64_t r0, int64_t r1, int64_t m, int64_t lda, const uint16_t* enc,
                const int64_t* seg_off, int32_t seg_cap, int64_t k, double scale, T* SA, int64_t ldsa, int accumulate,
                void* ws, size_t ws_bytes, void* stream) {
  constexpr int COLS = w_cols<T>();
  constexpr int64_t LDA_Q = 16 / (int64_t)sizeof(T);  // 16-byte row alignment
  if (d < 1 || m < 0 || k < 1 || lda < m || ldsa < m || seg_cap < W_HDR)
    return fail(SK_EINVAL, "sk_sparse_adjoint_wide: bad shape/leading dimension");
  if (r0 < 0 || r1 > d || r0 >= r1 || (r0 % W_R) != 0)
    return fail(SK_EINVAL, "sk_sparse_adjoint_wide: row block must be [r0, r1) within [0, d) with r0 % 128 == 0");
  if (m == 0) return SK_OK;
  if (!A || !SA || !enc || !seg_off) return fail(SK_EINVAL, "sk_sparse_adjoint_wide: null pointer");
  if ((reinterpret_cast<uintptr_t>(A) & 15) || (lda % LDA_Q))
    return fail(SK_EUNSUPPORTED, "sk_sparse_adjoint_wide: A must be 16-byte aligned with 16-byte rows");
  const int64_t rows = r1 - r0;
  const WPlan pl = wide_plan(rows, m, k, seg_cap, COLS, (int)sizeof(T));
  if (pl.smem > 227 * 1024) return fail(SK_EUNSUPPORTED, "sk_sparse_adjoint_wide: segment capacity too large");
  if (ws_bytes < pl.ws_bytes || !ws) return fail(SK_EINVAL, "sk_sparse_adjoint_wide: workspace too small");
  sm100::EncodeTiledFnT fn = sm100::encode_tiled_fn();
  if (!fn) return fail(SK_ECUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)m, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)lda * sizeof(T)};
  cuuint32_t box[2] = {(cuuint32_t)COLS, (cuuint32_t)W_R};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapDataType dt = sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  if (fn(&tm, dt, 2, const_cast<T*>(A), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return fail(SK_EINVAL, "sk_sparse_adjoint_wide: cannot describe A for TMA");
  WParams p{};
  p.d = rows;
  p.m = m;
  p.k = k;
  p.nchunks = pl.nchunks;
  p.ngroups = pl.ngroups;
  p.nslices = pl.nslices;
  p.npieces = pl.npieces;
  p.chunks_per_piece = pl.chunks_per_piece;
  p.chunk_base = r0 / W_R;
  p.stage_bytes = pl.stage_bytes;
  p.enc = enc;
  p.seg_off = seg_off;
  p.part = ws;
  cudaStream_t s = as_stream(stream);
  allow_smem(sparse_adjoint_wide<T>, pl.smem);
  sparse_adjoint_wide<T><<<dim3((unsigned)pl.ngroups, (unsigned)pl.nslices, (unsigned)pl.npieces),
                           (W_WARPS + 1) * 32, pl.smem, s>>>(tm, p);
  int st = check_launch("sk_sparse_adjoint_wide");
  if (st != SK_OK) return st;
  if constexpr (sizeof(T) == 4)
    return adjoint_reduce_f32(static_cast<const float*>(ws), pl.npieces, k, m, scale, SA, ldsa, accumulate, s);
  else
    return adjoint_reduce_f64(static_cast<const double*>(ws), pl.npieces, k, m, scale, SA, ldsa, accumulate, s);
}

}  // namespace
}  // namespace skb

extern "C" size_t sk_sparse_adjoint_wide_workspace_bytes(int64_t d, int64_t m, int64_t k) {
  if (d < 1 || m < 1 || k < 1) return 0;
  return wide_plan(d, m, k, 0).ws_bytes;
}

extern "C" size_t sk_sparse_adjoint_wide_workspace_bytes_f64(int64_t d, int64_t m, int64_t k) {
  if (d < 1 || m < 1 || k < 1) return 0;
  return wide_plan(d, m, k, 0, w_cols<double>(), 8).ws_bytes;
}

extern "C" int sk_sparse_adjoint_wide_rows(const float* A, int64_t d, int64_t r0, int64_t r1, int64_t m,
                                           int64_t lda, const uint16_t* enc, const int64_t* seg_off, int32_t seg_cap,
                                           int64_t k, double scale, float* SA, int64_t ldsa, int accumulate, void* ws,
                                           size_t ws_bytes, void* stream) {
  return wide_rows_t<float>(A, d, r0, r1, m, lda, enc, seg_off, seg_cap, k, scale, SA, ldsa, accumulate, ws, ws_bytes,
                            stream);
}

extern "C" int sk_sparse_adjoint_wide_rows_f64(const double* A, int64_t d, int64_t r0, int64_t r1, int64_t m,
                                               int64_t lda, const uint16_t* enc, const int64_t* seg_off,
                                               int32_t seg_cap, int64_t k, double scale, double* SA, int64_t ldsa,
                                               int accumulate, void* ws, size_t ws_bytes, void* stream) {
  return wide_rows_t<double>(A, d, r0, r1, m, lda, enc, seg_off, seg_cap, k, scale, SA, ldsa, accumulate, ws,
                             ws_bytes, stream);
}

extern "C" int sk_sparse_adjoint_wide(const float* A, int64_t d, int64_t m, int64_t lda, const uint16_t* enc,
                                      const int64_t* seg_off, int32_t seg_cap, int64_t k, double scale, float* SA,
                                      int64_t ldsa, int accumulate, void* ws, size_t ws_bytes, void* stream) {
  return sk_sparse_adjoint_wide_rows(A, d, 0, d, m, lda, enc, seg_off, seg_cap, k, scale, SA, ldsa, accumulate, ws,
                                     ws_bytes, stream);
}

extern "C" int sk_sparse_adjoint_wide_f64(const double* A, int64_t d, int64_t m, int64_t lda, const uint16_t* enc,
                                          const int64_t* seg_off, int32_t seg_cap, int64_t k, double scale, double* SA,
                                          int64_t ldsa, int accumulate, void* ws, size_t ws_bytes, void* stream) {
  return sk_sparse_adjoint_wide_rows_f64(A, d, 0, d, m, lda, enc, seg_off, seg_cap, k, scale, SA, ldsa, accumulate,
                                         ws, ws_bytes, stream);
}
