// Mixed-precision matrix-vector products for sketch-and-precondition LSQR (config 4 downstream):
// float32 A streamed once from HBM, float64 vectors and float64 accumulation (LSQR's residuals go
// below float32 epsilon). Replaces the widen-then-GEMV form (an f64 copy of every row block:
// 5x the HBM traffic of reading A once).
//   sk_gemv_f32_f64   : y = A v            (warp per row, v in shared memory)
//   sk_gemv_t_f32_f64 : z = A^T u          (thread per column over a row range, ordered float64
//                                           reduction of the per-range partials: deterministic)
#include <cstdlib>

#include "common.cuh"

namespace skb {
namespace {

constexpr int GV_THREADS = 256;

__global__ void __launch_bounds__(GV_THREADS)
    gemv_rows(const float* __restrict__ A, int64_t n, int64_t d, int64_t lda, const double* __restrict__ v,
              double* __restrict__ y, bool vec) {
  extern __shared__ double vs[];
  for (int64_t c = threadIdx.x; c < d; c += GV_THREADS) vs[c] = v[c];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t wstride = (int64_t)gridDim.x * (GV_THREADS / 32);
  for (int64_t r = (int64_t)blockIdx.x * (GV_THREADS / 32) + warp; r < n; r += wstride) {
    const float* a = A + r * lda;
    double acc0 = 0.0, acc1 = 0.0;
    if (vec) {
      int64_t c = 4 * lane;
      for (; c + 128 < d; c += 256) {  // two independent 16-byte loads in flight per lane
        const float4 x = __ldg(reinterpret_cast<const float4*>(a + c));
        const float4 x2 = __ldg(reinterpret_cast<const float4*>(a + c + 128));
        acc0 = fma((double)x.x, vs[c], acc0);
        acc0 = fma((double)x.y, vs[c + 1], acc0);
        acc0 = fma((double)x.z, vs[c + 2], acc0);
        acc0 = fma((double)x.w, vs[c + 3], acc0);
        acc1 = fma((double)x2.x, vs[c + 128], acc1);
        acc1 = fma((double)x2.y, vs[c + 129], acc1);
        acc1 = fma((double)x2.z, vs[c + 130], acc1);
        acc1 = fma((double)x2.w, vs[c + 131], acc1);
      }
      if (c < d) {
        const float4 x = __ldg(reinterpret_cast<const float4*>(a + c));
        acc0 = fma((double)x.x, vs[c], acc0);
        acc0 = fma((double)x.y, vs[c + 1], acc0);
        acc0 = fma((double)x.z, vs[c + 2], acc0);
        acc0 = fma((double)x.w, vs[c + 3], acc0);
      }
    } else {
      for (int64_t c = lane; c < d; c += 32) acc0 = fma((double)__ldg(a + c), vs[c], acc0);
    }
    double acc = acc0 + acc1;
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) y[r] = acc;
  }
}

// d = 128 * NQ (NQ <= 4): each lane keeps its 4 * NQ entries of v in registers (no shared-memory
// traffic per row) and loads its NQ 16-byte pieces of two rows at once (2 * NQ loads in flight)
template <int NQ>
__global__ void __launch_bounds__(GV_THREADS)
    gemv_rows_reg(const float* __restrict__ A, int64_t n, int64_t lda, const double* __restrict__ v,
                  double* __restrict__ y) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double vr[NQ][4];
#pragma unroll
  for (int q = 0; q < NQ; ++q)
#pragma unroll
    for (int c = 0; c < 4; ++c) vr[q][c] = v[128 * q + 4 * lane + c];
  const int64_t wstride = (int64_t)gridDim.x * (GV_THREADS / 32);
  for (int64_t r = (int64_t)blockIdx.x * (GV_THREADS / 32) + warp; r < n; r += 2 * wstride) {
    const int64_t r2 = r + wstride;
    const bool two = r2 < n;
    float4 x[NQ], x2[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      x[q] = __ldg(reinterpret_cast<const float4*>(A + r * lda + 128 * q + 4 * lane));
      x2[q] = two ? __ldg(reinterpret_cast<const float4*>(A + r2 * lda + 128 * q + 4 * lane)) : make_float4(0, 0, 0, 0);
    }
    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      a0 = fma((double)x[q].x, vr[q][0], a0);
      a1 = fma((double)x[q].y, vr[q][1], a1);
      a0 = fma((double)x[q].z, vr[q][2], a0);
      a1 = fma((double)x[q].w, vr[q][3], a1);
      b0 = fma((double)x2[q].x, vr[q][0], b0);
      b1 = fma((double)x2[q].y, vr[q][1], b1);
      b0 = fma((double)x2[q].z, vr[q][2], b0);
      b1 = fma((double)x2[q].w, vr[q][3], b1);
    }
    double sa = a0 + a1, sb = b0 + b1;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      sa += __shfl_xor_sync(0xffffffffu, sa, o);
      sb += __shfl_xor_sync(0xffffffffu, sb, o);
    }
    if (lane == 0) {
      y[r] = sa;
      if (two) y[r2] = sb;
    }
  }
}

// thread = 4 consecutive columns (one 16-byte load per row) over a range of rows, 4 rows in flight
__global__ void __launch_bounds__(GV_THREADS)
    gemv_cols_partial(const float* __restrict__ A, int64_t n, int64_t d, int64_t lda, const double* __restrict__ u,
                      int64_t rows_per_split, double* __restrict__ part, bool vec) {
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_split;
  const int64_t r1 = min(n, r0 + rows_per_split);
  if (c >= d) return;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  if (vec) {
    int64_t r = r0;
    for (; r + 4 <= r1; r += 4) {
      float4 x[4];
      double w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        x[q] = __ldg(reinterpret_cast<const float4*>(A + (r + q) * lda + c));
        w[q] = __ldg(u + r + q);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        acc[0] = fma((double)x[q].x, w[q], acc[0]);
        acc[1] = fma((double)x[q].y, w[q], acc[1]);
        acc[2] = fma((double)x[q].z, w[q], acc[2]);
        acc[3] = fma((double)x[q].w, w[q], acc[3]);
      }
    }
    for (; r < r1; ++r) {
      const float4 x = __ldg(reinterpret_cast<const float4*>(A + r * lda + c));
      const double w = __ldg(u + r);
      acc[0] = fma((double)x.x, w, acc[0]);
      acc[1] = fma((double)x.y, w, acc[1]);
      acc[2] = fma((double)x.z, w, acc[2]);
      acc[3] = fma((double)x.w, w, acc[3]);
    }
  } else {
    for (int64_t r = r0; r < r1; ++r) {
      const double w = __ldg(u + r);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (c + q < d) acc[q] = fma((double)__ldg(A + r * lda + c + q), w, acc[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (c + q < d) part[(int64_t)blockIdx.y * d + c + q] = acc[q];
}

// block = 32 columns x 32 warps: warp w sums splits w, w + 32, ... (4 loads in flight), then the 32
// warp sums are added in a fixed order (deterministic)
constexpr int RS_WARPS = 32;
__global__ void __launch_bounds__(RS_WARPS * 32)
    reduce_splits(const double* __restrict__ part, int nsplit, int64_t d, double* __restrict__ z) {
  __shared__ double sums[RS_WARPS][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t c = (int64_t)blockIdx.x * 32 + lane;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  if (c < d) {
    int i = warp;
    for (; i + 3 * RS_WARPS < nsplit; i += 4 * RS_WARPS) {
      s0 += part[(int64_t)i * d + c];
      s1 += part[(int64_t)(i + RS_WARPS) * d + c];
      s2 += part[(int64_t)(i + 2 * RS_WARPS) * d + c];
      s3 += part[(int64_t)(i + 3 * RS_WARPS) * d + c];
    }
    for (; i < nsplit; i += RS_WARPS) s0 += part[(int64_t)i * d + c];
  }
  sums[warp][lane] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  if (warp == 0 && c < d) {
    double s = 0.0;
#pragma unroll 8
    for (int w = 0; w < RS_WARPS; ++w) s += sums[w][lane];
    z[c] = s;
  }
}

// threads per column block: one per 4 columns, a warp multiple, at most GV_THREADS
int t_threads(int64_t d) {
  const int64_t t = ((d + 3) / 4 + 31) / 32 * 32;
  return (int)(t < GV_THREADS ? t : GV_THREADS);
}
int64_t t_colblocks(int64_t d) { return (d + 4 * t_threads(d) - 1) / (4 * t_threads(d)); }

int t_splits(int64_t n, int64_t d) {
  const int64_t colblocks = t_colblocks(d);
  int64_t s = (16 * (int64_t)sm_count() + colblocks - 1) / colblocks;
  if (s > n) s = n;
  if (s < 1) s = 1;
  return (int)s;
}

// One LSQR bidiagonalisation step in one pass over A (d = 128 * NQ):
//   u[r] <- (A v)[r] - alpha * u[r]   (written back),   part[split] = (A^T u_new, ||u_new||^2)
// Row r's update only needs row r of A, so the row that formed (A v)[r] is still in registers when
// u_new[r] * A[r, :] is added to the lane's column partials: both products of an LSQR iteration
// for one read of A (the two-kernel form reads it twice). Warps walk fixed row sets of the CTA's
// row range, then the CTA sums its 8 warps in a fixed order (deterministic with reduce_splits).
template <int NQ>
__global__ void __launch_bounds__(GV_THREADS)
    lsqr_step_rows(const float* __restrict__ A, int64_t n, int64_t lda, const double* __restrict__ v, double alpha,
                   double* __restrict__ u, int64_t rows_per_split, double* __restrict__ part, int64_t dp) {
  __shared__ double red[GV_THREADS / 32][4 * NQ * 32 + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double vr[NQ][4], zr[NQ][4];
#pragma unroll
  for (int q = 0; q < NQ; ++q)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      vr[q][c] = v[128 * q + 4 * lane + c];
      zr[q][c] = 0.0;
    }
  double b2 = 0.0;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_split;
  const int64_t r1 = min(n, r0 + rows_per_split);
  constexpr int W = GV_THREADS / 32;
  for (int64_t r = r0 + warp; r < r1; r += 2 * W) {
    const int64_t r2 = r + W;
    const bool two = r2 < r1;
    float4 x[NQ], x2[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      x[q] = __ldg(reinterpret_cast<const float4*>(A + r * lda + 128 * q + 4 * lane));
      x2[q] = two ? __ldg(reinterpret_cast<const float4*>(A + r2 * lda + 128 * q + 4 * lane)) : make_float4(0, 0, 0, 0);
    }
    const double ua = u[r], ub = two ? u[r2] : 0.0;
    double xa[NQ][4], xb[NQ][4];
    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      xa[q][0] = x[q].x; xa[q][1] = x[q].y; xa[q][2] = x[q].z; xa[q][3] = x[q].w;
      xb[q][0] = x2[q].x; xb[q][1] = x2[q].y; xb[q][2] = x2[q].z; xb[q][3] = x2[q].w;
      a0 = fma(xa[q][0], vr[q][0], a0);
      a1 = fma(xa[q][1], vr[q][1], a1);
      a0 = fma(xa[q][2], vr[q][2], a0);
      a1 = fma(xa[q][3], vr[q][3], a1);
      b0 = fma(xb[q][0], vr[q][0], b0);
      b1 = fma(xb[q][1], vr[q][1], b1);
      b0 = fma(xb[q][2], vr[q][2], b0);
      b1 = fma(xb[q][3], vr[q][3], b1);
    }
    double sa = a0 + a1, sb = b0 + b1;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      sa += __shfl_xor_sync(0xffffffffu, sa, o);
      sb += __shfl_xor_sync(0xffffffffu, sb, o);
    }
    const double na = sa - alpha * ua, nb = two ? sb - alpha * ub : 0.0;
    if (lane == 0) {
      u[r] = na;
      if (two) u[r2] = nb;
      b2 = fma(na, na, b2);
      b2 = fma(nb, nb, b2);
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
      for (int c = 0; c < 4; ++c) zr[q][c] = fma(nb, xb[q][c], fma(na, xa[q][c], zr[q][c]));
  }
  // CTA partial: warps in a fixed order
#pragma unroll
  for (int q = 0; q < NQ; ++q)
#pragma unroll
    for (int c = 0; c < 4; ++c) red[warp][128 * q + 4 * lane + c] = zr[q][c];
  if (lane == 0) red[warp][4 * NQ * 32] = b2;
  __syncthreads();
  double* out = part + (int64_t)blockIdx.x * dp;
  for (int c = threadIdx.x; c <= 4 * NQ * 32; c += GV_THREADS) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < W; ++w) s += red[w][c];
    out[c] = s;
  }
}

// Same step with the rows fed through a per-warp ring of bulk copies (cp.async.bulk, LS_SLOTS rows
// in flight per warp, no registers held by loads in flight): 2 CTAs per SM at <= 128 registers.
constexpr int LS_SLOTS = 4;
template <int NQ>
__global__ void __launch_bounds__(GV_THREADS, 2)
    lsqr_step_ring(const float* __restrict__ A, int64_t n, int64_t lda, const double* __restrict__ v, double alpha,
                   double* __restrict__ u, int64_t rows_per_split, double* __restrict__ part, int64_t dp) {
  constexpr int W = GV_THREADS / 32;
  constexpr uint32_t ROWB = 512u * NQ;  // bytes of one row (d = 128 NQ floats)
  extern __shared__ __align__(128) unsigned char ls_smem[];
  double* red = reinterpret_cast<double*>(ls_smem);  // reused after the row loop: [W][4 NQ 32 + 1]
  unsigned char* ring = ls_smem;
  __shared__ __align__(8) uint64_t bars[W][LS_SLOTS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_split;
  const int64_t r1 = min(n, r0 + rows_per_split);
  const int64_t nmine = r1 - r0 > warp ? (r1 - r0 - warp + W - 1) / W : 0;  // rows r0 + warp + W i
  unsigned char* wring = ring + (size_t)warp * LS_SLOTS * ROWB;
  const uint32_t wring_s = (uint32_t)__cvta_generic_to_shared(wring);
  if (lane == 0) {
    for (int s = 0; s < LS_SLOTS; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bars[warp][s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  auto issue = [&](int64_t i) {  // row i of this warp into slot i % LS_SLOTS
    const int s = (int)(i % LS_SLOTS);
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&bars[warp][s]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(ROWB) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     wring_s + (uint32_t)s * ROWB),
                 "l"(A + (r0 + warp + (int64_t)W * i) * lda), "r"(ROWB), "r"(bar)
                 : "memory");
  };
  if (lane == 0)
    for (int64_t i = 0; i < nmine && i < LS_SLOTS; ++i) issue(i);
  double vr[NQ][4], zr[NQ][4];
#pragma unroll
  for (int q = 0; q < NQ; ++q)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      vr[q][c] = v[128 * q + 4 * lane + c];
      zr[q][c] = 0.0;
    }
  double b2 = 0.0;
  for (int64_t i = 0; i < nmine; ++i) {
    const int s = (int)(i % LS_SLOTS);
    const uint32_t par = (uint32_t)((i / LS_SLOTS) & 1);
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&bars[warp][s]);
    asm volatile(
        "{\n\t.reg .pred P1;\n\tLSW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra LSW_%=;\n\t}" ::"r"(bar),
        "r"(par)
        : "memory");
    const int64_t r = r0 + warp + (int64_t)W * i;
    const double ur = u[r];
    double x[NQ][4];
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      float4 f;
      asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                   : "=f"(f.x), "=f"(f.y), "=f"(f.z), "=f"(f.w)
                   : "r"(wring_s + (uint32_t)s * ROWB + 512u * q + 16u * lane));
      x[q][0] = f.x; x[q][1] = f.y; x[q][2] = f.z; x[q][3] = f.w;
      a0 = fma(x[q][0], vr[q][0], a0);
      a1 = fma(x[q][1], vr[q][1], a1);
      a0 = fma(x[q][2], vr[q][2], a0);
      a1 = fma(x[q][3], vr[q][3], a1);
    }
    double sa = a0 + a1;
#pragma unroll
    for (int o = 16; o; o >>= 1) sa += __shfl_xor_sync(0xffffffffu, sa, o);
    // every lane's shared reads of slot s are complete (their values fed the reduction): refill it
    if (lane == 0 && i + LS_SLOTS < nmine) issue(i + LS_SLOTS);
    const double na = sa - alpha * ur;
    if (lane == 0) {
      u[r] = na;
      b2 = fma(na, na, b2);
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
      for (int c = 0; c < 4; ++c) zr[q][c] = fma(na, x[q][c], zr[q][c]);
  }
  __syncthreads();  // all rings drained before the buffer is reused for the reduction
  constexpr int RS = 4 * NQ * 32 + 1;
#pragma unroll
  for (int q = 0; q < NQ; ++q)
#pragma unroll
    for (int c = 0; c < 4; ++c) red[warp * RS + 128 * q + 4 * lane + c] = zr[q][c];
  if (lane == 0) red[warp * RS + 4 * NQ * 32] = b2;
  __syncthreads();
  double* out = part + (int64_t)blockIdx.x * dp;
  for (int c = threadIdx.x; c < RS; c += GV_THREADS) {
    double acc = 0.0;
#pragma unroll
    for (int w = 0; w < W; ++w) acc += red[w * RS + c];
    out[c] = acc;
  }
}

int lsqr_splits(int64_t n) {
  int64_t s = 4 * (int64_t)sm_count();  // one resident wave of 256-thread CTAs
  if (s > n) s = n;
  return (int)(s < 1 ? 1 : s);
}

}  // namespace
}  // namespace skb

extern "C" size_t sk_lsqr_step_f32_f64_workspace_bytes(int64_t n, int64_t d) {
  if (n < 1 || d < 1) return 0;
  return (size_t)skb::lsqr_splits(n) * (size_t)(d + 1) * sizeof(double);
}

// u <- A v - alpha u (in place); zb[0:d] = A^T u_new, zb[d] = ||u_new||^2 (float64, deterministic)
extern "C" int sk_lsqr_step_f32_f64(const float* A, int64_t n, int64_t d, int64_t lda, const double* v, double alpha,
                                    double* u, double* zb, double* ws, size_t ws_bytes, void* stream) {
  using namespace skb;
  if (n < 1 || d < 1 || lda < d) return fail(SK_EINVAL, "sk_lsqr_step_f32_f64: bad shape");
  if (!A || !v || !u || !zb) return fail(SK_EINVAL, "sk_lsqr_step_f32_f64: null pointer");
  if ((reinterpret_cast<uintptr_t>(A) & 15) || (lda % 4) || d % 128 || d > 512)
    return fail(SK_EUNSUPPORTED, "sk_lsqr_step_f32_f64: needs 16-byte aligned A, lda % 4 == 0, d = 128 q <= 512");
  const int nsplit = lsqr_splits(n);
  if (!ws || ws_bytes < (size_t)nsplit * (size_t)(d + 1) * sizeof(double))
    return fail(SK_EINVAL, "sk_lsqr_step_f32_f64: workspace too small");
  const int64_t rps = (n + nsplit - 1) / nsplit;
  cudaStream_t s = as_stream(stream);
  const char* ev = getenv("SKETCH_B200_LSQR_RING");
  if (!(ev && ev[0] == '0')) {
    const size_t smem = (size_t)(GV_THREADS / 32) * LS_SLOTS * 512 * (d / 128);
    int st = SK_OK;
    switch (d / 128) {
#define LS_CASE(Q)                                                                                             \
  case Q:                                                                                                      \
    allow_smem(lsqr_step_ring<Q>, smem);          \
    lsqr_step_ring<Q><<<(unsigned)nsplit, GV_THREADS, smem, s>>>(A, n, lda, v, alpha, u, rps, ws, d + 1);     \
    break;
      LS_CASE(1)
      LS_CASE(2)
      LS_CASE(3)
      default:
        LS_CASE(4)
#undef LS_CASE
    }
    st = check_launch("sk_lsqr_step_f32_f64");
    if (st != SK_OK) return st;
    reduce_splits<<<(unsigned)((d + 1 + 31) / 32), RS_WARPS * 32, 0, s>>>(ws, nsplit, d + 1, zb);
    return check_launch("sk_lsqr_step_f32_f64(reduce)");
  }
  switch (d / 128) {
    case 1: lsqr_step_rows<1><<<(unsigned)nsplit, GV_THREADS, 0, s>>>(A, n, lda, v, alpha, u, rps, ws, d + 1); break;
    case 2: lsqr_step_rows<2><<<(unsigned)nsplit, GV_THREADS, 0, s>>>(A, n, lda, v, alpha, u, rps, ws, d + 1); break;
    case 3: lsqr_step_rows<3><<<(unsigned)nsplit, GV_THREADS, 0, s>>>(A, n, lda, v, alpha, u, rps, ws, d + 1); break;
    default: lsqr_step_rows<4><<<(unsigned)nsplit, GV_THREADS, 0, s>>>(A, n, lda, v, alpha, u, rps, ws, d + 1); break;
  }
  int st = check_launch("sk_lsqr_step_f32_f64");
  if (st != SK_OK) return st;
  reduce_splits<<<(unsigned)((d + 1 + 31) / 32), RS_WARPS * 32, 0, s>>>(ws, nsplit, d + 1, zb);
  return check_launch("sk_lsqr_step_f32_f64(reduce)");
}

extern "C" int sk_gemv_f32_f64(const float* A, int64_t n, int64_t d, int64_t lda, const double* v, double* y,
                               void* stream) {
  using namespace skb;
  if (n < 0 || d < 1 || lda < d) return fail(SK_EINVAL, "sk_gemv_f32_f64: bad shape");
  if (n == 0) return SK_OK;
  if (!A || !v || !y) return fail(SK_EINVAL, "sk_gemv_f32_f64: null pointer");
  const size_t smem = (size_t)d * sizeof(double);
  if (smem > 200 * 1024) return fail(SK_EUNSUPPORTED, "sk_gemv_f32_f64: d too large for the shared vector");
  const bool vec = ((reinterpret_cast<uintptr_t>(A) & 15) == 0) && (lda % 4 == 0) && (d % 4 == 0);
  if (vec && d % 128 == 0 && d <= 512) {
    // one resident wave (64-register kernel: 4 CTAs of 256 threads per SM)
    int64_t g = (n + 15) / 16;
    if (g > 4 * (int64_t)sm_count()) g = 4 * (int64_t)sm_count();
    cudaStream_t st = as_stream(stream);
    switch (d / 128) {
      case 1: gemv_rows_reg<1><<<(unsigned)g, GV_THREADS, 0, st>>>(A, n, lda, v, y); break;
      case 2: gemv_rows_reg<2><<<(unsigned)g, GV_THREADS, 0, st>>>(A, n, lda, v, y); break;
      case 3: gemv_rows_reg<3><<<(unsigned)g, GV_THREADS, 0, st>>>(A, n, lda, v, y); break;
      default: gemv_rows_reg<4><<<(unsigned)g, GV_THREADS, 0, st>>>(A, n, lda, v, y); break;
    }
    return check_launch("sk_gemv_f32_f64");
  }
  allow_smem(gemv_rows, smem);
  int64_t grid = (n + 7) / 8;
  if (grid > 16 * (int64_t)sm_count()) grid = 16 * (int64_t)sm_count();
  gemv_rows<<<(unsigned)grid, GV_THREADS, smem, as_stream(stream)>>>(A, n, d, lda, v, y, vec);
  return check_launch("sk_gemv_f32_f64");
}

extern "C" size_t sk_gemv_t_f32_f64_workspace_bytes(int64_t n, int64_t d) {
  if (n < 1 || d < 1) return 0;
  return (size_t)skb::t_splits(n, d) * d * sizeof(double);
}

extern "C" int sk_gemv_t_f32_f64(const float* A, int64_t n, int64_t d, int64_t lda, const double* u, double* z,
                                 double* ws, size_t ws_bytes, void* stream) {
  using namespace skb;
  if (n < 0 || d < 1 || lda < d) return fail(SK_EINVAL, "sk_gemv_t_f32_f64: bad shape");
  if (!A || !u || !z) return fail(SK_EINVAL, "sk_gemv_t_f32_f64: null pointer");
  cudaStream_t s = as_stream(stream);
  if (n == 0) {
    cudaMemsetAsync(z, 0, (size_t)d * sizeof(double), s);
    return check_launch("sk_gemv_t_f32_f64");
  }
  const int nsplit = t_splits(n, d);
  if (!ws || ws_bytes < (size_t)nsplit * d * sizeof(double))
    return fail(SK_EINVAL, "sk_gemv_t_f32_f64: workspace too small");
  const int64_t rows_per_split = (n + nsplit - 1) / nsplit;
  const bool vec = ((reinterpret_cast<uintptr_t>(A) & 15) == 0) && (lda % 4 == 0) && (d % 4 == 0);
  dim3 grid((unsigned)t_colblocks(d), (unsigned)nsplit);
  gemv_cols_partial<<<grid, t_threads(d), 0, s>>>(A, n, d, lda, u, rows_per_split, ws, vec);
  int st = check_launch("sk_gemv_t_f32_f64");
  if (st != SK_OK) return st;
  reduce_splits<<<(unsigned)((d + 31) / 32), RS_WARPS * 32, 0, s>>>(ws, nsplit, d, z);
  return check_launch("sk_gemv_t_f32_f64(reduce)");
}
