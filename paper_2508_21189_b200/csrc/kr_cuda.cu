// K4c — Khatri-Rao apply on the CUDA cores, Omega never formed (float64, and float32 shapes the
// tcgen05 form cannot take: dl % 4 != 0 or a resident factor too large for shared memory).
//
//   right:   Y[r, j] = scale * sum_P W[P, j] * sum_q A[r, P*dl + q] * F[q, j]
//   adjoint: X[j, c] = scale * sum_P W[P, j] * sum_q F[q, j] * B[P*dl + q, c]   (B read in place)
//
// F (dl x k) is the Khatri-Rao product of the trailing factors and W (P x k) that of the leading
// ones (reference khatri_rao.py:62-74 contracts factor by factor; grouping them this way keeps the
// contraction a sequence of small GEMMs with a per-P column scaling).  float64 accumulates in
// float64 with FMA (the reference's dtype, parity 1e-12); float32 accumulates in float32 per P and
// in float64 across P.
//
// CTA = 256 threads, a 64 (rows r) x 64 (columns j) tile of the result, 4 x 4 per thread; A/B and F
// tiles of 16 q staged in shared memory.  The adjoint is the right apply of B^T: its tile loads are
// contiguous along c instead of q, and its result is written transposed.
#include "common.cuh"

namespace skb {

int gemm64_try(bool ta, const double* A, int64_t rows, int64_t P, int64_t dl, int64_t lda, const double* F,
               int64_t ldf, const double* W, int64_t ldw, int64_t k, double scale, double* Y, int64_t ldy,
               cudaStream_t s, const double* Fi = nullptr, const double* Wi = nullptr, int part = 0,
               int accumulate = 0, bool force = false);  // dense64.cu

namespace {

constexpr int TR = 64, TJ = 64, TQ = 16;

template <typename T, bool TA>
__global__ void __launch_bounds__(256) kr_cc_kernel(const T* __restrict__ A, int64_t rows, int64_t P, int64_t dl,
                                                    int64_t lda, const T* __restrict__ F, int64_t ldf,
                                                    const T* __restrict__ W, int64_t ldw, int64_t k, double scale,
                                                    T* __restrict__ Y, int64_t ldy) {
  using Acc = double;
  __shared__ T as[TQ][TR + 1];
  __shared__ T fs[TQ][TJ + 1];
  const int tid = threadIdx.x;
  const int tr = tid & 15, tj = tid >> 4;  // thread owns rows tr + 16 i, columns tj + 16 u
  const int64_t r0 = (int64_t)blockIdx.x * TR, j0 = (int64_t)blockIdx.y * TJ;
  Acc acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[i][u] = 0.0;
  for (int64_t pp = 0; pp < P; ++pp) {
    T part[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int u = 0; u < 4; ++u) part[i][u] = T(0);
    for (int64_t q0 = 0; q0 < dl; q0 += TQ) {
      // A tile: 16 q x 64 r (1024 values, 4 per thread)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int idx = tid + 256 * e;
        int qq, rr;
        if (TA) {  // B[P*dl + q][c]: contiguous along c
          qq = idx >> 6;
          rr = idx & 63;
        } else {   // A[r][P*dl + q]: contiguous along q
          rr = idx >> 4;
          qq = idx & 15;
        }
        const int64_t r = r0 + rr, q = q0 + qq;
        T v = T(0);
        if (r < rows && q < dl) v = TA ? A[(pp * dl + q) * lda + r] : A[r * lda + pp * dl + q];
        as[qq][rr] = v;
      }
      // F tile: 16 q x 64 j
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int idx = tid + 256 * e;
        const int qq = idx >> 6, jj = idx & 63;
        const int64_t q = q0 + qq, j = j0 + jj;
        fs[qq][jj] = (q < dl && j < k) ? F[q * ldf + j] : T(0);
      }
      __syncthreads();
#pragma unroll
      for (int qq = 0; qq < TQ; ++qq) {
        T a[4], f[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = as[qq][tr + 16 * i];
#pragma unroll
        for (int u = 0; u < 4; ++u) f[u] = fs[qq][tj + 16 * u];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int u = 0; u < 4; ++u) part[i][u] = fma(a[i], f[u], part[i][u]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t j = j0 + tj + 16 * u;
      const Acc w = j < k ? (W ? (Acc)W[pp * ldw + j] : 1.0) : 0.0;
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i][u] = fma(w, (Acc)part[i][u], acc[i][u]);
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = r0 + tr + 16 * i;
    if (r >= rows) continue;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t j = j0 + tj + 16 * u;
      if (j >= k) continue;
      const T v = (T)(acc[i][u] * scale);
      if (TA) Y[j * ldy + r] = v;
      else Y[r * ldy + j] = v;
    }
  }
}

template <typename T>
int kr_cc_launch(bool ta, const void* A, int64_t rows, int64_t P, int64_t dl, int64_t lda, const void* F, int64_t ldf,
                 const void* W, int64_t ldw, int64_t k, double scale, void* Y, int64_t ldy, cudaStream_t s) {
  const int64_t gx = (rows + TR - 1) / TR, gy = (k + TJ - 1) / TJ;
  if (gy > 65535) return fail(SK_EUNSUPPORTED, "sk_kr_cc: k too large");
  const dim3 grid((unsigned)gx, (unsigned)gy);
  if (ta)
    kr_cc_kernel<T, true><<<grid, 256, 0, s>>>(static_cast<const T*>(A), rows, P, dl, lda, static_cast<const T*>(F),
                                               ldf, static_cast<const T*>(W), ldw, k, scale, static_cast<T*>(Y), ldy);
  else
    kr_cc_kernel<T, false><<<grid, 256, 0, s>>>(static_cast<const T*>(A), rows, P, dl, lda, static_cast<const T*>(F),
                                                ldf, static_cast<const T*>(W), ldw, k, scale, static_cast<T*>(Y), ldy);
  return check_launch("sk_kr_cc");
}

int kr_cc(bool ta, int dtype, const void* A, int64_t rows, int64_t P, int64_t dl, int64_t lda, const void* F,
          int64_t ldf, const void* W, int64_t ldw, int64_t k, double scale, void* Y, int64_t ldy, void* stream) {
  if (rows < 0 || P < 1 || dl < 1 || k < 1 || ldf < k || (W && ldw < k)) return fail(SK_EINVAL, "sk_kr_cc: bad shape");
  if (!W && P != 1) return fail(SK_EINVAL, "sk_kr_cc: W may be NULL only for one block (P = 1)");
  if (ta ? (lda < rows || ldy < rows) : (lda < P * dl || ldy < k)) return fail(SK_EINVAL, "sk_kr_cc: bad leading dimension");
  if (rows == 0) return SK_OK;
  if (!A || !F || !Y) return fail(SK_EINVAL, "sk_kr_cc: null pointer");
  cudaStream_t s = as_stream(stream);
  if (dtype == SK_F64) {
    const int st = gemm64_try(ta, static_cast<const double*>(A), rows, P, dl, lda, static_cast<const double*>(F), ldf,
                              static_cast<const double*>(W), ldw, k, scale, static_cast<double*>(Y), ldy, s);
    if (st != 1) return st;
  }
  if (dtype == SK_F64) return kr_cc_launch<double>(ta, A, rows, P, dl, lda, F, ldf, W, ldw, k, scale, Y, ldy, s);
  if (dtype == SK_F32) return kr_cc_launch<float>(ta, A, rows, P, dl, lda, F, ldf, W, ldw, k, scale, Y, ldy, s);
  return fail(SK_EINVAL, "sk_kr_cc: dtype");
}

}  // namespace
}  // namespace skb

extern "C" int sk_kr_right_cc(int dtype, const void* A, int64_t n, int64_t P, int64_t dl, int64_t lda, const void* F,
                              int64_t ldf, const void* W, int64_t ldw, int64_t k, double scale, void* Y, int64_t ldy,
                              void* stream) {
  return skb::kr_cc(false, dtype, A, n, P, dl, lda, F, ldf, W, ldw, k, scale, Y, ldy, stream);
}

extern "C" int sk_kr_adjoint_cc(int dtype, const void* B, int64_t m, int64_t P, int64_t dl, int64_t ldb, const void* F,
                                int64_t ldf, const void* W, int64_t ldw, int64_t k, double scale, void* X, int64_t ldx,
                                void* stream) {
  return skb::kr_cc(true, dtype, B, m, P, dl, ldb, F, ldf, W, ldw, k, scale, X, ldx, stream);
}
