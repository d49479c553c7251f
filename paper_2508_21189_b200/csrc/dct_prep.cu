// DCT-III rows through one real inverse FFT (Makhoul): the half-spectrum preparation
//   V[r, k] = tw_k * (A[r, k] w_k - i A[r, N-k] w_{N-k}),  k = 0..N/2  (A[r, N] := 0)
// with w = D / s (the SRTT diagonal over the ortho weights) and tw_k = exp(i pi k / 2N), in one pass
// (complex64 for float32, complex128 for float64). The caller runs irfft(V, N) (cuFFT) and gathers
// the sampled outputs x_{2n} = v_n, x_{2n+1} = v_{N-1-n}. Serves SparseRttTM with the DCT transform,
// the reference's real-field default (src/sketch/rtt.py:92-93, 129-140).
#include "common.cuh"

namespace skb {
namespace {

template <typename T>
__global__ void dct3_prep_kernel(const T* __restrict__ A, int64_t n, int64_t N, int64_t lda, const T* __restrict__ w,
                                 const T* __restrict__ tw, T* __restrict__ V, int64_t ldv) {
  const int64_t h = N / 2, cols = h + 1, total = n * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / cols, k = idx % cols;
    const T* a = A + r * lda;
    const T re = a[k == N ? 0 : k] * w[k];
    const T im = (k == 0) ? T(0) : -(a[N - k] * w[N - k]);
    const T c = tw[2 * k], s = tw[2 * k + 1];
    T* v = V + r * ldv + 2 * k;
    v[0] = re * c - im * s;
    v[1] = re * s + im * c;
  }
}

template <typename T>
int run(const T* A, int64_t n, int64_t N, int64_t lda, const T* w, const T* tw, T* V, int64_t ldv, cudaStream_t s) {
  const int64_t total = n * (N / 2 + 1);
  int64_t grid = (total + 255) / 256;
  if (grid > 64 * (int64_t)sm_count()) grid = 64 * (int64_t)sm_count();
  dct3_prep_kernel<T><<<(unsigned)grid, 256, 0, s>>>(A, n, N, lda, w, tw, V, ldv);
  return check_launch("sk_dct3_prep");
}

}  // namespace
}  // namespace skb

extern "C" int sk_dct3_prep(int dtype, const void* A, int64_t n, int64_t N, int64_t lda, const void* w,
                            const void* tw, void* V, int64_t ldv, void* stream) {
  using namespace skb;
  if (n < 0 || N < 2 || (N % 2) || lda < N || ldv < N + 2) return fail(SK_EINVAL, "sk_dct3_prep: bad shape (even N)");
  if (n == 0) return SK_OK;
  if (!A || !w || !tw || !V) return fail(SK_EINVAL, "sk_dct3_prep: null pointer");
  cudaStream_t s = as_stream(stream);
  if (dtype == SK_F32)
    return run<float>(static_cast<const float*>(A), n, N, lda, static_cast<const float*>(w),
                      static_cast<const float*>(tw), static_cast<float*>(V), ldv, s);
  if (dtype == SK_F64)
    return run<double>(static_cast<const double*>(A), n, N, lda, static_cast<const double*>(w),
                       static_cast<const double*>(tw), static_cast<double*>(V), ldv, s);
  return fail(SK_EINVAL, "sk_dct3_prep: bad dtype");
}
