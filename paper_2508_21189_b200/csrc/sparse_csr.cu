// K1s — sparse A (CSR) times a sparse-sign Omega: Y = scale * A * Omega, Y dense n x k.
//
// Replaces `_SparseTM.apply_right` for SciPy-sparse A (src/sketch/sparse.py:63-66, `a @ self.matrix`
// followed by `.toarray()`), the path the reference's SuiteSparse experiments take: A is never
// densified. Omega is given by rows (CSR): for row j, int32 entries `c | neg << 31`; the common
// magnitude is folded into `scale`. One warp per row of A: lanes take the row's nonzeros
// A[i, j] in turn and scatter +-A[i, j] into the warp's k-wide accumulator row in shared memory
// for every entry of Omega's row j (shared-memory atomics), then the row is written out
// coalesced. When k is too wide for shared memory the warp scatters straight into Y (global
// atomics after a zero fill). The adjoint of a sparse B runs this on B^T (CSR of B^T).
#include "common.cuh"

namespace skb {
namespace {

constexpr int CSR_WARPS = 8;

template <typename T, bool SMEM>
__global__ void __launch_bounds__(CSR_WARPS * 32)
    sparse_right_csr(int64_t n, const int64_t* __restrict__ aptr, const int32_t* __restrict__ aidx,
                     const T* __restrict__ aval, const int32_t* __restrict__ optr, const int32_t* __restrict__ oent,
                     int64_t k, T scale, T* __restrict__ Y, int64_t ldy) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T* acc = SMEM ? reinterpret_cast<T*>(smem_raw) + (size_t)warp * k : nullptr;
  const int64_t wstride = (int64_t)gridDim.x * CSR_WARPS;
  for (int64_t row = (int64_t)blockIdx.x * CSR_WARPS + warp; row < n; row += wstride) {
    T* dst = SMEM ? acc : Y + row * ldy;
    if constexpr (SMEM) {
      for (int64_t c = lane; c < k; c += 32) acc[c] = T(0);
      __syncwarp();
    }
    const int64_t e0 = aptr[row], e1 = aptr[row + 1];
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const int32_t j = __ldg(aidx + e);
      const T v = __ldg(aval + e) * scale;
      const int32_t t1 = __ldg(optr + j + 1);
      for (int32_t t = __ldg(optr + j); t < t1; ++t) {
        const uint32_t u = (uint32_t)__ldg(oent + t);
        atomicAdd(dst + (u & 0x7fffffffu), (u >> 31) ? -v : v);
      }
    }
    if constexpr (SMEM) {
      __syncwarp();
      T* y = Y + row * ldy;
      for (int64_t c = lane; c < k; c += 32) y[c] = acc[c];
      __syncwarp();
    }
  }
}

template <typename T>
int run(int64_t n, int64_t d, const int64_t* aptr, const int32_t* aidx, const T* aval, const int32_t* optr,
        const int32_t* oent, int64_t k, double scale, T* Y, int64_t ldy, cudaStream_t s) {
  (void)d;
  const size_t smem = (size_t)CSR_WARPS * k * sizeof(T);
  int64_t grid = (n + CSR_WARPS - 1) / CSR_WARPS;
  if (smem <= 200 * 1024) {
    auto kern = sparse_right_csr<T, true>;
    allow_smem(kern, smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, CSR_WARPS * 32, smem);
    if (per_sm < 1) per_sm = 1;
    if (grid > (int64_t)per_sm * sm_count() * 4) grid = (int64_t)per_sm * sm_count() * 4;
    kern<<<(unsigned)grid, CSR_WARPS * 32, smem, s>>>(n, aptr, aidx, aval, optr, oent, k, (T)scale, Y, ldy);
  } else {
    // zero the n x k output (row by row when ldy > k), then scatter with global atomics
    if (ldy == k) {
      cudaMemsetAsync(Y, 0, (size_t)n * k * sizeof(T), s);
    } else {
      cudaMemset2DAsync(Y, (size_t)ldy * sizeof(T), 0, (size_t)k * sizeof(T), (size_t)n, s);
    }
    if (grid > 16 * (int64_t)sm_count()) grid = 16 * (int64_t)sm_count();
    sparse_right_csr<T, false><<<(unsigned)grid, CSR_WARPS * 32, 0, s>>>(n, aptr, aidx, aval, optr, oent, k,
                                                                          (T)scale, Y, ldy);
  }
  return check_launch("sk_sparse_right_csr");
}

}  // namespace
}  // namespace skb

extern "C" int sk_sparse_right_csr(int dtype, int64_t n, int64_t d, const int64_t* a_indptr, const int32_t* a_indices,
                                   const void* a_values, const int32_t* omega_indptr, const int32_t* omega_entries,
                                   int64_t k, double scale, void* Y, int64_t ldy, void* stream) {
  using namespace skb;
  if (n < 0 || d < 1 || k < 1 || ldy < k) return fail(SK_EINVAL, "sk_sparse_right_csr: bad shape/leading dimension");
  if (n == 0) return SK_OK;
  if (!a_indptr || !Y || !omega_indptr) return fail(SK_EINVAL, "sk_sparse_right_csr: null pointer");
  cudaStream_t s = as_stream(stream);
  if (dtype == SK_F32)
    return run<float>(n, d, a_indptr, a_indices, static_cast<const float*>(a_values), omega_indptr, omega_entries, k,
                      scale, static_cast<float*>(Y), ldy, s);
  if (dtype == SK_F64)
    return run<double>(n, d, a_indptr, a_indices, static_cast<const double*>(a_values), omega_indptr, omega_entries,
                       k, scale, static_cast<double*>(Y), ldy, s);
  return fail(SK_EINVAL, "sk_sparse_right_csr: bad dtype");
}
