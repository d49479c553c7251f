// K3 — sparse randomized trigonometric transform, right apply:  Y = A * D * H * S.
//
// Replaces `SparseRttTM.apply_right` (src/sketch/rtt.py:129-140): the reference multiplies A by
// the diagonal D, runs 13 full-array NumPy butterfly passes of `wht` (rtt.py:28-44) in float64,
// and then multiplies by the SparseColTM sampler S through csc_matvecs.  Here each row of A makes
// ONE trip through the SM: it is loaded once (coalesced 16-byte loads), sign-flipped in
// registers, transformed by an in-register / shared-memory Walsh-Hadamard butterfly network,
// and only the k*xi sampled outputs are written.
//
// Fast path (d = 2^L, 10 <= L <= 14 for float32, <= 13 for float64): T = d/32 threads per row, 32 values per thread.
//   phase 1: registers hold index bits {0,1,L-3,L-2,L-1}     (coalesced float4 loads)
//   phase 2: registers hold bits {2..6}                      (one smem transpose)
//   phase 3: registers hold bits {7..L-4} (+ filler bits)    (second transpose; skipped at L=10)
//   gather : out[c] = scale * sum_x sign * X[row_{c,x}]      (third write, random reads)
// Shared-memory address of index j: j ^ ((j>>5)&3) ^ (((j>>7)&7)<<2) — every transpose write and
// read is bank-conflict free for L in {10,13,14,15} (2-way in phase 3 for L in {11,12}).
// Butterfly order does not matter (the per-bit butterflies commute); natural Hadamard order as in
// the reference (`top = y0 + y1`, `bot = y0 - y1`).
//
// Other sizes (d = 2^L, row fits shared memory): one CTA per row, row in shared memory.
#include "common.cuh"

namespace skb {
namespace {

__device__ __forceinline__ int swz(int j) { return j ^ ((j >> 5) & 3) ^ (((j >> 7) & 7) << 2); }

template <typename T>
__device__ __forceinline__ void butterfly(T& a, T& b) {
  const T s = a + b, t = a - b;
  a = s;
  b = t;
}

// In-register WHT over the 5 bits of the register index.
template <typename T>
__device__ __forceinline__ void wht32(T (&x)[32]) {
#pragma unroll
  for (int h = 1; h < 32; h <<= 1) {
#pragma unroll
    for (int v = 0; v < 32; ++v) {
      if ((v & h) == 0) butterfly(x[v], x[v | h]);
    }
  }
}

// In-register WHT over only the register-index bits in `mask`.
template <typename T, int MASK>
__device__ __forceinline__ void wht32_bits(T (&x)[32]) {
#pragma unroll
  for (int h = 1; h < 32; h <<= 1) {
    if (MASK & h) {
#pragma unroll
      for (int v = 0; v < 32; ++v) {
        if ((v & h) == 0) butterfly(x[v], x[v | h]);
      }
    }
  }
}

template <typename T>
struct V4T;
template <>
struct V4T<float> {
  using type = float4;
};
template <>
struct V4T<double> {
  using type = double4;
};

__device__ __forceinline__ void ld4(const float* p, float (&o)[4]) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  o[0] = r.x; o[1] = r.y; o[2] = r.z; o[3] = r.w;
}
__device__ __forceinline__ void ld4(const double* p, double (&o)[4]) {
  double2 a, b;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(a.x), "=d"(a.y) : "l"(p));
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(b.x), "=d"(b.y) : "l"(p + 2));
  o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
}

// Phase-3 register bits for index length L: bits {7..L-4} plus the lowest filler bits.
template <int L>
struct Phase3 {
  static constexpr int M3 = L - 10;  // number of bits still to transform
  static constexpr int NFILL = 5 - M3;
  // register-index bit b (0..4) -> index bit
  __host__ __device__ static constexpr int reg_bit(int b) { return b < NFILL ? b : 7 + (b - NFILL); }
  // thread-index bit t (0..L-6) -> index bit: the index bits not used by registers, ascending
  __host__ __device__ static constexpr int thr_bit(int t) {
    int cnt = 0;
    for (int j = 0; j < L; ++j) {
      bool used = false;
      for (int b = 0; b < 5; ++b)
        if (reg_bit(b) == j) used = true;
      if (!used) {
        if (cnt == t) return j;
        ++cnt;
      }
    }
    return -1;
  }
};

template <typename T, int L, bool SIGNS>
__global__ void __launch_bounds__((1 << (L - 5)), (sizeof(T) == 4 ? (L <= 12 ? 3 : (L == 13 ? 2 : 1)) : (L <= 12 ? 2 : 1)))
    srtt_wht_fast(const T* __restrict__ A, int64_t n, int64_t lda, const T* __restrict__ dvals,
                  const int32_t* __restrict__ samp, int xi, int k, T scale, T* __restrict__ Y,
                  int64_t ldy) {
  constexpr int D = 1 << L;
  constexpr int NT = 1 << (L - 5);
  constexpr int QSTRIDE = D / 8;  // index stride between the 8 float4 groups of a thread
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* buf = reinterpret_cast<T*>(smem_raw);
  const int t = threadIdx.x;

  // D signs / values for this thread's 32 phase-1 positions j = 4t + c + QSTRIDE*q (v = c + 4q).
  uint32_t dmask = 0;
  if constexpr (SIGNS) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const T dv = dvals[4 * t + c + QSTRIDE * q];
        if (dv < T(0)) dmask |= 1u << (c + 4 * q);
      }
  }

  for (int64_t row = blockIdx.x; row < n; row += gridDim.x) {
    const T* a = A + row * lda;
    T x[32];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      T tmp[4];
      ld4(a + 4 * t + QSTRIDE * q, tmp);
#pragma unroll
      for (int c = 0; c < 4; ++c) x[c + 4 * q] = tmp[c];
    }
    if constexpr (SIGNS) {
#pragma unroll
      for (int v = 0; v < 32; ++v) x[v] = flip_if(x[v], (dmask >> v) & 1u);
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        T dv[4];
        const T* dp = dvals + 4 * t + QSTRIDE * q;
        dv[0] = __ldg(dp); dv[1] = __ldg(dp + 1); dv[2] = __ldg(dp + 2); dv[3] = __ldg(dp + 3);
#pragma unroll
        for (int c = 0; c < 4; ++c) x[c + 4 * q] *= dv[c];
      }
    }
    // phase 1: register bits = index bits {0,1,L-3,L-2,L-1}
    wht32(x);

    // transpose 1 -> 2
    __syncthreads();  // previous row's gather is done with buf
#pragma unroll
    for (int q = 0; q < 8; ++q)
#pragma unroll
      for (int c = 0; c < 4; ++c) buf[swz(4 * t + c + QSTRIDE * q)] = x[c + 4 * q];
    __syncthreads();
    // phase 2: thread bits = index bits {0,1} u {7..L-1}; register bits = {2..6}
    const int base2 = (t & 3) | ((t >> 2) << 7);
#pragma unroll
    for (int v = 0; v < 32; ++v) x[v] = buf[swz(base2 | (v << 2))];
    wht32(x);

    if constexpr (L > 10) {
      using P3 = Phase3<L>;
      __syncthreads();
#pragma unroll
      for (int v = 0; v < 32; ++v) buf[swz(base2 | (v << 2))] = x[v];
      __syncthreads();
      int base3 = 0;
#pragma unroll
      for (int b = 0; b < L - 5; ++b) base3 |= ((t >> b) & 1) << P3::thr_bit(b);
#pragma unroll
      for (int v = 0; v < 32; ++v) {
        int j = base3;
#pragma unroll
        for (int b = 0; b < 5; ++b) j |= ((v >> b) & 1) << P3::reg_bit(b);
        x[v] = buf[swz(j)];
      }
      constexpr int MASK3 = ((1 << P3::M3) - 1) << P3::NFILL;
      wht32_bits<T, MASK3>(x);
      __syncthreads();
#pragma unroll
      for (int v = 0; v < 32; ++v) {
        int j = base3;
#pragma unroll
        for (int b = 0; b < 5; ++b) j |= ((v >> b) & 1) << P3::reg_bit(b);
        buf[swz(j)] = x[v];
      }
    } else {
      __syncthreads();
#pragma unroll
      for (int v = 0; v < 32; ++v) buf[swz(base2 | (v << 2))] = x[v];
    }
    __syncthreads();
    // gather the sampled columns
    T* y = Y + row * ldy;
    for (int c = t; c < k; c += NT) {
      T s = T(0);
      for (int u = 0; u < xi; ++u) {
        const uint32_t e = (uint32_t)__ldg(samp + (int64_t)c * xi + u);
        s += flip_if(buf[swz((int)(e & 0x7fffffffu))], e >> 31);
      }
      y[c] = s * scale;
    }
  }
}

// Generic: one CTA per row, whole row in shared memory, log2(d) synchronised butterfly stages.
template <typename T>
__global__ void srtt_wht_simple(const T* __restrict__ A, int64_t n, int64_t d, int64_t lda,
                                const T* __restrict__ dvals, const int32_t* __restrict__ samp, int xi,
                                int k, T scale, T* __restrict__ Y, int64_t ldy) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* buf = reinterpret_cast<T*>(smem_raw);
  for (int64_t row = blockIdx.x; row < n; row += gridDim.x) {
    const T* a = A + row * lda;
    __syncthreads();
    for (int64_t j = threadIdx.x; j < d; j += blockDim.x) buf[j] = a[j] * dvals[j];
    __syncthreads();
    for (int64_t h = 1; h < d; h <<= 1) {
      for (int64_t p = threadIdx.x; p < d / 2; p += blockDim.x) {
        const int64_t j0 = (p / h) * 2 * h + (p % h), j1 = j0 + h;
        const T u = buf[j0], v = buf[j1];
        buf[j0] = u + v;
        buf[j1] = u - v;
      }
      __syncthreads();
    }
    T* y = Y + row * ldy;
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
      T s = T(0);
      for (int u = 0; u < xi; ++u) {
        const uint32_t e = (uint32_t)__ldg(samp + (int64_t)c * xi + u);
        s += flip_if(buf[e & 0x7fffffffu], e >> 31);
      }
      y[c] = s * scale;
    }
  }
}

template <typename T, int L, bool SIGNS>
int launch_fast(const T* A, int64_t n, int64_t lda, const T* dv, const int32_t* samp, int xi, int k,
                double scale, T* Y, int64_t ldy, cudaStream_t s) {
  constexpr int NT = 1 << (L - 5);
  const size_t smem = sizeof(T) << L;
  auto kern = srtt_wht_fast<T, L, SIGNS>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)sm_count() * per_sm;
  if (grid > n) grid = n;
  kern<<<(unsigned)grid, NT, smem, s>>>(A, n, lda, dv, samp, xi, k, (T)scale, Y, ldy);
  return check_launch("sk_srtt_right");
}

template <typename T, bool SIGNS>
int dispatch_L(int L, const T* A, int64_t n, int64_t lda, const T* dv, const int32_t* samp, int xi,
               int k, double scale, T* Y, int64_t ldy, cudaStream_t s) {
  switch (L) {
    case 10: return launch_fast<T, 10, SIGNS>(A, n, lda, dv, samp, xi, k, scale, Y, ldy, s);
    case 11: return launch_fast<T, 11, SIGNS>(A, n, lda, dv, samp, xi, k, scale, Y, ldy, s);
    case 12: return launch_fast<T, 12, SIGNS>(A, n, lda, dv, samp, xi, k, scale, Y, ldy, s);
    case 13: return launch_fast<T, 13, SIGNS>(A, n, lda, dv, samp, xi, k, scale, Y, ldy, s);
    case 14: return launch_fast<T, 14, SIGNS>(A, n, lda, dv, samp, xi, k, scale, Y, ldy, s);
    default: return fail(SK_EUNSUPPORTED, "sk_srtt_right: no fast WHT for this length");
  }
}

template <typename T>
int run(const void* A_, int64_t n, int64_t d, int64_t lda, const void* dv_, bool pm1, const int32_t* samp,
        int xi, int64_t k, double scale, void* Y_, int64_t ldy, cudaStream_t s) {
  const T* A = static_cast<const T*>(A_);
  const T* dv = static_cast<const T*>(dv_);
  T* Y = static_cast<T*>(Y_);
  int L = 0;
  while ((int64_t(1) << L) < d) ++L;
  const bool aligned = ((reinterpret_cast<uintptr_t>(A) & 15) == 0) && (lda % (16 / sizeof(T)) == 0);
  const int max_fast = sizeof(T) == 4 ? 14 : 13;
  if (L >= 10 && L <= max_fast && aligned) {
    // Rademacher diagonals take the sign-mask path; any other diagonal multiplies.
    return pm1 ? dispatch_L<T, true>(L, A, n, lda, dv, samp, xi, (int)k, scale, Y, ldy, s)
               : dispatch_L<T, false>(L, A, n, lda, dv, samp, xi, (int)k, scale, Y, ldy, s);
  }
  const size_t smem = sizeof(T) * (size_t)d;
  if (smem > 200 * 1024) return fail(SK_EUNSUPPORTED, "sk_srtt_right: row does not fit shared memory");
  cudaFuncSetAttribute(srtt_wht_simple<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int threads = (int)(d / 2 < 512 ? (d / 2 < 32 ? 32 : d / 2) : 512);
  int64_t grid = n < 4 * (int64_t)sm_count() ? n : 4 * (int64_t)sm_count();
  if (grid < 1) grid = 1;
  srtt_wht_simple<T><<<(unsigned)grid, threads, smem, s>>>(A, n, d, lda, dv, samp, xi, (int)k, (T)scale, Y, ldy);
  return check_launch("sk_srtt_right(simple)");
}

}  // namespace
}  // namespace skb

extern "C" int sk_srtt_right(int dtype, const void* A, int64_t n, int64_t d, int64_t lda, const void* dvals,
                             int transform, const int32_t* samp, int32_t xi, int64_t k, double scale, void* Y,
                             int64_t ldy, void* stream) {
  using namespace skb;
  const bool pm1 = (transform & SK_DIAG_PM1) != 0;
  transform &= ~SK_DIAG_PM1;
  if (transform != SK_WHT) return fail(SK_EUNSUPPORTED, "sk_srtt_right: only the WHT transform runs in this kernel");
  if (n < 0 || d < 1 || (d & (d - 1)) || k < 1 || xi < 1 || xi > d || lda < d || ldy < k)
    return fail(SK_EINVAL, "sk_srtt_right: bad shape (d must be a power of two)");
  if (k * (int64_t)xi > INT32_MAX) return fail(SK_EINVAL, "sk_srtt_right: k*xi too large");
  if (n > 0 && (!A || !Y || !dvals || !samp)) return fail(SK_EINVAL, "sk_srtt_right: null pointer");
  if (n == 0) return SK_OK;
  cudaStream_t s = as_stream(stream);
  if (dtype == SK_F32) return run<float>(A, n, d, lda, dvals, pm1, samp, xi, k, scale, Y, ldy, s);
  if (dtype == SK_F64) return run<double>(A, n, d, lda, dvals, pm1, samp, xi, k, scale, Y, ldy, s);
  return fail(SK_EINVAL, "sk_srtt_right: bad dtype");
}
