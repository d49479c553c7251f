// K3b — SRTT with the DCT transform (the reference's real-field default, src/sketch/rtt.py:92-93,
// 129-140):  Y[r, c] = scale * sum_x sign_{c,x} * DCT-III(A[r, :] D)[j_{c,x}]   for power-of-two d.
//
// One CTA per row (persistent over rows), everything in shared memory, no intermediate in HBM:
//   1. the raw row lands by one cp.async.bulk (prefetched while the previous row is transformed);
//   2. Makhoul's real-IFFT form of the DCT-III, folded with the split of a length-N real inverse FFT
//      into a length-M = N/2 complex one:  with Z = A D / s (s the ortho weights),
//         U_k = alpha_k (Z_k - i Z_{N-k}) + beta_k (Z_{M-k} + i Z_{M+k}),   k = 0..M-1  (Z_N := 0),
//      alpha_k = c_k (1 + i w^k), beta_k = conj(c_{M-k}) (1 - i w^k), c_k = e^{i pi k / 2N},
//      w = e^{2 pi i / N} (host tables, weights w = D / s folded into the load);
//   3. u = IDFT_M(U) by Stockham passes in shared memory (radix 16, plus one radix-4/8/32 pass when M is
//      not a power of 16), one butterfly group per thread, in place (loads, barrier, stores); each group
//      is an in-register DIF DFT; twiddles e^{2 pi i t / M} from a shared table;
//   4. the transformed row is v = (re u_0, im u_0, re u_1, ...) / N (u XOR-swizzled in shared memory)
//      and the DCT-III output is
//      x_{2n} = v_n, x_{2n+1} = v_{N-1-n}: the host maps every sampled output j to its index t in v,
//      so each of the k outputs gathers xi shared-memory values, signed, scaled, coalesced store.
// Replaces the cuFFT irfft + torch gather of round 1.  float32 d <= 16384, float64 d <= 8192.
#include "common.cuh"
#include "sm100.cuh"

namespace skb {
namespace {

// blockDim: 256 threads, 512 when d/2 = 8192 (one Stockham butterfly group per thread in every pass)

template <typename T>
struct C2 {
  T x, y;
};
template <typename T>
__device__ __forceinline__ C2<T> cmul(C2<T> a, C2<T> b) {
  return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
template <typename T>
__device__ __forceinline__ C2<T> cadd(C2<T> a, C2<T> b) {
  return {a.x + b.x, a.y + b.y};
}
template <typename T>
__device__ __forceinline__ C2<T> csub(C2<T> a, C2<T> b) {
  return {a.x - b.x, a.y - b.y};
}

// e^{2 pi i j / 32}, j < 32 (twiddles of the in-register DFTs, R | 32)
__constant__ double kW32c[32] = {
    1.0, 0.9807852804032304, 0.9238795325112867, 0.8314696123025452, 0.7071067811865476, 0.5555702330196023,
    0.38268343236508984, 0.19509032201612833, 0.0, -0.1950903220161282, -0.3826834323650897, -0.555570233019602,
    -0.7071067811865475, -0.8314696123025453, -0.9238795325112867, -0.9807852804032304, -1.0, -0.9807852804032304,
    -0.9238795325112868, -0.8314696123025455, -0.7071067811865477, -0.5555702330196022, -0.38268343236509034,
    -0.19509032201612866, 0.0, 0.1950903220161283, 0.38268343236509, 0.5555702330196018, 0.7071067811865474,
    0.8314696123025452, 0.9238795325112865, 0.9807852804032303};
__constant__ double kW32s[32] = {
    0.0, 0.19509032201612825, 0.3826834323650898, 0.5555702330196022, 0.7071067811865475, 0.8314696123025452,
    0.9238795325112867, 0.9807852804032304, 1.0, 0.9807852804032304, 0.9238795325112867, 0.8314696123025455,
    0.7071067811865476, 0.5555702330196022, 0.3826834323650899, 0.1950903220161286, 0.0, -0.19509032201612836,
    -0.38268343236508967, -0.555570233019602, -0.7071067811865475, -0.8314696123025452, -0.9238795325112865,
    -0.9807852804032303, -1.0, -0.9807852804032304, -0.9238795325112866, -0.8314696123025455, -0.7071067811865477,
    -0.5555702330196022, -0.3826834323650904, -0.19509032201612872};

__host__ __device__ constexpr int bitrev(int v, int bits) {
  int r = 0;
  for (int b = 0; b < bits; ++b) r |= ((v >> b) & 1) << (bits - 1 - b);
  return r;
}
__host__ __device__ constexpr int log2c(int v) { return v <= 1 ? 0 : 1 + log2c(v / 2); }

// in-register inverse DFT of length R (R | 32), decimation in frequency, in place: afterwards
// X_r sits in x[bitrev(r)]
template <typename T, int R>
__device__ __forceinline__ void dft_inv_dif(C2<T> (&x)[R]) {
#pragma unroll
  for (int span = R / 2; span >= 1; span /= 2) {
#pragma unroll
    for (int b = 0; b < R; b += 2 * span) {
#pragma unroll
      for (int j = 0; j < span; ++j) {
        const C2<T> a = x[b + j], c = x[b + j + span];
        x[b + j] = cadd(a, c);
        const C2<T> dlt = csub(a, c);
        const int e = j * (32 / (2 * span));  // W_{2 span}^j = W_32^(j * 32 / (2 span))
        x[b + j + span] = e ? cmul(dlt, C2<T>{(T)kW32c[e], (T)kW32s[e]}) : dlt;
      }
    }
  }
}

// u is stored XOR-swizzled at complex granularity: logical index i lives at sw(i) = i ^ ((i >> 4) & 15),
// so both the Stockham loads (consecutive i per lane) and the first pass's stores (i = 16 g + r) are
// bank-conflict free
__device__ __forceinline__ int sw(int i) { return i ^ ((i >> 4) & 15); }

// one Stockham pass of radix R on u (M complex, in shared memory), twiddles tw[t] = e^{2 pi i t / M}:
// element q of group g is multiplied by W^q with W = tw[k * M / (L R)] (k = g mod L; powers by a
// complex-multiply chain, one table read per group); one butterfly group per thread (blockDim >= M / R),
// in place (loads, barrier, stores, barrier)
template <typename T, int R>
__device__ __forceinline__ void stockham_pass(C2<T>* u, const C2<T>* tw, int M, int L) {
  const int G = M / R;
  const int g = threadIdx.x;
  const int stride_tw = M / (L * R);
  C2<T> v[R];
  const int k = g % L;
  if (g < G) {
    const C2<T> w1 = tw[k * stride_tw];
    C2<T> wq = w1;
    v[0] = u[sw(g)];
#pragma unroll
    for (int q = 1; q < R; ++q) {
      const C2<T> a = u[sw(g + q * G)];
      v[q] = k ? cmul(a, wq) : a;
      if (q + 1 < R) wq = cmul(wq, w1);
    }
    dft_inv_dif<T, R>(v);
  }
  __syncthreads();
  if (g < G) {
    constexpr int bits = log2c(R);
#pragma unroll
    for (int r = 0; r < R; ++r) u[sw((g - k) * R + k + r * L)] = v[bitrev(r, bits)];
  }
  __syncthreads();
}

template <typename T, int THREADS, int B>  // B = log2(M) % 4: the extra pass (0 none, 1 radix 32, 2 radix 4, 3 radix 8)
__global__ void __launch_bounds__(THREADS) srtt_dct_kernel(const T* __restrict__ A, int64_t n, int N, int64_t lda,
                                                               const T* __restrict__ w, const C2<T>* __restrict__ ab,
                                                               const C2<T>* __restrict__ twg,
                                                               const int32_t* __restrict__ samp, int xi, int k,
                                                               T scale, T* __restrict__ Y, int64_t ldy) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int M = N / 2;
  T* raw = reinterpret_cast<T*>(smem);                         // N reals (the bulk-copied row)
  C2<T>* u = reinterpret_cast<C2<T>*>(raw + N);                 // M complex
  C2<T>* tw = u + M;                                            // M twiddles
  uint64_t* bar = reinterpret_cast<uint64_t*>(tw + M);
  const int tid = threadIdx.x;
  for (int i = tid; i < M; i += blockDim.x) tw[i] = twg[i];
  if (tid == 0) {
    sm100::mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t row_bytes = (uint32_t)N * sizeof(T);
  int64_t r = blockIdx.x;
  uint32_t ph = 0;
  if (tid == 0 && r < n) {
    sm100::mbar_arrive_expect_tx(bar, row_bytes);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sm100::smem_u32(raw)),
                 "l"(A + r * lda), "r"(row_bytes), "r"(sm100::smem_u32(bar))
                 : "memory");
  }
  for (; r < n; r += gridDim.x) {
    sm100::mbar_wait(bar, ph);
    ph ^= 1;
    // 2. U_k from the raw row (weights w = D / s), Z_N := 0
    for (int kk = tid; kk < M; kk += blockDim.x) {
      const T z0 = raw[kk] * w[kk];
      const T zn = kk ? raw[N - kk] * w[N - kk] : T(0);
      const T zm = raw[M - kk] * w[M - kk];
      const T zp = raw[M + kk] * w[M + kk];
      const C2<T> al = ab[2 * kk], be = ab[2 * kk + 1];
      const C2<T> p = cmul(al, C2<T>{z0, -zn});
      const C2<T> q = cmul(be, C2<T>{zm, zp});
      u[sw(kk)] = cadd(p, q);
    }
    __syncthreads();
    // the raw buffer is free: prefetch the next row while this one is transformed
    const int64_t rn = r + gridDim.x;
    if (tid == 0 && rn < n) {
      sm100::mbar_arrive_expect_tx(bar, row_bytes);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sm100::smem_u32(raw)),
                   "l"(A + rn * lda), "r"(row_bytes), "r"(sm100::smem_u32(bar))
                   : "memory");
    }
    // 3. u = IDFT_M(U): M = 2^m, m = 4a + b: one pass of radix 4 (b = 2), 8 (b = 3) or 32 (b = 1, replacing
    //    a radix-16 pass), then radix-16 passes
    {
      int L = 1;
      if constexpr (B == 1) { stockham_pass<T, 32>(u, tw, M, L); L = 32; }
      if constexpr (B == 2) { stockham_pass<T, 4>(u, tw, M, L); L = 4; }
      if constexpr (B == 3) { stockham_pass<T, 8>(u, tw, M, L); L = 8; }
      while (L < M) {
        stockham_pass<T, 16>(u, tw, M, L);
        L *= 16;
      }
    }
    // 4. sampled outputs: v_t = (float view of u)[t]; scale includes 1 / N
    const T* v = reinterpret_cast<const T*>(u);
    T* y = Y + r * ldy;
    for (int c = tid; c < k; c += blockDim.x) {
      T s = T(0);
      for (int x = 0; x < xi; ++x) {
        const int32_t e = samp[c * xi + x];
        const int t = e & 0x7fffffff;
        const T val = v[2 * sw(t >> 1) + (t & 1)];
        s += (e < 0) ? -val : val;
      }
      y[c] = s * scale;
    }
    __syncthreads();
  }
}

template <typename T>
int dct_run(const T* A, int64_t n, int N, int64_t lda, const T* w, const T* ab, const T* tw, const int32_t* samp,
            int xi, int k, double scale, T* Y, int64_t ldy, cudaStream_t s) {
  const size_t smem = (size_t)N * sizeof(T) + (size_t)N * sizeof(T) + (size_t)N * sizeof(T) + 16;
  if (smem > 227 * 1024) return fail(SK_EUNSUPPORTED, "sk_srtt_dct_right: row too long for shared memory");
  using KernT = void (*)(const T*, int64_t, int, int64_t, const T*, const C2<T>*, const C2<T>*, const int32_t*, int,
                         int, T, T*, int64_t);
  const int b = (31 - __builtin_clz((unsigned)(N / 2))) & 3;
  const int threads = N / 2 > 4096 ? 512 : 256;  // one butterfly group per thread (M / 16 groups at most)
  KernT kern;
  if (threads == 512) {
    if constexpr (sizeof(T) == 8) return fail(SK_EUNSUPPORTED, "sk_srtt_dct_right: float64 needs d <= 8192");
    else kern = srtt_dct_kernel<T, 512, 1>;  // M = 8192 = 32 * 16 * 16
  } else {
    kern = b == 0 ? srtt_dct_kernel<T, 256, 0>
         : b == 1 ? srtt_dct_kernel<T, 256, 1>
         : b == 2 ? srtt_dct_kernel<T, 256, 2>
                  : srtt_dct_kernel<T, 256, 3>;
  }
  allow_smem(kern, smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)per_sm * sm_count();
  if (grid > n) grid = n;
  kern<<<(unsigned)grid, threads, smem, s>>>(A, n, N, lda, w, reinterpret_cast<const C2<T>*>(ab),
                                             reinterpret_cast<const C2<T>*>(tw), samp, xi, k, (T)scale, Y, ldy);
  return check_launch("sk_srtt_dct_right");
}

}  // namespace
}  // namespace skb

// ab: [M][2] complex (alpha_k, beta_k) interleaved re/im; tw: [M] complex e^{2 pi i t / M}; w: [N] = D / s;
// samp[c * xi + x] = t | neg << 31 with t the index in v of the sampled DCT output; scale includes 1 / N.
extern "C" int sk_srtt_dct_right(int dtype, const void* A, int64_t n, int64_t d, int64_t lda, const void* w,
                                 const void* ab, const void* tw, const int32_t* samp, int32_t xi, int64_t k,
                                 double scale, void* Y, int64_t ldy, void* stream) {
  using namespace skb;
  if (n < 0 || d < 32 || (d & (d - 1)) || lda < d || k < 1 || xi < 1 || ldy < k)
    return fail(SK_EINVAL, "sk_srtt_dct_right: bad shape (d a power of two >= 32)");
  if (n == 0) return SK_OK;
  if (!A || !w || !ab || !tw || !samp || !Y) return fail(SK_EINVAL, "sk_srtt_dct_right: null pointer");
  const size_t esz = dtype == SK_F64 ? 8 : 4;
  if ((reinterpret_cast<uintptr_t>(A) & 15) || ((lda * esz) & 15))
    return fail(SK_EINVAL, "sk_srtt_dct_right: rows must be 16-byte aligned");
  cudaStream_t s = as_stream(stream);
  if (dtype == SK_F32)
    return dct_run<float>(static_cast<const float*>(A), n, (int)d, lda, static_cast<const float*>(w),
                          static_cast<const float*>(ab), static_cast<const float*>(tw), samp, xi, (int)k, scale,
                          static_cast<float*>(Y), ldy, s);
  if (dtype == SK_F64)
    return dct_run<double>(static_cast<const double*>(A), n, (int)d, lda, static_cast<const double*>(w),
                           static_cast<const double*>(ab), static_cast<const double*>(tw), samp, xi, (int)k, scale,
                           static_cast<double*>(Y), ldy, s);
  return fail(SK_EINVAL, "sk_srtt_dct_right: dtype");
}

extern "C" int sk_srtt_dct_supported(int dtype, int64_t d) {
  if (d < 32 || (d & (d - 1))) return 0;
  const size_t esz = dtype == SK_F64 ? 8 : 4;
  return 3 * (size_t)d * esz + 16 <= 227 * 1024 ? 1 : 0;
}
