// K3b — SRTT with the DCT transform (the reference's real-field default, src/sketch/rtt.py:92-93,
// 129-140):  Y[r, c] = scale * sum_x sign_{c,x} * DCT-III(A[r, :] D)[j_{c,x}]   for power-of-two d.
//
// One CTA per row (persistent over rows, several CTAs per SM), everything in shared memory, no
// intermediate in HBM; a CTA keeps one row-sized buffer (plus ~3 KB of twiddles):
//   1. the raw row lands in it by one cp.async.bulk (issued as soon as the previous row's gather is done;
//      the other CTAs on the SM overlap the load);
//   2. Makhoul's real-IFFT form of the DCT-III, folded with the split of a length-N real inverse FFT
//      into a length-M = N/2 complex one:  with Z = A D / s (s the ortho weights),
//         U_k = alpha_k (Z_k - i Z_{N-k}) + beta_k (Z_{M-k} + i Z_{M+k}),   k = 0..M-1  (Z_N := 0),
//      alpha_k = c_k (1 + i w^k), beta_k = conj(c_{M-k}) (1 - i w^k), c_k = e^{i pi k / 2N},
//      w = e^{2 pi i / N} = c^4 (c_k from two short shared tables formed by sincospi at CTA start; the
//      weights w = D / s folded into the load, a +-1 diagonal as a shared sign mask); every thread forms
//      its U_k in registers before any is stored, because u overwrites the raw row in place;
//   3. u = IDFT_M(U) by Stockham passes in shared memory (radix 16, plus one radix-4/8/32 pass when M is
//      not a power of 16), one butterfly group per thread, in place (loads, barrier, stores); each group
//      is an in-register DIF DFT; twiddles e^{2 pi i t / M} as products of two short shared tables;
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

// a * e^{2 pi i e / 32} with e a compile-time constant after unrolling: quarter turns are swaps and
// negations, odd multiples of pi/4 two multiplies, the rest a complex multiply by literals
template <typename T>
__device__ __forceinline__ C2<T> mul_w32(C2<T> a, int e) {
  constexpr double r2 = 0.70710678118654752440;
  switch (e & 31) {
    case 0: return a;
    case 8: return {-a.y, a.x};
    case 16: return {-a.x, -a.y};
    case 24: return {a.y, -a.x};
    case 4: return {(T)r2 * (a.x - a.y), (T)r2 * (a.x + a.y)};
    case 12: return {(T)(-r2) * (a.x + a.y), (T)r2 * (a.x - a.y)};
    case 20: return {(T)r2 * (a.y - a.x), (T)(-r2) * (a.x + a.y)};
    case 28: return {(T)r2 * (a.x + a.y), (T)r2 * (a.y - a.x)};
    case 1: return cmul(a, C2<T>{(T)(0.9807852804032304), (T)(0.19509032201612825)});
    case 2: return cmul(a, C2<T>{(T)(0.9238795325112867), (T)(0.3826834323650898)});
    case 3: return cmul(a, C2<T>{(T)(0.8314696123025452), (T)(0.5555702330196022)});
    case 5: return cmul(a, C2<T>{(T)(0.5555702330196023), (T)(0.8314696123025452)});
    case 6: return cmul(a, C2<T>{(T)(0.38268343236508984), (T)(0.9238795325112867)});
    case 7: return cmul(a, C2<T>{(T)(0.19509032201612833), (T)(0.9807852804032304)});
    case 9: return cmul(a, C2<T>{(T)(-0.1950903220161282), (T)(0.9807852804032304)});
    case 10: return cmul(a, C2<T>{(T)(-0.3826834323650897), (T)(0.9238795325112867)});
    case 11: return cmul(a, C2<T>{(T)(-0.555570233019602), (T)(0.8314696123025455)});
    case 13: return cmul(a, C2<T>{(T)(-0.8314696123025453), (T)(0.5555702330196022)});
    case 14: return cmul(a, C2<T>{(T)(-0.9238795325112867), (T)(0.3826834323650899)});
    case 15: return cmul(a, C2<T>{(T)(-0.9807852804032304), (T)(0.1950903220161286)});
    case 17: return cmul(a, C2<T>{(T)(-0.9807852804032304), (T)(-0.19509032201612836)});
    case 18: return cmul(a, C2<T>{(T)(-0.9238795325112868), (T)(-0.38268343236508967)});
    case 19: return cmul(a, C2<T>{(T)(-0.8314696123025455), (T)(-0.555570233019602)});
    case 21: return cmul(a, C2<T>{(T)(-0.5555702330196022), (T)(-0.8314696123025452)});
    case 22: return cmul(a, C2<T>{(T)(-0.38268343236509034), (T)(-0.9238795325112865)});
    case 23: return cmul(a, C2<T>{(T)(-0.19509032201612866), (T)(-0.9807852804032303)});
    case 25: return cmul(a, C2<T>{(T)(0.1950903220161283), (T)(-0.9807852804032304)});
    case 26: return cmul(a, C2<T>{(T)(0.38268343236509), (T)(-0.9238795325112866)});
    case 27: return cmul(a, C2<T>{(T)(0.5555702330196018), (T)(-0.8314696123025455)});
    case 29: return cmul(a, C2<T>{(T)(0.8314696123025452), (T)(-0.5555702330196022)});
    case 30: return cmul(a, C2<T>{(T)(0.9238795325112865), (T)(-0.3826834323650904)});
    case 31: return cmul(a, C2<T>{(T)(0.9807852804032303), (T)(-0.19509032201612872)});
    default: return a;
  }
}

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
        x[b + j + span] = mul_w32(dlt, e);
      }
    }
  }
}

// u is stored XOR-swizzled at complex granularity: logical index i lives at sw(i) = i ^ ((i >> 4) & 15),
// so both the Stockham loads (consecutive i per lane) and the first pass's stores (i = 16 g + r) are
// bank-conflict free
__device__ __forceinline__ int sw(int i) { return i ^ ((i >> 4) & 15); }

// twiddle e^{2 pi i t / M} from two short shared tables: t0[l] = e^{2 pi i l / M} (l < 64) and
// t1[h] = e^{2 pi i 64 h / M}, so the CTA keeps ~3 KB of twiddles instead of M complex values
template <typename T>
__device__ __forceinline__ C2<T> twid(const C2<T>* t0, const C2<T>* t1, int t) {
  return t < 64 ? t0[t] : cmul(t1[t >> 6], t0[t & 63]);
}

// one Stockham pass of radix R on u (M complex, in shared memory): element q of group g is multiplied
// by W^q with W = e^{2 pi i k / (L R)} (k = g mod L; powers by a complex-multiply chain, one twiddle per
// group); one butterfly group per thread (blockDim >= M / R), in place (loads, barrier, stores, barrier)
template <typename T, int R>
__device__ __forceinline__ void stockham_pass(C2<T>* u, const C2<T>* t0, const C2<T>* t1, int M, int L) {
  const int G = M / R;
  const int g = threadIdx.x;
  const int stride_tw = M / (L * R);
  C2<T> v[R];
  const int k = g % L;
  if (g < G) {
    const C2<T> w1 = twid(t0, t1, k * stride_tw);
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

template <typename T>
__device__ __forceinline__ C2<T> cis_pi(double x) {  // e^{i pi x}
  double s, c;
  sincospi(x, &s, &c);
  return {(T)c, (T)s};
}

template <typename T, int THREADS, int B>  // B = log2(M) % 4: the extra pass (0 none, 1 radix 32, 2 radix 4, 3 radix 8)
__global__ void __launch_bounds__(THREADS, THREADS == 512 ? 1 : 2)
    srtt_dct_kernel(const T* __restrict__ A, int64_t n, int N, int64_t lda, const T* __restrict__ w,
                    const int32_t* __restrict__ samp, int xi, int k, T scale, T* __restrict__ Y, int64_t ldy) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int M = N / 2;
  const int nt1 = M >= 64 ? M / 64 : 1;
  C2<T>* u = reinterpret_cast<C2<T>*>(smem);  // M complex; the raw row (N reals) lands here
  const T* raw = reinterpret_cast<const T*>(smem);
  C2<T>* t0 = u + M;                          // e^{2 pi i l / M}, l < 64
  C2<T>* t1 = t0 + 64;                        // e^{2 pi i 64 h / M}, h < M / 64
  C2<T>* r0 = t1 + nt1;                       // c_l = e^{i pi l / 2N}, l < 64
  C2<T>* r1 = r0 + 64;                        // e^{i pi 64 h / 2N}, h < M / 64
  C2<T>* q0 = r1 + nt1;                       // c_l^5 = e^{i 5 pi l / 2N}, l < 64
  C2<T>* q1 = q0 + 64;                        // e^{i 5 pi 64 h / 2N}, h < M / 64
  uint32_t* sbits = reinterpret_cast<uint32_t*>(q1 + nt1);  // sign of w[i], N bits
  uint64_t* bar = reinterpret_cast<uint64_t*>(sbits + ((N / 32 + 1) & ~1));  // 8-byte aligned
  const int tid = threadIdx.x;
  // every trig table is formed here (sincospi, float64), ~3 KB per CTA: no table is re-read from L2
  for (int i = tid; i < 64; i += THREADS) {
    t0[i] = cis_pi<T>(2.0 * (i < M ? i : 0) / M);
    r0[i] = cis_pi<T>((double)i / (2.0 * N));
    q0[i] = cis_pi<T>(5.0 * i / (2.0 * N));
  }
  for (int i = tid; i < nt1; i += THREADS) {
    t1[i] = cis_pi<T>(M >= 64 ? 128.0 * i / M : 0.0);
    r1[i] = cis_pi<T>(64.0 * i / (2.0 * N));
    q1[i] = cis_pi<T>(5.0 * 64.0 * i / (2.0 * N));
  }
  // w = D / s: with a +-1 diagonal |w| is one value past index 0, so the signs go to a bit mask and
  // the loads below never touch the table (any other w is read as given)
  const T wm0 = fabs(w[0]), wm1 = fabs(w[1]);
  bool uni = true;
  for (int i = tid; i < N; i += THREADS) {
    const T v = w[i];
    const unsigned bits = __ballot_sync(0xffffffffu, v < T(0));
    if ((i & 31) == 0) sbits[i >> 5] = bits;
    if (i > 0 && fabs(v) != wm1) uni = false;
  }
  uni = __syncthreads_and(uni);
  auto wv = [=](int i) -> T {
    if (!uni) return w[i];
    const T m = i ? wm1 : wm0;
    return ((sbits[i >> 5] >> (i & 31)) & 1u) ? -m : m;
  };
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
    // 2. U_k from the raw row (weights w = D / s), Z_N := 0.  The row and u share the buffer, so every
    //    thread forms its U_k in registers first, then a barrier, then the stores.  U_k and U_{M-k} read
    //    the same four inputs; with c = c_k, c5 = c_k^5 (om = c^4): alpha_k = c + i c5,
    //    beta_k = e^{-i pi/4} (c - i c5), alpha_{M-k} = e^{i pi/4} conj(alpha_k),
    //    beta_{M-k} = e^{-i pi/4} conj(beta_k).  Pairs k = 1 .. M/2 - 1; k = 0 and M/2 by threads 0, 1.
    constexpr int PPT = 8;  // (M/2 - 1) / THREADS <= 8 for every supported (d, THREADS)
    // the thread index re-read per row: the pair indices below are row-invariant, and hoisting their
    // address / weight arithmetic out of the row loop only spills it to local memory
    int tr;
    asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tr));
    const C2<T> ep = {(T)0.70710678118654752440, (T)0.70710678118654752440};  // e^{i pi / 4}
    const C2<T> em = {ep.x, -ep.y};
    C2<T> ua[PPT], ub[PPT];
#pragma unroll
    for (int i = 0; i < PPT; ++i) {
      const int kk = 1 + tr + i * THREADS;
      if (kk < M / 2) {
        const T za = raw[kk] * wv(kk), zb = raw[N - kk] * wv(N - kk);
        const T zc = raw[M - kk] * wv(M - kk), ze = raw[M + kk] * wv(M + kk);
        const C2<T> c = twid(r0, r1, kk), c5 = twid(q0, q1, kk);
        const C2<T> al = {c.x - c5.y, c.y + c5.x};
        const C2<T> be = cmul(em, C2<T>{c.x + c5.y, c.y - c5.x});
        ua[i] = cadd(cmul(al, C2<T>{za, -zb}), cmul(be, C2<T>{zc, ze}));
        const C2<T> al2 = cmul(ep, C2<T>{al.x, -al.y}), be2 = cmul(em, C2<T>{be.x, -be.y});
        ub[i] = cadd(cmul(al2, C2<T>{zc, -ze}), cmul(be2, C2<T>{za, zb}));
      }
    }
    C2<T> ux = {T(0), T(0)};
    const int kx = tid == 0 ? 0 : M / 2;  // threads 0 and 1
    if (tid < 2) {
      const T z0 = raw[kx] * wv(kx), zn = kx ? raw[N - kx] * wv(N - kx) : T(0);
      const T zm = raw[M - kx] * wv(M - kx), zp = raw[M + kx] * wv(M + kx);
      const C2<T> c = twid(r0, r1, kx), c5 = twid(q0, q1, kx);
      const C2<T> al = {c.x - c5.y, c.y + c5.x};
      const C2<T> be = cmul(em, C2<T>{c.x + c5.y, c.y - c5.x});
      ux = cadd(cmul(al, C2<T>{z0, -zn}), cmul(be, C2<T>{zm, zp}));
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < PPT; ++i) {
      const int kk = 1 + tid + i * THREADS;
      if (kk < M / 2) {
        u[sw(kk)] = ua[i];
        u[sw(M - kk)] = ub[i];
      }
    }
    if (tid < 2) u[sw(kx)] = ux;
    __syncthreads();
    // 3. u = IDFT_M(U): M = 2^m, m = 4a + b: one pass of radix 4 (b = 2), 8 (b = 3) or 32 (b = 1, replacing
    //    a radix-16 pass), then radix-16 passes
    {
      int L = 1;
      if constexpr (B == 1) { stockham_pass<T, 32>(u, t0, t1, M, L); L = 32; }
      if constexpr (B == 2) { stockham_pass<T, 4>(u, t0, t1, M, L); L = 4; }
      if constexpr (B == 3) { stockham_pass<T, 8>(u, t0, t1, M, L); L = 8; }
      while (L < M) {
        stockham_pass<T, 16>(u, t0, t1, M, L);
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
    // u is free: the CTA's next row lands in it (other CTAs on the SM overlap this load)
    const int64_t rn = r + gridDim.x;
    if (tid == 0 && rn < n) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      sm100::mbar_arrive_expect_tx(bar, row_bytes);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sm100::smem_u32(u)),
                   "l"(A + rn * lda), "r"(row_bytes), "r"(sm100::smem_u32(bar))
                   : "memory");
    }
  }
}

size_t dct_smem(int64_t N, size_t esz) {
  const int64_t M = N / 2;
  return (size_t)N * esz + (size_t)(64 + (M >= 64 ? M / 64 : 1)) * 3 * 2 * esz + (size_t)((N / 32 + 1) & ~1) * 4 + 16;
}

template <typename T>
int dct_run(const T* A, int64_t n, int N, int64_t lda, const T* w, const int32_t* samp, int xi, int k, double scale,
            T* Y, int64_t ldy, cudaStream_t s) {
  const size_t smem = dct_smem(N, sizeof(T));
  if (smem > 227 * 1024) return fail(SK_EUNSUPPORTED, "sk_srtt_dct_right: row too long for shared memory");
  using KernT = void (*)(const T*, int64_t, int, int64_t, const T*, const int32_t*, int, int, T, T*, int64_t);
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
  kern<<<(unsigned)grid, threads, smem, s>>>(A, n, N, lda, w, samp, xi, k, (T)scale, Y, ldy);
  return check_launch("sk_srtt_dct_right");
}

}  // namespace
}  // namespace skb

// w: [N] = D / s; samp[c * xi + x] = t | neg << 31 with t the index in v of the sampled DCT output;
// scale includes 1 / N.  The trig tables are formed on the device.
extern "C" int sk_srtt_dct_right(int dtype, const void* A, int64_t n, int64_t d, int64_t lda, const void* w,
                                 const int32_t* samp, int32_t xi, int64_t k, double scale, void* Y, int64_t ldy,
                                 void* stream) {
  using namespace skb;
  if (n < 0 || d < 32 || (d & (d - 1)) || lda < d || k < 1 || xi < 1 || ldy < k)
    return fail(SK_EINVAL, "sk_srtt_dct_right: bad shape (d a power of two >= 32)");
  if (n == 0) return SK_OK;
  if (!A || !w || !samp || !Y) return fail(SK_EINVAL, "sk_srtt_dct_right: null pointer");
  const size_t esz = dtype == SK_F64 ? 8 : 4;
  if ((reinterpret_cast<uintptr_t>(A) & 15) || ((lda * esz) & 15))
    return fail(SK_EINVAL, "sk_srtt_dct_right: rows must be 16-byte aligned");
  cudaStream_t s = as_stream(stream);
  if (dtype == SK_F32)
    return dct_run<float>(static_cast<const float*>(A), n, (int)d, lda, static_cast<const float*>(w), samp, xi,
                          (int)k, scale, static_cast<float*>(Y), ldy, s);
  if (dtype == SK_F64)
    return dct_run<double>(static_cast<const double*>(A), n, (int)d, lda, static_cast<const double*>(w), samp, xi,
                           (int)k, scale, static_cast<double*>(Y), ldy, s);
  return fail(SK_EINVAL, "sk_srtt_dct_right: dtype");
}

extern "C" int sk_srtt_dct_supported(int dtype, int64_t d) {
  if (d < 32 || (d & (d - 1))) return 0;
  if (dtype == SK_F64 ? d > 8192 : d > 16384) return 0;  // one butterfly group per thread (<= 512 threads)
  return skb::dct_smem(d, dtype == SK_F64 ? 8 : 4) <= 227 * 1024 ? 1 : 0;
}
