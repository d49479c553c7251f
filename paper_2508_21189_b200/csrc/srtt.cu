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
// Small rows (d = 2^L, 32 <= d <= 512): one warp per row (shuffle butterflies).
// Other sizes (d = 2^L, row fits shared memory): one CTA per row, row in shared memory.
#include <stdlib.h>

#include "common.cuh"

namespace skb {
int launch_srtt_tc(int L, const float* A, int64_t n, int64_t lda, const float* dv, const int32_t* samp, int xi, int k,
                   double scale, float* Y, int64_t ldy, cudaStream_t s);
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

// One-instruction bulk prefetch of [p, p + bytes) into L2 (TMA unit; bytes % 16 == 0).
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

template <typename T, int L, bool SIGNS>
__global__ void __launch_bounds__((1 << (L - 5)), (sizeof(T) == 4 ? (L <= 12 ? 3 : (L == 13 ? 2 : 1)) : (L <= 12 ? 2 : (L == 13 ? 2 : 1))))
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
    // the CTA's next row heads for L2 while this one is transformed (its loads then hit L2)
    if (t == 0 && row + gridDim.x < n && ((reinterpret_cast<uintptr_t>(a) & 15) == 0) && ((lda * sizeof(T)) & 15) == 0)
      prefetch_l2_bulk(a + gridDim.x * lda, (uint32_t)(D * sizeof(T)));
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


// ---------------------------------------------------------------------------------------------
// Float64 wide path (d = 8192, +-1 diagonal): 128 threads per row and 64 values per thread (128
// registers), so 12 of the 13 butterfly stages run in two register phases with ONE shared-memory
// transpose between them, and the last stage (index bit 7) is folded into the sampled gather:
//   phase 1: registers hold index bits {0, 8..12}    (32 coalesced 16-byte loads per thread)
//   phase 2: registers hold bits {1..6}              (one transpose; each thread writes back the
//            same positions it read, so no barrier between the read and the write-back)
//   gather : out = sum_x sign (X[j & ~128] +- X[j | 128])  (bit 7: top = sum, bottom = difference)
// The 3-phase fast path moves every row through shared memory five times (≈4200 wavefronts per
// row at config-2 shape, shared memory 64 % busy, 1.52 ms); this one three times: 1.07 ms (4.0 TB/s),
// latency-bound at 8 warps per SM (long-scoreboard on the row loads, float64 add chains).
// SKETCH_B200_SRTT64=3 selects the 3-phase kernel.
// Shared address of index j: j ^ (((j >> 7) & 7) << 1): the phase-1 16-byte stores and the phase-2
// 8-byte accesses are conflict free.
__device__ __forceinline__ int swz64(int j) { return j ^ (((j >> 7) & 7) << 1); }

__device__ __forceinline__ void wht64_regs(double (&x)[64]) {
#pragma unroll
  for (int h = 1; h < 64; h <<= 1) {
#pragma unroll
    for (int v = 0; v < 64; ++v) {
      if ((v & h) == 0) butterfly(x[v], x[v | h]);
    }
  }
}

template <int MINB>
__global__ void __launch_bounds__(128, MINB)
    srtt_wht64_wide(const double* __restrict__ A, int64_t n, int64_t lda, const double* __restrict__ dvals,
                    const int32_t* __restrict__ samp, int xi, int k, double scale, double* __restrict__ Y,
                    int64_t ldy) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* buf = reinterpret_cast<double*>(smem_raw);
  const int t = threadIdx.x, w = t >> 5, l = t & 31;
  const int base1 = 2 * l + 64 * w;              // phase-1 index of register pair q: base1 + 256 q
  const int base2 = (t & 1) | ((t >> 1) << 7);   // phase-2 index of register r: base2 | (r << 1)
  uint64_t dmask = 0;                            // D < 0 at the phase-1 positions (register e + 2 q)
#pragma unroll 1
  for (int q = 0; q < 32; ++q)
    for (int e = 0; e < 2; ++e)
      if (dvals[base1 + 256 * q + e] < 0.0) dmask |= 1ull << (e + 2 * q);
  for (int64_t row = blockIdx.x; row < n; row += gridDim.x) {
    const double* a = A + row * lda;
    if (t == 0 && row + gridDim.x < n)
      prefetch_l2_bulk(a + gridDim.x * lda, 8192u * 8u);  // the CTA's next row heads for L2
    double x[64];
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      double2 v;
      asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y)
                   : "l"(a + base1 + 256 * q));
      x[2 * q] = v.x;
      x[2 * q + 1] = v.y;
    }
#pragma unroll
    for (int r = 0; r < 64; ++r) x[r] = flip_if(x[r], (uint32_t)((dmask >> r) & 1u));
    wht64_regs(x);
    __syncthreads();  // the previous row's gather is done with buf
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      double* dst = buf + swz64(base1 + 256 * q);
      asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "d"(x[2 * q]),
                   "d"(x[2 * q + 1])
                   : "memory");
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 64; ++r) x[r] = buf[swz64(base2 | (r << 1))];
    wht64_regs(x);
#pragma unroll
    for (int r = 0; r < 64; ++r) buf[swz64(base2 | (r << 1))] = x[r];
    __syncthreads();
    double* y = Y + row * ldy;
    for (int c = t; c < k; c += 128) {
      double sacc = 0.0;
      for (int u = 0; u < xi; ++u) {
        const uint32_t e = (uint32_t)__ldg(samp + (int64_t)c * xi + u);
        const int j = (int)(e & 0x7fffffffu);
        const double x0 = buf[swz64(j & ~128)], x1 = buf[swz64(j | 128)];
        sacc += flip_if((j & 128) ? x0 - x1 : x0 + x1, e >> 31);
      }
      y[c] = sacc * scale;
    }
  }
}

template <int MINB>
int launch_wide64_t(const double* A, int64_t n, int64_t lda, const double* dv, const int32_t* samp, int xi, int k,
                    double scale, double* Y, int64_t ldy, cudaStream_t s) {
  const size_t smem = 8192 * sizeof(double);
  allow_smem(srtt_wht64_wide<MINB>, smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, srtt_wht64_wide<MINB>, 128, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)sm_count() * per_sm;
  if (grid > n) grid = n;
  srtt_wht64_wide<MINB><<<(unsigned)grid, 128, smem, s>>>(A, n, lda, dv, samp, xi, k, scale, Y, ldy);
  return check_launch("sk_srtt_right(f64 wide)");
}
// two CTAs per SM (254 registers): three (168 registers) spill the values and ran 1.15 vs 1.07 ms
int launch_wide64(const double* A, int64_t n, int64_t lda, const double* dv, const int32_t* samp, int xi, int k,
                  double scale, double* Y, int64_t ldy, cudaStream_t s) {
  return launch_wide64_t<2>(A, n, lda, dv, samp, xi, k, scale, Y, ldy, s);
}

// ---------------------------------------------------------------------------------------------
// Wide fast path (float32, +-1 diagonal, d = 2^L, 12 <= L <= 14): T = d/128 threads per row and
// 128 values per thread held as 64 packed float pairs, so 12 of the 13 (L=13) butterfly stages run
// as Blackwell FADD2/FSUB2 (add.rn.f32x2) on register pairs.
//   phase 1: registers hold index bits {0,1} u {L-5..L-1}   (32 coalesced float4 loads / thread)
//   phase 2: registers hold bits {0,1} u {2..6}             (one float4 shared-memory transpose;
//            each thread then owns 128 consecutive indices, so the write-back needs no barrier)
//   gather : remaining bits {7..L-6} are folded into the sampled gather: each sampled output is a
//            +-sum of 2^(L-12) transposed values.
// Shared address of index j: j ^ (((j >> 7) & 7) << 2) — float4 writes and reads conflict free.
// ---------------------------------------------------------------------------------------------
typedef unsigned long long u64;

__device__ __forceinline__ u64 f2add(u64 a, u64 b) {
  u64 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 f2sub(u64 a, u64 b) {
  u64 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 pk(float lo, float hi) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void upk(u64 p, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(p));
}
__device__ __forceinline__ int swz4(int j) { return j ^ (((j >> 7) & 7) << 2); }



template <int L>
struct WideCfg {
  static constexpr int T = 1 << (L - 7);
  static constexpr int MINB = L == 12 ? 8 : (L == 13 ? 4 : 2);
};

template <int L>
__global__ void __launch_bounds__(WideCfg<L>::T, WideCfg<L>::MINB)
    srtt_wht_wide(const float* __restrict__ A, int64_t n, int64_t lda, const float* __restrict__ dvals,
                  const int32_t* __restrict__ samp, int xi, int k, float scale, float* __restrict__ Y,
                  int64_t ldy) {
  constexpr int T = WideCfg<L>::T;
  constexpr int QS = 4 * T;        // index stride of the 32 float4 groups in phase 1
  constexpr int M3 = L - 12;       // bits folded into the gather
  constexpr int PF = 2;            // rows of L2 prefetch distance per CTA
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* buf = reinterpret_cast<float*>(smem_raw);
  const int t = threadIdx.x;

  // sign bits of D at this thread's 128 phase-1 positions: bit (4q + c) <-> j = 4t + c + QS*q
  uint32_t dm[4] = {0u, 0u, 0u, 0u};
#pragma unroll
  for (int q = 0; q < 32; ++q) {
    const float4 dv = *reinterpret_cast<const float4*>(dvals + 4 * t + QS * q);
    const uint32_t b = (dv.x < 0.f ? 1u : 0u) | (dv.y < 0.f ? 2u : 0u) | (dv.z < 0.f ? 4u : 0u) | (dv.w < 0.f ? 8u : 0u);
    dm[q >> 3] |= b << (4 * (q & 7));
  }

  if (t == 0) {
    for (int j = 0; j < PF; ++j)
      if (blockIdx.x + (int64_t)j * gridDim.x < n) prefetch_l2_bulk(A + (blockIdx.x + (int64_t)j * gridDim.x) * lda, 4u << L);
  }
  u64 p[64];
  auto load_row = [&](int64_t row) {
    const float* a = A + row * lda;
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      float v[4];
      ld4(a + 4 * t + QS * q, v);
      p[2 * q] = pk(v[0], v[1]);
      p[2 * q + 1] = pk(v[2], v[3]);
    }
  };
  for (int64_t row = blockIdx.x; row < n; row += gridDim.x) {
    // keep the DRAM stream busy: the CTA's row PF iterations ahead goes to L2 now
    if (t == 0 && row + (int64_t)PF * gridDim.x < n) prefetch_l2_bulk(A + (row + (int64_t)PF * gridDim.x) * lda, 4u << L);
    load_row(row);
    // sign flip (D) and the stage on index bit 0
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      float v[4];
      upk(p[2 * q], v[0], v[1]);
      upk(p[2 * q + 1], v[2], v[3]);
      const uint32_t w = dm[q >> 3] >> (4 * (q & 7));
      v[0] = __int_as_float(__float_as_int(v[0]) ^ (w << 31));
      v[1] = __int_as_float(__float_as_int(v[1]) ^ ((w << 30) & 0x80000000u));
      v[2] = __int_as_float(__float_as_int(v[2]) ^ ((w << 29) & 0x80000000u));
      v[3] = __int_as_float(__float_as_int(v[3]) ^ ((w << 28) & 0x80000000u));
      p[2 * q] = pk(v[0] + v[1], v[0] - v[1]);
      p[2 * q + 1] = pk(v[2] + v[3], v[2] - v[3]);
    }
    // stage on index bit 1 (pair index bit 0), then the 5 q bits (pair index bits 1..5)
#pragma unroll
    for (int h = 1; h < 64; h <<= 1) {
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        if ((i & h) == 0) {
          const u64 s = f2add(p[i], p[i | h]);
          const u64 d = f2sub(p[i], p[i | h]);
          p[i] = s;
          p[i | h] = d;
        }
      }
    }
    __syncthreads();  // the previous row's gather has finished reading buf
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      float v[4];
      upk(p[2 * q], v[0], v[1]);
      upk(p[2 * q + 1], v[2], v[3]);
      *reinterpret_cast<float4*>(buf + swz4(4 * t + QS * q)) = make_float4(v[0], v[1], v[2], v[3]);
    }
    __syncthreads();
    // phase 2: this thread owns indices 128t .. 128t+127 (bits 0..6)
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      const float4 v = *reinterpret_cast<const float4*>(buf + swz4(128 * t + 4 * u));
      p[2 * u] = pk(v.x, v.y);
      p[2 * u + 1] = pk(v.z, v.w);
    }
#pragma unroll
    for (int h = 2; h < 64; h <<= 1) {
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        if ((i & h) == 0) {
          const u64 s = f2add(p[i], p[i | h]);
          const u64 d = f2sub(p[i], p[i | h]);
          p[i] = s;
          p[i | h] = d;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      float v[4];
      upk(p[2 * u], v[0], v[1]);
      upk(p[2 * u + 1], v[2], v[3]);
      *reinterpret_cast<float4*>(buf + swz4(128 * t + 4 * u)) = make_float4(v[0], v[1], v[2], v[3]);
    }
    __syncthreads();
    // gather with the last M3 stages folded in
    float* y = Y + row * ldy;
    for (int c = t; c < k; c += T) {
      float s = 0.f;
      for (int x = 0; x < xi; ++x) {
        const uint32_t e = (uint32_t)__ldg(samp + (int64_t)c * xi + x);
        const int r = (int)(e & 0x7fffffffu);
        float acc;
        if constexpr (M3 == 0) {
          acc = buf[swz4(r)];
        } else {
          constexpr int MK = ((1 << M3) - 1) << 7;
          const int rb = r & ~MK, rh = (r >> 7) & ((1 << M3) - 1);
          acc = 0.f;
#pragma unroll
          for (int u = 0; u < (1 << M3); ++u) {
            const float z = buf[swz4(rb | (u << 7))];
            acc += flip_if(z, (uint32_t)(__popc(u & rh) & 1));
          }
        }
        s += flip_if(acc, e >> 31);
      }
      y[c] = s * scale;
    }
  }
}

template <int L>
int launch_wide(const float* A, int64_t n, int64_t lda, const float* dv, const int32_t* samp, int xi, int k,
                double scale, float* Y, int64_t ldy, cudaStream_t s) {
  constexpr int T = WideCfg<L>::T;
  const size_t smem = sizeof(float) << L;
  auto kern = srtt_wht_wide<L>;
  allow_smem(kern, smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)sm_count() * per_sm;
  if (grid > n) grid = n;
  kern<<<(unsigned)grid, T, smem, s>>>(A, n, lda, dv, samp, xi, k, (float)scale, Y, ldy);
  return check_launch("sk_srtt_right(wide)");
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

// Small rows (d = 2^L, 5 <= L <= 9): one warp per row, V = d/32 consecutive values per lane.
// In-register butterflies over the low log2(V) index bits, shuffle butterflies over the 5 lane
// bits, then the warp's transformed row goes to a private shared-memory buffer for the sampled
// gather (coalesced row loads, one HBM pass, no CTA barrier).
template <typename T, int L, bool SIGNS, bool VEC>
__global__ void __launch_bounds__(256)
    srtt_wht_warp(const T* __restrict__ A, int64_t n, int64_t lda, const T* __restrict__ dvals,
                  const int32_t* __restrict__ samp, int xi, int k, T scale, T* __restrict__ Y, int64_t ldy) {
  constexpr int D = 1 << L, V = D / 32, NV = 16 / sizeof(T);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T* buf = reinterpret_cast<T*>(smem_raw) + warp * D;
  T dv[V];
  uint32_t dmask = 0;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    dv[v] = dvals[lane * V + v];
    if (dv[v] < T(0)) dmask |= 1u << v;
  }
  const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; row < n; row += wstride) {
    const T* a = A + row * lda + lane * V;
    T x[V];
    if constexpr (VEC && (V % NV) == 0) {
#pragma unroll
      for (int q = 0; q < V / NV; ++q) {
        T tmp[NV];
        if constexpr (sizeof(T) == 4) {
          const float4 f = __ldg(reinterpret_cast<const float4*>(a) + q);
          tmp[0] = f.x; tmp[1] = f.y; tmp[2] = f.z; tmp[3] = f.w;
        } else {
          const double2 f = __ldg(reinterpret_cast<const double2*>(a) + q);
          tmp[0] = f.x; tmp[1] = f.y;
        }
#pragma unroll
        for (int c = 0; c < NV; ++c) x[q * NV + c] = tmp[c];
      }
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v) x[v] = __ldg(a + v);
    }
#pragma unroll
    for (int v = 0; v < V; ++v) x[v] = SIGNS ? flip_if(x[v], (dmask >> v) & 1u) : x[v] * dv[v];
#pragma unroll
    for (int h = 1; h < V; h <<= 1)
#pragma unroll
      for (int v = 0; v < V; ++v)
        if ((v & h) == 0) butterfly(x[v], x[v | h]);
#pragma unroll
    for (int h = 1; h < 32; h <<= 1) {
      const bool bottom = (lane & h) != 0;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const T o = __shfl_xor_sync(0xffffffffu, x[v], h);
        x[v] = bottom ? o - x[v] : x[v] + o;
      }
    }
    __syncwarp();  // previous row's gather is done with buf
#pragma unroll
    for (int v = 0; v < V; ++v) buf[lane * V + v] = x[v];
    __syncwarp();
    T* y = Y + row * ldy;
    for (int c = lane; c < k; c += 32) {
      T acc = T(0);
      for (int u = 0; u < xi; ++u) {
        const uint32_t e = (uint32_t)__ldg(samp + (int64_t)c * xi + u);
        acc += flip_if(buf[e & 0x7fffffffu], e >> 31);
      }
      y[c] = acc * scale;
    }
  }
}

template <typename T, int L, bool SIGNS>
int launch_warp(const T* A, int64_t n, int64_t lda, const T* dv, const int32_t* samp, int xi, int k, double scale,
                T* Y, int64_t ldy, bool vec, cudaStream_t s) {
  const size_t smem = sizeof(T) * ((size_t)8 << L);
  auto kern = vec ? srtt_wht_warp<T, L, SIGNS, true> : srtt_wht_warp<T, L, SIGNS, false>;
  allow_smem(kern, smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)sm_count() * per_sm;
  const int64_t need = (n + 7) / 8;
  if (grid > need) grid = need;
  kern<<<(unsigned)grid, 256, smem, s>>>(A, n, lda, dv, samp, xi, k, (T)scale, Y, ldy);
  return check_launch("sk_srtt_right(warp)");
}

template <typename T, bool SIGNS>
int dispatch_warp(int L, const T* A, int64_t n, int64_t lda, const T* dv, const int32_t* samp, int xi, int k,
                  double scale, T* Y, int64_t ldy, bool vec, cudaStream_t s) {
  switch (L) {
    case 5: return launch_warp<T, 5, SIGNS>(A, n, lda, dv, samp, xi, k, scale, Y, ldy, vec, s);
    case 6: return launch_warp<T, 6, SIGNS>(A, n, lda, dv, samp, xi, k, scale, Y, ldy, vec, s);
    case 7: return launch_warp<T, 7, SIGNS>(A, n, lda, dv, samp, xi, k, scale, Y, ldy, vec, s);
    case 8: return launch_warp<T, 8, SIGNS>(A, n, lda, dv, samp, xi, k, scale, Y, ldy, vec, s);
    case 9: return launch_warp<T, 9, SIGNS>(A, n, lda, dv, samp, xi, k, scale, Y, ldy, vec, s);
    default: return fail(SK_EUNSUPPORTED, "sk_srtt_right: no warp WHT for this length");
  }
}

template <typename T, int L, bool SIGNS>
int launch_fast(const T* A, int64_t n, int64_t lda, const T* dv, const int32_t* samp, int xi, int k,
                double scale, T* Y, int64_t ldy, cudaStream_t s) {
  constexpr int NT = 1 << (L - 5);
  const size_t smem = sizeof(T) << L;
  auto kern = srtt_wht_fast<T, L, SIGNS>;
  allow_smem(kern, smem);
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

// SKETCH_B200_SRTT=regs forces the CUDA-core kernel (A/B comparisons); default: tensor cores at d = 8192
bool srtt_tc_enabled() {
  const char* e = getenv("SKETCH_B200_SRTT");
  return !(e && e[0] == 'r');
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
  if constexpr (sizeof(T) == 4) {
    const bool dv_aligned = (reinterpret_cast<uintptr_t>(dv) & 15) == 0;
    if (pm1 && aligned && dv_aligned && L >= 11 && L <= 14) {
      const float* Af = reinterpret_cast<const float*>(A);
      const float* dvf = reinterpret_cast<const float*>(dv);
      float* Yf = reinterpret_cast<float*>(Y);
      // tensor cores for d = 4096, 8192 (at d = 2048 the per-row epilogue and gather dominate: the
      // CUDA-core kernel is faster, 40 % vs 32 % of HBM)
      if (L >= 12 && L <= 13 && srtt_tc_enabled())
        return launch_srtt_tc(L, Af, n, lda, dvf, samp, xi, (int)k, scale, Yf, ldy, s);
      if (L == 11) return dispatch_L<float, true>(L, A, n, lda, dv, samp, xi, (int)k, scale, Y, ldy, s);
      if (L == 12) return launch_wide<12>(Af, n, lda, dvf, samp, xi, (int)k, scale, Yf, ldy, s);
      if (L == 13) return launch_wide<13>(Af, n, lda, dvf, samp, xi, (int)k, scale, Yf, ldy, s);
      return launch_wide<14>(Af, n, lda, dvf, samp, xi, (int)k, scale, Yf, ldy, s);
    }
  }
  if constexpr (sizeof(T) == 8) {
    const char* e = getenv("SKETCH_B200_SRTT64");
    if (pm1 && aligned && L == 13 && (int64_t(1) << L) == d && !(e && e[0] == '3'))
      return launch_wide64(reinterpret_cast<const double*>(A), n, lda, reinterpret_cast<const double*>(dv), samp,
                           xi, (int)k, scale, reinterpret_cast<double*>(Y), ldy, s);
  }
  const int max_fast = sizeof(T) == 4 ? 14 : 13;
  if (L >= 10 && L <= max_fast && aligned) {
    // Rademacher diagonals take the sign-mask path; any other diagonal multiplies.
    return pm1 ? dispatch_L<T, true>(L, A, n, lda, dv, samp, xi, (int)k, scale, Y, ldy, s)
               : dispatch_L<T, false>(L, A, n, lda, dv, samp, xi, (int)k, scale, Y, ldy, s);
  }
  if (L >= 5 && L <= 9 && (int64_t(1) << L) == d) {
    const bool dv_aligned = (reinterpret_cast<uintptr_t>(dv) & 15) == 0;
    const bool vec = aligned && dv_aligned;
    return pm1 ? dispatch_warp<T, true>(L, A, n, lda, dv, samp, xi, (int)k, scale, Y, ldy, vec, s)
               : dispatch_warp<T, false>(L, A, n, lda, dv, samp, xi, (int)k, scale, Y, ldy, vec, s);
  }
  const size_t smem = sizeof(T) * (size_t)d;
  if (smem > 200 * 1024) return fail(SK_EUNSUPPORTED, "sk_srtt_right: row does not fit shared memory");
  allow_smem(srtt_wht_simple<T>, smem);
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
