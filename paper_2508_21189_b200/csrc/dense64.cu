// K5d — float64 dense and Khatri-Rao applies on the FP64 tensor cores (DMMA, mma.sync m8n8k4 .f64).
//
// The reference computes every apply in float64 (core/containers.py:41-46; sketch/base.py:75-79,
// khatri_rao.py:158-164), so NumPy callers of the drop-in land here for the Gaussian family, the
// Khatri-Rao family and the adjoints of materialised operators:
//
//   C[M x N] = scale * opA(M x K) * opB(K x N)
//     opA = A (row-major M x K)              or A^T with A stored K x M (TA: the adjoint's B^T)
//     opB = B (row-major K x N, dense)       or the Khatri-Rao tile  B[P*dl + q, n] = W[P, n] * F[q, n]
//                                               synthesised in shared memory (KR: Omega never formed)
//     C   = row-major M x N                  or stored transposed (TC: the adjoint writes X = C^T)
//
// CTA = GM x GN warps, warp tile 32 x 32 of m8n8k4 DMMAs (16 independent accumulators per k step):
// 128 x 64 CTA tiles of 8 warps, K in stages of 16 through a 3-deep cp.async ring (one CTA barrier
// per stage), two CTAs per SM.  Shared tiles are padded to a row stride = 4 (mod 16) doubles so
// the fragment loads (8 rows x 4 k, or 4 k x 8 columns, per half-warp) hit 16 distinct bank pairs.  The Khatri-Rao tile goes through registers (F and W loads
// issued before the stage's MMAs, the product stored after them).  Accumulation is float64 (DMMA is
// an IEEE fma chain per element), so parity with the reference holds to rounding (~1e-15).
#include <cuda_runtime.h>

#include <cstdlib>

#include "common.cuh"

namespace skb {
namespace {

constexpr int BK_DEF = 32;
constexpr int STAGES_DEF = 3;

__device__ __forceinline__ void cp16(uint32_t dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// m8n8k4 .f64 (SASS DMMA.8x8x4; the larger .f64 shapes are sequences of it): A a0 at (g, t), B b0 at
// (t, g), C (c0, c1) at (g, 2t + {0, 1})   [g = lane / 4, t = lane % 4]
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

struct G64 {
  const double* A;
  int64_t M, K, lda;
  const double* B;  // dense opB (K x N, ldb) when W == nullptr, else F (dl x N, ldb)
  int64_t ldb;
  const double* W;  // Khatri-Rao leading weights (P x N, ldw) or nullptr
  int64_t ldw, dl;
  const double* Bi;  // complex Khatri-Rao: imaginary planes of F and W (same strides)
  const double* Wi;
  int part;          // complex Khatri-Rao: 0 = Re(W F), 1 = Im(W F)
  int accumulate;    // C += instead of C =
  int64_t N;
  double scale;
  double* C;
  int64_t ldc;
};

template <bool TA, bool TC, bool KR, int WM, int WN, int GM, int GN, bool CPLX = false, int BK = BK_DEF,
          int STAGES = STAGES_DEF, int MINB = 1>
__global__ void __launch_bounds__(GM * GN * 32, MINB) gemm64_kernel(const G64 p) {
  constexpr int THREADS = GM * GN * 32;
  constexpr int BM = GM * WM, BN = GN * WN;
  constexpr int SA = TA ? BM + 4 : BK + 4;  // A tile row stride (doubles): [BK][BM+4] or [BM][BK+4]
  constexpr int SB = BN + 4;                // B tile [BK][BN+4]
  constexpr int A_ELEMS = TA ? BK * SA : BM * SA;
  constexpr int B_ELEMS = BK * SB;
  extern __shared__ __align__(16) double sm64[];
  double* as = sm64;                            // [STAGES][A_ELEMS]
  double* bs = sm64 + STAGES * A_ELEMS;         // [STAGES][B_ELEMS]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp % GM, wn = warp / GM;
  const int g = lane >> 2, t = lane & 3;
  const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
  const int KT = (int)((p.K + BK - 1) / BK);
  // a warp whose 32 x 32 block lies wholly outside the result only loads (edge tiles: k = 200 on
  // 128-column tiles computes 224 columns, not 256)
  const bool busy = m0 + wm * WM < p.M && n0 + wn * WN < p.N;

  // ---- stage loaders
  auto load_a = [&](int kt, int slot) {
    const uint32_t base = su32(as + slot * A_ELEMS);
    const int64_t k0 = (int64_t)kt * BK;
    if (!TA) {  // BM rows x BK doubles (chunks of 2)
#pragma unroll
      for (int e = 0; e < BM * (BK / 2) / THREADS; ++e) {
        const int c = tid + THREADS * e, r = c / (BK / 2), ch = c % (BK / 2);
        const int64_t m = m0 + r, k = k0 + 2 * ch;
        const int64_t valid = (m < p.M) ? min((int64_t)2, max((int64_t)0, p.K - k)) : 0;
        const double* src = valid ? p.A + m * p.lda + k : p.A;
        cp16(base + (uint32_t)(r * SA + 2 * ch) * 8u, src, (int)valid * 8);
      }
    } else {    // BK rows (k) x BM doubles
#pragma unroll
      for (int e = 0; e < BK * BM / 2 / THREADS; ++e) {
        const int c = tid + THREADS * e, r = c / (BM / 2), ch = c % (BM / 2);
        const int64_t k = k0 + r, m = m0 + 2 * ch;
        const int64_t valid = (k < p.K) ? min((int64_t)2, max((int64_t)0, p.M - m)) : 0;
        const double* src = valid ? p.A + k * p.lda + m : p.A;
        cp16(base + (uint32_t)(r * SA + 2 * ch) * 8u, src, (int)valid * 8);
      }
    }
  };
  auto load_b = [&](int kt, int slot) {  // dense opB
    const uint32_t base = su32(bs + slot * B_ELEMS);
    const int64_t k0 = (int64_t)kt * BK;
#pragma unroll
    for (int e = 0; e < BK * BN / 2 / THREADS; ++e) {
      const int c = tid + THREADS * e, r = c / (BN / 2), ch = c % (BN / 2);
      const int64_t k = k0 + r, n = n0 + 2 * ch;
      const int64_t valid = (k < p.K) ? min((int64_t)2, max((int64_t)0, p.N - n)) : 0;
      const double* src = valid ? p.B + k * p.ldb + n : p.B;
      cp16(base + (uint32_t)(r * SB + 2 * ch) * 8u, src, (int)valid * 8);
    }
  };
  // Khatri-Rao opB through registers: fetch (F row q, W row P) pairs, multiply, store
  constexpr int KRV = KR ? BK * BN / 2 / THREADS : 1;
  double2 fr[KRV], wr[KRV];
  auto fetch_kr = [&](int kt) {
#pragma unroll
    for (int e = 0; e < KRV; ++e) {
      const int c = tid + THREADS * e, r = c / (BN / 2), ch = c % (BN / 2);
      const int64_t k = (int64_t)kt * BK + r, n = n0 + 2 * ch;
      fr[e] = make_double2(0.0, 0.0);
      wr[e] = make_double2(0.0, 0.0);
      if (k < p.K && n < p.N) {
        const int64_t P = k / p.dl, q = k - P * p.dl;
        const double* f = p.B + q * p.ldb + n;
        const double* w = p.W + P * p.ldw + n;
        if (n + 1 < p.N) {
          fr[e] = __ldg(reinterpret_cast<const double2*>(f));
          wr[e] = __ldg(reinterpret_cast<const double2*>(w));
        } else {
          fr[e].x = __ldg(f);
          wr[e].x = __ldg(w);
        }
        if (CPLX) {  // (wr + i wi)(fr + i fi): keep the requested part as fr * 1
          double2 fi = make_double2(0.0, 0.0), wi = make_double2(0.0, 0.0);
          const double* f2 = p.Bi + q * p.ldb + n;
          const double* w2 = p.Wi + P * p.ldw + n;
          if (n + 1 < p.N) {
            fi = __ldg(reinterpret_cast<const double2*>(f2));
            wi = __ldg(reinterpret_cast<const double2*>(w2));
          } else {
            fi.x = __ldg(f2);
            wi.x = __ldg(w2);
          }
          const double2 a = fr[e], b = wr[e];
          fr[e] = p.part ? make_double2(b.x * fi.x + wi.x * a.x, b.y * fi.y + wi.y * a.y)
                         : make_double2(b.x * a.x - wi.x * fi.x, b.y * a.y - wi.y * fi.y);
          wr[e] = make_double2(1.0, 1.0);
        }
      }
    }
  };
  auto store_kr = [&](int slot) {
    double* b = bs + slot * B_ELEMS;
#pragma unroll
    for (int e = 0; e < KRV; ++e) {
      const int c = tid + THREADS * e, r = c / (BN / 2), ch = c % (BN / 2);
      *reinterpret_cast<double2*>(b + r * SB + 2 * ch) = make_double2(fr[e].x * wr[e].x, fr[e].y * wr[e].y);
    }
  };

  double acc[WM / 8][WN / 8][2];
#pragma unroll
  for (int i = 0; i < WM / 8; ++i)
#pragma unroll
    for (int j = 0; j < WN / 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // prologue: stages 0 .. STAGES-2
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) {
      load_a(s, s);
      if (KR) {
        fetch_kr(s);
        store_kr(s);
      } else {
        load_b(s, s);
      }
    }
    cp_commit();
  }

  for (int kt = 0; kt < KT; ++kt) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    const int nk = kt + STAGES - 1, ns = nk % STAGES;
    if (nk < KT) {
      load_a(nk, ns);
      if (KR) fetch_kr(nk);
      else load_b(nk, ns);
    }
    cp_commit();

    const int slot = kt % STAGES;
    const double* a_t = as + slot * A_ELEMS;
    const double* b_t = bs + slot * B_ELEMS;
#pragma unroll
    for (int kk = 0; kk < (busy ? BK : 0); kk += 4) {  // consecutive DMMAs write distinct accumulators
      double af[WM / 8], bf[WN / 8];
#pragma unroll
      for (int i = 0; i < WM / 8; ++i) {
        const int m = wm * WM + i * 8 + g, k = kk + t;
        af[i] = TA ? a_t[k * SA + m] : a_t[m * SA + k];
      }
#pragma unroll
      for (int j = 0; j < WN / 8; ++j) bf[j] = b_t[(kk + t) * SB + wn * WN + j * 8 + g];
#pragma unroll
      for (int i = 0; i < WM / 8; ++i)
#pragma unroll
        for (int j = 0; j < WN / 8; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    if (KR && nk < KT) store_kr(ns);  // the slot was last read in iteration kt - 1 (barrier above)
  }
  cp_wait<0>();

  // ---- epilogue: (c0, c1) at (row g, columns 2t, 2t + 1) of each 8 x 8 block
#pragma unroll
  for (int i = 0; i < WM / 8; ++i) {
    const int64_t m = m0 + wm * WM + i * 8 + g;
    if (m >= p.M) continue;
#pragma unroll
    for (int j = 0; j < WN / 8; ++j) {
      const int64_t n = n0 + wn * WN + j * 8 + 2 * t;
      const double v0 = acc[i][j][0] * p.scale, v1 = acc[i][j][1] * p.scale;
      if (TC) {
        double* c0 = p.C + n * p.ldc + m;
        if (n < p.N) *c0 = p.accumulate ? *c0 + v0 : v0;
        if (n + 1 < p.N) c0[p.ldc] = p.accumulate ? c0[p.ldc] + v1 : v1;
      } else {
        double* c = p.C + m * p.ldc + n;
        if (n + 1 < p.N && ((reinterpret_cast<uintptr_t>(c) & 15) == 0)) {
          double2 v = make_double2(v0, v1);
          if (p.accumulate) {
            const double2 o = *reinterpret_cast<const double2*>(c);
            v.x += o.x;
            v.y += o.y;
          }
          *reinterpret_cast<double2*>(c) = v;
        } else {
          if (n < p.N) c[0] = p.accumulate ? c[0] + v0 : v0;
          if (n + 1 < p.N) c[1] = p.accumulate ? c[1] + v1 : v1;
        }
      }
    }
  }
}

template <bool TA, bool TC, bool KR, int WM, int WN, int GM, int GN, bool CPLX = false, int BK = BK_DEF,
          int STAGES = STAGES_DEF, int MINB = 1>
int launch64(const G64& p, cudaStream_t s) {
  constexpr int BM = GM * WM, BN = GN * WN;
  constexpr int SA = TA ? BM + 4 : BK + 4;
  constexpr int A_ELEMS = TA ? BK * SA : BM * SA;
  constexpr int B_ELEMS = BK * (BN + 4);
  const size_t smem = (size_t)STAGES * (A_ELEMS + B_ELEMS) * sizeof(double);
  auto kern = gemm64_kernel<TA, TC, KR, WM, WN, GM, GN, CPLX, BK, STAGES, MINB>;
  allow_smem(kern, smem);
  const int64_t gx = (p.M + BM - 1) / BM, gy = (p.N + BN - 1) / BN;
  if (gy > 65535 || gx > 0x7fffffff) return fail(SK_EUNSUPPORTED, "sk_gemm64: grid too large");
  kern<<<dim3((unsigned)gx, (unsigned)gy), GM * GN * 32, smem, s>>>(p);
  return check_launch("sk_gemm64");
}

template <bool TA, bool TC, bool KR>
int pick_tile(const G64& p, cudaStream_t s) {
  if (KR && p.Bi) return launch64<TA, TC, KR, 32, 32, 4, 2, true, 16, 3, 2>(p, s);  // complex synthesis
  // 128 x 64 tiles of 8 warps, 16-deep stages, two CTAs per SM (one CTA's barrier wait is the other's
  // issue slot, and twice the tiles per wave): 32.6 TFLOP/s at k = 512 and 25.0 on the Khatri-Rao
  // config-5 shape, against 31.3 / 21.5 for 128 x 128 tiles of 16 warps with 32-deep stages
  return launch64<TA, TC, KR, 32, 32, 4, 2, false, 16, 3, 2>(p, s);
}

}  // namespace

// float64 GEMM engine entry used by sk_kr_right_cc / sk_kr_adjoint_cc (kr_cuda.cu).  Returns 1 if the
// shape/alignment is not taken (the caller then runs the CUDA-core kernel), else an SK status.
int gemm64_try(bool ta, const double* A, int64_t rows, int64_t P, int64_t dl, int64_t lda, const double* F,
               int64_t ldf, const double* W, int64_t ldw, int64_t k, double scale, double* Y, int64_t ldy,
               cudaStream_t s, const double* Fi, const double* Wi, int part, int accumulate, bool force) {
  // force: the complex-plane entry points (no CUDA-core alternative); otherwise 1 = not taken
  const auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  const bool cplx = Fi != nullptr;
  if (!force && (rows < 64 || k < 8)) return 1;  // tiny products: the CUDA-core tiles waste less
  if (!al16(A) || (lda & 1) || !al16(F) || (ldf & 1) || (W && (!al16(W) || (ldw & 1))) ||
      (cplx && (!al16(Fi) || !W || !Wi || !al16(Wi))))
    return force ? fail(SK_EINVAL, "sk_kr_*_z: 16-byte aligned planes, even row strides") : 1;
  G64 p{};
  p.A = A;
  p.M = rows;
  p.K = P * dl;
  p.lda = lda;
  p.B = F;
  p.ldb = ldf;
  p.W = W;
  p.ldw = ldw;
  p.dl = dl;
  p.N = k;
  p.scale = scale;
  p.C = Y;
  p.ldc = ldy;
  p.Bi = Fi;
  p.Wi = Wi;
  p.part = part;
  p.accumulate = accumulate;
  const bool kr = W != nullptr;
  if (ta) return kr ? pick_tile<true, true, true>(p, s) : pick_tile<true, true, false>(p, s);
  return kr ? pick_tile<false, false, true>(p, s) : pick_tile<false, false, false>(p, s);
}

}  // namespace skb

// float64 GEMM engine on the planes of a complex Omega (the complex fields of the reference: its
// default Khatri-Rao base is complex_spherical, Gaussian and SRTT have complex variants).
extern "C" int sk_kr_right_z(const double* A, int64_t n, int64_t P, int64_t dl, int64_t lda, const double* Fr,
                             const double* Fi, int64_t ldf, const double* Wr, const double* Wi, int64_t ldw, int64_t k,
                             int part, double scale, int accumulate, double* Y, int64_t ldy, void* stream) {
  using namespace skb;
  if (n < 0 || P < 1 || dl < 1 || k < 1 || ldf < k || lda < P * dl || ldy < k || (Wr && ldw < k) || part < 0 ||
      part > 1 || (!Wr && P != 1) || (!Wr && Fi))
    return fail(SK_EINVAL, "sk_kr_right_z: bad shape");
  if (n == 0) return SK_OK;
  if (!A || !Fr || !Y || (Wr && (!Fi || !Wi))) return fail(SK_EINVAL, "sk_kr_right_z: null pointer");
  return gemm64_try(false, A, n, P, dl, lda, Fr, ldf, Wr, ldw, k, scale, Y, ldy, as_stream(stream), Fi, Wi, part,
                    accumulate ? 1 : 0, true);
}

extern "C" int sk_kr_adjoint_z(const double* B, int64_t m, int64_t P, int64_t dl, int64_t ldb, const double* Fr,
                               const double* Fi, int64_t ldf, const double* Wr, const double* Wi, int64_t ldw,
                               int64_t k, int part, double scale, int accumulate, double* X, int64_t ldx,
                               void* stream) {
  using namespace skb;
  if (m < 0 || P < 1 || dl < 1 || k < 1 || ldf < k || ldb < m || ldx < m || (Wr && ldw < k) || part < 0 ||
      part > 1 || (!Wr && P != 1) || (!Wr && Fi))
    return fail(SK_EINVAL, "sk_kr_adjoint_z: bad shape");
  if (m == 0) return SK_OK;
  if (!B || !Fr || !X || (Wr && (!Fi || !Wi))) return fail(SK_EINVAL, "sk_kr_adjoint_z: null pointer");
  return gemm64_try(true, B, m, P, dl, ldb, Fr, ldf, Wr, ldw, k, scale, X, ldx, as_stream(stream), Fi, Wi, part,
                    accumulate ? 1 : 0, true);
}
