// K2 — sparse-sign adjoint apply  SA = scale * Omega^T * A  (Omega: d x k, exactly zeta +-1 per row).
//
// Replaces `_SparseTM.apply_adjoint` = `self.matrix.conj().T @ b` (src/sketch/sparse.py:68-78),
// which SciPy runs single-threaded through csc_matvecs after upcasting float32 input to a float64
// copy.  Gather formulation, every output element a register accumulator:
//
//   CTA  = a 32-column slice of A (lane = column) x a block of CB = W*CPW output rows c
//          x a contiguous range of row chunks (row split).
//   chunk = R rows of A (x 32 columns) staged in shared memory ([r][32]: conflict-free rows).
//   warp = CPW output rows c; for each bcsc entry (r, sign) of (chunk, c): acc += +-A_s[r][lane].
//   The next chunk is prefetched into registers while the current one is consumed.
//   Row splits write partial sums to a workspace; a second kernel adds them in a fixed order
//   (deterministic, float64 for the float64 path) and applies `scale` / `accumulate`.
#include "common.cuh"

namespace skb {
namespace {

constexpr int kWarps = 16;
constexpr int kCols = 32;

template <typename T>
constexpr int adj_chunk_rows() {
  return sizeof(T) == 4 ? 512 : 256;
}

template <typename T>
struct Vec16;
template <>
struct Vec16<float> {
  using type = float4;
  static constexpr int n = 4;
};
template <>
struct Vec16<double> {
  using type = double2;
  static constexpr int n = 2;
};

template <typename T, int CPW, int R, bool VEC>
__global__ void __launch_bounds__(kWarps * 32, 1)
    sparse_adjoint_kernel(const T* __restrict__ A, int64_t d, int64_t m, int64_t lda,
                          const int32_t* __restrict__ ptr, const uint16_t* __restrict__ ent, int64_t k,
                          int nchunks, int chunks_per_split, T* __restrict__ part, int64_t part_split_stride,
                          int64_t ldp) {
  using V = typename Vec16<T>::type;
  constexpr int NV = Vec16<T>::n;
  constexpr int NT = kWarps * 32;
  constexpr int VEC_PER_ROW = kCols / NV;
  constexpr int VPT = R * VEC_PER_ROW / NT;
  constexpr int SPT = R * kCols / NT;
  constexpr int CB = kWarps * CPW;
  static_assert((R * VEC_PER_ROW) % NT == 0, "tile");

  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* As = reinterpret_cast<T*>(smem_raw);  // [R][32]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t m0 = (int64_t)blockIdx.x * kCols;
  const int64_t cb0 = (int64_t)blockIdx.y * CB;
  const int split = blockIdx.z;
  const int h_begin = split * chunks_per_split;
  const int h_end = min(nchunks, h_begin + chunks_per_split);

  V pre[VEC ? VPT : 1];
  T pres[VEC ? 1 : SPT];
  auto load_chunk = [&](int h) {
    const int64_t r0 = (int64_t)h * R;
    if constexpr (VEC) {
#pragma unroll
      for (int j = 0; j < VPT; ++j) {
        const int q = tid + j * NT;
        const int r = q / VEC_PER_ROW, cv = q % VEC_PER_ROW;
        const int64_t row = r0 + r, col = m0 + cv * NV;
        pre[j] = (row < d && col < m) ? __ldg(reinterpret_cast<const V*>(A + row * lda + col)) : V{};
      }
    } else {
#pragma unroll
      for (int j = 0; j < SPT; ++j) {
        const int q = tid + j * NT;
        const int r = q / kCols, cc = q % kCols;
        const int64_t row = r0 + r, col = m0 + cc;
        pres[j] = (row < d && col < m) ? A[row * lda + col] : T(0);
      }
    }
  };
  auto store_chunk = [&]() {
    if constexpr (VEC) {
#pragma unroll
      for (int j = 0; j < VPT; ++j) {
        const int q = tid + j * NT;
        reinterpret_cast<V*>(As)[q] = pre[j];
      }
    } else {
#pragma unroll
      for (int j = 0; j < SPT; ++j) As[tid + j * NT] = pres[j];
    }
  };

  T acc[CPW];
#pragma unroll
  for (int j = 0; j < CPW; ++j) acc[j] = T(0);

  if (h_begin < h_end) load_chunk(h_begin);
  for (int h = h_begin; h < h_end; ++h) {
    __syncthreads();
    store_chunk();
    __syncthreads();
    if (h + 1 < h_end) load_chunk(h + 1);

    int my_lo = 0, my_hi = 0;
    if (lane < CPW) {
      const int64_t c = cb0 + warp + (int64_t)kWarps * lane;
      if (c < k) {
        my_lo = __ldg(ptr + (int64_t)h * k + c);
        my_hi = __ldg(ptr + (int64_t)h * k + c + 1);
      }
    }
#pragma unroll
    for (int j = 0; j < CPW; ++j) {
      const int lo = __shfl_sync(0xffffffffu, my_lo, j);
      const int hi = __shfl_sync(0xffffffffu, my_hi, j);
      T s0 = T(0), s1 = T(0), s2 = T(0), s3 = T(0);
      for (int base = lo; base < hi; base += 32) {
        const int cnt = min(32, hi - base);
        const uint32_t my_e = (lane < cnt) ? (uint32_t)__ldg(ent + base + lane) : 0u;
        int t = 0;
        for (; t + 4 <= cnt; t += 4) {
          const uint32_t e0 = __shfl_sync(0xffffffffu, my_e, t);
          const uint32_t e1 = __shfl_sync(0xffffffffu, my_e, t + 1);
          const uint32_t e2 = __shfl_sync(0xffffffffu, my_e, t + 2);
          const uint32_t e3 = __shfl_sync(0xffffffffu, my_e, t + 3);
          s0 += flip_if(As[(e0 >> 1) * kCols + lane], e0 & 1u);
          s1 += flip_if(As[(e1 >> 1) * kCols + lane], e1 & 1u);
          s2 += flip_if(As[(e2 >> 1) * kCols + lane], e2 & 1u);
          s3 += flip_if(As[(e3 >> 1) * kCols + lane], e3 & 1u);
        }
        for (; t < cnt; ++t) {
          const uint32_t e0 = __shfl_sync(0xffffffffu, my_e, t);
          s0 += flip_if(As[(e0 >> 1) * kCols + lane], e0 & 1u);
        }
      }
      acc[j] += (s0 + s1) + (s2 + s3);
    }
  }

  // partial[split][c][m]: for fixed c the 32 lanes write 32 consecutive columns (coalesced).
  T* p = part + (int64_t)split * part_split_stride;
  const int64_t col = m0 + lane;
  if (col < m) {
#pragma unroll
    for (int j = 0; j < CPW; ++j) {
      const int64_t c = cb0 + warp + (int64_t)kWarps * j;
      if (c < k) p[c * ldp + col] = acc[j];
    }
  }
}

// SA[c][col] (+)= scale * sum_s part[s][c][col], summed in split order.
template <typename T>
__global__ void adjoint_reduce(const T* __restrict__ part, int nsplit, int64_t split_stride, int64_t ldp,
                               int64_t k, int64_t m, T scale, T* __restrict__ SA, int64_t ldsa, int accumulate) {
  const int64_t total = k * m;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = idx / m, col = idx % m;
    double s = 0.0;
    for (int q = 0; q < nsplit; ++q) s += (double)part[q * split_stride + c * ldp + col];
    T v = (T)(s * (double)scale);
    if (accumulate) v += SA[c * ldsa + col];
    SA[c * ldsa + col] = v;
  }
}

struct Plan {
  int cpw, nchunks, nsplit, chunks_per_split, grid_x, grid_y;
};

template <typename T>
Plan make_plan(int64_t d, int64_t m, int64_t k) {
  constexpr int R = adj_chunk_rows<T>();
  Plan p{};
  const int64_t need = (k + kWarps - 1) / kWarps;
  p.cpw = need <= 4 ? 4 : (need <= 8 ? 8 : 16);
  const int64_t cb = (int64_t)kWarps * p.cpw;
  p.nchunks = (int)((d + R - 1) / R);
  p.grid_x = (int)((m + kCols - 1) / kCols);
  p.grid_y = (int)((k + cb - 1) / cb);
  const int64_t tiles = (int64_t)p.grid_x * p.grid_y;
  const int64_t target = 2 * (int64_t)sm_count();
  int64_t nsplit = (target + tiles - 1) / tiles;
  if (nsplit > p.nchunks) nsplit = p.nchunks;
  if (nsplit < 1) nsplit = 1;
  p.chunks_per_split = (int)((p.nchunks + nsplit - 1) / nsplit);
  p.nsplit = (int)((p.nchunks + p.chunks_per_split - 1) / p.chunks_per_split);
  return p;
}

template <typename T, int CPW, bool VEC>
int launch_t(const Plan& pl, const T* A, int64_t d, int64_t m, int64_t lda, const int32_t* ptr,
             const uint16_t* ent, int64_t k, T* part, cudaStream_t s) {
  constexpr int R = adj_chunk_rows<T>();
  const size_t smem = (size_t)R * kCols * sizeof(T);
  auto kern = sparse_adjoint_kernel<T, CPW, R, VEC>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid(pl.grid_x, pl.grid_y, pl.nsplit);
  kern<<<grid, kWarps * 32, smem, s>>>(A, d, m, lda, ptr, ent, k, pl.nchunks, pl.chunks_per_split, part,
                                       k * m, m);
  return check_launch("sk_sparse_adjoint");
}

template <typename T>
int run(const void* A_, int64_t d, int64_t m, int64_t lda, const int32_t* ptr, const uint16_t* ent, int64_t k,
        double scale, void* SA_, int64_t ldsa, int accumulate, void* ws, size_t ws_bytes, cudaStream_t s) {
  const T* A = static_cast<const T*>(A_);
  T* SA = static_cast<T*>(SA_);
  const Plan pl = make_plan<T>(d, m, k);
  const size_t need = (size_t)pl.nsplit * k * m * sizeof(T);
  if (ws_bytes < need || ws == nullptr) return fail(SK_EINVAL, "sk_sparse_adjoint: workspace too small");
  T* part = static_cast<T*>(ws);
  constexpr int NV = 16 / sizeof(T);
  const bool vec = ((reinterpret_cast<uintptr_t>(A) & 15) == 0) && (lda % NV == 0) && (m % NV == 0);
  int st;
#define SKB_ADJ(CPW)                                                                   \
  st = vec ? launch_t<T, CPW, true>(pl, A, d, m, lda, ptr, ent, k, part, s)             \
           : launch_t<T, CPW, false>(pl, A, d, m, lda, ptr, ent, k, part, s)
  if (pl.cpw == 4) {
    SKB_ADJ(4);
  } else if (pl.cpw == 8) {
    SKB_ADJ(8);
  } else {
    SKB_ADJ(16);
  }
#undef SKB_ADJ
  if (st != SK_OK) return st;
  const int64_t total = k * m;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 8 * (int64_t)sm_count()) blocks = 8 * (int64_t)sm_count();
  adjoint_reduce<T><<<(unsigned)blocks, 256, 0, s>>>(part, pl.nsplit, k * m, m, k, m, (T)scale, SA, ldsa, accumulate);
  return check_launch("sk_sparse_adjoint(reduce)");
}

}  // namespace
}  // namespace skb

extern "C" int sk_sparse_adjoint_chunk_rows(int dtype, int64_t d, int64_t k) {
  (void)d;
  (void)k;
  if (dtype == SK_F32) return skb::adj_chunk_rows<float>();
  if (dtype == SK_F64) return skb::adj_chunk_rows<double>();
  return skb::fail(SK_EINVAL, "sk_sparse_adjoint_chunk_rows: bad dtype");
}

extern "C" size_t sk_sparse_adjoint_workspace_bytes(int dtype, int64_t d, int64_t m, int64_t k) {
  if (d < 1 || m < 1 || k < 1) return 0;
  if (dtype == SK_F32) return (size_t)skb::make_plan<float>(d, m, k).nsplit * k * m * sizeof(float);
  if (dtype == SK_F64) return (size_t)skb::make_plan<double>(d, m, k).nsplit * k * m * sizeof(double);
  return 0;
}

extern "C" int sk_sparse_adjoint(int dtype, const void* A, int64_t d, int64_t m, int64_t lda, const int32_t* ptr,
                                 const uint16_t* ent, int32_t chunk_rows, int64_t k, double scale, void* SA,
                                 int64_t ldsa, int accumulate, void* ws, size_t ws_bytes, void* stream) {
  using namespace skb;
  if (d < 1 || m < 0 || k < 1 || lda < m || ldsa < m) return fail(SK_EINVAL, "sk_sparse_adjoint: bad shape/leading dimension");
  if (dtype != SK_F32 && dtype != SK_F64) return fail(SK_EINVAL, "sk_sparse_adjoint: bad dtype");
  if (chunk_rows != sk_sparse_adjoint_chunk_rows(dtype, d, k))
    return fail(SK_EINVAL, "sk_sparse_adjoint: chunk_rows does not match sk_sparse_adjoint_chunk_rows");
  if (m == 0) return SK_OK;
  if (!A || !SA || !ptr) return fail(SK_EINVAL, "sk_sparse_adjoint: null pointer");
  cudaStream_t s = as_stream(stream);
  return dtype == SK_F32 ? run<float>(A, d, m, lda, ptr, ent, k, scale, SA, ldsa, accumulate, ws, ws_bytes, s)
                         : run<double>(A, d, m, lda, ptr, ent, k, scale, SA, ldsa, accumulate, ws, ws_bytes, s);
}
