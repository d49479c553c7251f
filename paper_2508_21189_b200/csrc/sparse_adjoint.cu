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
#include <cuda.h>

#include "common.cuh"
#include "sm100.cuh"

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
  // the (row, column) position advances by the grid stride: no 64-bit divide / modulo per element
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i0 >= total) return;
  int64_t c = i0 / m, col = i0 - c * m;
  const int64_t dc = stride / m, dcol = stride - dc * m;
  for (int64_t idx = i0; idx < total; idx += stride) {
    double s = 0.0;
    for (int q = 0; q < nsplit; ++q) s += (double)part[q * split_stride + c * ldp + col];
    T v = (T)(s * (double)scale);
    if (accumulate) v += SA[c * ldsa + col];
    SA[c * ldsa + col] = v;
    c += dc;
    col += dcol;
    if (col >= m) {
      col -= m;
      ++c;
    }
  }
}


// ---------------------------------------------------------------------------------------------
// v2 (float32): one CTA = a 32-column slice x a group of 1024 output rows c x a piece of the row
// chunks.  A chunks (512 rows x 32 columns = 64 KB) arrive by TMA, together with the chunk's bcsc
// pointer segment and entry segment (bulk copies), into a 2-stage ring; one producer thread runs
// ahead.  Warp w owns the 64 output rows cg*1024 + 64w + j: per (chunk, c) it walks the entry list
// (uniform shared loads), and every lane adds +-A_s[row][lane] into its register accumulator.
// Lanes read one 128-byte row per entry: conflict free.  Pieces write partials; an ordered float64
// reduction forms SA.
// ---------------------------------------------------------------------------------------------
constexpr int V2_R = 512;          // rows per chunk (== adj_chunk_rows<float>)
constexpr int V2_CW = 64;          // output rows per warp
constexpr int V2_CG = kWarps * V2_CW;  // output rows per CTA (1024)

struct V2Params {
  int64_t d, m, k;
  int nchunks, nslices, ngroups, npieces, chunks_per_piece;
  const int32_t* ptr;        // padded by >= 4 entries
  const uint16_t* ent;
  const int32_t* seg;        // [nchunks][ngroups][2]: aligned entry start (multiple of 8), entry count (mult of 8)
  int ent_cap;               // max entries (multiple of 8) of any (chunk, group) segment
  float* part;               // [npieces][k][m]
};

__global__ void __launch_bounds__((kWarps + 1) * 32, 1)
    sparse_adjoint_v2(const __grid_constant__ CUtensorMap tm_a, const V2Params p) {
  using namespace sm100;
  extern __shared__ uint8_t smem_dyn[];
  // keep the pointer derived from the __shared__ array (integer offset) so accesses stay LDS/STS
  uint8_t* smem = smem_dyn + ((1024u - (sm100::smem_u32(smem_dyn) & 1023u)) & 1023u);
  constexpr uint32_t A_BYTES = V2_R * 32 * 4;
  constexpr uint32_t PTR_BYTES = (V2_CG + 4) * 4;  // 1028 ints (>= 1025, multiple of 16 bytes)
  const uint32_t ent_bytes = (uint32_t)p.ent_cap * 2;
  const uint32_t stage_bytes = (A_BYTES + PTR_BYTES + ent_bytes + 1023) & ~1023u;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + 2 * stage_bytes);
  uint64_t* empty = full + 2;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int role = blockIdx.x % (p.nslices * p.ngroups);
  const int piece = blockIdx.x / (p.nslices * p.ngroups);
  const int slice = role % p.nslices, grp = role / p.nslices;
  const int h0 = piece * p.chunks_per_piece;
  const int h1 = min(p.nchunks, h0 + p.chunks_per_piece);
  const int64_t cb = (int64_t)grp * V2_CG;

  if (tid == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWarps);
    }
    fence_mbar_init();
    tma_prefetch_desc(&tm_a);
  }
  __syncthreads();

  if (warp == kWarps) {
    // producer warp (one thread): runs ahead by up to 2 chunks
    if (lane != 0) return;
    int s = 0;
    uint32_t ph = 0;
    for (int h = h0; h < h1; ++h) {
      mbar_wait(&empty[s], ph ^ 1);
      uint8_t* st = smem + (size_t)s * stage_bytes;
      const int32_t e0 = __ldg(p.seg + ((int64_t)h * p.ngroups + grp) * 2);
      const int32_t en = __ldg(p.seg + ((int64_t)h * p.ngroups + grp) * 2 + 1);
      mbar_arrive_expect_tx(&full[s], A_BYTES + PTR_BYTES + (uint32_t)en * 2);
      tma_load_2d(st, &tm_a, &full[s], slice * 32, h * V2_R);
      tma_load_2d(st + A_BYTES / 2, &tm_a, &full[s], slice * 32, h * V2_R + V2_R / 2);
      const int32_t* psrc = p.ptr + (int64_t)h * p.k + cb;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(st + A_BYTES)),
                   "l"(psrc), "r"(PTR_BYTES), "r"(smem_u32(&full[s]))
                   : "memory");
      if (en > 0) {
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(st + A_BYTES + PTR_BYTES)),
                     "l"(p.ent + e0), "r"((uint32_t)en * 2), "r"(smem_u32(&full[s]))
                     : "memory");
      }
      if (++s == 2) { s = 0; ph ^= 1; }
    }
    return;
  }

  float acc[V2_CW];
#pragma unroll
  for (int j = 0; j < V2_CW; ++j) acc[j] = 0.f;
  int s = 0;
  uint32_t ph = 0;
  const int cw0 = warp * V2_CW;  // this warp's first output row within the group
  for (int h = h0; h < h1; ++h) {
    mbar_wait(&full[s], ph);
    const uint8_t* st = smem + (size_t)s * stage_bytes;
    const float* As = reinterpret_cast<const float*>(st);
    const int32_t* ps = reinterpret_cast<const int32_t*>(st + A_BYTES);
    const uint16_t* es = reinterpret_cast<const uint16_t*>(st + A_BYTES + PTR_BYTES);
    const int32_t e0 = __ldg(p.seg + ((int64_t)h * p.ngroups + grp) * 2);
    if (cb + cw0 < p.k) {
      const int nc = (int)min((int64_t)V2_CW, p.k - cb - cw0);
      int e = ps[cw0] - e0;
      // byte address of A_s[0][lane]; an entry u = (row << 1) | neg maps to row * 128 = (u << 6) & 0xff80
      const uint32_t abase = smem_u32(As) + lane * 4;
      const uint32_t ebase = smem_u32(es);
#pragma unroll
      for (int j = 0; j < V2_CW; ++j) {
        const int hi = (j < nc) ? ps[cw0 + j + 1] - e0 : e;
        float a0 = 0.f, a1 = 0.f;
        for (; e + 2 <= hi; e += 2) {  // pairs: two independent row loads in flight
          uint32_t u0, u1;
          if (e & 1) {  // warp-uniform: odd start, two 16-bit loads
            asm volatile("ld.shared.u16 %0, [%1];" : "=r"(u0) : "r"(ebase + 2u * e));
            asm volatile("ld.shared.u16 %0, [%1];" : "=r"(u1) : "r"(ebase + 2u * e + 2u));
          } else {      // even start: one aligned 32-bit load carries both entries
            uint32_t u01;
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(u01) : "r"(ebase + 2u * e));
            u0 = u01 & 0xffffu;
            u1 = u01 >> 16;
          }
          float v0, v1;
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v0) : "r"(abase + ((u0 << 6) & 0xff80u)));
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v1) : "r"(abase + ((u1 << 6) & 0xff80u)));
          a0 += flip_if(v0, u0 & 1u);
          a1 += flip_if(v1, u1 & 1u);
        }
        if (e < hi) {
          uint32_t u0;
          asm volatile("ld.shared.u16 %0, [%1];" : "=r"(u0) : "r"(ebase + 2u * e));
          float v0;
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v0) : "r"(abase + ((u0 << 6) & 0xff80u)));
          a0 += flip_if(v0, u0 & 1u);
          ++e;
        }
        acc[j] += a0 + a1;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == 2) { s = 0; ph ^= 1; }
  }
  const int64_t col = (int64_t)slice * 32 + lane;
  if (col < p.m) {
    float* out = p.part + (int64_t)piece * p.k * p.m;
#pragma unroll
    for (int j = 0; j < V2_CW; ++j) {
      const int64_t c = cb + cw0 + j;
      if (c < p.k) out[c * p.m + col] = acc[j];
    }
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
  allow_smem(kern, smem);
  dim3 grid(pl.grid_x, pl.grid_y, pl.nsplit);
  kern<<<grid, kWarps * 32, smem, s>>>(A, d, m, lda, ptr, ent, k, pl.nchunks, pl.chunks_per_split, part,
                                       k * m, m);
  return check_launch("sk_sparse_adjoint");
}

typedef CUresult (*EncodeTiledFnA)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFnA encode_fn_a() {
  // resolved once (thread-safe static initialisation: trials may run on a host thread pool)
  static const EncodeTiledFnA fn = [] {
    void* q = nullptr;
    cudaDriverEntryPointQueryResult r;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &q, cudaEnableDefault, &r) == cudaSuccess &&
        r == cudaDriverEntryPointSuccess)
      return reinterpret_cast<EncodeTiledFnA>(q);
    return static_cast<EncodeTiledFnA>(nullptr);
  }();
  ensure_context();
  return fn;
}

struct V2Plan {
  int nslices, ngroups, npieces, chunks_per_piece, nchunks;
  size_t smem, ws_bytes;
};

V2Plan v2_plan(int64_t d, int64_t m, int64_t k, int ent_cap) {
  V2Plan pl{};
  pl.nchunks = (int)((d + V2_R - 1) / V2_R);
  pl.nslices = (int)((m + 31) / 32);
  pl.ngroups = (int)((k + V2_CG - 1) / V2_CG);
  const int roles = pl.nslices * pl.ngroups;
  int pieces = (2 * sm_count() + roles - 1) / roles;
  if (pieces > pl.nchunks) pieces = pl.nchunks;
  if (pieces < 1) pieces = 1;
  pl.chunks_per_piece = (pl.nchunks + pieces - 1) / pieces;
  pl.npieces = (pl.nchunks + pl.chunks_per_piece - 1) / pl.chunks_per_piece;
  const size_t stage = ((size_t)V2_R * 32 * 4 + (V2_CG + 4) * 4 + (size_t)ent_cap * 2 + 1023) & ~(size_t)1023;
  pl.smem = 1024 + 2 * stage + 64;
  pl.ws_bytes = (size_t)pl.npieces * k * m * sizeof(float);
  return pl;
}

bool v2_ok(int64_t d, int64_t m, int64_t k, const float* A, int64_t lda, const int32_t* seg, int ent_cap) {
  if (!seg || ent_cap < 0 || (ent_cap & 7)) return false;
  if ((reinterpret_cast<uintptr_t>(A) & 15) || (lda & 3) || m < 16) return false;
  if (k % 4) return false;  // 16-byte aligned pointer segments
  return v2_plan(d, m, k, ent_cap).smem <= 227 * 1024;
}

int run_v2(const float* A, int64_t d, int64_t m, int64_t lda, const int32_t* ptr, const uint16_t* ent,
           const int32_t* seg, int ent_cap, int64_t k, double scale, float* SA, int64_t ldsa, int accumulate, void* ws,
           size_t ws_bytes, cudaStream_t s) {
  const V2Plan pl = v2_plan(d, m, k, ent_cap);
  if (ws_bytes < pl.ws_bytes || !ws) return fail(SK_EINVAL, "sk_sparse_adjoint: workspace too small");
  EncodeTiledFnA fn = encode_fn_a();
  if (!fn) return fail(SK_ECUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)m, (cuuint64_t)d};
  cuuint64_t strides[1] = {(cuuint64_t)lda * 4};
  cuuint32_t box[2] = {32, (cuuint32_t)(V2_R / 2)};
  cuuint32_t estr[2] = {1, 1};
  if (fn(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(A), dims, strides, box, estr,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return fail(SK_EINVAL, "sk_sparse_adjoint: cannot describe A for TMA");
  V2Params p{};
  p.d = d;
  p.m = m;
  p.k = k;
  p.nchunks = pl.nchunks;
  p.nslices = pl.nslices;
  p.ngroups = pl.ngroups;
  p.npieces = pl.npieces;
  p.chunks_per_piece = pl.chunks_per_piece;
  p.ptr = ptr;
  p.ent = ent;
  p.seg = seg;
  p.ent_cap = ent_cap;
  p.part = static_cast<float*>(ws);
  allow_smem(sparse_adjoint_v2, pl.smem);
  const int grid = pl.nslices * pl.ngroups * pl.npieces;
  sparse_adjoint_v2<<<grid, (kWarps + 1) * 32, pl.smem, s>>>(tm, p);
  int st = check_launch("sk_sparse_adjoint(v2)");
  if (st != SK_OK) return st;
  const int64_t total = k * m;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 8 * (int64_t)sm_count()) blocks = 8 * (int64_t)sm_count();
  adjoint_reduce<float><<<(unsigned)blocks, 256, 0, s>>>(p.part, pl.npieces, k * m, m, k, m, (float)scale, SA, ldsa,
                                                         accumulate);
  return check_launch("sk_sparse_adjoint(reduce)");
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

int adjoint_reduce_f32(const float* part, int npieces, int64_t k, int64_t m, double scale, float* SA, int64_t ldsa,
                       int accumulate, cudaStream_t s) {
  const int64_t total = k * m;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 8 * (int64_t)sm_count()) blocks = 8 * (int64_t)sm_count();
  adjoint_reduce<float><<<(unsigned)blocks, 256, 0, s>>>(part, npieces, k * m, m, k, m, (float)scale, SA, ldsa,
                                                         accumulate);
  return check_launch("sk_sparse_adjoint(reduce)");
}

int adjoint_reduce_f64(const double* part, int npieces, int64_t k, int64_t m, double scale, double* SA, int64_t ldsa,
                       int accumulate, cudaStream_t s) {
  const int64_t total = k * m;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 8 * (int64_t)sm_count()) blocks = 8 * (int64_t)sm_count();
  adjoint_reduce<double><<<(unsigned)blocks, 256, 0, s>>>(part, npieces, k * m, m, k, m, scale, SA, ldsa, accumulate);
  return check_launch("sk_sparse_adjoint(reduce)");
}

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
  if (dtype == SK_F32) {
    const size_t a = (size_t)skb::make_plan<float>(d, m, k).nsplit * k * m * sizeof(float);
    const size_t b = skb::v2_plan(d, m, k, 0).ws_bytes;
    return a > b ? a : b;
  }
  if (dtype == SK_F64) return (size_t)skb::make_plan<double>(d, m, k).nsplit * k * m * sizeof(double);
  return 0;
}

extern "C" int sk_sparse_adjoint(int dtype, const void* A, int64_t d, int64_t m, int64_t lda, const int32_t* ptr,
                                 const uint16_t* ent, int32_t chunk_rows, const int32_t* seg, int32_t ent_cap,
                                 int64_t k, double scale, void* SA, int64_t ldsa, int accumulate, void* ws,
                                 size_t ws_bytes, void* stream) {
  using namespace skb;
  if (d < 1 || m < 0 || k < 1 || lda < m || ldsa < m) return fail(SK_EINVAL, "sk_sparse_adjoint: bad shape/leading dimension");
  if (dtype != SK_F32 && dtype != SK_F64) return fail(SK_EINVAL, "sk_sparse_adjoint: bad dtype");
  if (chunk_rows != sk_sparse_adjoint_chunk_rows(dtype, d, k))
    return fail(SK_EINVAL, "sk_sparse_adjoint: chunk_rows does not match sk_sparse_adjoint_chunk_rows");
  if (m == 0) return SK_OK;
  if (!A || !SA || !ptr) return fail(SK_EINVAL, "sk_sparse_adjoint: null pointer");
  cudaStream_t s = as_stream(stream);
  if (dtype == SK_F32 && v2_ok(d, m, k, static_cast<const float*>(A), lda, seg, ent_cap))
    return run_v2(static_cast<const float*>(A), d, m, lda, ptr, ent, seg, ent_cap, k, scale, static_cast<float*>(SA),
                  ldsa, accumulate, ws, ws_bytes, s);
  return dtype == SK_F32 ? run<float>(A, d, m, lda, ptr, ent, k, scale, SA, ldsa, accumulate, ws, ws_bytes, s)
                         : run<double>(A, d, m, lda, ptr, ent, k, scale, SA, ldsa, accumulate, ws, ws_bytes, s);
}
