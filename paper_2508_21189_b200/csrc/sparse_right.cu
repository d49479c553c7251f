// K1 — sparse-sign right apply  Y = scale * A * Omega  (Omega: exactly zeta +-1 per row).
//
// Replaces the reference `_SparseTM.apply_right` (src/sketch/sparse.py:63-66), which SciPy runs
// as csc_matvecs over Omega^T after copying A transposed.  Here A is streamed from HBM exactly
// once, row-tile by row-tile, and every output element is a register accumulator:
//
//   CTA   = 32 rows of A (one per lane) x a block of CB = W*CPW output columns.
//   warp  = CPW consecutive output columns c (c = cb0 + warp*CPW + j); lane = row.
//   chunk = R consecutive columns of A (rows of Omega) staged in shared memory, XOR-swizzled so
//           that (a) 16-byte vector stores of a row segment and (b) the gather pattern "32 lanes
//           = 32 rows, same column r" are both bank-conflict free.
//   Omega = bcsc lists: for chunk h and column c, uint16 entries (local_r << 1) | neg.
//   The next chunk is prefetched into registers (LDG.128, L1 no-allocate) while the current
//   one is consumed, so HBM reads overlap the shared-memory gathers.
//
// Bytes per launch (algorithmic): n*d*sizeof(T) read + n*k*sizeof(T) written.
#include <stdlib.h>

#include <type_traits>

#include "common.cuh"

namespace skb {
namespace {

constexpr int kRowsPerTile = 32;

template <typename T>
struct VecOf;
template <>
struct VecOf<float> {
  using type = float4;
  static constexpr int n = 4;
};
template <>
struct VecOf<double> {
  using type = double2;
  static constexpr int n = 2;
};

__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}

// Permute a vector so that component q lands at q ^ key (key < n): XOR swizzle inside a 16 B block.
__device__ __forceinline__ float4 xor_perm(float4 v, int key) {
  if (key & 1) { float t = v.x; v.x = v.y; v.y = t; t = v.z; v.z = v.w; v.w = t; }
  if (key & 2) { float t = v.x; v.x = v.z; v.z = t; t = v.y; v.y = v.w; v.w = t; }
  return v;
}
__device__ __forceinline__ double2 xor_perm(double2 v, int key) {
  if (key & 1) { double t = v.x; v.x = v.y; v.y = t; }
  return v;
}

template <typename T>
__device__ __forceinline__ T lds_t(uint32_t addr);
template <>
__device__ __forceinline__ float lds_t<float>(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
template <>
__device__ __forceinline__ double lds_t<double>(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}

template <typename T, int W, int CPW, int R, bool VEC, bool OMS>
__global__ void __launch_bounds__(W * 32, 1)
    sparse_right_kernel(const T* __restrict__ A, int64_t n, int64_t d, int64_t lda,
                        const int32_t* __restrict__ ptr, const uint16_t* __restrict__ ent,
                        int64_t k, int nchunks, int nnz, uint32_t omega_off, T scale, T* __restrict__ Y,
                        int64_t ldy) {
  using V4 = typename VecOf<T>::type;
  constexpr int NV = VecOf<T>::n;               // elements per 16 B vector
  constexpr int NT = W * 32;                    // threads
  constexpr int VEC_PER_ROW = R / NV;
  constexpr int VPT = kRowsPerTile * VEC_PER_ROW / NT;  // prefetch vectors per thread
  constexpr int SPT = kRowsPerTile * R / NT;            // scalar elements per thread (!VEC)
  constexpr int CB = W * CPW;
  static_assert(R % 32 == 0 && (kRowsPerTile * VEC_PER_ROW) % NT == 0, "tile shape");

  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* As = reinterpret_cast<T*>(smem_raw);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // 1-D grid, column blocks fastest: the CTAs that share a row tile run back to back, so the
  // tile is read from DRAM once and from L2 by the others
  const int ncb = (int)((k + CB - 1) / CB);
  const int64_t row0 = (int64_t)(blockIdx.x / ncb) * kRowsPerTile;
  const int64_t cb0 = (int64_t)(blockIdx.x % ncb) * CB;

  V4 pre[VEC ? VPT : 1];
  T pres[VEC ? 1 : SPT];

  // VEC: vector j of a thread is row tid / VEC_PER_ROW + j * (NT / VEC_PER_ROW), column (tid % VEC_PER_ROW) * NV
  // of the chunk: one base pointer and a row-validity mask per thread, 64-bit adds per chunk.
  static_assert(!VEC || NT % VEC_PER_ROW == 0, "prefetch mapping");
  constexpr int ROWS_PER_PASS = VEC ? NT / VEC_PER_ROW : 1;
  const int64_t vrow0 = row0 + tid / VEC_PER_ROW;
  const int64_t vcol = (int64_t)(tid % VEC_PER_ROW) * NV;
  const T* vbase = A + vrow0 * lda + vcol;
  uint32_t vrows_ok = 0;
#pragma unroll
  for (int j = 0; j < (VEC ? VPT : 1); ++j)
    if (vrow0 + (int64_t)j * ROWS_PER_PASS < n) vrows_ok |= 1u << j;
  auto load_chunk = [&](int h) {
    const int64_t c0 = (int64_t)h * R;
    if constexpr (VEC) {
      const bool col_ok = vcol + c0 < d;
      const T* p = vbase + c0;
#pragma unroll
      for (int j = 0; j < VPT; ++j) {
        if (col_ok && ((vrows_ok >> j) & 1u)) {
          pre[j] = ld_stream(reinterpret_cast<const V4*>(p + (int64_t)j * ROWS_PER_PASS * lda));
        } else {
          pre[j] = V4{};
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < SPT; ++j) {
        const int q = tid + j * NT;
        const int i = q / R, cc = q % R;
        const int64_t row = row0 + i, col = c0 + cc;
        pres[j] = (row < n && col < d) ? A[row * lda + col] : T(0);
      }
    }
  };
  // every prefetch vector of a thread lies in rows of the same residue mod NV (NT is a multiple of
  // NV * VEC_PER_ROW), so the in-vector permutation is one warp-uniform choice per chunk
  static_assert(!VEC || (NT / VEC_PER_ROW) % NV == 0, "row residue per thread");
  auto store_vecs = [&](T* dst, auto key_c) {
    constexpr int KEY = decltype(key_c)::value;
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
      const int q = tid + j * NT;
      const int i = q / VEC_PER_ROW, cv = q % VEC_PER_ROW;
      const int blk = (cv * NV) ^ (i & 31 & ~(NV - 1));
      *reinterpret_cast<V4*>(dst + i * R + blk) = xor_perm(pre[j], KEY);
    }
  };
  auto store_chunk = [&](T* dst) {
    if constexpr (VEC) {
      const int key = (tid / VEC_PER_ROW) & (NV - 1);
      if (key == 0) store_vecs(dst, std::integral_constant<int, 0>{});
      else if (key == 1) store_vecs(dst, std::integral_constant<int, 1>{});
      else if constexpr (NV == 4) {
        if (key == 2) store_vecs(dst, std::integral_constant<int, 2>{});
        else store_vecs(dst, std::integral_constant<int, 3>{});
      }
    } else {
#pragma unroll
      for (int j = 0; j < SPT; ++j) {
        const int q = tid + j * NT;
        const int i = q / R, cc = q % R;
        dst[i * R + (cc ^ (i & 31))] = pres[j];
      }
    }
  };

  T acc[CPW];
#pragma unroll
  for (int j = 0; j < CPW; ++j) acc[j] = T(0);

  // OMS: the whole bcsc encoding of Omega sits in shared memory (small Omega, e.g. config 1:
  // 48 KB); entry and pointer reads are then uniform shared loads (broadcast, no L1 traffic).
  const int nptr = nchunks * (int)k + 1;
  int32_t* ptr_s = reinterpret_cast<int32_t*>(smem_raw + omega_off);
  uint16_t* ent_s = reinterpret_cast<uint16_t*>(ptr_s + ((nptr + 3) & ~3));
  // OMS entries are re-coded while staged: (local_r * sizeof(T)) | (neg << 15), so the swizzled
  // byte address inside the tile is one LOP3, (u & RMASK) ^ LXOR (rows are R * sizeof(T) = 2 KB apart
  // and the swizzle XORs the lane into the low 5 bits of local_r).
  constexpr uint32_t SH = sizeof(T) == 8 ? 3u : 2u;
  constexpr uint32_t RMASK = (uint32_t)(R - 1) << SH;
  static_assert(R * sizeof(T) == 2048, "row stride of the staged tile");
  if constexpr (OMS) {
    for (int i = tid; i < nptr; i += NT) ptr_s[i] = __ldg(ptr + i);
    for (int i = tid; i < nnz; i += NT) {
      const uint32_t e = __ldg(ent + i);
      ent_s[i] = (uint16_t)(((e >> 1) << SH) | ((e & 1u) << 15));
    }
  }
  const uint32_t tile_s0 = (uint32_t)__cvta_generic_to_shared(smem_raw);
  const uint32_t lxor = ((uint32_t)lane << 11) | ((uint32_t)lane << SH);
  auto P = [&](int64_t i) -> int { return OMS ? ptr_s[i] : __ldg(ptr + i); };
  auto E = [&](int i) -> uint32_t { return OMS ? (uint32_t)ent_s[i] : (uint32_t)__ldg(ent + i); };

  // two staged tiles: chunk h lives in As + (h & 1) * TILE; the next chunk is stored into the other
  // tile right after this one is consumed, so one barrier per chunk separates the two
  constexpr int TILE = kRowsPerTile * R;
  load_chunk(0);
  store_chunk(As);
  if (nchunks > 1) load_chunk(1);
  __syncthreads();
  for (int h = 0; h < nchunks; ++h) {
    T* const cur = As + (h & 1) * TILE;
    const T* my_row = cur + lane * R;
    const uint32_t tile_s = tile_s0 + (uint32_t)((h & 1) * TILE * sizeof(T));

    // warp w owns the CPW consecutive columns cb0 + w * CPW + j: their CPW + 1 offsets are adjacent
    const int64_t cw = cb0 + (int64_t)warp * CPW;
    int bounds[CPW + 1];
#pragma unroll
    for (int j = 0; j <= CPW; ++j) bounds[j] = (cw + j <= k) ? P((int64_t)h * k + cw + j) : 0;
#pragma unroll
    for (int j = 0; j < CPW; ++j) {
      int lo = 0, hi = 0;
      if (cw + j < k) {
        lo = bounds[j];
        hi = bounds[j + 1];
      }
      T s0 = T(0), s1 = T(0);
      int e = lo;
      if constexpr (OMS) {
        for (; e + 2 <= hi; e += 2) {
          const uint32_t u0 = ent_s[e], u1 = ent_s[e + 1];
          s0 += flip_if(lds_t<T>(tile_s + ((u0 & RMASK) ^ lxor)), u0 >> 15);
          s1 += flip_if(lds_t<T>(tile_s + ((u1 & RMASK) ^ lxor)), u1 >> 15);
        }
        if (e < hi) {
          const uint32_t u0 = ent_s[e];
          s0 += flip_if(lds_t<T>(tile_s + ((u0 & RMASK) ^ lxor)), u0 >> 15);
        }
      } else {
        for (; e + 2 <= hi; e += 2) {
          const uint32_t e0 = E(e), e1 = E(e + 1);
          s0 += flip_if(my_row[(e0 >> 1) ^ lane], e0 & 1u);
          s1 += flip_if(my_row[(e1 >> 1) ^ lane], e1 & 1u);
        }
        if (e < hi) {
          const uint32_t e0 = E(e);
          s0 += flip_if(my_row[(e0 >> 1) ^ lane], e0 & 1u);
        }
      }
      acc[j] += s0 + s1;
    }
    if (h + 1 < nchunks) {
      store_chunk(As + ((h + 1) & 1) * TILE);
      if (h + 2 < nchunks) load_chunk(h + 2);
    }
    __syncthreads();
  }

  // Epilogue: stage the 32 x CB tile through shared memory, then coalesced row stores.
  __syncthreads();
  constexpr int YS = CB + 1;
  T* Ys = As;
#pragma unroll
  for (int j = 0; j < CPW; ++j) Ys[lane * YS + warp * CPW + j] = acc[j] * scale;
  __syncthreads();
  for (int idx = tid; idx < kRowsPerTile * CB; idx += NT) {
    const int i = idx / CB, cl = idx % CB;
    const int64_t row = row0 + i, c = cb0 + cl;
    if (row < n && c < k) Y[row * ldy + c] = Ys[i * YS + cl];
  }
}

// ---------------------------------------------------------------------------------------------
// Persistent form (used whenever the CTA's share of Omega fits in shared memory, e.g. config 1).
// One CTA per SM, fixed column block cb = blockIdx.x % ncb, row tiles blockIdx.x / ncb + i * (grid /
// ncb). Omega's entries for the column block are staged once per CTA as 32-bit words
// (local_r << SH) | (neg << 31), each column's list starting at an even slot so pairs come in one
// 8-byte broadcast load, with per-(chunk, column) start offsets (bit 0 = odd count). The
// double-buffered chunk stream runs across tile boundaries; a finished tile's accumulators go
// straight from registers to Y (lane = row, CPW consecutive columns).
template <typename T>
__device__ __forceinline__ T xor_sign(T v, uint32_t u);
template <>
__device__ __forceinline__ float xor_sign<float>(float v, uint32_t u) {
  return __uint_as_float(__float_as_uint(v) ^ (u & 0x80000000u));
}
template <>
__device__ __forceinline__ double xor_sign<double>(double v, uint32_t u) {
  return __hiloint2double(__double2hiint(v) ^ (int)(u & 0x80000000u), __double2loint(v));
}
__device__ __forceinline__ uint2 lds_u2(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint32_t lds_u1(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ int4 lds_i4(uint32_t addr) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

template <int CB>
constexpr int lp_stride() {
  return CB + 4;  // CB + 1 offsets per chunk, padded to a 16-byte multiple
}

template <typename T, int W, int CPW, int R>
__global__ void __launch_bounds__(W * 32, 1)
    sparse_right_persistent(const T* __restrict__ A, int64_t n, int64_t d, int64_t lda, const int32_t* __restrict__ ptr,
                            const uint16_t* __restrict__ ent, int64_t k, int nchunks, int ncb, int64_t ntiles,
                            uint32_t lp_off, uint32_t ent_off, T scale, T* __restrict__ Y, int64_t ldy) {
  using V4 = typename VecOf<T>::type;
  constexpr int NV = VecOf<T>::n;
  constexpr int NT = W * 32;
  constexpr int VEC_PER_ROW = R / NV;
  constexpr int VPT = kRowsPerTile * VEC_PER_ROW / NT;
  constexpr int ROWS_PER_PASS = NT / VEC_PER_ROW;
  constexpr int CB = W * CPW;
  constexpr int LPS = lp_stride<CB>();
  constexpr int TILE = kRowsPerTile * R;
  constexpr uint32_t SH = sizeof(T) == 8 ? 3u : 2u;
  constexpr uint32_t RMASK = (uint32_t)(R - 1) << SH;
  static_assert(R * sizeof(T) == 2048, "row stride of the staged tile");
  static_assert(NT % VEC_PER_ROW == 0 && (NT / VEC_PER_ROW) % NV == 0, "prefetch mapping");
  static_assert(CPW % 4 == 0, "vector loads of the column offsets");

  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* As = reinterpret_cast<T*>(smem_raw);
  int32_t* lp = reinterpret_cast<int32_t*>(smem_raw + lp_off);
  uint32_t* lent = reinterpret_cast<uint32_t*>(smem_raw + ent_off);
  __shared__ int32_t warp_tot[W];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cb = (int)(blockIdx.x % (unsigned)ncb);
  const int64_t nper = gridDim.x / ncb;
  const int64_t first_tile = blockIdx.x / ncb;
  const int64_t c0 = (int64_t)cb * CB;

  // ---- stage Omega's column block: padded counts, block-wide exclusive scan, offsets, entries
  {
    const int items = nchunks * CB;
    const int per = (items + NT - 1) / NT;
    const int i0 = min(items, tid * per), i1 = min(items, i0 + per);
    auto count = [&](int i) -> int {
      const int h = i / CB, j = i % CB;
      const int64_t c = c0 + j;
      if (c >= k) return 0;
      return __ldg(ptr + (int64_t)h * k + c + 1) - __ldg(ptr + (int64_t)h * k + c);
    };
    int mine = 0;
    for (int i = i0; i < i1; ++i) {
      const int c = count(i);
      mine += c + (c & 1);
    }
    // exclusive scan of the per-thread sums
    int incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    int base = 0;
    for (int w = 0; w < warp; ++w) base += warp_tot[w];
    int run = base + incl - mine;
    for (int i = i0; i < i1; ++i) {
      const int h = i / CB, j = i % CB;
      const int c = count(i);
      lp[h * LPS + j] = run | (c & 1);
      if (c > 0) {
        const int64_t g0 = __ldg(ptr + (int64_t)h * k + c0 + j);
        for (int q = 0; q < c; ++q) {
          const uint32_t e = __ldg(ent + g0 + q);
          lent[run + q] = ((e >> 1) << SH) | ((e & 1u) << 31);
        }
      }
      run += c + (c & 1);
      if (j == CB - 1) lp[h * LPS + CB] = run;  // end of chunk h's lists
    }
  }

  // ---- chunk stream over this CTA's tiles (cursors advance incrementally: no divisions)
  const int64_t my_tiles = first_tile < ntiles ? (ntiles - first_tile + nper - 1) / nper : 0;
  const int64_t steps = my_tiles * nchunks;
  const int vr = tid / VEC_PER_ROW;
  const int vcol = (tid % VEC_PER_ROW) * NV;
  V4 pre[VPT];
  // loader cursor: tile lt, chunk lh; per-tile base pointer and row-validity mask
  int64_t lt = first_tile;
  int lh = 0;
  const T* lbase = nullptr;
  uint32_t lrows = 0;
  auto set_tile = [&]() {
    const int64_t r = lt * kRowsPerTile + vr;
    lbase = A + r * lda + vcol;
    lrows = 0;
#pragma unroll
    for (int j = 0; j < VPT; ++j)
      if (r + (int64_t)j * ROWS_PER_PASS < n) lrows |= 1u << j;
  };
  auto load_next = [&]() {
    // rows past n and columns past d keep stale values: only lanes of invalid rows read them,
    // and Omega never references columns >= d
    const T* p = lbase + (int64_t)lh * R;
    const bool col_ok = (int64_t)lh * R + vcol < d;
#pragma unroll
    for (int j = 0; j < VPT; ++j)
      if (col_ok && ((lrows >> j) & 1u)) pre[j] = ld_stream(reinterpret_cast<const V4*>(p + (int64_t)j * ROWS_PER_PASS * lda));
    if (++lh == nchunks) {
      lh = 0;
      lt += nper;
      set_tile();
    }
  };
  auto store_vecs = [&](T* dst, auto key_c) {
    constexpr int KEY = decltype(key_c)::value;
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
      const int q = tid + j * NT;
      const int i = q / VEC_PER_ROW, cv = q % VEC_PER_ROW;
      const int blk = (cv * NV) ^ (i & 31 & ~(NV - 1));
      *reinterpret_cast<V4*>(dst + i * R + blk) = xor_perm(pre[j], KEY);
    }
  };
  auto store_step = [&](T* dst) {
    const int key = vr & (NV - 1);
    if (key == 0) store_vecs(dst, std::integral_constant<int, 0>{});
    else if (key == 1) store_vecs(dst, std::integral_constant<int, 1>{});
    else if constexpr (NV == 4) {
      if (key == 2) store_vecs(dst, std::integral_constant<int, 2>{});
      else store_vecs(dst, std::integral_constant<int, 3>{});
    }
  };

  if (steps > 0) {
    set_tile();
    load_next();
    store_step(As);
    if (steps > 1) load_next();
  }
  __syncthreads();

  const uint32_t tile_s0 = (uint32_t)__cvta_generic_to_shared(smem_raw);
  const uint32_t lp_s = (uint32_t)__cvta_generic_to_shared(lp) + 4u * (uint32_t)(warp * CPW);
  const uint32_t ent_s = (uint32_t)__cvta_generic_to_shared(lent);
  const uint32_t lxor = ((uint32_t)lane << 11) | ((uint32_t)lane << SH);
  T acc[CPW];
#pragma unroll
  for (int j = 0; j < CPW; ++j) acc[j] = T(0);

  int h = 0;
  int64_t ct = first_tile;  // compute cursor
  for (int64_t st = 0; st < steps; ++st) {
    const uint32_t tile_s = tile_s0 + ((uint32_t)st & 1u) * (uint32_t)(TILE * sizeof(T));
    int bnd[CPW + 4];
    const uint32_t lp_h = lp_s + 4u * (uint32_t)(h * LPS);
#pragma unroll
    for (int q = 0; q < CPW + 4; q += 4) {
      const int4 b4 = lds_i4(lp_h + 4u * (uint32_t)q);
      bnd[q] = b4.x;
      bnd[q + 1] = b4.y;
      bnd[q + 2] = b4.z;
      bnd[q + 3] = b4.w;
    }
#pragma unroll
    for (int j = 0; j < CPW; ++j) {
      const int e0 = bnd[j] & ~1;
      const int e1 = (bnd[j + 1] & ~1) - (bnd[j] & 1);
      T s0 = T(0), s1 = T(0);
      int e = e0;
#pragma unroll 1
      for (; e + 2 <= e1; e += 2) {
        const uint2 u = lds_u2(ent_s + 4u * (uint32_t)e);
        s0 += xor_sign(lds_t<T>(tile_s + ((u.x & RMASK) ^ lxor)), u.x);
        s1 += xor_sign(lds_t<T>(tile_s + ((u.y & RMASK) ^ lxor)), u.y);
      }
      if (e < e1) {
        const uint32_t u = lds_u1(ent_s + 4u * (uint32_t)e);
        s0 += xor_sign(lds_t<T>(tile_s + ((u & RMASK) ^ lxor)), u);
      }
      acc[j] += s0 + s1;
    }
    if (++h == nchunks) {
      // tile done: scaled accumulators straight to Y, then restart
      h = 0;
      const int64_t row = ct * kRowsPerTile + lane;
      const int64_t cw = c0 + (int64_t)warp * CPW;
      if (row < n) {
        T* y = Y + row * ldy + cw;
#pragma unroll
        for (int j = 0; j < CPW; ++j)
          if (cw + j < k) y[j] = acc[j] * scale;
      }
#pragma unroll
      for (int j = 0; j < CPW; ++j) acc[j] = T(0);
      ct += nper;
    }
    if (st + 1 < steps) {
      store_step(As + ((st + 1) & 1) * TILE);
      if (st + 2 < steps) load_next();
    }
    __syncthreads();
  }
}

constexpr int kWarps = 16;

template <typename T>
constexpr int chunk_rows_for() {
  return sizeof(T) == 4 ? 512 : 256;
}

template <typename T, int CPW, bool VEC>
int launch_t(const T* A, int64_t n, int64_t d, int64_t lda, const int32_t* ptr, const uint16_t* ent,
             int64_t nnz, int64_t k, double scale, T* Y, int64_t ldy, cudaStream_t s) {
  constexpr int R = chunk_rows_for<T>();
  constexpr int CB = kWarps * CPW;
  const int nchunks = (int)((d + R - 1) / R);
  const size_t tile_bytes = 2 * (size_t)kRowsPerTile * R * sizeof(T);  // double-buffered tile
  const size_t ys_bytes = (size_t)kRowsPerTile * (CB + 1) * sizeof(T);
  const size_t base = ((tile_bytes > ys_bytes ? tile_bytes : ys_bytes) + 15) & ~(size_t)15;
  // the whole encoding of a small Omega is staged in shared memory (nnz supplied by the caller)
  const int64_t nptr = (int64_t)nchunks * k + 1;
  const size_t ptr_bytes = (size_t)((nptr + 3) & ~3) * 4;
  const size_t oms_bytes = nnz > 0 ? ptr_bytes + (size_t)nnz * 2 : (size_t)1 << 30;
  const unsigned grid = (unsigned)(((n + kRowsPerTile - 1) / kRowsPerTile) * ((k + CB - 1) / CB));
  // persistent form when the column block's lists fit beside the two tiles (bound: every list
  // padded by one slot)
  {
    constexpr int LPS = lp_stride<CB>();
    const size_t lp_bytes = (size_t)nchunks * LPS * 4;
    const size_t ent_bytes = nnz > 0 ? ((size_t)nnz + (size_t)nchunks * CB + 3) / 4 * 16 : (size_t)1 << 30;
    const size_t smem = tile_bytes + lp_bytes + ent_bytes;
    const char* ov = getenv("SKETCH_B200_K1_CLASSIC");
    const bool off = ov && ov[0] == '1';
    if (VEC && !off && smem <= 220 * 1024) {
      // 32 warps x CPW / 2 columns (same column block): twice the warps to hide the shared-load chains
      constexpr int W2 = (CPW >= 8) ? 2 * kWarps : kWarps;
      constexpr int CPW2 = (CPW >= 8) ? CPW / 2 : CPW;
      static_assert(W2 * CPW2 == CB, "column block");
      auto kern = sparse_right_persistent<T, W2, CPW2, R>;
      const int nthreads = W2 * 32;
      allow_smem(kern, smem);
      const int ncb = (int)((k + CB - 1) / CB);
      const int64_t ntiles = (n + kRowsPerTile - 1) / kRowsPerTile;
      int64_t per_cb = sm_count() / ncb;
      if (per_cb < 1) per_cb = 1;
      if (per_cb > ntiles) per_cb = ntiles;
      kern<<<(unsigned)(per_cb * ncb), nthreads, smem, s>>>(A, n, d, lda, ptr, ent, k, nchunks, ncb, ntiles,
                                                           (uint32_t)tile_bytes, (uint32_t)(tile_bytes + lp_bytes),
                                                           (T)scale, Y, ldy);
      return check_launch("sk_sparse_right");
    }
  }
  if (base + oms_bytes <= 200 * 1024) {
    const size_t smem = base + oms_bytes;
    auto kern = sparse_right_kernel<T, kWarps, CPW, R, VEC, true>;
    allow_smem(kern, smem);
    kern<<<grid, kWarps * 32, smem, s>>>(A, n, d, lda, ptr, ent, k, nchunks, (int)nnz, (uint32_t)base, (T)scale, Y,
                                         ldy);
  } else {
    auto kern = sparse_right_kernel<T, kWarps, CPW, R, VEC, false>;
    allow_smem(kern, base);
    kern<<<grid, kWarps * 32, base, s>>>(A, n, d, lda, ptr, ent, k, nchunks, 0, (uint32_t)base, (T)scale, Y, ldy);
  }
  return check_launch("sk_sparse_right");
}

template <typename T>
int dispatch(const void* A_, int64_t n, int64_t d, int64_t lda, const int32_t* ptr, const uint16_t* ent,
             int64_t nnz, int64_t k, double scale, void* Y_, int64_t ldy, cudaStream_t s) {
  const T* A = static_cast<const T*>(A_);
  T* Y = static_cast<T*>(Y_);
  constexpr int NV = 16 / sizeof(T);
  const bool vec = ((reinterpret_cast<uintptr_t>(A) & 15) == 0) && (lda % NV == 0) && (d % NV == 0);
  int64_t need = (k + kWarps - 1) / kWarps;
  // split the output columns over more CTAs when there are few row tiles (wave balance)
  const int64_t tiles = (n + kRowsPerTile - 1) / kRowsPerTile;
  if (tiles < 8 * (int64_t)sm_count() && need > 8) need = 8;
  if (const char* ov = getenv("SKETCH_B200_K1_NEED")) need = atoi(ov);  // A/B experiments
  if (need <= 4) return vec ? launch_t<T, 4, true>(A, n, d, lda, ptr, ent, nnz, k, scale, Y, ldy, s)
                            : launch_t<T, 4, false>(A, n, d, lda, ptr, ent, nnz, k, scale, Y, ldy, s);
  if (need <= 8) return vec ? launch_t<T, 8, true>(A, n, d, lda, ptr, ent, nnz, k, scale, Y, ldy, s)
                            : launch_t<T, 8, false>(A, n, d, lda, ptr, ent, nnz, k, scale, Y, ldy, s);
  return vec ? launch_t<T, 16, true>(A, n, d, lda, ptr, ent, nnz, k, scale, Y, ldy, s)
             : launch_t<T, 16, false>(A, n, d, lda, ptr, ent, nnz, k, scale, Y, ldy, s);
}

}  // namespace
}  // namespace skb

extern "C" int sk_sparse_right_chunk_rows(int dtype, int64_t d, int64_t k) {
  (void)d;
  (void)k;
  if (dtype == SK_F32) return skb::chunk_rows_for<float>();
  if (dtype == SK_F64) return skb::chunk_rows_for<double>();
  return skb::fail(SK_EINVAL, "sk_sparse_right_chunk_rows: bad dtype");
}

extern "C" int sk_sparse_right(int dtype, const void* A, int64_t n, int64_t d, int64_t lda,
                               const int32_t* ptr, const uint16_t* ent, int32_t chunk_rows, int64_t nnz,
                               int64_t k, double scale, void* Y, int64_t ldy, void* stream) {
  using namespace skb;
  if (n < 0 || d < 1 || k < 1 || lda < d || ldy < k) return fail(SK_EINVAL, "sk_sparse_right: bad shape/leading dimension");
  if (n > 0 && (!A || !Y || !ptr)) return fail(SK_EINVAL, "sk_sparse_right: null pointer");
  if (dtype != SK_F32 && dtype != SK_F64) return fail(SK_EINVAL, "sk_sparse_right: bad dtype");
  if (chunk_rows != sk_sparse_right_chunk_rows(dtype, d, k))
    return fail(SK_EINVAL, "sk_sparse_right: chunk_rows does not match sk_sparse_right_chunk_rows");
  if (n == 0) return SK_OK;
  cudaStream_t s = as_stream(stream);
  return dtype == SK_F32 ? dispatch<float>(A, n, d, lda, ptr, ent, nnz, k, scale, Y, ldy, s)
                         : dispatch<double>(A, n, d, lda, ptr, ent, nnz, k, scale, Y, ldy, s);
}
