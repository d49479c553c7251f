// K1c — sparse-sign right apply  Y = scale * A * Omega  with lanes = output columns
// (BASELINE config 1: A 16384 x 4096 f64, Omega 4096 x 256 with zeta = 4 +-1 per row).
//
// Replaces `_SparseTM.apply_right` = `a @ self.matrix` (reference src/sketch/sparse.py:63-66).
// K1r (sparse_right_ring.cu) maps lanes to rows of A and walks each output column's short list per
// 128-row unit of Omega: ~29 instructions per warp-entry, issue-bound at 35-40 % of HBM.  Here the
// roles flip:
//
//   * lane = one output column j (8 warps = 256 columns per CTA); lane j keeps the WHOLE list of
//     Omega's column j in registers for the kernel's lifetime, as half byte offsets into a row of A
//     with the entry's sign in bit 31 (positions padded to the warp's longest list, a multiple of 8;
//     the padding reads a zeroed 128-byte pad after the row).
//   * lane 0 of warp 0 streams pairs of whole rows of A (one cp.async.bulk of d * sizeof(T) per
//     row) into a ring of two-row slots (no producer warp: 8 warps leave 255 registers per thread
//     for the lists).  Per slot each lane sums +-A[row, r] over its list for both rows: one address
//     (base + 2 q) per entry, two shared loads (the second row at + pitch), two sign XORs, two adds
//     into four independent accumulators per row — Y[row, j] needs no cross-lane reduction and no
//     per-column loop control.
//   * shared-memory bank conflicts of the per-lane gathers are removed at encoding time: Omega is
//     fixed, so the host scheduler (sk_sparse_right_cols_encode) orders every lane's list such that
//     at each position the lanes of a conflict group (16 lanes for float64 — one 128-byte wavefront
//     of 8-byte loads — 32 for float32) read distinct 8 / 4-byte bank slots where it can (a matching
//     of lanes to slots per position); columns are dealt to lanes by list length, a local search
//     then swaps lane slots while that lowers positions + unavoidable conflicts, and the warps of a
//     CTA are placed so each scheduler pairs a long-list warp with a short one.
//
// Config 1 (float64): 0.100 ms back to back = 88 % of the HBM copy peak (K1r: 0.215 ms).
//
// Bytes per launch (algorithmic): n * d * sizeof(T) read + n * k * sizeof(T) written.  The floor is
// shared memory: every (row, entry) pair is one lane-load (8 B for float64), plus the row's landing.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <functional>
#include <numeric>
#include <vector>

#include "common.cuh"
#include "sm100.cuh"

namespace skb {
namespace {

constexpr int C_WARPS = 8;                    // consumer warps per CTA (256 output columns)
constexpr int C_COLS = C_WARPS * 32;          // columns per group (CTA)
constexpr int C_THREADS = C_WARPS * 32;       // lane 0 of warp 0 also issues the row copies
constexpr int C_MAX_STAGES = 8;
constexpr size_t C_SMEM_BUDGET = 200 * 1024;
constexpr uint32_t C_PAD_BYTES = 128;         // zeroed pad after each row (dummy entries)
constexpr int C_ROWS = 2;                     // rows of A per ring slot (one entry address feeds both)

struct ColsParams {
  const void* A;
  int64_t n, d, lda;      // lda in elements
  const uint32_t* ent;    // [ngroups * C_WARPS][maxp][32]: byte offset | neg << 31
  const int32_t* colmap;  // [ngroups * C_WARPS * 32]: output column of each lane, -1 = none
  const int32_t* tw;      // [ngroups * C_WARPS]: positions of each warp (multiple of 8)
  int ngroups, nrb, stages;
  uint32_t stage_bytes;
  double scale;
  void* Y;
  int64_t ldy;
  int accumulate;
};

__device__ __forceinline__ double lds_val(uint32_t a, double*) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float lds_val(uint32_t a, float*) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
// sbit = 0 or 0x80000000: flip the sign of v
__device__ __forceinline__ double flip_hi(double v, uint32_t sbit) {
  return __hiloint2double(__double2hiint(v) ^ (int)sbit, __double2loint(v));
}
__device__ __forceinline__ float flip_hi(float v, uint32_t sbit) { return __int_as_float(__float_as_int(v) ^ sbit); }

__device__ __forceinline__ void bulk_row(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// addr = base + 2 * q: the doubling drops the sign bit (bit 31) of an entry q = offset / 2 | neg << 31.
// Opaque to the compiler, so it is not hoisted out of the row loop as 96 extra registers.
__device__ __forceinline__ uint32_t entry_addr(uint32_t q, uint32_t base) {
  uint32_t a;
  asm("mad.lo.u32 %0, %1, 2, %2;" : "=r"(a) : "r"(q), "r"(base));
  return a;
}

template <typename T, int MAXP>
__global__ void __launch_bounds__(C_THREADS, 1) sparse_right_cols_kernel(const ColsParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)p.stages * p.stage_bytes);
  uint64_t* empty = full + C_MAX_STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x % p.ngroups;
  const int rb = blockIdx.x / p.ngroups;
  const int64_t r0 = p.n * rb / p.nrb, r1 = p.n * (rb + 1) / p.nrb;
  const uint32_t row_bytes = (uint32_t)(p.d * (int64_t)sizeof(T));
  const uint32_t pitch = p.stage_bytes / C_ROWS;  // one row + its pad, multiple of 128
  const uint32_t ring = sm100::smem_u32(smem);

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], C_WARPS);
    }
    sm100::fence_mbar_init();
  }
  // the pad after every row of a slot reads as zero (the bulk copies never write it)
  for (int i = threadIdx.x; i < p.stages * C_ROWS * (int)(C_PAD_BYTES / 4); i += blockDim.x) {
    const int s = i / (C_PAD_BYTES / 4), q = i % (C_PAD_BYTES / 4);
    reinterpret_cast<uint32_t*>(smem + (size_t)s * pitch + row_bytes)[q] = 0u;
  }
  __syncthreads();

  const int wg = g * C_WARPS + warp;
  uint32_t e[MAXP];
  {
    const uint32_t* ep = p.ent + (size_t)wg * MAXP * 32 + lane;
#pragma unroll
    for (int i = 0; i < MAXP; ++i) e[i] = __ldg(ep + i * 32);
  }
  const int npos = __ldg(p.tw + wg);
  const int col = __ldg(p.colmap + wg * 32 + lane);
  T* ybase = static_cast<T*>(p.Y) + (col >= 0 ? col : 0);  // stores only when col >= 0
  const T scale = (T)p.scale;
  // row copies: issued by lane 0 of warp 0 (the warp with the longest lists, so the slot it refills
  // — released by every warp after the previous pair of rows — is normally free when it asks)
  const bool producer = (threadIdx.x == 0);
  const int64_t step = p.lda * (int64_t)sizeof(T);
  const uint8_t* src = static_cast<const uint8_t*>(p.A) + r0 * step;
  const int64_t nslots = (r1 - r0 + C_ROWS - 1) / C_ROWS;
  int64_t sp = 0;  // next slot to fill
  int ps = 0;
  uint32_t pph = 0;
  auto issue = [&]() {
    const int64_t rr = r0 + sp * C_ROWS;
    const uint32_t nr = (uint32_t)(r1 - rr < C_ROWS ? r1 - rr : C_ROWS);
    sm100::mbar_wait(&empty[ps], pph ^ 1);
    sm100::mbar_arrive_expect_tx(&full[ps], nr * row_bytes);
    for (uint32_t i = 0; i < nr; ++i) {
      bulk_row(ring + (uint32_t)ps * p.stage_bytes + i * pitch, src, row_bytes, sm100::smem_u32(&full[ps]));
      src += step;
    }
    ++sp;
    if (++ps == p.stages) {
      ps = 0;
      pph ^= 1;
    }
  };
  if (producer)
    while (sp < nslots && sp < p.stages - 1) issue();
  int s = 0;
  uint32_t ph = 0;
  for (int64_t slot = 0; slot < nslots; ++slot) {
    if (producer && sp < nslots) issue();  // slot + stages - 1 into the ring slot the previous one used
    sm100::mbar_wait(&full[s], ph);
    const uint32_t base = ring + (uint32_t)s * p.stage_bytes;
    // rows 2*slot and 2*slot + 1 of the range (the second is ignored past the end): one address per
    // entry feeds both rows (the second at +pitch)
    T a[2][4];
#pragma unroll
    for (int j = 0; j < 4; ++j) a[0][j] = a[1][j] = T(0);
#pragma unroll
    for (int b = 0; b < MAXP / 8; ++b) {
      if (b * 8 >= npos) break;  // warp-uniform
      T x[2][8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t ad = entry_addr(e[8 * b + i], base);
        x[0][i] = lds_val(ad, (T*)nullptr);
        x[1][i] = lds_val(ad + pitch, (T*)nullptr);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t sb = e[8 * b + i] & 0x80000000u;
        a[0][i & 3] += flip_hi(x[0][i], sb);
        a[1][i & 3] += flip_hi(x[1][i], sb);
      }
    }
    const T y0 = ((a[0][0] + a[0][1]) + (a[0][2] + a[0][3])) * scale;
    const T y1 = ((a[1][0] + a[1][1]) + (a[1][2] + a[1][3])) * scale;
    __syncwarp();  // every lane's loads of this slot have returned (y depends on all of them)
    if (lane == 0) sm100::mbar_arrive(&empty[s]);
    if (col >= 0) {
      const int64_t r = r0 + slot * C_ROWS;
      T* yp = ybase + r * p.ldy;
      *yp = p.accumulate ? *yp + y0 : y0;
      if (r + 1 < r1) {
        yp += p.ldy;
        *yp = p.accumulate ? *yp + y1 : y1;
      }
    }
    if (++s == p.stages) {
      s = 0;
      ph ^= 1;
    }
  }
}

template <typename T>
int elem_classes() {
  return (int)(128 / sizeof(T));  // bank slots of one 128-byte wavefront
}
inline int conflict_lanes(int dtype) { return dtype == SK_F64 ? 16 : 32; }
inline size_t elem_size(int dtype) { return dtype == SK_F64 ? 8 : 4; }

uint32_t stage_bytes_for(int dtype, int64_t d) {
  const size_t b = (size_t)d * elem_size(dtype) + C_PAD_BYTES;
  return (uint32_t)(C_ROWS * ((b + 127) & ~(size_t)127));
}
int stages_for(int dtype, int64_t d) {
  const size_t sb = stage_bytes_for(dtype, d);
  const size_t room = C_SMEM_BUDGET - 2 * C_MAX_STAGES * 8;
  return (int)std::min<size_t>(C_MAX_STAGES, room / sb);
}
bool maxp_ok(int maxp) { return maxp == 32 || maxp == 64 || maxp == 96 || maxp == 128; }

template <typename T, int MAXP>
int cols_launch(const ColsParams& p, int grid, size_t smem, cudaStream_t s) {
  allow_smem(sparse_right_cols_kernel<T, MAXP>, smem);
  sparse_right_cols_kernel<T, MAXP><<<grid, C_THREADS, smem, s>>>(p);
  return check_launch("sk_sparse_right_cols");
}
template <typename T>
int cols_dispatch(int maxp, const ColsParams& p, int grid, size_t smem, cudaStream_t s) {
  switch (maxp) {
    case 32: return cols_launch<T, 32>(p, grid, smem, s);
    case 64: return cols_launch<T, 64>(p, grid, smem, s);
    case 96: return cols_launch<T, 96>(p, grid, smem, s);
    default: return cols_launch<T, 128>(p, grid, smem, s);
  }
}

}  // namespace
}  // namespace skb

// ------------------------------------------------------------------------------------ C ABI
extern "C" int sk_sparse_right_cols_groups(int64_t k) { return k < 1 ? 0 : (int)((k + skb::C_COLS - 1) / skb::C_COLS); }

extern "C" int sk_sparse_right_cols_supported(int dtype, int64_t d, int64_t k, int32_t maxp) {
  if ((dtype != SK_F32 && dtype != SK_F64) || d < 1 || k < 1 || !skb::maxp_ok(maxp)) return 0;
  const size_t es = skb::elem_size(dtype);
  if (((size_t)d * es) % 16 != 0 || (size_t)d * es + 16 > (size_t)0x7fffffff) return 0;
  return skb::stages_for(dtype, d) >= 2 ? 1 : 0;
}

// Column-to-lane assignment, per-warp position counts and (ent != NULL) the scheduled entries.
// colmap: [groups * 256], tw: [groups * 8], ent: [groups * 8][maxp][32] with maxp >= *need.
extern "C" int sk_sparse_right_cols_encode(int dtype, int64_t d, int64_t k, int64_t nnz, const int64_t* rows,
                                           const int64_t* cols, const uint8_t* neg, int32_t maxp, uint32_t* ent,
                                           int32_t* colmap, int32_t* tw, int32_t* need) {
  using namespace skb;
  if ((dtype != SK_F32 && dtype != SK_F64) || d < 1 || k < 1 || nnz < 0 || !colmap || !tw || !need ||
      (nnz > 0 && (!rows || !cols || !neg)))
    return fail(SK_EINVAL, "sk_sparse_right_cols_encode: bad arguments");
  const size_t es = elem_size(dtype);
  if ((size_t)(d + 32) * es > (size_t)0x7fffffff)
    return fail(SK_EINVAL, "sk_sparse_right_cols_encode: row too long for 31-bit offsets");
  const int ngroups = sk_sparse_right_cols_groups(k);
  const int nwarps = ngroups * C_WARPS;
  std::vector<int64_t> cnt((size_t)k, 0);
  for (int64_t i = 0; i < nnz; ++i) {
    if (rows[i] < 0 || rows[i] >= d || cols[i] < 0 || cols[i] >= k)
      return fail(SK_EINVAL, "sk_sparse_right_cols_encode: index out of range");
    ++cnt[(size_t)cols[i]];
  }
  // columns dealt to lanes by decreasing list length (stable), so each warp's lists are near-equal
  std::vector<int64_t> order((size_t)k);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return cnt[(size_t)a] > cnt[(size_t)b]; });
  order.resize((size_t)nwarps * 32, -1);  // empty lanes at the end
  {
    // Local search over the lane slots: per warp, cost = groups * positions (one wavefront per
    // conflict group and position) + the entries of a bank class beyond the positions in each group
    // (the conflicts no schedule avoids).  Swaps of two slots (within a window of the sorted order)
    // are kept when they lower the cost; deterministic, so both encode calls agree.
    const int Cc = (int)(128 / es), Lg = conflict_lanes(dtype), G = 32 / Lg;
    std::vector<int32_t> hist((size_t)k * Cc, 0);
    for (int64_t i = 0; i < nnz; ++i) ++hist[(size_t)cols[i] * Cc + (size_t)(rows[i] % Cc)];
    auto len_of = [&](int64_t c) -> int64_t { return c < 0 ? 0 : cnt[(size_t)c]; };
    // incremental state: per conflict group its bank-class degrees, per warp its lane lengths
    const int nslots = nwarps * 32;
    const int ngrp = nwarps * G;
    std::vector<int64_t> deg((size_t)ngrp * Cc, 0);
    for (int i = 0; i < nslots; ++i) {
      const int64_t c = order[(size_t)i];
      if (c >= 0)
        for (int b = 0; b < Cc; ++b) deg[(size_t)(i / Lg) * Cc + b] += hist[(size_t)c * Cc + b];
    }
    auto warp_T = [&](int w) -> int64_t {
      int64_t m = 0;
      for (int l = 0; l < 32; ++l) m = std::max(m, len_of(order[(size_t)w * 32 + l]));
      return (m + 7) / 8 * 8;
    };
    auto warp_cost = [&](int w, int64_t T) -> int64_t {
      int64_t cost = G * T;
      for (int g = w * G; g < (w + 1) * G; ++g)
        for (int b = 0; b < Cc; ++b) cost += std::max<int64_t>(0, deg[(size_t)g * Cc + b] - T);
      return cost;
    };
    auto move = [&](int slot, int64_t c, int sign) {  // add / remove column c's classes at slot's group
      if (c < 0) return;
      int64_t* dg = &deg[(size_t)(slot / Lg) * Cc];
      const int32_t* hc = &hist[(size_t)c * Cc];
      for (int b = 0; b < Cc; ++b) dg[b] += sign * hc[b];
    };
    std::vector<int64_t> wc((size_t)nwarps);
    for (int w = 0; w < nwarps; ++w) wc[(size_t)w] = warp_cost(w, warp_T(w));
    const int window = 64;
    for (int pass = 0; pass < 3; ++pass) {
      bool improved = false;
      for (int i = 0; i < nslots; ++i)
        for (int j = i + 1; j < std::min(nslots, i + window); ++j) {
          const int wi = i / 32, wj = j / 32;
          if (i / Lg == j / Lg) continue;  // same conflict group: no change
          const int64_t ci0 = order[(size_t)i], cj0 = order[(size_t)j];
          if (ci0 < 0 && cj0 < 0) continue;
          move(i, ci0, -1), move(j, cj0, -1), move(i, cj0, 1), move(j, ci0, 1);
          std::swap(order[(size_t)i], order[(size_t)j]);
          const int64_t ci = warp_cost(wi, warp_T(wi)), cj = wi == wj ? ci : warp_cost(wj, warp_T(wj));
          const int64_t before = wc[(size_t)wi] + (wi == wj ? 0 : wc[(size_t)wj]);
          const int64_t after = ci + (wi == wj ? 0 : cj);
          if (after < before) {
            wc[(size_t)wi] = ci;
            wc[(size_t)wj] = cj;
            improved = true;
          } else {
            std::swap(order[(size_t)i], order[(size_t)j]);
            move(i, cj0, -1), move(j, ci0, -1), move(i, ci0, 1), move(j, cj0, 1);
          }
        }
      if (!improved) break;
    }
  }
  {
    // within each CTA group, put warps on the 4 schedulers (warp id % 4) so a long-list warp shares
    // its scheduler with a short-list one: ranks by max list length -> ids 0, 1, 2, 3, 7, 6, 5, 4
    // (config 1: 0.1007 -> 0.1000 ms)
    for (int g = 0; g < ngroups; ++g) {
      std::vector<std::pair<int64_t, int>> wl;
      for (int w = 0; w < C_WARPS; ++w) {
        int64_t m = 0;
        for (int l = 0; l < 32; ++l) {
          const int64_t c = order[(size_t)(g * C_WARPS + w) * 32 + l];
          m = std::max<int64_t>(m, c < 0 ? 0 : cnt[(size_t)c]);
        }
        wl.push_back({-m, w});
      }
      std::stable_sort(wl.begin(), wl.end());
      static const int slot_of_rank[C_WARPS] = {0, 1, 2, 3, 7, 6, 5, 4};
      std::vector<int64_t> tmp((size_t)C_WARPS * 32);
      for (int r = 0; r < C_WARPS; ++r)
        for (int l = 0; l < 32; ++l)
          tmp[(size_t)slot_of_rank[r] * 32 + l] = order[(size_t)(g * C_WARPS + wl[(size_t)r].second) * 32 + l];
      std::copy(tmp.begin(), tmp.end(), order.begin() + (size_t)g * C_WARPS * 32);
    }
  }
  std::vector<int64_t> lane_len((size_t)nwarps * 32, 0);
  for (int i = 0; i < nwarps * 32; ++i) {
    colmap[i] = (int32_t)order[(size_t)i];
    lane_len[(size_t)i] = order[(size_t)i] >= 0 ? cnt[(size_t)order[(size_t)i]] : 0;
  }
  int32_t mx = 0;
  for (int w = 0; w < nwarps; ++w) {
    int64_t m = 0;
    for (int l = 0; l < 32; ++l) m = std::max(m, lane_len[(size_t)w * 32 + l]);
    if (m > (1 << 28)) return fail(SK_EINVAL, "sk_sparse_right_cols_encode: column list too long");
    tw[w] = (int32_t)((m + 7) / 8 * 8);
    mx = std::max(mx, tw[w]);
  }
  *need = mx;
  if (!ent) return SK_OK;
  if (maxp < mx) return fail(SK_EINVAL, "sk_sparse_right_cols_encode: maxp below the longest warp's positions");

  // per-lane buckets by bank class
  const int C = (int)(128 / es);
  const int L = conflict_lanes(dtype);
  std::vector<int32_t> lane_of((size_t)k, 0);
  for (int i = 0; i < nwarps * 32; ++i)
    if (order[(size_t)i] >= 0) lane_of[(size_t)order[(size_t)i]] = i;
  // entries grouped by lane then class: value = byte offset | neg << 31
  std::vector<std::vector<std::vector<uint32_t>>> buckets((size_t)nwarps * 32, std::vector<std::vector<uint32_t>>(C));
  for (int64_t i = 0; i < nnz; ++i) {
    const int ln = lane_of[(size_t)cols[i]];
    const uint32_t v = (uint32_t)((uint64_t)rows[i] * es / 2) | (neg[i] ? 0x80000000u : 0u);
    buckets[(size_t)ln][(size_t)(rows[i] % C)].push_back(v);
  }
  for (auto& lb : buckets)
    for (auto& b : lb) std::sort(b.begin(), b.end(), std::greater<uint32_t>());  // pop_back = smallest offset
  const int dmod = (int)(d % C);
  auto dummy = [&](int cls) -> uint32_t { return (uint32_t)((uint64_t)(d + ((cls - dmod + C) % C)) * es / 2); };

  // Per position, a bipartite matching of lanes to bank classes (Kuhn's augmenting paths): lanes
  // whose remaining entries equal the positions left must take a real entry, the others take one
  // when a class is free for it (else a dummy in a free class, using their slack), so that as many
  // lanes as possible read distinct classes.  Unmatched forced lanes take their least-used class.
  std::vector<int> cls_of((size_t)L), lane_at((size_t)C), used((size_t)C), seen((size_t)C);
  std::vector<int64_t> rem((size_t)L);
  std::vector<std::vector<int>> pref((size_t)L);
  for (int w = 0; w < nwarps; ++w) {
    uint32_t* ew = ent + (size_t)w * maxp * 32;
    for (int t = tw[w]; t < maxp; ++t)
      for (int l = 0; l < 32; ++l) ew[(size_t)t * 32 + l] = dummy(l % C);
    for (int l0 = 0; l0 < 32; l0 += L) {
      auto bucket = [&](int j, int c) -> std::vector<uint32_t>& { return buckets[(size_t)w * 32 + l0 + j][(size_t)c]; };
      for (int j = 0; j < L; ++j) rem[(size_t)j] = lane_len[(size_t)w * 32 + l0 + j];
      const int T = tw[w];
      for (int t = 0; t < T; ++t) {
        const int64_t left = T - t;
        std::fill(cls_of.begin(), cls_of.end(), -1);
        std::fill(lane_at.begin(), lane_at.end(), -1);
        for (int j = 0; j < L; ++j) {  // real classes, fullest bucket first
          auto& pj = pref[(size_t)j];
          pj.clear();
          for (int c = 0; c < C; ++c)
            if (!bucket(j, c).empty()) pj.push_back(c);
          std::stable_sort(pj.begin(), pj.end(), [&](int a2, int b2) { return bucket(j, a2).size() > bucket(j, b2).size(); });
        }
        std::function<bool(int)> augment = [&](int j) -> bool {
          for (int c : pref[(size_t)j]) {
            if (seen[(size_t)c]) continue;
            seen[(size_t)c] = 1;
            if (lane_at[(size_t)c] < 0 || augment(lane_at[(size_t)c])) {
              lane_at[(size_t)c] = j;
              cls_of[(size_t)j] = c;
              return true;
            }
          }
          return false;
        };
        for (int pass = 0; pass < 2; ++pass)  // forced lanes first, then lanes with slack
          for (int j = 0; j < L; ++j) {
            if (rem[(size_t)j] == 0 || (rem[(size_t)j] >= left) != (pass == 0)) continue;
            std::fill(seen.begin(), seen.end(), 0);
            augment(j);
          }
        std::fill(used.begin(), used.end(), 0);
        for (int c = 0; c < C; ++c)
          if (lane_at[(size_t)c] >= 0) used[(size_t)c] = 1;
        for (int j = 0; j < L; ++j) {
          uint32_t v;
          int c = cls_of[(size_t)j];
          if (c < 0 && rem[(size_t)j] > 0 && rem[(size_t)j] >= left) {  // forced and unmatched: conflict
            int mu = 1 << 30;
            for (int c2 = 0; c2 < C; ++c2)
              if (!bucket(j, c2).empty() && used[(size_t)c2] < mu) {
                mu = used[(size_t)c2];
                c = c2;
              }
          }
          if (c >= 0) {
            v = bucket(j, c).back();
            bucket(j, c).pop_back();
            --rem[(size_t)j];
          } else {  // dummy in the least-used class
            int mu = 1 << 30;
            for (int c2 = 0; c2 < C; ++c2)
              if (used[(size_t)c2] < mu) {
                mu = used[(size_t)c2];
                c = c2;
              }
            v = dummy(c);
          }
          ++used[(size_t)c];
          if (cls_of[(size_t)j] >= 0) --used[(size_t)c], used[(size_t)c] = std::max(used[(size_t)c], 1);
          ew[(size_t)t * 32 + l0 + j] = v;
        }
      }
    }
  }
  return SK_OK;
}

extern "C" int sk_sparse_right_cols(int dtype, const void* A, int64_t n, int64_t d, int64_t lda, const uint32_t* ent,
                                    const int32_t* colmap, const int32_t* tw, int64_t k, int32_t maxp, double scale,
                                    void* Y, int64_t ldy, int accumulate, void* stream) {
  using namespace skb;
  if (n < 0 || d < 1 || k < 1 || lda < d || ldy < k) return fail(SK_EINVAL, "sk_sparse_right_cols: bad shape");
  if (!sk_sparse_right_cols_supported(dtype, d, k, maxp))
    return fail(SK_EUNSUPPORTED, "sk_sparse_right_cols: unsupported dtype / row length / maxp");
  if (n == 0) return SK_OK;
  if (!A || !ent || !colmap || !tw || !Y) return fail(SK_EINVAL, "sk_sparse_right_cols: null pointer");
  const size_t es = elem_size(dtype);
  if ((reinterpret_cast<uintptr_t>(A) & 15) || ((size_t)lda * es) % 16 || (reinterpret_cast<uintptr_t>(Y) % es))
    return fail(SK_EINVAL, "sk_sparse_right_cols: A and its rows 16-byte aligned, Y element-aligned");
  ColsParams p{};
  p.A = A;
  p.n = n;
  p.d = d;
  p.lda = lda;
  p.ent = ent;
  p.colmap = colmap;
  p.tw = tw;
  p.ngroups = sk_sparse_right_cols_groups(k);
  p.nrb = (int)std::max<int64_t>(1, std::min<int64_t>(n, std::max(1, sm_count() / p.ngroups)));
  p.stages = stages_for(dtype, d);
  p.stage_bytes = stage_bytes_for(dtype, d);
  p.scale = scale;
  p.Y = Y;
  p.ldy = ldy;
  p.accumulate = accumulate ? 1 : 0;
  const size_t smem = (size_t)p.stages * p.stage_bytes + 2 * C_MAX_STAGES * 8;
  const int grid = p.ngroups * p.nrb;
  cudaStream_t s = as_stream(stream);
  return dtype == SK_F64 ? cols_dispatch<double>(maxp, p, grid, smem, s) : cols_dispatch<float>(maxp, p, grid, smem, s);
}
