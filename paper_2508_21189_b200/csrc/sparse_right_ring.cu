// K1r — float64 sparse-sign right apply  Y = scale * A * Omega  on a warp-specialised ring
// (BASELINE config 1: A 16384 x 4096 f64, Omega 4096 x 256 with zeta = 4 +-1 per row).
//
// Replaces `_SparseTM.apply_right` = `a @ self.matrix` (reference src/sketch/sparse.py:63-66).
// Round-1 K1 (csrc/sparse_right.cu) staged each chunk of A through registers with a CTA barrier per
// chunk: the Poisson spread of entries per warp left the fast warps waiting (30 % of HBM).  Here:
//
//   * 2 producer warps copy each 64-row x 64-column chunk of A (32 KB) into a 4-stage shared-memory
//     ring with 8-byte cp.async (no registers held), XOR-swizzled at 8-byte granularity:
//     element (row, r) at row * 512 + ((r ^ (row & 15)) << 3), so the gather "32 lanes = 32 rows,
//     same column r" hits 16 distinct bank pairs per half-warp (conflict-free);
//     `cp.async.mbarrier.arrive.noinc` completes the stage's full barrier.
//   * 16 consumer warps own 16 output columns each (k <= 256); lane = rows l and l + 32 of the tile,
//     so every Omega entry feeds two independent gathers and two float64 adds (register
//     accumulators).  Entries come from per-(chunk, warp) segments staged once in shared memory:
//     16 column counts (uint8) then uint16 entries stage << 15 | r << 3 | neg; one consumer pass takes
//     two stages (a 128-row unit of Omega: ~2 entries per column, so the per-column loop overhead is
//     paid half as often).  Warps release stages through the empty barriers (16 arrivals): no
//     CTA-wide barrier, a slow warp may lag by up to one unit.
//   * stream-K: CTA c walks the global chunk range [c L, (c + 1) L) over (tile, chunk) pairs
//     (L >= chunks per tile), so every SM streams the same number of bytes.  A tile cut between
//     two CTAs: CTA c processes its tail part first and publishes it (ws[c], flag[c] = 16 warps);
//     CTA c - 1 reaches the head part last, adds ws[c] and writes Y (deterministic order).
//
// Bytes per launch (algorithmic): n * d * 8 read + n * k * 8 written.
#include <cuda_runtime.h>

#include "common.cuh"
#include "sm100.cuh"

namespace skb {
namespace {

constexpr int RR = 64;          // rows per tile (2 per lane)
constexpr int RC = 64;          // columns of A (rows of Omega) per stage
constexpr int UC = 2 * RC;      // per unit: a consumer pass takes two stages (amortises the column loops)
constexpr int STAGES = 4;  // even: a unit's two stages are adjacent (one base address per unit)
constexpr int STAGE_BYTES = RR * RC * 8;  // 32 KB
constexpr int NPROD = 2;        // producer warps (64 threads: one column of the chunk each)
constexpr int NCONS = 16;       // consumer warps
constexpr int CPW = 16;         // output columns per consumer warp
constexpr int THREADS = (NPROD + NCONS) * 32;

struct RingParams {
  const double* A;
  int64_t n, d, lda;
  int k;
  const uint8_t* lists;     // segments (16-byte units), seg[h * NCONS + w] = offset of (chunk h, warp w)
  const uint32_t* seg;      // [nchunks * NCONS + 1]
  int nchunks;              // units per tile = ceil(d / UC)
  int64_t total;            // tiles * nchunks
  int64_t L;                // units per CTA
  double scale;
  double* Y;
  int64_t ldy;
  double* ws;               // [grid][RR][256] tail partials
  int* flags;               // [grid] (zeroed before the launch)
  int accumulate;           // Y += (a column slab of a wider Omega) instead of Y =
};

__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(valid ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(sm100::smem_u32(bar)) : "memory");
}
__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint4 lds_v4(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double flip(double v, uint32_t neg) {
  return __hiloint2double(__double2hiint(v) ^ (int)(neg << 31), __double2loint(v));
}

__global__ void __launch_bounds__(THREADS, 1) sparse_right_ring_kernel(const RingParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int nseg_bytes = (int)p.seg[p.nchunks * NCONS] * 16;
  const int nseg = p.nchunks * NCONS + 1;
  uint8_t* ring = smem;
  uint8_t* lists = smem + STAGES * STAGE_BYTES;
  uint32_t* seg_s = reinterpret_cast<uint32_t*>(lists + nseg_bytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(seg_s + ((nseg + 3) & ~3));
  uint64_t* empty = full + STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      sm100::mbar_init(&full[s], NPROD * 32);
      sm100::mbar_init(&empty[s], NCONS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // Omega's segments: staged once per CTA (16-byte vector copies)
  for (int i = threadIdx.x; i < nseg_bytes / 16; i += THREADS)
    reinterpret_cast<uint4*>(lists)[i] = __ldg(reinterpret_cast<const uint4*>(p.lists) + i);
  for (int i = threadIdx.x; i < nseg; i += THREADS) seg_s[i] = __ldg(p.seg + i);
  __syncthreads();

  const int64_t g0 = (int64_t)blockIdx.x * p.L;
  const int64_t g1 = min(p.total, g0 + p.L);
  const uint32_t ring_u32 = sm100::smem_u32(ring);

  if (warp < NPROD) {
    // ---------------------------------------------------------------- producers (cp.async ring)
    // thread pc = column pc of the chunk, all 64 rows (row-major A: each warp copies 256 contiguous
    // bytes of one row per step); destination (row, pc) -> row * 512 + ((pc ^ (row & 15)) << 3)
    const int pc = threadIdx.x;  // 0..63
    uint32_t xo[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) xo[i] = (uint32_t)((pc ^ i) << 3);
    int s = 0;
    uint32_t ph = 0;
    int64_t t = g0 / p.nchunks;
    int h = (int)(g0 - t * p.nchunks);
    for (int64_t g = g0; g < g1; ++g) {
      const int64_t rows_left = p.n - t * RR;  // rows valid while row < rows_left
#pragma unroll 1
      for (int sub = 0; sub < 2; ++sub) {
        const int64_t col = (int64_t)h * UC + sub * RC + pc;
        const double* src = p.A + t * RR * p.lda + col;
        const bool col_ok = col < p.d;
        sm100::mbar_wait(&empty[s], ph ^ 1);
        const uint32_t st = ring_u32 + (uint32_t)s * STAGE_BYTES;
#pragma unroll
        for (int row = 0; row < RR; ++row) {
          const bool ok = col_ok && row < rows_left;
          cp_async8(st + (uint32_t)row * (RC * 8) + xo[row & 15], ok ? src : p.A, ok);
          src += p.lda;
        }
        cp_async_arrive_noinc(&full[s]);
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
      if (++h == p.nchunks) { h = 0; ++t; }
    }
  } else {
    // ---------------------------------------------------------------- consumers
    const int w = warp - NPROD;
    double acc0[CPW], acc1[CPW];
#pragma unroll
    for (int j = 0; j < CPW; ++j) acc0[j] = acc1[j] = 0.0;
    const uint32_t lists_u32 = sm100::smem_u32(lists);
    const uint32_t lane_off = (uint32_t)lane * (RC * 8);
    const uint32_t lane_x8 = (uint32_t)(lane & 15) << 3;
    int s = 0;
    uint32_t ph = 0;

    auto flush = [&](int64_t t, int hs, int he) {
      const int64_t r0 = t * RR + lane, r1 = r0 + 32;
      const int c0 = w * CPW;
      double* part = p.ws + (int64_t)blockIdx.x * RR * 256;
      if (hs > 0) {
        // tail part (this CTA's first segment): publish for the CTA that holds the head part
#pragma unroll
        for (int j = 0; j < CPW; ++j) {
          part[(int64_t)lane * 256 + c0 + j] = acc0[j];
          part[(int64_t)(lane + 32) * 256 + c0 + j] = acc1[j];
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(p.flags + blockIdx.x, 1);
        return;
      }
      if (he < p.nchunks) {
        // head part (this CTA's last segment): add the successor's tail partial
        const int* fl = p.flags + blockIdx.x + 1;
        if (lane == 0)
          while (ld_acquire(fl) < NCONS) __nanosleep(64);
        __syncwarp();
        const double* q = p.ws + (int64_t)(blockIdx.x + 1) * RR * 256;
#pragma unroll
        for (int j = 0; j < CPW; ++j) {
          acc0[j] += q[(int64_t)lane * 256 + c0 + j];
          acc1[j] += q[(int64_t)(lane + 32) * 256 + c0 + j];
        }
      }
      double* y0 = p.Y + r0 * p.ldy + c0;
      double* y1 = y0 + 32 * p.ldy;
      const int kc = p.k - c0;
      const bool ok0 = r0 < p.n, ok1 = r1 < p.n;
      if (p.accumulate) {
#pragma unroll
        for (int j = 0; j < CPW; ++j) {
          if (j < kc) {
            if (ok0) y0[j] += acc0[j] * p.scale;
            if (ok1) y1[j] += acc1[j] * p.scale;
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < CPW; ++j) {
          if (j < kc) {
            if (ok0) y0[j] = acc0[j] * p.scale;
            if (ok1) y1[j] = acc1[j] * p.scale;
          }
        }
      }
    };

    // tile segments of this CTA's chunk range: [hs, he) of tile t, accumulators reset per segment
    for (int64_t g = g0; g < g1;) {
      const int64_t t = g / p.nchunks;
      const int hs = (int)(g - t * p.nchunks);
      const int he = (int)min((int64_t)p.nchunks, hs + (g1 - g));
#pragma unroll
      for (int j = 0; j < CPW; ++j) acc0[j] = acc1[j] = 0.0;
      for (int h = hs; h < he; ++h) {
        // this warp's segment of unit h (stages s, s + 1): 16 uint8 counts, then uint16 entries
        // stage << 15 | (row % 64) << 3 | neg: the byte offset of the row's column in the unit, so a
        // gather address is one XOR with the lane's swizzle and one add
        const uint32_t sb = lists_u32 + seg_s[h * NCONS + w] * 16u;
        const uint4 cnt = lds_v4(sb);
        uint32_t e = sb + 16;
        sm100::mbar_wait(&full[s], ph);
        sm100::mbar_wait(&full[s + 1], ph);
        const uint32_t a0 = ring_u32 + (uint32_t)s * STAGE_BYTES + lane_off;
        const uint32_t cw[4] = {cnt.x, cnt.y, cnt.z, cnt.w};
#pragma unroll
        for (int j = 0; j < CPW; ++j) {
          const uint32_t nj = (cw[j >> 2] >> (8 * (j & 3))) & 0xffu;
          const uint32_t eend = e + 2 * nj;
          for (; e + 2 < eend; e += 4) {  // two entries in flight
            const uint32_t en0 = lds_u16(e), en1 = lds_u16(e + 2);
            const uint32_t ad0 = a0 + ((en0 & 0xfff8u) ^ lane_x8), ad1 = a0 + ((en1 & 0xfff8u) ^ lane_x8);
            const double x0 = lds_f64(ad0), y0 = lds_f64(ad0 + 32u * RC * 8u);
            const double x1 = lds_f64(ad1), y1 = lds_f64(ad1 + 32u * RC * 8u);
            acc0[j] += flip(x0, en0 & 1u) + flip(x1, en1 & 1u);
            acc1[j] += flip(y0, en0 & 1u) + flip(y1, en1 & 1u);
          }
          if (e < eend) {
            const uint32_t en = lds_u16(e);
            const uint32_t addr = a0 + ((en & 0xfff8u) ^ lane_x8);
            acc0[j] += flip(lds_f64(addr), en & 1u);
            acc1[j] += flip(lds_f64(addr + 32u * RC * 8u), en & 1u);
            e += 2;
          }
        }
        __syncwarp();
        if (lane == 0) {
          sm100::mbar_arrive(&empty[s]);
          sm100::mbar_arrive(&empty[s + 1]);
        }
        s += 2;
        if (s == STAGES) { s = 0; ph ^= 1; }
      }
      flush(t, hs, he);
      g += he - hs;
    }
  }
}

}  // namespace
}  // namespace skb

// ------------------------------------------------------------------------------------ C ABI
namespace skb {
namespace {
size_t ring_smem(int64_t d, int64_t seg_bytes) {
  const int64_t nseg = ((d + UC - 1) / UC) * NCONS + 1;
  return (size_t)STAGES * STAGE_BYTES + (size_t)((seg_bytes + 15) & ~15) + (size_t)((nseg + 3) & ~3) * 4 +
         2 * STAGES * 8;
}
// stream-K split: grid and chunks per CTA (every CTA spans at least one tile, so a tile is cut
// between at most two CTAs)
void ring_grid(int64_t n, int64_t d, int* grid, int64_t* L, int64_t* total) {
  const int nchunks = (int)((d + UC - 1) / UC);
  const int64_t tiles = (n + RR - 1) / RR;
  *total = tiles * nchunks;
  int64_t l = (*total + sm_count() - 1) / sm_count();
  if (l < nchunks) l = nchunks;
  *L = l;
  *grid = (int)((*total + l - 1) / l);
}
}  // namespace
}  // namespace skb

// segment layout: see the kernel comment; seg has ceil(d / 64) * 16 + 1 entries (16-byte units)
extern "C" int sk_sparse_right_ring_supported(int dtype, int64_t d, int64_t k, int64_t seg_bytes) {
  const size_t smem = skb::ring_smem(d, seg_bytes);
  return (dtype == SK_F64 && k >= 1 && k <= skb::NCONS * skb::CPW && d >= 1 && smem <= 227 * 1024) ? 1 : 0;
}

extern "C" size_t sk_sparse_right_ring_workspace_bytes(int64_t n, int64_t d) {
  if (n < 1 || d < 1) return 0;
  int grid;
  int64_t L, total;
  skb::ring_grid(n, d, &grid, &L, &total);
  return (size_t)grid * (skb::RR * 256 * sizeof(double) + sizeof(int));
}

namespace skb {
namespace {
int ring_run(const double* A, int64_t n, int64_t d, int64_t lda, const uint8_t* lists, const uint32_t* seg,
             int64_t seg_bytes, int64_t k, double scale, double* Y, int64_t ldy, int accumulate, void* ws,
             size_t ws_bytes, void* stream) {
  if (n < 0 || d < 1 || k < 1 || lda < d || ldy < k) return fail(SK_EINVAL, "sk_sparse_right_ring: bad shape");
  if (!sk_sparse_right_ring_supported(SK_F64, d, k, seg_bytes))
    return fail(SK_EUNSUPPORTED, "sk_sparse_right_ring: k > 256 or segments too large for shared memory");
  if (n == 0) return SK_OK;
  if (!A || !lists || !seg || !Y) return fail(SK_EINVAL, "sk_sparse_right_ring: null pointer");
  if ((reinterpret_cast<uintptr_t>(A) & 7) || (reinterpret_cast<uintptr_t>(lists) & 15))
    return fail(SK_EINVAL, "sk_sparse_right_ring: A 8-byte and lists 16-byte aligned");
  int grid;
  int64_t L, total;
  ring_grid(n, d, &grid, &L, &total);
  const size_t need = (size_t)grid * (RR * 256 * sizeof(double) + sizeof(int));
  if (!ws || ws_bytes < need) return fail(SK_EINVAL, "sk_sparse_right_ring: workspace too small");
  double* part = static_cast<double*>(ws);
  int* flags = reinterpret_cast<int*>(part + (size_t)grid * RR * 256);
  cudaStream_t s = as_stream(stream);
  if (cudaMemsetAsync(flags, 0, (size_t)grid * sizeof(int), s) != cudaSuccess)
    return check_launch("sk_sparse_right_ring");
  RingParams p{};
  p.A = A;
  p.n = n;
  p.d = d;
  p.lda = lda;
  p.k = (int)k;
  p.lists = lists;
  p.seg = seg;
  p.nchunks = (int)((d + UC - 1) / UC);
  p.total = total;
  p.L = L;
  p.scale = scale;
  p.Y = Y;
  p.ldy = ldy;
  p.ws = part;
  p.flags = flags;
  p.accumulate = accumulate;
  const size_t smem = ring_smem(d, seg_bytes);
  allow_smem(sparse_right_ring_kernel, smem);
  sparse_right_ring_kernel<<<grid, THREADS, smem, s>>>(p);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, sparse_right_ring_kernel);
    return fail(SK_ECUDA, std::string("sk_sparse_right_ring: ") + cudaGetErrorString(e) + " (regs " +
                              std::to_string(fa.numRegs) + ", max threads " + std::to_string(fa.maxThreadsPerBlock) +
                              ", smem " + std::to_string(smem) + ")");
  }
  return SK_OK;
}
}  // namespace
}  // namespace skb

extern "C" int sk_sparse_right_ring(const double* A, int64_t n, int64_t d, int64_t lda, const uint8_t* lists,
                                    const uint32_t* seg, int64_t seg_bytes, int64_t k, double scale, double* Y,
                                    int64_t ldy, void* ws, size_t ws_bytes, void* stream) {
  return skb::ring_run(A, n, d, lda, lists, seg, seg_bytes, k, scale, Y, ldy, 0, ws, ws_bytes, stream);
}

extern "C" int sk_sparse_right_ring_slab(const double* A, int64_t n, int64_t d, int64_t lda, const uint8_t* lists,
                                         const uint32_t* seg, int64_t seg_bytes, int64_t k, double scale, double* Y,
                                         int64_t ldy, int accumulate, void* ws, size_t ws_bytes, void* stream) {
  return skb::ring_run(A, n, d, lda, lists, seg, seg_bytes, k, scale, Y, ldy, accumulate ? 1 : 0, ws, ws_bytes,
                       stream);
}
