// Microbenchmark: read-modify-write of single TMEM columns by warps (tcgen05.ld/st 32x32b.x1),
// the access pattern of a TMEM-accumulator scatter (one output row per column, 32 lanes = 32
// input columns). Each warp updates B columns per batch (ld x B, wait::ld, FADD x B, st x B,
// wait::st). Reports quadrant-updates per SM per cycle.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/tmem_rmw tools/micro/tmem_rmw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int B, bool WAIT_ST>
__global__ void __launch_bounds__(512, 1) tmem_rmw(int iters, float* out, long long* cycles) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot + ((uint32_t)(32 * (warp & 3)) << 16);
  // warps of a quadrant own disjoint column sets: column = 4 * x + (warp >> 2)
  uint32_t h = 0x9E3779B9u * (warp + 1);
  float v = 1.0f + lane;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t col[B], r[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      h = h * 1664525u + 1013904223u;
      col[b] = ((h >> 10) & 127u) * 4u + (uint32_t)(warp >> 2);
    }
#pragma unroll
    for (int b = 0; b < B; ++b)
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r[b]) : "r"(tmem + col[b]));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int b = 0; b < B; ++b) r[b] = __float_as_uint(__uint_as_float(r[b]) + v);
#pragma unroll
    for (int b = 0; b < B; ++b)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + col[b]), "r"(r[b]));
    if (WAIT_ST) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  long long t1 = clock64();
  uint32_t x;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(x) : "r"(tmem));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  out[blockIdx.x * 512 + threadIdx.x] = __uint_as_float(x);
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

template <int B, bool W>
void run(int sms) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, sms * 512 * 4);
  cudaMalloc(&cyc, sms * 8);
  const int iters = 4000;
  tmem_rmw<B, W><<<sms, 512>>>(iters, out, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  tmem_rmw<B, W><<<sms, 512>>>(iters, out, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double upd = 16.0 * iters * B;  // quadrant-updates per SM
  printf("B=%2d wait_st=%d: %.3f ms, %.2f cycles per quadrant-update per SM (clock64), err=%s\n", B, (int)W, ms,
         (double)c / upd, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<4, true>(sms);
  run<8, true>(sms);
  run<16, true>(sms);
  run<8, false>(sms);
  run<16, false>(sms);
  return 0;
}
