// Microbenchmark: read bandwidth of a persistent per-SM TMA bulk-copy ring (no compute), to size
// the SRTT row ring. nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_ring tma_ring.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void ring(const uint8_t* A, int64_t nchunks, int chunk, int ns, unsigned* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)ns * chunk);
  uint64_t* empty = full + ns;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ns; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0; uint32_t ph = 0;
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
      asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}" ::"r"(su32(&empty[s])), "r"(ph ^ 1));
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(chunk));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(sm + (size_t)s * chunk)), "l"(A + c * chunk), "r"(chunk), "r"(su32(&full[s])) : "memory");
      if (++s == ns) { s = 0; ph ^= 1; }
    }
  } else if (threadIdx.x == 32) {
    int s = 0; uint32_t ph = 0; unsigned acc = 0;
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
      asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}" ::"r"(su32(&full[s])), "r"(ph));
      acc += *reinterpret_cast<volatile unsigned*>(sm + (size_t)s * chunk);
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])));
      if (++s == ns) { s = 0; ph ^= 1; }
    }
    if (acc == 0x12345678) sink[0] = acc;
  }
}

// same ring, rows of 32 KB loaded as 4 tensor boxes of [64 lines][128 B] (stride 512 B, SWIZZLE_128B)
__global__ void ring4d(const __grid_constant__ CUtensorMap m, int64_t nrows, int ns, unsigned* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int chunk = 32768;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)ns * chunk);
  uint64_t* empty = full + ns;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ns; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0; uint32_t ph = 0;
    for (int64_t c = blockIdx.x; c < nrows; c += gridDim.x) {
      asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}" ::"r"(su32(&empty[s])), "r"(ph ^ 1));
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(chunk));
      for (int p = 0; p < 4; ++p)
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                     ::"r"(su32(sm + (size_t)s * chunk + p * 8192)), "l"(&m), "r"(0), "r"(p), "r"(0), "r"((int)c), "r"(su32(&full[s])) : "memory");
      if (++s == ns) { s = 0; ph ^= 1; }
    }
  } else if (threadIdx.x == 32) {
    int s = 0; uint32_t ph = 0; unsigned acc = 0;
    for (int64_t c = blockIdx.x; c < nrows; c += gridDim.x) {
      asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}" ::"r"(su32(&full[s])), "r"(ph));
      acc += *reinterpret_cast<volatile unsigned*>(sm + (size_t)s * chunk);
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])));
      if (++s == ns) { s = 0; ph ^= 1; }
    }
    if (acc == 0x12345678) sink[0] = acc;
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const size_t bytes = (size_t)2 << 30;
  uint8_t* A; unsigned* sink;
  cudaMalloc(&A, bytes); cudaMalloc(&sink, 4);
  cudaMemset(A, 1, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int chunks[] = {32768};
  for (int chunk : chunks) {
    for (int ns = 2; ns <= 12; ns += (ns < 6 ? 1 : 2)) {
      size_t smem = (size_t)ns * chunk + 2 * ns * 8;
      if (smem > 227 * 1024) continue;
      int64_t n = bytes / chunk;
      for (int grid : {sms, 2 * sms}) {
        if (grid == 2 * sms && smem > 113 * 1024) continue;
        for (int i = 0; i < 2; ++i) ring<<<grid, 64, smem>>>(A, n, chunk, ns, sink);
        cudaEventRecord(e0);
        for (int i = 0; i < 10; ++i) ring<<<grid, 64, smem>>>(A, n, chunk, ns, sink);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("chunk %6d ns %2d grid %4d  inflight/SM %4zu KB  %.4f ms  %.0f GB/s\n", chunk, ns, grid,
               (size_t)ns * chunk * (grid / sms) / 1024, ms / 10, bytes / (ms / 10) / 1e6);
      }
    }
  }
  {
    void* ptr = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q);
    EncFn fn = (EncFn)ptr;
    int64_t nrows = bytes / 32768;
    for (int l2p = 0; l2p < 4; ++l2p) {
      CUtensorMap m;
      cuuint64_t dims[4] = {32, 4, 64, (cuuint64_t)nrows};
      cuuint64_t strides[3] = {128, 512, 32768};
      cuuint32_t box[4] = {32, 1, 64, 1};
      cuuint32_t estr[4] = {1, 1, 1, 1};
      CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, A, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, (CUtensorMapL2promotion)l2p, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); break; }
      cudaFuncSetAttribute(ring4d, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      for (int ns = 3; ns <= 6; ++ns) {
        size_t smem = (size_t)ns * 32768 + 2 * ns * 8;
        for (int i = 0; i < 2; ++i) ring4d<<<sms, 64, smem>>>(m, nrows, ns, sink);
        cudaEventRecord(e0);
        for (int i = 0; i < 10; ++i) ring4d<<<sms, 64, smem>>>(m, nrows, ns, sink);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("4d rows l2promo %d ns %d  %.4f ms  %.0f GB/s\n", l2p, ns, ms / 10, bytes / (ms / 10) / 1e6);
      }
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(err));
  return 0;
}
