// Semantics check of the TMA row gather (cp.async.bulk.tensor.2d ... tile::gather4): which bytes land
// where for a 2-D float32 tensor map with box {W cols, 1 row}.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/micro/gather4_test tools/micro/gather4_test.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void g4(const __grid_constant__ CUtensorMap tm, int c, int r0, int r1, int r2, int r3, float* out, int n) {
  extern __shared__ __align__(1024) float buf[];
  __shared__ uint64_t bar;
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(buf);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(n * 4));
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5, %6}], [%7];" ::"r"(d),
        "l"(&tm), "r"(c), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(b)
        : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(b));
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = buf[i];
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int rows = 1000, cols = 512;
  std::vector<float> h((size_t)rows * cols);
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j) h[(size_t)i * cols + j] = (float)(i * 1000 + j);
  float *dA, *dO;
  cudaMalloc(&dA, h.size() * 4);
  cudaMemcpy(dA, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&dO, 4096 * 4);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncFn enc = (EncFn)fp;
  for (int W : {128, 256}) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
    cuuint32_t box[2] = {(cuuint32_t)W, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dA, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("W=%d encode=%d\n", W, (int)r);
    const int n = 4 * W;
    g4<<<1, 128, n * 4 + 1024>>>(tm, 128, 5, 900, 3, 999, dO, n);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> o(n);
    cudaMemcpy(o.data(), dO, n * 4, cudaMemcpyDeviceToHost);
    printf("  err=%s  out[0]=%g out[1]=%g out[W-1]=%g out[W]=%g out[2W]=%g out[3W]=%g out[4W-1]=%g\n",
           cudaGetErrorString(e), o[0], o[1], o[W - 1], o[W], o[2 * W], o[3 * W], o[n - 1]);
  }
  return 0;
}
