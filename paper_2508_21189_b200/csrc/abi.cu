// Library identity, error strings and device queries of the sketch_b200 C ABI.
#include <atomic>
#include <mutex>
#include <map>
#include <string>
#include <utility>

#include "common.cuh"

namespace skb {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int sm_count() {
  static std::atomic<int> cache[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  int v = cache[dev].load(std::memory_order_relaxed);
  if (v == 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    cache[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

void ensure_context() {
  thread_local int bound = -1;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev == bound) return;
  if (cudaSetDevice(dev) == cudaSuccess) bound = dev;
}

cudaError_t allow_dynamic_smem(const void* kern, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> granted;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  size_t& have = granted[{dev, kern}];
  if (smem <= have) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) have = smem;
  return e;
}

}  // namespace skb

extern "C" int sk_abi_version(void) { return SK_ABI_VERSION; }

extern "C" const char* sk_last_error(void) { return skb::g_last_error.c_str(); }

extern "C" int sk_device_sm_count(int device) {
  int v = 0;
  cudaError_t e = cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) return skb::fail(SK_ECUDA, std::string("sk_device_sm_count: ") + cudaGetErrorString(e));
  return v;
}
