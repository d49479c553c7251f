// Library identity, error strings and device queries of the sketch_b200 C ABI.
#include <mutex>
#include <string>

#include "common.cuh"

namespace skb {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int sm_count() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (cache[dev] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    cache[dev] = v;
  }
  return cache[dev];
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
