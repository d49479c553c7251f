// Shared helpers for the sketch_b200 C ABI: status handling, error strings, launch checks.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "sketch_b200.h"

namespace skb {

// Thread-local last error (sk_last_error); set by fail().
void set_error(const std::string& msg);

inline int fail(int status, const std::string& msg) {
  set_error(msg);
  return status;
}

inline int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    return fail(SK_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
  return SK_OK;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// SM count of the current device (cached per device).
int sm_count();

// Bind the current device's primary context to the calling host thread (once per thread and device).
// The runtime binds it lazily on the first runtime call that needs it; driver-API calls made before
// that (cuTensorMapEncodeTiled) would fail with "invalid context" on a fresh thread (thread pools).
void ensure_context();

// Raise a kernel's dynamic shared-memory limit on the current device to at least `smem`.  The limit
// only ever grows (per device and kernel, under a lock): setting it per launch to that launch's
// size would let one host thread shrink it under another's launch of the same kernel.
cudaError_t allow_dynamic_smem(const void* kern, size_t smem);
template <typename K>
inline cudaError_t allow_smem(K* kern, size_t smem) {
  return allow_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
}

template <typename T>
struct DT;
template <>
struct DT<float> {
  static constexpr int id = SK_F32;
};
template <>
struct DT<double> {
  static constexpr int id = SK_F64;
};

__device__ __forceinline__ float flip_if(float v, uint32_t neg) {
  return __int_as_float(__float_as_int(v) ^ (neg << 31));
}
__device__ __forceinline__ double flip_if(double v, uint32_t neg) {
  return __longlong_as_double(__double_as_longlong(v) ^ ((unsigned long long)neg << 63));
}

}  // namespace skb
