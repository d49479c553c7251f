// Device-side NumPy Philox stream: the 32-bit outputs of numpy.random.Philox (Philox4x64-10) at
// any stream position, so test matrices are drawn on the GPU bit-identically to the reference's
// host draws.
//
// NumPy's generator (numpy/random/src/philox/philox.h): next_uint64 increments the 256-bit counter
// and then emits the 4 words of philox4x64_10(counter, key) in order; next_uint32 splits each
// 64-bit word into its low then its high half. A fresh generator starts with an empty buffer, so
// 32-bit output number p comes from word (p / 2) % 4 of the block for counter + 1 + p / 8, half
// p % 2. Each thread produces the 8 outputs of one block.
#include "common.cuh"

namespace skb {
namespace {

__device__ __forceinline__ void mulhilo64(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
  lo = a * b;
  hi = __umul64hi(a, b);
}

__device__ __forceinline__ void philox4x64_10(uint64_t (&c)[4], uint64_t k0, uint64_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo64(0xD2E7470EE14C6C93ull, c[0], hi0, lo0);
    mulhilo64(0xCA5A826395121157ull, c[2], hi1, lo1);
    const uint64_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += 0x9E3779B97F4A7C15ull;
    k1 += 0xBB67AE8584CAA73Bull;
  }
}

// out[i] = 32-bit output number (first + i) of the stream, i < count; first % 8 == 0.
__global__ void philox_u32_kernel(uint64_t k0, uint64_t k1, uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3,
                                  uint64_t first_block, int64_t count, uint32_t* __restrict__ out) {
  const int64_t nblocks = (count + 7) / 8;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nblocks;
       b += (int64_t)gridDim.x * blockDim.x) {
    // counter + 1 + first_block + b (256-bit add with carry)
    const uint64_t add = 1ull + first_block + (uint64_t)b;
    uint64_t c[4];
    c[0] = c0 + add;
    uint64_t carry = c[0] < add ? 1ull : 0ull;
    c[1] = c1 + carry;
    carry = (carry && c[1] == 0) ? 1ull : 0ull;
    c[2] = c2 + carry;
    carry = (carry && c[2] == 0) ? 1ull : 0ull;
    c[3] = c3 + carry;
    philox4x64_10(c, k0, k1);
    const int64_t base = b * 8;
    if (base + 8 <= count) {
      uint4* o = reinterpret_cast<uint4*>(out + base);
      o[0] = make_uint4((uint32_t)c[0], (uint32_t)(c[0] >> 32), (uint32_t)c[1], (uint32_t)(c[1] >> 32));
      o[1] = make_uint4((uint32_t)c[2], (uint32_t)(c[2] >> 32), (uint32_t)c[3], (uint32_t)(c[3] >> 32));
    } else {
#pragma unroll
      for (int w = 0; w < 8; ++w)
        if (base + w < count) out[base + w] = (uint32_t)(c[w >> 1] >> (32 * (w & 1)));
    }
  }
}

}  // namespace
}  // namespace skb

extern "C" int sk_philox_u32(const uint64_t* key2, const uint64_t* counter4, uint64_t first, int64_t count,
                             uint32_t* out, void* stream) {
  using namespace skb;
  if (!key2 || !counter4 || (count > 0 && !out) || count < 0) return fail(SK_EINVAL, "sk_philox_u32: bad arguments");
  if (first % 8) return fail(SK_EINVAL, "sk_philox_u32: first must be a multiple of 8");
  if ((reinterpret_cast<uintptr_t>(out) & 15) != 0) return fail(SK_EINVAL, "sk_philox_u32: out must be 16-byte aligned");
  if (count == 0) return SK_OK;
  const int64_t nblocks = (count + 7) / 8;
  int64_t grid = (nblocks + 255) / 256;
  if (grid > 32 * (int64_t)sm_count()) grid = 32 * (int64_t)sm_count();
  philox_u32_kernel<<<(unsigned)grid, 256, 0, as_stream(stream)>>>(key2[0], key2[1], counter4[0], counter4[1],
                                                                    counter4[2], counter4[3], first / 8, count, out);
  return check_launch("sk_philox_u32");
}
