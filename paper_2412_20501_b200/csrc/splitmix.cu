// SplitMix64 -> uniform fp64 -> fp32 -> bf16 (RNE) input generator, bit-exact
// with ringsim.rng (pkg/src/ringsim/rng.py:25-53) followed by the canonical
// bf16 rounding used on both sides of every parity check.  Lets each rank
// materialise only its own shard of a 1M-token input on the device.
#include <cuda_bf16.h>

#include "tr_internal.h"

namespace tr {

__global__ void __launch_bounds__(256) splitmix_bf16_kernel(uint64_t seed, int64_t first,
                                                            int64_t count, double low,
                                                            double span,
                                                            __nv_bfloat16* __restrict__ dst) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < count; j += stride) {
    uint64_t z = seed + static_cast<uint64_t>(first + j + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    const double u = static_cast<double>(z >> 11) * 0x1.0p-53;
    const double x = __dadd_rn(low, __dmul_rn(span, u));
    dst[j] = __float2bfloat16_rn(__double2float_rn(x));
  }
}

int launch_splitmix(uint64_t seed, int64_t first, int64_t count, double low, double high,
                    void* dst, cudaStream_t s) {
  if (count <= 0) return TR_OK;
  const int64_t blocks = std::min<int64_t>((count + 255) / 256, 148 * 32);
  splitmix_bf16_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(
      seed, first, count, low, high - low, static_cast<__nv_bfloat16*>(dst));
  return cuda_status(cudaGetLastError(), "splitmix launch");
}

}  // namespace tr
