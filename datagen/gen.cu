// gen.cu -- the CUDA twin of datagen/__init__.py: same counter-based
// generator, bit-identical output (integer arithmetic plus one correctly
// rounded fp32 multiply and an integer RNE bf16 rounding).  Holds no attention
// arithmetic; used by bench.py / tests to create large synthetic inputs on the
// device.  C ABI:
//   int datagen_fill(void* dst, long long count, unsigned long long key,
//                    long long start, int bf16, float inv_sigma, cudaStream_t stream);
// writes elements [start, start + count) of stream `key` (bf16 bits when
// bf16 == 1, fp16 bits when bf16 == 2, else fp32).  Returns a cudaError_t value.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace {
constexpr uint64_t G = 0x9E3779B97F4A7C15ull;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ int64_t fields(uint64_t w) {
  return (int64_t)(w & 0xFFFF) + (int64_t)((w >> 16) & 0xFFFF) + (int64_t)((w >> 32) & 0xFFFF) + (int64_t)(w >> 48);
}

__global__ void fill_kernel(void* dst, long long count, uint64_t key, long long start, int bf16, float inv_sigma) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    const uint64_t idx = (uint64_t)(start + i);
    const uint64_t base = key + (2ull * idx + 1ull) * G;
    const int64_t s = fields(mix64(base)) + fields(mix64(base + G)) - 4 * 65535;
    const float x = __fmul_rn((float)s, inv_sigma);  // (float)s is exact: |s| < 2^24
    if (bf16 == 2) {
      static_cast<__half*>(dst)[i] = __float2half_rn(x);
    } else if (bf16) {
      const uint32_t b = __float_as_uint(x);
      const uint32_t r = (b + 0x7FFFu + ((b >> 16) & 1u)) >> 16;
      static_cast<uint16_t*>(dst)[i] = (uint16_t)r;
    } else {
      static_cast<float*>(dst)[i] = x;
    }
  }
}
}  // namespace

extern "C" __attribute__((visibility("default"))) int datagen_fill(void* dst, long long count, unsigned long long key, long long start, int bf16,
                            float inv_sigma, cudaStream_t stream) {
  if (count <= 0) return 0;
  long long blocks = (count + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  fill_kernel<<<(unsigned)blocks, 256, 0, stream>>>(dst, count, key, start, bf16, inv_sigma);
  return (int)cudaGetLastError();
}
