// exp_mix.cu -- throughput of the softmax exp-phase instruction mix with one
// warp per SMSP (4 warps/CTA, 1 CTA/SM): per element FFMA (scale - max),
// MUFU.EX2, FADD (row sum), and a bf16x2 pack every two elements.
#include <cstdio>
#include <cstdint>
#include "ptx.cuh"
using namespace attn;

__device__ __forceinline__ float ex2_poly_b(float x) {
  const float xc = fmaxf(x, -127.f);
  const float t = xc + 12582912.f;
  const float f = xc - (t - 12582912.f);
  float p = fmaf(0.05517109f, f, 0.24261115f);
  p = fmaf(p, f, 0.6932611f);
  p = fmaf(p, f, 0.99992806f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

template <int kMode>
__global__ void __launch_bounds__(128, 1) k(float* out, int iters, float c, float m) {
  float x[128];
  for (int i = 0; i < 128; ++i) x[i] = 0.001f * (threadIdx.x + i);
  float s0 = 0.f, s1 = 0.f;
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int e = 0; e < 64; ++e) {
      float p0, p1;
      if (kMode == 0) {            // full mix
        p0 = ex2_approx(fmaf(x[2 * e], c, -m));
        p1 = ex2_approx(fmaf(x[2 * e + 1], c, -m));
        s0 += p0; s1 += p1;
        acc ^= pack_bf16x2(p0, p1);
      } else if (kMode == 1) {     // ex2 only (dependent on x through the FFMA)
        p0 = ex2_approx(fmaf(x[2 * e], c, -m));
        p1 = ex2_approx(fmaf(x[2 * e + 1], c, -m));
        acc += __float_as_uint(p0) + __float_as_uint(p1);
      } else if (kMode >= 3) {     // full mix, every kMode-th pair on the FMA pipe (poly)
        const float a0 = fmaf(x[2 * e], c, -m), a1 = fmaf(x[2 * e + 1], c, -m);
        if (e % kMode == kMode - 1) {
          p0 = ex2_poly_b(a0);
          p1 = ex2_poly_b(a1);
        } else {
          p0 = ex2_approx(a0);
          p1 = ex2_approx(a1);
        }
        s0 += p0; s1 += p1;
        acc ^= pack_bf16x2(p0, p1);
      } else {                     // mix without the pack
        p0 = ex2_approx(fmaf(x[2 * e], c, -m));
        p1 = ex2_approx(fmaf(x[2 * e + 1], c, -m));
        s0 += p0; s1 += p1;
      }
    }
    m += 1e-7f;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (float)(t1 - t0) / iters;
  if (s0 + s1 == 1234.5f || acc == 12345u) out[1000 + threadIdx.x] = s0;
}
int main() {
  float* d; cudaMalloc(&d, 4096 * 4);
  const char* names[7] = {"FFMA+EX2+FADD+F2FP", "FFMA+EX2", "FFMA+EX2+FADD", "full, 1/3 poly", "full, 1/4 poly", "full, 1/5 poly", "full, 1/8 poly"};
  for (int mode = 0; mode < 7; ++mode) {
    auto kern = mode == 0 ? k<0> : (mode == 1 ? k<1> : (mode == 2 ? k<2> : (mode == 3 ? k<3> : (mode == 4 ? k<4> : (mode == 5 ? k<5> : k<8>)))));
    kern<<<148, 128>>>(d, 10, 1.4427f, 0.5f);
    kern<<<148, 128>>>(d, 2000, 1.4427f, 0.5f);
    cudaError_t e = cudaDeviceSynchronize();
    float h; cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
    printf("%-22s %s cycles per 128 elements/thread: %.1f  (MUFU bound 1024)\n", names[mode], cudaGetErrorString(e), h);
  }
}
