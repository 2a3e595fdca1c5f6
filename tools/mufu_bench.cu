// mufu_bench.cu -- MUFU ex2 throughput: f32 vs packed f16x2 / bf16x2 (results per SM per clock).
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
template <int kMode>
__global__ void k(float* out, int iters) {
  uint32_t a[8];
  float f[8];
  for (int i = 0; i < 8; ++i) { f[i] = -0.001f * (threadIdx.x + i); a[i] = 0x3c00bc00u + i; }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (kMode == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i]));
      if (kMode == 1) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[i]));
      if (kMode == 2) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i]));
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += f[i] + __uint_as_float(a[i]);
  if (threadIdx.x == 0) out[blockIdx.x] = (float)(t1 - t0);
  if (s == 1234.5f) out[1000] = s;
}
int main() {
  float* d; cudaMalloc(&d, 4096 * 4);
  const char* names[3] = {"ex2.f32", "ex2.f16x2", "ex2.bf16x2"};
  for (int m = 0; m < 3; ++m) {
    int iters = 2000;
    auto kern = m == 0 ? k<0> : (m == 1 ? k<1> : k<2>);
    kern<<<148, 512>>>(d, 10);
    kern<<<148, 512>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    float h; cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
    double inst = 512.0 * iters * 8;                 // thread-instructions per SM
    double res = inst * (m == 0 ? 1 : 2);            // results per SM
    printf("%-11s %s  thread-instr/clk/SM %.2f  results/clk/SM %.2f\n", names[m], cudaGetErrorString(e), inst / h, res / h);
  }
}
