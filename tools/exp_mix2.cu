// exp_mix2.cu -- softmax exp-phase mix under kernel-like conditions:
// kW softmax warps per SM sub-partition (4*kW warps/CTA, 1 CTA/SM), P packed to
// bf16x2 and stored to shared memory in the swizzled UMMA layout (as the
// P-in-shared-memory kernel does), optional interference warps running the
// row-max phase (FMNMX3 over 128 registers).  Reports SM cycles per 128x128
// tile-equivalent of exponentials (MUFU bound: 1024).
#include <cstdio>
#include <cstdint>
#include "ptx.cuh"
using namespace attn;

__device__ __forceinline__ float ex2_poly_b(float x) {   // degree-3 2^x on the FMA pipe (as fwd_tc.cu)
  const float xc = fmaxf(x, -127.f);
  const float t = xc + 12582912.f;
  const float f = xc - (t - 12582912.f);
  float p = fmaf(0.05517109f, f, 0.24261115f);
  p = fmaf(p, f, 0.6932611f);
  p = fmaf(p, f, 0.99992806f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

template <int kW, bool kStore, int kMaxWarps, bool kMma = false, int kPoly = 0>
__global__ void __launch_bounds__(128 * kW + 32 * kMaxWarps + (kMma ? 32 : 0), 1) k(float* out, int iters, float c, float m) {
  extern __shared__ __align__(1024) uint8_t sp[];   // 64 KiB dynamic
  __shared__ volatile int done;
  if (threadIdx.x == 0) done = 0;
  __syncthreads();
  const int warp = threadIdx.x / 32;
  __shared__ uint32_t tslot;
  __shared__ uint64_t mbar;
  if (kMma) {
    if (warp == 4 * kW + kMaxWarps) {
      tmem_alloc<512>(&tslot);
      if (threadIdx.x % 32 == 0) { mbar_init(&mbar, 1); fence_mbarrier_init(); }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 4 * kW + kMaxWarps) {   // tensor core kept busy: SS M128 N128 K16 MMAs until the exps finish
      const uint32_t tmem = tslot;
      if (threadIdx.x % 32 == 0) {
        const uint32_t idesc = idesc_bf16_f32(128, 128, 0, 0);
        const uint32_t sa = smem_u32(sp), sb = smem_u32(sp + 32768);
        uint32_t ph = 0;
        while (!done) {
          for (int kk = 0; kk < 32; ++kk)
            mma_ss(tmem, smem_desc_sw128(sa + (kk & 1) * 16384 + (kk & 3) * 32, 16, 1024),
                   smem_desc_sw128(sb + (kk & 1) * 16384 + (kk & 3) * 32, 16, 1024), idesc, 1);
          mma_commit(&mbar);
          mbar_wait(&mbar, ph);
          ph ^= 1;
        }
      }
      __syncwarp();
      tc_fence_after();
      tmem_dealloc<512>(tmem);
      return;
    }
  }
  float x[128];
  for (int i = 0; i < 128; ++i) x[i] = 0.001f * (threadIdx.x + i);
  if (warp >= 4 * kW) {      // interference: max phase over fresh registers
    float mx = 0.f;
    while (!done) {
#pragma unroll
      for (int i = 0; i < 128; i += 2) mx = fmaxf(mx, fmaxf(x[i], x[i + 1]));
      x[mx > 1e30f ? 0 : 1] += 1e-9f;
    }
    if (mx == 1234.f) out[2000] = mx;
    return;
  }
  const int r = threadIdx.x & 127;
  uint8_t* base = sp + (threadIdx.x >= 128 ? 32768 : 0);
  float s0 = 0.f, s1 = 0.f;
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c0 = 0; c0 < 128; c0 += 32) {
      uint32_t pk[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        float p0, p1;
        if (kPoly > 0 && e % kPoly == kPoly - 1) {
          p0 = ex2_poly_b(fmaf(x[c0 + 2 * e], c, -m));
          p1 = ex2_poly_b(fmaf(x[c0 + 2 * e + 1], c, -m));
        } else {
          p0 = ex2_approx(fmaf(x[c0 + 2 * e], c, -m));
          p1 = ex2_approx(fmaf(x[c0 + 2 * e + 1], c, -m));
        }
        s0 += p0; s1 += p1;
        pk[e] = pack_bf16x2(p0, p1);
      }
      if (kStore) {
        uint8_t* rowp = base + (c0 >> 6) * 16384 + r * 128;
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const int ch = ((c0 & 63) >> 3) + q4;
          *reinterpret_cast<uint4*>(rowp + ((ch ^ (r & 7)) << 4)) = make_uint4(pk[4 * q4], pk[4 * q4 + 1], pk[4 * q4 + 2], pk[4 * q4 + 3]);
        }
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) acc ^= pk[e];
      }
    }
    m += 1e-7f;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) {
    out[blockIdx.x] = (float)(t1 - t0) / iters;
    done = 1;
  }
  if (s0 + s1 == 1234.5f || acc == 12345u) out[1000 + threadIdx.x] = s0;
}

template <int kW, bool kStore, int kMaxWarps, bool kMma = false, int kPoly = 0>
void run(const char* name, float* d) {
  auto kern = k<kW, kStore, kMaxWarps, kMma, kPoly>;
  const int threads = 128 * kW + 32 * kMaxWarps + (kMma ? 32 : 0);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  kern<<<148, threads, 65536>>>(d, 10, 1.4427f, 0.5f);
  kern<<<148, threads, 65536>>>(d, 1000, 1.4427f, 0.5f);
  cudaError_t e = cudaDeviceSynchronize();
  float h; cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
  // each softmax warp handled 128 elements/thread per iteration; kW tiles of 128 rows per iteration
  printf("%-40s %s  cycles per 128x128 tile: %.1f  (MUFU bound 1024)\n", name, cudaGetErrorString(e), h / kW);
}

int main() {
  float* d; cudaMalloc(&d, 4096 * 4);
  run<1, false, 0>("1 warp/SMSP, no store", d);
  run<1, true, 0>("1 warp/SMSP, STS P", d);
  run<2, false, 0>("2 warps/SMSP, no store", d);
  run<2, true, 0>("2 warps/SMSP, STS P", d);
  run<1, true, 4>("1 warp/SMSP, STS P, +4 max warps", d);
  run<2, true, 4>("2 warps/SMSP, STS P, +4 max warps", d);
  run<1, true, 0, true>("1 warp/SMSP, STS P, +MMA", d);
  run<2, true, 0, true>("2 warps/SMSP, STS P, +MMA", d);
  run<1, true, 4, true>("1 warp/SMSP, STS P, +4 max, +MMA", d);
  run<1, true, 0, true, 4>("1 warp, STS, MMA, poly 1/4", d);
  run<1, true, 0, true, 8>("1 warp, STS, MMA, poly 1/8", d);
  run<1, true, 0, true, 16>("1 warp, STS, MMA, poly 1/16", d);
  run<2, true, 0, true, 4>("2 warps, STS, MMA, poly 1/4", d);
  run<2, true, 0, true, 8>("2 warps, STS, MMA, poly 1/8", d);
}
