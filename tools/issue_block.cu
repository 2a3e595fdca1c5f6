// issue_block.cu -- does a warp blocked in tcgen05.mma issue slow the OTHER warps of its SM
// sub-partition?  One CTA per SM: warps 0-3 run a fixed softmax-like mix (FFMA2, MUFU ex2,
// F2FP, STS; one warp per SMSP), a sixth warp issues a long stream of M128 N128 K16 MMAs in
// one of several ways.  Prints each worker warp's duration (cycles, mean over SMs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2510_08726_b200/csrc \
//        tools/issue_block.cu -o build/issue_block && build/issue_block
#include <cstdio>
#include "ptx.cuh"
using namespace attn;

constexpr int kMmas = 768;
__device__ int g_fence;

// Eight MMAs into one accumulator from ONE asm block (one elect.sync for the batch).
__device__ __forceinline__ void mma8_ss(uint32_t d, const uint64_t (&a)[8], const uint64_t (&b)[8], uint32_t idesc,
                                        uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p, q, e;\n .reg .b32 r;\n setp.ne.b32 p, %2, 0;\n setp.eq.b32 q, %2, %2;\n"
      " elect.sync r|e, 0xffffffff;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %3, %11, %1, p;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %4, %12, %1, q;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %5, %13, %1, q;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %6, %14, %1, q;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %7, %15, %1, q;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %8, %16, %1, q;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %9, %17, %1, q;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %10, %18, %1, q;\n}\n" ::"r"(d),
      "r"(idesc), "r"(acc), "l"(a[0]), "l"(a[1]), "l"(a[2]), "l"(a[3]), "l"(a[4]), "l"(a[5]), "l"(a[6]), "l"(a[7]),
      "l"(b[0]), "l"(b[1]), "l"(b[2]), "l"(b[3]), "l"(b[4]), "l"(b[5]), "l"(b[6]), "l"(b[7])
      : "memory");
}

__device__ __forceinline__ void work(int iters, float seed, uint8_t* st, float* sink) {
  float a[8], s0 = 0.f, s1 = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + i * 0.01f;
  for (int it = 0; it < iters; ++it) {
    uint32_t pk[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float x0, x1;
      fma2_bc(x0, x1, a[2 * e], a[2 * e + 1], 0.999f, -0.5f);
      const float p0 = ex2_approx(x0), p1 = ex2_approx(x1);
      add2_acc(s0, s1, p0, p1);
      pk[e] = pack_bf16x2(p0, p1);
      a[2 * e] = x0 * 0.5f + 0.25f;
      a[2 * e + 1] = x1 * 0.5f + 0.25f;
    }
    *reinterpret_cast<uint4*>(st + ((it & 7) << 4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    if (g_fence && (it & 15) == 15) fence_proxy_async_smem();   // P-tile hand-off as in the kernel
  }
  *sink = s0 + s1;
}

// mode: 0 issuer idle; 1 warp-wide elect issue (kernel style); 2 lane-0 branch issue;
//       3 warp-wide, N = 256 (half the instructions); 4 warp-wide with commit+try_wait every 4 MMAs
template <int NW, bool kLow>   // NW worker warps; issuer = warp NW (highest id) or warp 0 (kLow)
__global__ void __launch_bounds__(320, 1) k(int mode, int iters, long long* out, float* sink) {
  constexpr int kIssuerWarp = kLow ? 0 : NW;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int alloc_warp = NW + 1;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbarrier_init(); }
  if (warp == alloc_warp) tmem_alloc<512>(&tslot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tslot;
  long long t0 = clock64();
  if (warp == kIssuerWarp) {
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 65536);
    const uint32_t id128 = idesc_bf16_f32(128, 128, 0, 0), id256 = idesc_bf16_f32(128, 256, 0, 0);
    if (mode == 1 || mode == 4) {
      for (int m = 0; m < kMmas; ++m) {
        const int kk = m & 7;
        mma_ss_warp(tmem + ((m >> 3) & 1) * 128, smem_desc_sw128(sa + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                    smem_desc_sw128(sb + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024), id128, kk > 0);
        if (mode == 4 && (m & 3) == 3) {
          mma_commit_warp(&bar);
          mbar_wait(&bar, (m >> 2) & 1);
        }
      }
    } else if (mode == 2) {
      if (lane == 0)
        for (int m = 0; m < kMmas; ++m) {
          const int kk = m & 7;
          mma_ss(tmem + ((m >> 3) & 1) * 128, smem_desc_sw128(sa + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                 smem_desc_sw128(sb + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024), id128, kk > 0);
        }
      __syncwarp();
    } else if (mode == 5) {
      const uint64_t da = smem_desc_sw128(sa, 16, 1024), db = smem_desc_sw128(sb, 16, 1024);
      for (int g = 0; g < kMmas / 8; ++g) {
        uint64_t a[8], b[8];
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          a[kk] = da + (uint64_t)((kk >> 2) * 1024 + (kk & 3) * 2);
          b[kk] = db + (uint64_t)((kk >> 2) * 1024 + (kk & 3) * 2);
        }
        mma8_ss(tmem + (g & 1) * 128, a, b, id128, 0u);
      }
    } else if (mode == 3) {
      for (int m = 0; m < kMmas / 2; ++m) {
        const int kk = m & 7;
        mma_ss_warp(tmem + ((m >> 3) & 1) * 256, smem_desc_sw128(sa + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                    smem_desc_sw128(sb + (kk >> 2) * 32768 + (kk & 3) * 32, 16, 1024), id256, kk > 0);
      }
    }
    mma_commit_warp(&bar);
    mbar_wait(&bar, mode == 4 ? ((kMmas / 4) & 1) : 0);
  } else if (warp <= NW) {
    work(iters, (float)threadIdx.x * 1e-3f, smem + 131072 + warp * 256 + (lane & 1) * 128, sink + blockIdx.x * 320 + threadIdx.x);
  }
  long long t1 = clock64();
  if (lane == 0) out[blockIdx.x * 10 + warp] = t1 - t0;
  tc_fence_before(); __syncthreads();
  if (warp == alloc_warp) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

template <int NW, bool kLow>
void run(const char* name, int mode, int iters) {
  long long* d; float* sink;
  cudaMalloc(&d, 148 * 10 * sizeof(long long));
  cudaMemset(d, 0, 148 * 10 * sizeof(long long));
  cudaMalloc(&sink, 148 * 320 * sizeof(float));
  constexpr int nthr = (NW + 2) * 32;
  cudaFuncSetAttribute(k<NW, kLow>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  k<NW, kLow><<<148, nthr, 160 * 1024>>>(mode, iters, d, sink);
  k<NW, kLow><<<148, nthr, 160 * 1024>>>(mode, iters, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148 * 10];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double m[10] = {0};
  for (int b = 0; b < 148; ++b) for (int w = 0; w < 10; ++w) m[w] += h[b * 10 + w] / 148.0;
  printf("%-36s %s issuer w%d: ", name, cudaGetErrorString(e), kLow ? 0 : NW);
  for (int w = 0; w < NW + 1; ++w) printf("w%d=%6.0f ", w, m[w]);
  printf("\n");
  cudaFree(d); cudaFree(sink);
}

int main() {
  const int iters = 700;
  for (int f = 0; f < 2; ++f) {
  cudaMemcpyToSymbol(g_fence, &f, sizeof(int));
  printf("--- workers fence.proxy.async every 16 iterations: %d\n", f);
  run<4, false>("4w mode0 issuer idle", 0, iters);
  run<4, false>("4w mode1 warp-wide elect", 1, iters);
  run<4, false>("4w mode2 lane0 branch", 2, iters);
  run<4, false>("4w mode3 warp-wide N256", 3, iters);
  run<4, false>("4w mode4 commit+wait per 4", 4, iters);
  run<4, true>("4w low-id issuer mode1", 1, iters);
  run<4, false>("4w mode5 batched elect x8", 5, iters);
  run<8, false>("8w mode0 issuer idle", 0, iters);
  run<8, false>("8w mode1 warp-wide elect", 1, iters);
  run<8, false>("8w mode2 lane0 branch", 2, iters);
  run<8, false>("8w mode3 N256", 3, iters);
  run<8, true>("8w low-id issuer mode1", 1, iters);
  run<8, false>("8w mode5 batched elect x8", 5, iters);
  }
  return 0;
}
