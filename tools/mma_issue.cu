// mma_issue.cu -- does issuing tcgen05.mma block?  Times the issue of one group
// of 8 M128N128K16 MMAs and its completion (commit -> mbarrier), repeated.
#include <cstdio>
#include "ptx.cuh"
using namespace attn;

__global__ void __launch_bounds__(128, 1) k(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbarrier_init(); }
  if (warp == 0) tmem_alloc<512>(&tslot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_bf16_f32(128, 128, 0, 0);
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 32768);
    for (int rep = 0; rep < 6; ++rep) {
      long long t0 = clock64();
      const int groups = rep < 3 ? 1 : 4;
      for (int g = 0; g < groups; ++g)
        for (int kk = 0; kk < 8; ++kk)
          mma_ss(tmem + (g & 1) * 128, smem_desc_sw128(sa + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                 smem_desc_sw128(sb + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024), idesc, kk > 0);
      long long t1 = clock64();
      mma_commit(&bar);
      long long t2 = clock64();
      mbar_wait_spin(&bar, rep & 1);
      long long t3 = clock64();
      if (blockIdx.x == 0) { out[rep * 4 + 0] = groups; out[rep * 4 + 1] = t1 - t0; out[rep * 4 + 2] = t2 - t1; out[rep * 4 + 3] = t3 - t0; }
    }
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}
int main() {
  long long *d, h[24];
  cudaMalloc(&d, sizeof(h));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  k<<<148, 128, 96 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%s\n", cudaGetErrorString(e));
  for (int r = 0; r < 6; ++r) printf("groups=%lld issue=%lld commit=%lld total(issue->done)=%lld\n", h[r*4], h[r*4+1], h[r*4+2], h[r*4+3]);
}
