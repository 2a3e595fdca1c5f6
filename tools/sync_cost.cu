// sync_cost.cu -- cycles of mbarrier test_wait / try_wait on a completed phase and of
// tcgen05.fence::after_thread_sync, with the tensor pipe idle and busy.
#include <cstdio>
#include "ptx.cuh"
using namespace attn;

__global__ void __launch_bounds__(128, 1) k(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&bar2, 1); fence_mbarrier_init(); }
  if (warp == 0) tmem_alloc<512>(&tslot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    mbar_arrive(&bar);  // phase 0 complete
    const uint32_t idesc = idesc_bf16_f32(128, 128, 0, 0);
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 32768);
    long long r[12];
    for (int busy = 0; busy < 2; ++busy) {
      if (busy)
        for (int kk = 0; kk < 8; ++kk)
          mma_ss(tmem, smem_desc_sw128(sa + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                 smem_desc_sw128(sb + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024), idesc, kk > 0);
      long long t0 = clock64();
      mbar_wait_spin(&bar, 0);
      long long t1 = clock64();
      mbar_wait(&bar, 0);
      long long t2 = clock64();
      tc_fence_after();
      long long t3 = clock64();
      mbar_wait_spin(&bar, 0);
      tc_fence_after();
      long long t4 = clock64();
      long long t5 = clock64();
      r[busy * 6 + 0] = t1 - t0; r[busy * 6 + 1] = t2 - t1; r[busy * 6 + 2] = t3 - t2; r[busy * 6 + 3] = t4 - t3;
      r[busy * 6 + 4] = t5 - t4;
      mma_commit(&bar2);
      mbar_wait_spin(&bar2, busy);
      r[busy * 6 + 5] = clock64() - t5;
    }
    if (blockIdx.x == 0) for (int i = 0; i < 12; ++i) out[i] = r[i];
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}
int main() {
  long long *d, h[12];
  cudaMalloc(&d, sizeof(h));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  k<<<148, 128, 96 * 1024>>>(d);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const char* n[6] = {"test_wait(done)", "try_wait(done)", "fence::after", "test_wait+fence", "clock pair", "commit->done"};
  for (int b = 0; b < 2; ++b) { printf(b ? "tensor busy:\n" : "tensor idle:\n"); for (int i = 0; i < 6; ++i) printf("  %-18s %lld\n", n[i], h[b * 6 + i]); }
}
