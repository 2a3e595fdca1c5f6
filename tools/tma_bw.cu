// tma_bw.cu -- per-SM TMA load throughput and latency from an L2-resident K/V-like tensor.
// One CTA per SM; a producer lane streams 32 KiB tiles (two 64-column SW128 boxes of 128 rows,
// the prefill kernel's K/V tile) through an R-slot ring, a consumer warp frees each slot as soon
// as it lands (no compute).  Prints bytes/clk/SM and the mean issue->landed latency.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2510_08726_b200/csrc \
//        tools/tma_bw.cu -o build/tma_bw -lcuda && build/tma_bw
#include <cuda.h>
#include <cstdio>
#include "ptx.cuh"
using namespace attn;

constexpr int kTileBytes = 32768;

// mma: 0 none; 1 SS M128 N128 K16 back to back (A, B 64 KiB after the ring); 2 TS (A in TMEM);
//      3 SS M128 N256
__device__ volatile int g_stop[148];
template <int R>
__global__ void __launch_bounds__(384, 1) k(const __grid_constant__ CUtensorMap tm, int ntiles, int S, long long* out,
                                            int mma, int hbm_mode, int st_mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[R], empty[R];
  __shared__ long long t_issue[R];
  __shared__ uint32_t tslot;
  __shared__ volatile int stop;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < R; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    fence_mbarrier_init();
    stop = 0;
  }
  if (warp == 3) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 2) {
    if (mma) {
      const uint32_t sa = smem_u32(smem + R * kTileBytes), sb = sa + 32768;
      const uint32_t id = idesc_bf16_f32(128, mma == 3 ? 256 : 128, 0, 0);
      const uint64_t da = smem_desc_sw128(sa, 16, 1024), db = smem_desc_sw128(sb, 16, 1024);
      int n = 0;
      while (!stop) {
        uint64_t a[8], b[8];
        uint32_t ta[8];
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          a[kk] = da + (uint64_t)((kk >> 2) * 1024 + (kk & 3) * 2);
          b[kk] = db + (uint64_t)((kk >> 2) * 1024 + (kk & 3) * 2);
          ta[kk] = tmem + 256 + kk * 8;
        }
        if (mma == 2) mma_ts_x8(tmem + (n & 1) * 128, ta, b, id, 0u);
        else mma_ss_x8(tmem + (mma == 3 ? 0 : (n & 1) * 128), a, b, id, 0u);
        ++n;
      }
      mma_commit_warp(&empty[0]);   // (drain: any barrier; the kernel ends after this)
    }
  }
  if (warp >= 4 && st_mode) {   // 8 warps of P-like 16-byte swizzled stores (st_mode 2: paced)
    uint8_t* base = smem + R * kTileBytes + 65536;
    const int row = threadIdx.x & 127;
    uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
    while (!stop) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(base + row * 128 + ((c ^ (row & 7)) << 4))),
                     "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
        v.y += 1;
      }
      if (st_mode == 2) __nanosleep(100);
    }
  }
  // hbm_mode 1: every CTA streams its own heads; 2: groups of 16 CTAs stream the same fresh heads in
  // lockstep (the prefill kernel's q-blocks of one head); 3: as 2 plus an L2 prefetch 4 tiles ahead
  const int head = hbm_mode == 1 ? blockIdx.x : hbm_mode >= 2 ? blockIdx.x / 16 : blockIdx.x % 16;
  const int tiles_per_pass = S / 128;
  long long t0 = clock64(), lat = 0;
  if (warp == 0 && lane == 0) {
    const uint64_t pol = policy_evict_last();
    for (int i = 0; i < ntiles; ++i) {
      mbar_wait_spin(&empty[i % R], ((i / R) & 1) ^ 1);
      t_issue[i % R] = clock64();
      mbar_arrive_expect_tx(&full[i % R], kTileBytes);
      uint8_t* dst = smem + (i % R) * kTileBytes;
      const int row = (i % tiles_per_pass) * 128;
      const int hh = hbm_mode == 1 ? head + 148 * (i / tiles_per_pass) : hbm_mode >= 2 ? head + 10 * (i / tiles_per_pass) : head;
      if (hbm_mode == 3 && i + 4 < ntiles) {
        const int i4 = i + 4, r4 = (i4 % tiles_per_pass) * 128, h4 = head + 10 * (i4 / tiles_per_pass);
        for (int bx = 0; bx < 2; ++bx) tma_prefetch_4d(&tm, bx * 64, r4, h4, 0);
      }
      for (int bx = 0; bx < 2; ++bx) tma_load_4d(&tm, &full[i % R], dst + bx * 16384, bx * 64, row, hh, 0, pol);
    }
  } else if (warp == 1 && lane == 0) {
    for (int i = 0; i < ntiles; ++i) {
      mbar_wait_spin(&full[i % R], (i / R) & 1);
      lat += clock64() - t_issue[i % R];
      mbar_arrive(&empty[i % R]);
    }
    out[blockIdx.x * 2] = clock64() - t0;
    out[blockIdx.x * 2 + 1] = lat / ntiles;
    stop = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 3) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

template <int R>
void run(const CUtensorMap& tm, int S, int ntiles, int mma = 0, int hbm = 0, int st = 0) {
  long long* d;
  cudaMalloc(&d, 148 * 2 * sizeof(long long));
  const int smem = R * kTileBytes + 65536 + 32768;
  cudaFuncSetAttribute(k<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 2; ++rep) k<R><<<148, 384, smem>>>(tm, ntiles, S, d, mma, hbm, st);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148 * 2];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double cyc = 0, lat = 0;
  for (int b = 0; b < 148; ++b) { cyc += h[2 * b] / 148.0; lat += h[2 * b + 1] / 148.0; }
  printf("st %d mode %d mma %d ring %d x 32 KiB: %s  %.1f B/clk/SM (%.2f TB/s chip at 1.965 GHz)  mean issue->landed %.0f cyc\n", st, hbm, mma, R,
         cudaGetErrorString(e), (double)ntiles * kTileBytes / cyc, (double)ntiles * kTileBytes / cyc * 148 * 1.965e9 / 1e12,
         lat);
  cudaFree(d);
}

int main() {
  const int H = 148 * 4, S = 4096, D = 128;   // 620 MB: hbm mode streams 4 heads per CTA
  void* buf;
  cudaMalloc(&buf, (size_t)H * S * D * 2);
  cudaMemset(buf, 0, (size_t)H * S * D * 2);
  CUtensorMap tm;
  cuuint64_t dims[4] = {(cuuint64_t)D, (cuuint64_t)S, (cuuint64_t)H, 1};
  cuuint64_t strides[3] = {(cuuint64_t)D * 2, (cuuint64_t)S * D * 2, (cuuint64_t)H * S * D * 2};
  cuuint32_t box[4] = {64, 128, 1, 1}, estr[4] = {1, 1, 1, 1};
  CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, dims, strides, box, estr,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  const int ntiles = 512;
  run<3>(tm, S, ntiles, 0, 0, 0);
  run<3>(tm, S, 128, 0, 1, 0);
  run<3>(tm, S, 128, 0, 2, 0);
  run<3>(tm, S, 128, 0, 3, 0);
  run<3>(tm, S, 128, 1, 2, 1);
  run<3>(tm, S, 128, 1, 3, 1);
  return 0;
}
