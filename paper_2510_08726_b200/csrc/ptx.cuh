// ptx.cuh -- thin inline-PTX wrappers for sm_100a: mbarrier, TMA (bulk tensor
// and 1-D bulk copies), tcgen05 (TMEM alloc, MMA, commit, ld/st, fences),
// plus the UMMA shared-memory / instruction descriptors.
//
// Descriptor bit layouts follow the sm_100 tcgen05 matrix-descriptor and
// instruction-descriptor formats (PTX ISA 8.6 "tcgen05 ... descriptors").
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

#ifndef ATTN_WATCHDOG_SPINS
#define ATTN_WATCHDOG_SPINS (1u << 26)
#endif
// The watchdog traps a wait that never completes (a hung kernel becomes a launch error).  Its
// printf (block, thread, barrier) is a debug option: the vprintf call inside every wait loop
// makes the hot loops respect the call ABI, which costs registers (spills) in the prefill kernels.
#ifndef ATTN_WATCHDOG_PRINTF
#define ATTN_WATCHDOG_PRINTF 0
#endif

namespace attn {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t warp_id() { return threadIdx.x >> 5; }
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n .reg .b32 r;\n .reg .pred p;\n elect.sync r|p, 0xffffffff;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(pred));
  return pred != 0;
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbarrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Blocking wait with a watchdog: a protocol bug traps (error reported to the
// host) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t spins = 0;
  while (!mbar_try_wait(bar, parity)) {
    if (++spins > ATTN_WATCHDOG_SPINS) {
#if ATTN_WATCHDOG_PRINTF
      printf("attn watchdog: block (%d,%d,%d) thread %d stuck on mbarrier %p parity %u\n", blockIdx.x,
             blockIdx.y, blockIdx.z, threadIdx.x, bar, parity);
#endif
      __trap();
    }
  }
}

// Polling wait (mbarrier.test_wait): no suspend/wake-up latency; for the
// single-thread producer / MMA roles that sit on their own high-priority warps.
__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
  uint32_t spins = 0;
  while (!mbar_test_wait(bar, parity)) {
    if (++spins > 16u * ATTN_WATCHDOG_SPINS) {
#if ATTN_WATCHDOG_PRINTF
      printf("attn watchdog (spin): block (%d,%d,%d) thread %d stuck on mbarrier %p parity %u\n", blockIdx.x,
             blockIdx.y, blockIdx.z, threadIdx.x, bar, parity);
#endif
      __trap();
    }
  }
}

// ---------------------------------------------------------------- named barriers
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ void named_bar_arrive(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------- TMA
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(m) : "memory");
}
__device__ __forceinline__ void tma_load_4d(const CUtensorMap* m, uint64_t* bar, void* dst, int c0, int c1,
                                            int c2, int c3, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(smem_u32(dst)),
      "l"(m), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "l"(policy)
      : "memory");
}
// Bring a tensor tile into L2 ahead of its TMA load (no shared memory involved).
__device__ __forceinline__ void tma_prefetch_4d(const CUtensorMap* m, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global [%0, {%1, %2, %3, %4}];" ::"l"(m), "r"(c0), "r"(c1),
               "r"(c2), "r"(c3)
               : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* m, const void* src, int c0, int c1, int c2,
                                             int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(m),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// 1-D bulk copy global -> shared, completion counted in bytes on `bar`.
__device__ __forceinline__ void bulk_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                             uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
      "%4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// ---------------------------------------------------------------- tcgen05
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem) {  // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {  // whole warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem]^T-ish per descriptors (kind::f16, bf16 in, fp32 acc).
__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// A operand from TMEM.
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Warp-wide variants: every lane executes the instruction with warp-uniform
// operands and one elected lane issues it, so the compiler keeps descriptors
// in uniform registers (no per-lane broadcast loop around each MMA).
__device__ __forceinline__ void mma_ss_warp(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p, e;\n .reg .b32 r;\n setp.ne.b32 p, %4, 0;\n elect.sync r|e, 0xffffffff;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_ts_warp(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p, e;\n .reg .b32 r;\n setp.ne.b32 p, %4, 0;\n elect.sync r|e, 0xffffffff;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// A whole K loop of one accumulator (4 or 8 MMAs) from ONE asm block with ONE elect.sync.
// Per-MMA elect.sync makes ptxas wrap every UTCHMMA in its own elect/branch loop; with another
// warp on the sub-partition that issue stream ran at ~140 cycles per M128 N128 K16 MMA (64 is
// the tensor rate) and stole ~20 % of the sub-partition's issue slots.  The batched form issues
// at the tensor rate and costs the neighbour warps ~3 % (tools/issue_block.cu, r2).
// `acc` = 0: the first MMA overwrites D (enable-input-d false), the rest accumulate.
#define ATTN_MMA_BATCH_HEAD                                                                   \
  "{\n .reg .pred p, q, e;\n .reg .b32 r;\n setp.ne.b32 p, %2, 0;\n setp.eq.b32 q, %2, %2;\n" \
  " elect.sync r|e, 0xffffffff;\n"
__device__ __forceinline__ void mma_ss_x8(uint32_t d, const uint64_t (&a)[8], const uint64_t (&b)[8], uint32_t idesc,
                                          uint32_t acc) {
  asm volatile(ATTN_MMA_BATCH_HEAD
               " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %3, %11, %1, p;\n"
               " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %4, %12, %1, q;\n"
               " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %5, %13, %1, q;\n"
               " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %6, %14, %1, q;\n"
               " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %7, %15, %1, q;\n"
               " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %8, %16, %1, q;\n"
               " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %9, %17, %1, q;\n"
               " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %10, %18, %1, q;\n}\n" ::"r"(d),
               "r"(idesc), "r"(acc), "l"(a[0]), "l"(a[1]), "l"(a[2]), "l"(a[3]), "l"(a[4]), "l"(a[5]), "l"(a[6]),
               "l"(a[7]), "l"(b[0]), "l"(b[1]), "l"(b[2]), "l"(b[3]), "l"(b[4]), "l"(b[5]), "l"(b[6]), "l"(b[7])
               : "memory");
}
__device__ __forceinline__ void mma_ss_x4(uint32_t d, const uint64_t (&a)[4], const uint64_t (&b)[4], uint32_t idesc,
                                          uint32_t acc) {
  asm volatile(ATTN_MMA_BATCH_HEAD
               " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %3, %7, %1, p;\n"
               " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %4, %8, %1, q;\n"
               " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %5, %9, %1, q;\n"
               " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %6, %10, %1, q;\n}\n" ::"r"(d),
               "r"(idesc), "r"(acc), "l"(a[0]), "l"(a[1]), "l"(a[2]), "l"(a[3]), "l"(b[0]), "l"(b[1]), "l"(b[2]),
               "l"(b[3])
               : "memory");
}
// A operand from TMEM (a[k] = TMEM addresses).
__device__ __forceinline__ void mma_ts_x4(uint32_t d, const uint32_t (&a)[4], const uint64_t (&b)[4], uint32_t idesc,
                                          uint32_t acc) {
  asm volatile(ATTN_MMA_BATCH_HEAD
               " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%3], %7, %1, p;\n"
               " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%4], %8, %1, q;\n"
               " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%5], %9, %1, q;\n"
               " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%6], %10, %1, q;\n}\n" ::"r"(d),
               "r"(idesc), "r"(acc), "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "l"(b[0]), "l"(b[1]), "l"(b[2]),
               "l"(b[3])
               : "memory");
}
__device__ __forceinline__ void mma_ts_x8(uint32_t d, const uint32_t (&a)[8], const uint64_t (&b)[8], uint32_t idesc,
                                          uint32_t acc) {
  asm volatile(ATTN_MMA_BATCH_HEAD
               " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%3], %11, %1, p;\n"
               " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%4], %12, %1, q;\n"
               " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%5], %13, %1, q;\n"
               " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%6], %14, %1, q;\n"
               " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%7], %15, %1, q;\n"
               " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%8], %16, %1, q;\n"
               " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%9], %17, %1, q;\n"
               " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%10], %18, %1, q;\n}\n" ::"r"(d),
               "r"(idesc), "r"(acc), "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]),
               "r"(a[7]), "l"(b[0]), "l"(b[1]), "l"(b[2]), "l"(b[3]), "l"(b[4]), "l"(b[5]), "l"(b[6]), "l"(b[7])
               : "memory");
}
#undef ATTN_MMA_BATCH_HEAD

__device__ __forceinline__ void mma_commit_warp(uint64_t* bar) {
  asm volatile(
      "{\n .reg .pred e;\n .reg .b32 r;\n elect.sync r|e, 0xffffffff;\n"
      " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(bar))
      : "memory");
}

// Arrive (once) on `bar` when all previously issued tcgen05 async ops of this thread complete.
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// 32 lanes x 32 columns of 32-bit: thread t of the warp gets columns [c, c+32) of lane (base + t).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
      "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
      "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ---------------------------------------------------------------- descriptors
// Shared-memory matrix descriptor, 128-byte swizzle (layout type 2), sm_100 version 1.
//   start: smem byte address; lbo/sbo: byte offsets (multiples of 16).
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t start, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((start >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;  // descriptor version (sm_100)
  d |= 2ull << 61;  // SWIZZLE_128B
  return d;
}
// Shared-memory matrix descriptor, no swizzle, K-major: core matrices of 8 rows x 16 B stored
// contiguously (128 B); lbo = byte stride between core matrices along K, sbo = along M/N.
__device__ __forceinline__ uint64_t smem_desc_nosw(uint32_t start, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((start >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;  // descriptor version (sm_100); layout type 0 = SWIZZLE_NONE
  return d;
}
// Instruction descriptor for kind::f16 with fp16 (fmt 0) or bf16 (fmt 1) A/B and fp32 D.
__host__ __device__ constexpr uint32_t idesc_f16_f32(uint32_t M, uint32_t N, uint32_t a_mn, uint32_t b_mn,
                                                     bool bf16) {
  return (1u << 4) | ((bf16 ? 1u : 0u) << 7) | ((bf16 ? 1u : 0u) << 10) | (a_mn << 15) | (b_mn << 16) |
         ((N >> 3) << 17) | ((M >> 4) << 24);
}
// Instruction descriptor for kind::f16 with bf16 A/B and fp32 D.
//   a_mn / b_mn: 1 if the operand is MN-major (else K-major).
__host__ __device__ constexpr uint32_t idesc_bf16_f32(uint32_t M, uint32_t N, uint32_t a_mn, uint32_t b_mn) {
  return (1u << 4)            // D format f32
         | (1u << 7)          // A format bf16
         | (1u << 10)         // B format bf16
         | (a_mn << 15) | (b_mn << 16) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

// ---------------------------------------------------------------- math helpers
// Packed fp32x2 arithmetic (sm_100: FFMA2 / FADD2 -- one issue slot for two lanes' worth).
__device__ __forceinline__ unsigned long long f32x2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f32x2_split(unsigned long long r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
// (d0, d1) = (a0, a1) * b + c
__device__ __forceinline__ void fma2_bc(float& d0, float& d1, float a0, float a1, float b, float c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f32x2(a0, a1)), "l"(f32x2(b, b)), "l"(f32x2(c, c)));
  f32x2_split(d, d0, d1);
}
// (s0, s1) += (a0, a1)
__device__ __forceinline__ void add2_acc(float& s0, float& s1, float a0, float a1) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f32x2(s0, s1)), "l"(f32x2(a0, a1)));
  f32x2_split(d, s0, s1);
}

// 2^a0, 2^a1 on the FMA/ALU pipes (MUFU offload, FA4-style): a = k + f with k = round(a)
// (the 1.5*2^23 + 127 add leaves k + 127 in the low mantissa bits), 2^f by a degree-3
// minimax polynomial on f in [-1/2, 1/2] (relative error 7.5e-5, below the 2^-9 half-ulp
// of the bf16 / 2^-11 of the fp16 P it feeds), times 2^k built in the exponent field.
// a is clamped to >= -127, where 2^k's bit pattern is +0.0: masked (-inf) inputs give an
// exact 0 like ex2.approx; otherwise a < -126 underflows to <= 2^-126 (true value
// < 2^-126).  Packed f32x2 arithmetic: 9 FMA-pipe / 4 ALU instructions per pair.
__device__ __forceinline__ void ex2_poly2(float a0, float a1, float& r0, float& r1) {
  constexpr float kMagic = 12582912.f + 127.f;   // 1.5 * 2^23 + 127
  const float c0 = fmaxf(a0, -127.f), c1 = fmaxf(a1, -127.f);
  unsigned long long t, u, f, p;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(f32x2(c0, c1)), "l"(f32x2(kMagic, kMagic)));
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(u) : "l"(t), "l"(f32x2(kMagic, kMagic)));
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(f) : "l"(f32x2(c0, c1)), "l"(u));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(p) : "l"(f), "l"(f32x2(0.05517109f, 0.05517109f)),
      "l"(f32x2(0.24261115f, 0.24261115f)));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(p) : "l"(p), "l"(f), "l"(f32x2(0.6932611f, 0.6932611f)));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(p) : "l"(p), "l"(f), "l"(f32x2(0.99992806f, 0.99992806f)));
  float t0, t1;
  f32x2_split(t, t0, t1);
  const unsigned long long sc = f32x2(__uint_as_float(__float_as_uint(t0) << 23), __uint_as_float(__float_as_uint(t1) << 23));
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(p), "l"(sc));
  f32x2_split(r, r0, r1);
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

__device__ __forceinline__ uint32_t pack_f16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
// 16-bit packing in the element type of the kernel (bf16 or fp16), RNE.
template <bool kF16>
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  if constexpr (kF16) return pack_f16x2(lo, hi);
  else return pack_bf16x2(lo, hi);
}
// x rounded (RNE) to the kernel's 16-bit element type, as a float.
template <bool kF16>
__device__ __forceinline__ float round16(float x) {
  const uint32_t u = pack2<kF16>(x, 0.f) & 0xFFFFu;
  if constexpr (kF16) {
    float f;
    asm("{ .reg .f16 h; mov.b16 h, %1; cvt.f32.f16 %0, h; }" : "=f"(f) : "h"((unsigned short)u));
    return f;
  } else {
    return __uint_as_float(u << 16);
  }
}

}  // namespace attn
