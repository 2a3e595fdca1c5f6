// kernels.h -- internal (non-ABI) launch interface between the host layer
// (api.cu) and the kernels.  Not installed; no torch types anywhere.
#pragma once
#include <atomic>
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace attn {

// cudaFuncSetAttribute(max dynamic smem) once per (kernel, device): it costs
// ~1 us of host time per launch otherwise (visible on small, launch-bound shapes).
template <auto kKern>
inline cudaError_t set_smem_once(int bytes) {
  static std::atomic<unsigned long long> done{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  const unsigned long long bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_relaxed) & bit) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kKern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit);
  return e;
}

// Variant parameters shared by all kernels, pre-converted on the host to the
// log2 domain the kernels compute in (exp(x) = exp2(x * log2 e)).
struct VariantParams {
  float scale;          // softmax scale on q.k
  float scale_log2;     // scale * log2(e)
  float softcap;        // 0 = off
  float softcap_log2;   // softcap * log2(e)
  float scale_over_cap; // scale / softcap
  const float* alibi;   // natural-units slopes [Hq] or nullptr
  int causal;
  int window_left, window_right;
  long long q_off;      // absolute position of query row 0
  long long kv_off;     // absolute position of local key 0
  unsigned* repair_events;   // nullable [ATTN_REPAIR_SLOTS] (attn_debug_repair_counters)
};

struct Shape {
  int B, Hq, Hkv, Sq, Skv, D;
  // Prefill KV split (NEXT-2, small grids): kv_splits CTAs per (q-block, hq, b), split s
  // owning KV tiles [s*kv_split_tiles, (s+1)*kv_split_tiles); outputs go to batch index
  // s*B + b of a partial [kv_splits*B] output.  kv_splits <= 1: off.
  int kv_splits = 1, kv_split_tiles = 0;
  // fp32 output of normalised partials (KV split, context-parallel prefill): when set the
  // prefill kernels write O / l as fp32 [kv_splits*B][Hq][Sq][D] (dense) here instead of
  // storing the 16-bit output through tm_o.
  float* o_part = nullptr;
};

// ------------------------------------------------------------ tcgen05 prefill
struct FwdTcArgs {
  Shape s;
  bool f16;    // fp16 inputs/outputs (else bf16)
  VariantParams v;
  float* lse;  // nullable, [B][Hq][Sq]
  CUtensorMap tm_q, tm_k, tm_v, tm_o;
};
cudaError_t launch_fwd_tc(const FwdTcArgs& a, cudaStream_t stream, int* launches);
int fwd_kv_tile_keys(int D);   // KV tile width (keys) of the prefill kernel: the K/V TMA box rows

// ------------------------------------------------------------ fp32 SIMT forward
struct FwdSimtArgs {
  Shape s;
  VariantParams v;
  const float* q; const float* k; const float* v_; float* o;
  long long q_sb, q_sh, q_ss, k_sb, k_sh, k_ss, v_sb, v_sh, v_ss, o_sb, o_sh, o_ss;
  float* lse;
};
cudaError_t launch_fwd_simt(const FwdSimtArgs& a, cudaStream_t stream, int* launches);

// ------------------------------------------------------------ split-KV decode
struct PartsView {
  float* m; float* l; float* o;
  int num_parts;
  long long m_sp, m_sb, m_sh, o_sp, o_sb, o_sh;
};
struct DecodeArgs {
  Shape s;
  bool f16;                     // fp16 inputs (else bf16)
  VariantParams v;
  const uint16_t* q;            // bf16 / fp16 bits
  long long q_sb, q_sh, q_ss;
  int num_splits, split_len;    // keys per split (multiple of the stage size)
  PartsView parts;              // destination of the local-section triples
  CUtensorMap tm_k, tm_v;       // [D x Skv x Hkv x B], box (D, NK)
  // Fused Eq. 8 global section (tickets != nullptr): the last CTA of each (b, hkv)
  // combines the splits and writes O / lse.  tickets: [B][Hkv], zero on entry and exit.
  unsigned* tickets;
  int out_f16;                  // output dtype: 1 fp16, 0 bf16
  void* o; long long o_sb, o_sh, o_ss;
  float* lse;                   // nullable [B][Hq][Sq]
  // packed != nullptr (Sq == 1): the fused global section writes the UN-normalised merged
  // triple of each (b, hq) -- O_acc at [0, D), m (natural log) at D, l at D + 1 of row
  // (b * Hq + hq) * (D + 2) -- instead of O / lse (the send buffer of the KV-sharded decode).
  float* packed;
};
cudaError_t launch_decode(const DecodeArgs& a, cudaStream_t stream, int* launches);
int decode_stage_keys(int G, int D);
int decode_fused_max_splits(int rows, int D);   // largest split count the fused combine can stage

// ------------------------------------------------------------ combine (Eq. 8)
struct CombineArgs {
  int B, H, D;
  PartsView in;
  int out_bf16;                 // 1: bf16 out, 2: fp16 out, 0: fp32 out
  void* o; long long o_sb, o_sh;  // nullable
  float* lse;                   // nullable [B][H]
  PartsView acc;                // acc.m == nullptr => not written
};
cudaError_t launch_combine(const CombineArgs& a, cudaStream_t stream, int* launches);

// ------------------------------------------------------------ merge of normalised partials (Eq. 8)
struct MergeArgs {
  int P, D;
  long long rows;
  int in_dtype, out_dtype;       // 0 bf16, 1 fp32, 2 fp16 (attn_dtype values)
  const void* o_in; long long o_sp, o_sr;
  const float* lse_in; long long l_sp;
  void* o_out; long long o_out_sr;
  float* lse_out;
  // out_Sq > 0: row r = (b * out_H + h) * out_Sq + i is written at
  // o_out + b*o_out_sb + h*o_out_sh + i*o_out_sr (a strided [B][H][Sq][D] output)
  int out_H = 0, out_Sq = 0; long long o_out_sb = 0, o_out_sh = 0;
};
cudaError_t launch_merge(const MergeArgs& a, cudaStream_t stream, int* launches);

// ------------------------------------------------------------ NEXT-4: softmax rows (Fig. 2 chain)
struct SoftmaxRowsArgs {
  long long rows;
  int cols;
  int dtype;                    // attn_dtype value
  const void* x; long long x_stride;
  void* y; long long y_stride;  // nullable
  float* row_max;               // nullable
  float* row_sum;               // nullable
};
cudaError_t launch_softmax_rows(const SoftmaxRowsArgs& a, cudaStream_t stream, int* launches);

}  // namespace attn
