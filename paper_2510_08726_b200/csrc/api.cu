// api.cu -- host side of the C ABI declared in include/attn.h: argument
// validation (synchronous status codes, no exceptions), TMA descriptor
// construction (cuTensorMapEncodeTiled through the runtime's driver entry
// point, so the library links no libcuda), and kernel dispatch.  No device
// memory is allocated here and the host never synchronises.
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>

#include <dlfcn.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <mutex>

#include "../../include/attn.h"
#include "kernels.h"

namespace {

thread_local char g_err[512] = "";
thread_local int g_launches = 0;
thread_local unsigned* g_repair_events = nullptr;   // attn_debug_repair_counters

attn_status fail(attn_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return s;
}

#define CHECK_ARG(cond, ...) \
  do {                       \
    if (!(cond)) return fail(ATTN_ERR_INVALID_ARGUMENT, __VA_ARGS__); \
  } while (0)

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// 4-D bf16 map over [B][H][S][D] (dims listed innermost first), box (box_d, box_s, 1, 1).
attn_status make_map(CUtensorMap* m, const attn_tensor& t, int B, int H, int S, int D, int box_d, int box_s,
                     bool swizzle128, bool f16 = false) {
  EncodeFn enc = get_encode();
  if (!enc) return fail(ATTN_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[4] = {(cuuint64_t)D, (cuuint64_t)S, (cuuint64_t)H, (cuuint64_t)B};
  cuuint64_t strides[3] = {(cuuint64_t)t.stride_s * 2, (cuuint64_t)t.stride_h * 2, (cuuint64_t)t.stride_b * 2};
  cuuint32_t box[4] = {(cuuint32_t)box_d, (cuuint32_t)box_s, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(m, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, t.ptr, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ATTN_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return ATTN_OK;
}

attn_status check_tensor(const attn_tensor& t, const char* name, int elem_bytes, int B, int H, int S) {
  if (t.ptr == nullptr) return fail(ATTN_ERR_INVALID_ARGUMENT, "%s: null pointer", name);
  if (t.stride_b < 0 || t.stride_h < 0 || t.stride_s < 0)
    return fail(ATTN_ERR_INVALID_ARGUMENT, "%s: negative stride", name);
  if (elem_bytes == 2) {
    if ((reinterpret_cast<uintptr_t>(t.ptr) & 15) != 0)
      return fail(ATTN_ERR_ALIGNMENT, "%s: base pointer must be 16-byte aligned", name);
    if ((B > 1 && t.stride_b % 8) || (H > 1 && t.stride_h % 8) || (S > 1 && t.stride_s % 8))
      return fail(ATTN_ERR_ALIGNMENT, "%s: strides must be multiples of 8 elements (16 bytes)", name);
  } else if ((reinterpret_cast<uintptr_t>(t.ptr) & 3) != 0) {
    return fail(ATTN_ERR_ALIGNMENT, "%s: base pointer must be 4-byte aligned", name);
  }
  return ATTN_OK;
}

attn_status check_problem(const attn_problem* p, attn::VariantParams* vp) {
  CHECK_ARG(p != nullptr, "problem is NULL");
  CHECK_ARG(p->batch >= 1 && p->heads_q >= 1 && p->heads_kv >= 1 && p->seqlen_q >= 1 && p->seqlen_kv >= 1 &&
                p->head_dim >= 1,
            "all extents must be >= 1");
  CHECK_ARG(p->heads_q % p->heads_kv == 0, "heads_q (%d) must be a multiple of heads_kv (%d)", p->heads_q,
            p->heads_kv);
  CHECK_ARG(isfinite(p->scale) && p->scale > 0.f, "scale must be finite and > 0");
  CHECK_ARG(isfinite(p->softcap) && p->softcap >= 0.f, "softcap must be finite and >= 0");
  CHECK_ARG(p->window_left >= -1 && p->window_right >= -1, "window bounds must be >= -1");
  CHECK_ARG(p->causal == 0 || p->causal == 1, "causal must be 0 or 1");
  CHECK_ARG(p->dtype == ATTN_BF16 || p->dtype == ATTN_FP32 || p->dtype == ATTN_FP16, "unknown dtype");
  const int64_t total = p->seqlen_kv_total == 0 ? p->seqlen_kv : p->seqlen_kv_total;
  CHECK_ARG(p->kv_pos_offset >= 0 && p->kv_pos_offset + p->seqlen_kv <= total,
            "need 0 <= kv_pos_offset and kv_pos_offset + seqlen_kv <= seqlen_kv_total");
  CHECK_ARG(total < (1LL << 30) && p->seqlen_q < (1 << 30), "sequence too long");
  const int64_t qoff = p->q_pos_offset == ATTN_Q_POS_DEFAULT ? total - p->seqlen_q : p->q_pos_offset;
  CHECK_ARG(qoff > -(1LL << 30) && qoff < (1LL << 30), "q_pos_offset out of range");
  const float log2e = 1.4426950408889634f;
  vp->scale = p->scale;
  vp->scale_log2 = p->scale * log2e;
  vp->softcap = p->softcap;
  vp->softcap_log2 = p->softcap * log2e;
  vp->scale_over_cap = p->softcap > 0.f ? p->scale / p->softcap : 0.f;
  vp->alibi = p->alibi_slopes;
  vp->causal = p->causal;
  vp->window_left = p->window_left;
  vp->window_right = p->window_right;
  vp->q_off = qoff;
  vp->kv_off = p->kv_pos_offset;
  vp->repair_events = g_repair_events;
  return ATTN_OK;
}

attn_status cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return ATTN_OK;
  return fail(ATTN_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

int sm_count_cached() {   // of the CURRENT device (one cached value per device ordinal)
  static std::atomic<int> cache[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  int n = cache[dev & 63].load(std::memory_order_relaxed);
  if (n == 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) n = 148;
    cache[dev & 63].store(n, std::memory_order_relaxed);
  }
  return n;
}

attn::Shape shape_of(const attn_problem* p) {
  return attn::Shape{p->batch, p->heads_q, p->heads_kv, p->seqlen_q, p->seqlen_kv, p->head_dim};
}

}  // namespace

extern "C" {

int attn_abi_version(void) { return ATTN_ABI_VERSION; }
const char* attn_last_error(void) { return g_err; }
int attn_last_launch_count(void) { return g_launches; }
void attn_debug_repair_counters(unsigned int* counters) { g_repair_events = counters; }

const char* attn_status_string(attn_status s) {
  switch (s) {
    case ATTN_OK: return "ok";
    case ATTN_ERR_INVALID_ARGUMENT: return "invalid argument";
    case ATTN_ERR_UNSUPPORTED: return "unsupported";
    case ATTN_ERR_ALIGNMENT: return "alignment";
    case ATTN_ERR_WORKSPACE_TOO_SMALL: return "workspace too small";
    case ATTN_ERR_CUDA: return "cuda error";
    case ATTN_ERR_NCCL: return "nccl error";
  }
  return "unknown status";
}

attn_status attn_fused_fwd(const attn_problem* prob, attn_tensor q, attn_tensor k, attn_tensor v, attn_tensor o,
                           float* lse, attn_stream_t stream) {
  return attn_fused_fwd_splitkv(prob, q, k, v, o, lse, 1, nullptr, 0, stream);
}

int32_t attn_fused_fwd_default_splits(const attn_problem* p, int32_t sm_count) {
  if (p == nullptr || p->dtype == ATTN_FP32 || p->batch < 1 || p->heads_q < 1 || p->seqlen_q < 1) return 1;
  if (sm_count <= 0) sm_count = sm_count_cached();
  const int64_t units = (int64_t)p->batch * p->heads_q * ((p->seqlen_q + 255) / 256);
  const int64_t ntiles = (p->seqlen_kv + 127) / 128;
  // Measured on the Table 3 grid (tools/sweep.py --table3): a split pays for its merge
  // launch only with >= 4 splits of >= 4 KV tiles each (s_kv >= 2048 at s_q <= 256:
  // 28.7 -> 20.8 us); fewer / shorter splits were slower than the plain kernel.
  int64_t splits = sm_count / units;
  if (splits > ntiles / 4) splits = ntiles / 4;
  if (splits > 16) splits = 16;
  return splits < 4 ? 1 : (int32_t)splits;
}

size_t attn_fused_fwd_workspace_bytes(const attn_problem* p, int32_t num_splits) {
  if (p == nullptr) return 0;
  if (num_splits <= 0) num_splits = attn_fused_fwd_default_splits(p, 0);
  if (num_splits <= 1) return 0;
  const size_t rows = (size_t)num_splits * p->batch * p->heads_q * p->seqlen_q;
  auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
  return up(rows * p->head_dim * 4) + up(rows * 4);   // partial O (fp32, normalised), partial lse (fp32)
}

attn_status attn_fused_fwd_splitkv(const attn_problem* prob, attn_tensor q, attn_tensor k, attn_tensor v,
                                   attn_tensor o, float* lse, int32_t num_splits, void* workspace,
                                   size_t workspace_bytes, attn_stream_t stream) {
  g_err[0] = 0;
  attn::VariantParams vp;
  attn_status st = check_problem(prob, &vp);
  if (st != ATTN_OK) return st;
  const attn_problem& p = *prob;
  if (num_splits < 0) return fail(ATTN_ERR_INVALID_ARGUMENT, "num_splits must be >= 0");
  if (num_splits == 0) num_splits = attn_fused_fwd_default_splits(prob, 0);
  const int eb = p.dtype == ATTN_FP32 ? 4 : 2;
  if ((st = check_tensor(q, "q", eb, p.batch, p.heads_q, p.seqlen_q)) != ATTN_OK) return st;
  if ((st = check_tensor(k, "k", eb, p.batch, p.heads_kv, p.seqlen_kv)) != ATTN_OK) return st;
  if ((st = check_tensor(v, "v", eb, p.batch, p.heads_kv, p.seqlen_kv)) != ATTN_OK) return st;
  if ((st = check_tensor(o, "o", eb, p.batch, p.heads_q, p.seqlen_q)) != ATTN_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int launches = 0;
  if (p.dtype == ATTN_BF16 || p.dtype == ATTN_FP16) {
    if (p.head_dim != 64 && p.head_dim != 128)
      return fail(ATTN_ERR_UNSUPPORTED, "bf16/fp16 head_dim must be 64 or 128 (got %d)", p.head_dim);
    attn::FwdTcArgs a;
    a.s = shape_of(prob);
    a.f16 = p.dtype == ATTN_FP16;
    a.v = vp;
    a.lse = lse;
    if ((st = make_map(&a.tm_q, q, p.batch, p.heads_q, p.seqlen_q, p.head_dim, 64, 128, true, a.f16)) != ATTN_OK) return st;
    const int bn = attn::fwd_kv_tile_keys(p.head_dim);
    if ((st = make_map(&a.tm_k, k, p.batch, p.heads_kv, p.seqlen_kv, p.head_dim, 64, bn, true, a.f16)) != ATTN_OK) return st;
    if ((st = make_map(&a.tm_v, v, p.batch, p.heads_kv, p.seqlen_kv, p.head_dim, 64, bn, true, a.f16)) != ATTN_OK) return st;
    // (the prefill kernels prefetch tm_o even when they write fp32 partials: always a valid map)
    if ((st = make_map(&a.tm_o, o, p.batch, p.heads_q, p.seqlen_q, p.head_dim, 64, 128, true, a.f16)) != ATTN_OK) return st;
    if (num_splits <= 1)
      return (st = cuda_status(attn::launch_fwd_tc(a, s, &launches), "fwd_tc launch")) == ATTN_OK
                 ? (g_launches = launches, ATTN_OK) : st;
    // KV split: fp32 normalised partial (O_s, lse_s) per split into the workspace, then Eq. 8
    const size_t need = attn_fused_fwd_workspace_bytes(prob, num_splits);
    if (workspace == nullptr || workspace_bytes < need)
      return fail(ATTN_ERR_WORKSPACE_TOO_SMALL, "workspace needs %zu bytes", need);
    if ((reinterpret_cast<uintptr_t>(workspace) & 255) != 0)
      return fail(ATTN_ERR_ALIGNMENT, "workspace must be 256-byte aligned");
    const long long rows = (long long)p.batch * p.heads_q * p.seqlen_q;
    const size_t obytes = (((size_t)num_splits * rows * p.head_dim * 4) + 255) & ~size_t(255);
    float* po = static_cast<float*>(workspace);
    float* plse = reinterpret_cast<float*>(static_cast<char*>(workspace) + obytes);
    const int ntiles = (p.seqlen_kv + 127) / 128;
    a.s.kv_splits = num_splits;
    a.s.kv_split_tiles = (ntiles + num_splits - 1) / num_splits;
    a.s.o_part = po;
    a.lse = plse;
    if ((st = cuda_status(attn::launch_fwd_tc(a, s, &launches), "fwd_tc launch")) != ATTN_OK) return st;
    attn::MergeArgs m{};
    m.P = num_splits;
    m.D = p.head_dim;
    m.rows = rows;
    m.in_dtype = ATTN_FP32;
    m.out_dtype = p.dtype;
    m.o_in = po;
    m.o_sp = rows * p.head_dim;
    m.o_sr = p.head_dim;
    m.lse_in = plse;
    m.l_sp = rows;
    m.o_out = o.ptr;
    m.o_out_sr = o.stride_s;
    m.out_H = p.heads_q;
    m.out_Sq = p.seqlen_q;
    m.o_out_sb = o.stride_b;
    m.o_out_sh = o.stride_h;
    m.lse_out = lse;
    if ((st = cuda_status(attn::launch_merge(m, s, &launches), "merge launch")) != ATTN_OK) return st;
    g_launches = launches;
    return ATTN_OK;
  }
  if (num_splits > 1) return fail(ATTN_ERR_UNSUPPORTED, "the fp32 path has no KV split");
  if (p.head_dim > 256) return fail(ATTN_ERR_UNSUPPORTED, "fp32 head_dim must be <= 256");
  attn::FwdSimtArgs a;
  a.s = shape_of(prob);
  a.v = vp;
  a.q = static_cast<const float*>(q.ptr);
  a.k = static_cast<const float*>(k.ptr);
  a.v_ = static_cast<const float*>(v.ptr);
  a.o = static_cast<float*>(o.ptr);
  a.q_sb = q.stride_b; a.q_sh = q.stride_h; a.q_ss = q.stride_s;
  a.k_sb = k.stride_b; a.k_sh = k.stride_h; a.k_ss = k.stride_s;
  a.v_sb = v.stride_b; a.v_sh = v.stride_h; a.v_ss = v.stride_s;
  a.o_sb = o.stride_b; a.o_sh = o.stride_h; a.o_ss = o.stride_s;
  a.lse = lse;
  st = cuda_status(attn::launch_fwd_simt(a, s, &launches), "fwd_simt launch");
  if (st == ATTN_OK) g_launches = launches;
  return st;
}

attn_status attn_fused_fwd_partial(const attn_problem* prob, attn_tensor q, attn_tensor k, attn_tensor v,
                                   float* o_part, float* lse, attn_stream_t stream) {
  g_err[0] = 0;
  attn::VariantParams vp;
  attn_status st = check_problem(prob, &vp);
  if (st != ATTN_OK) return st;
  const attn_problem& p = *prob;
  if (p.dtype != ATTN_BF16 && p.dtype != ATTN_FP16)
    return fail(ATTN_ERR_UNSUPPORTED, "attn_fused_fwd_partial takes bf16 / fp16 inputs (fp32: use attn_fused_fwd)");
  if (p.head_dim != 64 && p.head_dim != 128)
    return fail(ATTN_ERR_UNSUPPORTED, "bf16/fp16 head_dim must be 64 or 128 (got %d)", p.head_dim);
  CHECK_ARG(o_part != nullptr && lse != nullptr, "o_part and lse are required");
  if ((reinterpret_cast<uintptr_t>(o_part) & 15) != 0) return fail(ATTN_ERR_ALIGNMENT, "o_part must be 16-byte aligned");
  if ((st = check_tensor(q, "q", 2, p.batch, p.heads_q, p.seqlen_q)) != ATTN_OK) return st;
  if ((st = check_tensor(k, "k", 2, p.batch, p.heads_kv, p.seqlen_kv)) != ATTN_OK) return st;
  if ((st = check_tensor(v, "v", 2, p.batch, p.heads_kv, p.seqlen_kv)) != ATTN_OK) return st;
  attn::FwdTcArgs a;
  a.s = shape_of(prob);
  a.f16 = p.dtype == ATTN_FP16;
  a.v = vp;
  a.lse = lse;
  a.s.o_part = o_part;
  if ((st = make_map(&a.tm_q, q, p.batch, p.heads_q, p.seqlen_q, p.head_dim, 64, 128, true, a.f16)) != ATTN_OK) return st;
  const int bn = attn::fwd_kv_tile_keys(p.head_dim);
  if ((st = make_map(&a.tm_k, k, p.batch, p.heads_kv, p.seqlen_kv, p.head_dim, 64, bn, true, a.f16)) != ATTN_OK) return st;
  if ((st = make_map(&a.tm_v, v, p.batch, p.heads_kv, p.seqlen_kv, p.head_dim, 64, bn, true, a.f16)) != ATTN_OK) return st;
  a.tm_o = a.tm_q;   // never stored through (prefetched only)
  int launches = 0;
  st = cuda_status(attn::launch_fwd_tc(a, reinterpret_cast<cudaStream_t>(stream), &launches), "fwd_tc launch");
  if (st == ATTN_OK) g_launches = launches;
  return st;
}

int32_t attn_splitkv_default_splits(const attn_problem* p, int32_t sm_count) {
  if (p == nullptr || p->batch < 1 || p->heads_kv < 1 || p->seqlen_kv < 1) return 1;
  if (sm_count <= 0) sm_count = sm_count_cached();
  const int nk = attn::decode_stage_keys(p->heads_q / p->heads_kv, p->head_dim);
  const int64_t units = (int64_t)p->batch * p->heads_kv;
  // The largest split count with at most ONE (b, hkv, split) CTA per SM: measured on B200
  // (tools/decode_splits.py) this streams K/V fastest (B = 1..16: 6.2-7.2 TB/s), while two
  // per SM or a partial second wave lose 5-20 %.
  int64_t splits = sm_count / units;
  // With >= 64 (b, hkv) groups the floor leaves SMs idle (B = 8: 128 of 148; B = 16: 128) while
  // two decode CTAs fit per SM, so round UP (<= 2 per SM, all resident): measured r1k
  // (profiles/r1k_decode_splits.txt) B = 8 6954 -> 7131, B = 16 6974 -> 7146 GB/s; below 64
  // groups rounding up loses (B = 1: 6352 -> 6088, B = 2: 6783 -> 6536, B = 4: 6869 -> 6795).
  if (units >= 64 && units < sm_count) splits = (sm_count + units - 1) / units;
  const int64_t max_splits = (p->seqlen_kv + nk - 1) / nk;
  if (splits > max_splits) splits = max_splits;
  if (splits < 1) splits = 1;
  return (int32_t)splits;
}

size_t attn_splitkv_workspace_bytes(const attn_problem* p, int32_t num_splits) {
  if (p == nullptr) return 0;
  if (num_splits <= 0) num_splits = attn_splitkv_default_splits(p, 0);
  const size_t rows = (size_t)num_splits * p->batch * p->heads_q * (p->seqlen_q > 1 ? p->seqlen_q : 1);
  auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
  // the fused combine's arrival tickets [B][Hkv] (zero between calls), then m | l | O partials
  return up((size_t)p->batch * p->heads_kv * 4) + up(rows * 4) * 2 + up(rows * p->head_dim * 4);
}

}  // extern "C"

namespace {
// attn_splitkv_decode, and (packed != NULL) its fused form that ends in the un-normalised
// packed triple of attn_splitkv_decode_packed.
attn_status decode_impl(const attn_problem* prob, attn_tensor q, attn_tensor k, attn_tensor v, int32_t num_splits,
                        void* workspace, size_t workspace_bytes, const attn_parts* parts_out, attn_tensor o,
                        float* lse, float* packed, attn_stream_t stream) {
  g_err[0] = 0;
  attn::VariantParams vp;
  attn_status st = check_problem(prob, &vp);
  if (st != ATTN_OK) return st;
  const attn_problem& p = *prob;
  if (p.dtype == ATTN_FP32) return fail(ATTN_ERR_UNSUPPORTED, "decode supports bf16 and fp16 only");
  if (p.head_dim != 64 && p.head_dim != 128)
    return fail(ATTN_ERR_UNSUPPORTED, "decode head_dim must be 64 or 128 (got %d)", p.head_dim);
  const int G = p.heads_q / p.heads_kv;
  const int Sq = p.seqlen_q;
  // the G * Sq (head, query) rows of a KV group are packed into one 16-row mma tile
  if ((int64_t)G * Sq > 16)
    return fail(ATTN_ERR_UNSUPPORTED, "decode packs G * seqlen_q <= 16 rows (got %d x %d); use attn_fused_fwd",
                G, Sq);
  CHECK_ARG(parts_out != nullptr || o.ptr != nullptr || packed != nullptr, "decode needs parts_out or o");
  if (packed != nullptr && (Sq != 1 || parts_out != nullptr || o.ptr != nullptr))
    return fail(ATTN_ERR_UNSUPPORTED, "the packed triple output needs seqlen_q == 1 and no other output");
  if (Sq > 1 && parts_out != nullptr)
    return fail(ATTN_ERR_UNSUPPORTED, "parts_out (a per-(b, h) triple) needs seqlen_q == 1");
  if (num_splits < 0) return fail(ATTN_ERR_INVALID_ARGUMENT, "num_splits must be >= 0");
  if (num_splits == 0) num_splits = attn_splitkv_default_splits(prob, 0);
  if (Sq > 1 && num_splits > attn::decode_fused_max_splits(G * Sq, p.head_dim))
    return fail(ATTN_ERR_UNSUPPORTED, "seqlen_q > 1 supports at most %d splits",
                attn::decode_fused_max_splits(G * Sq, p.head_dim));
  if ((st = check_tensor(q, "q", 2, p.batch, p.heads_q, Sq)) != ATTN_OK) return st;
  if ((st = check_tensor(k, "k", 2, p.batch, p.heads_kv, p.seqlen_kv)) != ATTN_OK) return st;
  if ((st = check_tensor(v, "v", 2, p.batch, p.heads_kv, p.seqlen_kv)) != ATTN_OK) return st;
  if (o.ptr != nullptr && (st = check_tensor(o, "o", 2, p.batch, p.heads_q, Sq)) != ATTN_OK) return st;

  attn::DecodeArgs a{};
  a.s = shape_of(prob);
  a.f16 = p.dtype == ATTN_FP16;
  a.v = vp;
  a.q = static_cast<const uint16_t*>(q.ptr);
  a.q_sb = q.stride_b;
  a.q_sh = q.stride_h;
  a.q_ss = q.stride_s;
  const int nk = attn::decode_stage_keys(G, p.head_dim);
  a.num_splits = num_splits;
  const int64_t per = (p.seqlen_kv + num_splits - 1) / num_splits;
  a.split_len = (int)(((per + nk - 1) / nk) * nk);
  if (parts_out != nullptr) {
    CHECK_ARG(parts_out->m && parts_out->l && parts_out->o, "parts_out has a null array");
    CHECK_ARG(parts_out->num_parts == num_splits, "parts_out->num_parts (%d) must equal the split count (%d)",
              parts_out->num_parts, num_splits);
    a.parts = attn::PartsView{parts_out->m, parts_out->l, parts_out->o, num_splits,
                              parts_out->m_stride_part, parts_out->m_stride_b, parts_out->m_stride_h,
                              parts_out->o_stride_part, parts_out->o_stride_b, parts_out->o_stride_h};
  } else {
    const size_t need = attn_splitkv_workspace_bytes(prob, num_splits);
    if (workspace == nullptr || workspace_bytes < need)
      return fail(ATTN_ERR_WORKSPACE_TOO_SMALL, "workspace needs %zu bytes", need);
    const size_t rows = (size_t)num_splits * p.batch * p.heads_q * Sq;
    auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
    char* const w0 = static_cast<char*>(workspace);
    char* w = w0 + up((size_t)p.batch * p.heads_kv * 4);   // after the ticket block
    float* m = reinterpret_cast<float*>(w);
    float* l = reinterpret_cast<float*>(w + up(rows * 4));
    float* ob = reinterpret_cast<float*>(w + 2 * up(rows * 4));
    // [split][b][hq][i] (m, l) and [split][b][hq][i][d] (O); the kernel adds i (and i * D)
    const long long bhs = (long long)p.batch * p.heads_q * Sq;
    a.parts = attn::PartsView{m, l, ob, num_splits, bhs, (long long)p.heads_q * Sq, Sq, bhs * p.head_dim,
                              (long long)p.heads_q * Sq * p.head_dim, (long long)Sq * p.head_dim};
    // Fused Eq. 8 combine (last CTA per (b, hkv)) when the output is wanted and the
    // split weights fit the kernel's staging area; else the separate combine kernel.
    if ((o.ptr != nullptr || packed != nullptr) && num_splits <= attn::decode_fused_max_splits(G * Sq, p.head_dim)) {
      a.tickets = reinterpret_cast<unsigned*>(w0);
      a.out_f16 = p.dtype == ATTN_FP16 ? 1 : 0;
      a.o = o.ptr;
      a.o_sb = o.stride_b;
      a.o_sh = o.stride_h;
      a.o_ss = o.stride_s;
      a.lse = lse;
      a.packed = packed;
    } else if (packed != nullptr) {
      return fail(ATTN_ERR_UNSUPPORTED, "packed output needs num_splits <= %d",
                  attn::decode_fused_max_splits(G * Sq, p.head_dim));
    }
  }
  if ((st = make_map(&a.tm_k, k, p.batch, p.heads_kv, p.seqlen_kv, p.head_dim, 64, nk, true, a.f16)) != ATTN_OK) return st;
  if ((st = make_map(&a.tm_v, v, p.batch, p.heads_kv, p.seqlen_kv, p.head_dim, 64, nk, true, a.f16)) != ATTN_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int launches = 0;
  st = cuda_status(attn::launch_decode(a, s, &launches), "decode launch");
  if (st != ATTN_OK) return st;
  if (o.ptr != nullptr && a.tickets == nullptr) {
    attn::CombineArgs c{};
    c.B = p.batch;
    c.H = p.heads_q;
    c.D = p.head_dim;
    c.in = a.parts;
    c.out_bf16 = a.f16 ? 2 : 1;
    c.o = o.ptr;
    c.o_sb = o.stride_b;
    c.o_sh = o.stride_h;
    c.lse = lse;
    c.acc.m = nullptr;
    st = cuda_status(attn::launch_combine(c, s, &launches), "combine launch");
  }
  if (st == ATTN_OK) g_launches = launches;
  return st;
}
}  // namespace

extern "C" {

attn_status attn_splitkv_decode(const attn_problem* prob, attn_tensor q, attn_tensor k, attn_tensor v,
                                int32_t num_splits, void* workspace, size_t workspace_bytes,
                                const attn_parts* parts_out, attn_tensor o, float* lse, attn_stream_t stream) {
  return decode_impl(prob, q, k, v, num_splits, workspace, workspace_bytes, parts_out, o, lse, nullptr, stream);
}

attn_status attn_splitkv_decode_packed(const attn_problem* prob, attn_tensor q, attn_tensor k, attn_tensor v,
                                       int32_t num_splits, void* workspace, size_t workspace_bytes, float* packed,
                                       attn_stream_t stream) {
  if (packed == nullptr) {
    g_err[0] = 0;
    return fail(ATTN_ERR_INVALID_ARGUMENT, "packed is NULL");
  }
  const attn_tensor none{nullptr, 0, 0, 0};
  return decode_impl(prob, q, k, v, num_splits, workspace, workspace_bytes, nullptr, none, nullptr, packed, stream);
}

attn_status attn_combine(int32_t batch, int32_t heads, int32_t head_dim, const attn_parts* in,
                         attn_dtype out_dtype, attn_tensor o, float* lse, const attn_parts* acc_out,
                         attn_stream_t stream) {
  g_err[0] = 0;
  CHECK_ARG(batch >= 1 && heads >= 1 && head_dim >= 1, "extents must be >= 1");
  if (head_dim > 256) return fail(ATTN_ERR_UNSUPPORTED, "combine head_dim must be <= 256");
  CHECK_ARG(in != nullptr && in->m && in->l && in->o && in->num_parts >= 1, "bad input parts");
  CHECK_ARG(o.ptr != nullptr || lse != nullptr || acc_out != nullptr, "no output requested");
  CHECK_ARG(out_dtype == ATTN_BF16 || out_dtype == ATTN_FP32 || out_dtype == ATTN_FP16, "unknown out dtype");
  if (acc_out) CHECK_ARG(acc_out->m && acc_out->l && acc_out->o && acc_out->num_parts == 1, "bad acc_out");
  attn::CombineArgs c{};
  c.B = batch;
  c.H = heads;
  c.D = head_dim;
  c.in = attn::PartsView{in->m, in->l, in->o, in->num_parts, in->m_stride_part, in->m_stride_b, in->m_stride_h,
                         in->o_stride_part, in->o_stride_b, in->o_stride_h};
  c.out_bf16 = out_dtype == ATTN_BF16 ? 1 : (out_dtype == ATTN_FP16 ? 2 : 0);
  c.o = o.ptr;
  c.o_sb = o.stride_b;
  c.o_sh = o.stride_h;
  c.lse = lse;
  if (acc_out)
    c.acc = attn::PartsView{acc_out->m, acc_out->l, acc_out->o, 1, 0, acc_out->m_stride_b, acc_out->m_stride_h,
                            0, acc_out->o_stride_b, acc_out->o_stride_h};
  else
    c.acc.m = nullptr;
  int launches = 0;
  attn_status st = cuda_status(attn::launch_combine(c, reinterpret_cast<cudaStream_t>(stream), &launches),
                               "combine launch");
  if (st == ATTN_OK) g_launches = launches;
  return st;
}

attn_status attn_merge_partials(int32_t num_parts, int64_t rows, int32_t head_dim, attn_dtype in_dtype,
                                const void* o_in, int64_t o_stride_part, int64_t o_stride_row, const float* lse_in,
                                int64_t lse_stride_part, attn_dtype out_dtype, void* o_out, int64_t o_out_stride_row,
                                float* lse_out, attn_stream_t stream) {
  g_err[0] = 0;
  CHECK_ARG(num_parts >= 1 && rows >= 1 && head_dim >= 1, "extents must be >= 1");
  if (head_dim > 256) return fail(ATTN_ERR_UNSUPPORTED, "merge head_dim must be <= 256");
  CHECK_ARG(o_in != nullptr && lse_in != nullptr, "null input");
  CHECK_ARG(o_out != nullptr || lse_out != nullptr, "no output requested");
  auto dt_ok = [](attn_dtype d) { return d == ATTN_BF16 || d == ATTN_FP32 || d == ATTN_FP16; };
  CHECK_ARG(dt_ok(in_dtype) && dt_ok(out_dtype), "unknown dtype");
  attn::MergeArgs m{};
  m.P = num_parts;
  m.D = head_dim;
  m.rows = rows;
  m.in_dtype = in_dtype;
  m.out_dtype = out_dtype;
  m.o_in = o_in;
  m.o_sp = o_stride_part;
  m.o_sr = o_stride_row;
  m.lse_in = lse_in;
  m.l_sp = lse_stride_part;
  m.o_out = o_out;
  m.o_out_sr = o_out_stride_row;
  m.lse_out = lse_out;
  int launches = 0;
  attn_status st = cuda_status(attn::launch_merge(m, reinterpret_cast<cudaStream_t>(stream), &launches),
                               "merge launch");
  if (st == ATTN_OK) g_launches = launches;
  return st;
}

attn_status attn_softmax_rows(int64_t rows, int32_t cols, attn_dtype dtype, const void* x, int64_t x_stride_row,
                              void* y, int64_t y_stride_row, float* row_max, float* row_sum, attn_stream_t stream) {
  g_err[0] = 0;
  CHECK_ARG(rows >= 1 && cols >= 1, "extents must be >= 1");
  CHECK_ARG(rows < (1LL << 31), "too many rows");
  CHECK_ARG(dtype == ATTN_BF16 || dtype == ATTN_FP32 || dtype == ATTN_FP16, "unknown dtype");
  CHECK_ARG(x != nullptr, "x is NULL");
  CHECK_ARG(y != nullptr || row_max != nullptr || row_sum != nullptr, "no output requested");
  const int eb = dtype == ATTN_FP32 ? 4 : 2;
  CHECK_ARG(x_stride_row >= cols && (y == nullptr || y_stride_row >= cols), "row stride smaller than cols");
  if ((reinterpret_cast<uintptr_t>(x) & 15) || ((x_stride_row * eb) & 15) ||
      (y != nullptr && ((reinterpret_cast<uintptr_t>(y) & 15) || ((y_stride_row * eb) & 15))))
    return fail(ATTN_ERR_ALIGNMENT, "x / y must be 16-byte aligned with 16-byte-multiple row strides");
  attn::SoftmaxRowsArgs s{rows, cols, (int)dtype, x, x_stride_row, y, y_stride_row, row_max, row_sum};
  int launches = 0;
  attn_status st = cuda_status(attn::launch_softmax_rows(s, reinterpret_cast<cudaStream_t>(stream), &launches),
                               "softmax_rows launch");
  if (st == ATTN_OK) g_launches = launches;
  return st;
}

// ---------------------------------------------------------------- multi-GPU decode (NCCL, loaded at run time)
namespace {
struct NcclApi {
  using Uid = struct { char internal[128]; };
  int (*get_unique_id)(Uid*) = nullptr;
  int (*comm_init_rank)(void** comm, int nranks, Uid id, int rank) = nullptr;
  int (*comm_destroy)(void* comm) = nullptr;
  int (*all_gather)(const void* send, void* recv, size_t count, int dtype, void* comm, cudaStream_t s) = nullptr;
  const char* (*error_string)(int) = nullptr;
  bool ok = false;
};
const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_gather && api.error_string;
  });
  return api;
}
struct Comm {
  void* nc;
  int nranks, rank;
};
constexpr int kNcclFloat32 = 7;   // ncclFloat32 in nccl.h's ncclDataType_t
attn_status nccl_status(int r, const char* what) {
  if (r == 0) return ATTN_OK;
  return fail(ATTN_ERR_NCCL, "%s: %s", what, nccl().error_string ? nccl().error_string(r) : "?");
}
size_t up256(size_t x) { return (x + 255) & ~size_t(255); }
}  // namespace

attn_status attn_nccl_get_unique_id(void* id_out) {
  g_err[0] = 0;
  CHECK_ARG(id_out != nullptr, "id_out is NULL");
  if (!nccl().ok) return fail(ATTN_ERR_NCCL, "libnccl.so.2 not loadable");
  NcclApi::Uid id;
  attn_status st = nccl_status(nccl().get_unique_id(&id), "ncclGetUniqueId");
  if (st == ATTN_OK) memcpy(id_out, id.internal, sizeof(id.internal));
  return st;
}

attn_status attn_nccl_comm_init(void** comm, int32_t nranks, int32_t rank, const void* nccl_unique_id) {
  g_err[0] = 0;
  CHECK_ARG(comm != nullptr && nccl_unique_id != nullptr, "null argument");
  CHECK_ARG(nranks >= 1 && rank >= 0 && rank < nranks, "bad nranks / rank (%d / %d)", nranks, rank);
  if (!nccl().ok) return fail(ATTN_ERR_NCCL, "libnccl.so.2 not loadable");
  NcclApi::Uid id;
  memcpy(id.internal, nccl_unique_id, sizeof(id.internal));
  void* nc = nullptr;
  attn_status st = nccl_status(nccl().comm_init_rank(&nc, nranks, id, rank), "ncclCommInitRank");
  if (st != ATTN_OK) return st;
  *comm = new Comm{nc, nranks, rank};
  return ATTN_OK;
}

attn_status attn_nccl_comm_destroy(void* comm) {
  g_err[0] = 0;
  if (comm == nullptr) return ATTN_OK;
  Comm* c = static_cast<Comm*>(comm);
  attn_status st = nccl().ok ? nccl_status(nccl().comm_destroy(c->nc), "ncclCommDestroy") : ATTN_OK;
  delete c;
  return st;
}

size_t attn_decode_kv_sharded_workspace_bytes(const attn_problem* p, int32_t nranks) {
  if (p == nullptr || nranks < 1) return 0;
  const int32_t splits = attn_splitkv_default_splits(p, 0);
  const size_t packed = (size_t)p->batch * p->heads_q * (p->head_dim + 2);
  // [split-decode workspace: tickets | m | l | O] [send: packed triples] [recv: nranks x packed]
  return attn_splitkv_workspace_bytes(p, splits) + up256(packed * 4) * (1 + (size_t)nranks);
}

attn_status attn_decode_kv_sharded(void* comm, const attn_problem* local, attn_tensor q, attn_tensor k_shard,
                                   attn_tensor v_shard, void* workspace, size_t workspace_bytes, attn_tensor o,
                                   float* lse, attn_stream_t stream) {
  g_err[0] = 0;
  CHECK_ARG(comm != nullptr && local != nullptr, "null comm / problem");
  CHECK_ARG(o.ptr != nullptr, "o is NULL");
  const Comm* c = static_cast<const Comm*>(comm);
  const size_t need = attn_decode_kv_sharded_workspace_bytes(local, c->nranks);
  if (workspace == nullptr || workspace_bytes < need)
    return fail(ATTN_ERR_WORKSPACE_TOO_SMALL, "workspace needs %zu bytes", need);
  if ((reinterpret_cast<uintptr_t>(workspace) & 255) != 0)
    return fail(ATTN_ERR_ALIGNMENT, "workspace must be 256-byte aligned");
  const attn_problem& p = *local;
  const int32_t splits = attn_splitkv_default_splits(local, 0);
  const size_t dec_ws = attn_splitkv_workspace_bytes(local, splits);
  const long long bh = (long long)p.batch * p.heads_q, D = p.head_dim, W = D + 2;
  char* w = static_cast<char*>(workspace);
  float* send = reinterpret_cast<float*>(w + dec_ws);
  float* recv = reinterpret_cast<float*>(reinterpret_cast<char*>(send) + up256(bh * W * 4));
  const attn_tensor none{nullptr, 0, 0, 0};
  int launches = 0;
  attn_status st;
  // 1. local section over this rank's keys, its splits merged by the fused global section of the
  //    same launch into one UN-normalised triple per (b, hq), packed [B][Hq][D+2] (send buffer)
  if (splits <= attn::decode_fused_max_splits(p.heads_q / p.heads_kv, p.head_dim)) {
    st = decode_impl(local, q, k_shard, v_shard, splits, w, dec_ws, nullptr, none, nullptr, send, stream);
    if (st != ATTN_OK) return st;
    launches = g_launches;
  } else {   // too many splits to stage in the kernel: raw triples, then a separate merge
    const size_t rows = (size_t)splits * p.batch * p.heads_q;
    char* w1 = w + up256((size_t)p.batch * p.heads_kv * 4);
    float* pm = reinterpret_cast<float*>(w1);
    float* pl = reinterpret_cast<float*>(w1 + up256(rows * 4));
    float* po = reinterpret_cast<float*>(w1 + 2 * up256(rows * 4));
    const attn_parts parts{pm, pl, po, splits, bh, p.heads_q, 1, bh * D, (int64_t)p.heads_q * D, D};
    st = decode_impl(local, q, k_shard, v_shard, splits, nullptr, 0, &parts, none, nullptr, nullptr, stream);
    if (st != ATTN_OK) return st;
    launches = g_launches;
    const attn_parts packed{send + D, send + D + 1, send, 1, 0, p.heads_q * W, W, 0, p.heads_q * W, W};
    st = attn_combine(p.batch, p.heads_q, p.head_dim, &parts, p.dtype, none, nullptr, &packed, stream);
    if (st != ATTN_OK) return st;
    launches += g_launches;
  }
  // 2. all-gather the packed triples
  st = nccl_status(nccl().all_gather(send, recv, (size_t)bh * W, kNcclFloat32, c->nc,
                                     reinterpret_cast<cudaStream_t>(stream)), "ncclAllGather");
  if (st != ATTN_OK) return st;
  // 3. Eq. 8 over the ranks' triples
  const attn_parts gathered{recv + D, recv + D + 1, recv, c->nranks, bh * W, p.heads_q * W, W,
                            bh * W, p.heads_q * W, W};
  st = attn_combine(p.batch, p.heads_q, p.head_dim, &gathered, p.dtype, o, lse, nullptr, stream);
  if (st != ATTN_OK) return st;
  g_launches = launches + g_launches;
  return ATTN_OK;
}

}  // extern "C"
