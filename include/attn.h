/*
 * attn.h -- C ABI of the B200 (sm_100a) fused-attention hot path of
 * Neptune (arXiv 2510.08726): the reduction chain S = Q K^T -> score_mod/mask
 * -> row max -> exp -> row sum -> O = P V computed in ONE naive-fusion pass
 * over KV tiles with the algebraic repair term exp(m_old - m_new)
 * ("Rolling Update", Alg. 1; tile form Fig. 19), and
 * its loop-fission form for decoding with a repaired combine of partial
 * (m, l, O) triples ("Split-K Update", Alg. 2; Fig. 5,
 * P:706-722; Eq. 8).  P:n = line n of the paper's PAPER.md.
 *
 * The operation every entry point computes is Fig. 8's compute definition
 * extended with the Table 1 variants:
 *
 *   x[i,j]   = scale * <q_i, k_j>                      (batch_matmul)
 *   x[i,j]   = softcap * tanh(x / softcap)  if softcap > 0      (SoftCap)
 *   x[i,j]  -= alibi_slopes[hq] * |qpos(i) - kpos(j)|  if slopes (ALiBi)
 *   x[i,j]   = -inf  unless allowed(i,j)               (if_then_else)
 *   O[i,:]   = sum_j exp(x[i,j] - m_i) v_j / sum_j exp(x[i,j] - m_i),
 *              m_i = max_j x[i,j]
 *   lse[i]   = m_i + ln(sum_j exp(x[i,j] - m_i))
 *
 *   qpos(i) = q_pos_offset + i,  kpos(j) = kv_pos_offset + j,
 *   allowed = (!causal || kpos <= qpos)
 *             && (window_left  < 0 || qpos - kpos <= window_left)
 *             && (window_right < 0 || kpos - qpos <= window_right).
 *   GQA: query head hq reads KV head hq / (heads_q / heads_kv).
 *   A row with no allowed key has O = 0 and lse = -inf.
 *
 * Readings of points the paper leaves open are listed in DESIGN.md §2
 * (R1..R12) and are binding for this ABI.
 *
 * Conventions for every call
 * --------------------------
 * - Tensors are caller-owned DEVICE memory, logical layout [B][H][S][D]
 *   ("BHSD", Fig. 8's (B, N, S, H)) described by attn_tensor:
 *   element strides for b, h, s; the D dimension must be contiguous.
 *   bf16/fp16 tensors: base 16-byte aligned, strides multiples of 8 elements
 *   (TMA requirement) -- else ATTN_ERR_ALIGNMENT.
 * - Calls are asynchronous on `stream`; they never synchronise the host and
 *   never allocate device memory, so they are CUDA-graph capturable.
 * - Argument checks are synchronous and return a status; nothing is launched
 *   when a check fails.  Launch failures map to ATTN_ERR_CUDA.  The detail
 *   string of the last failure on the calling thread is attn_last_error().
 * - There is no CPU fallback: unsupported combinations return
 *   ATTN_ERR_UNSUPPORTED.
 */
#ifndef ATTN_H_
#define ATTN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ATTN_ABI_VERSION 1

#if defined(__GNUC__)
#define ATTN_API __attribute__((visibility("default")))
#else
#define ATTN_API
#endif

typedef struct CUstream_st* attn_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
  ATTN_OK = 0,
  ATTN_ERR_INVALID_ARGUMENT = 1,
  ATTN_ERR_UNSUPPORTED = 2,
  ATTN_ERR_ALIGNMENT = 3,
  ATTN_ERR_WORKSPACE_TOO_SMALL = 4,
  ATTN_ERR_CUDA = 5,
  ATTN_ERR_NCCL = 6 /* NCCL missing (libnccl.so.2 not loadable) or an NCCL call failed */
} attn_status;

typedef enum {
  ATTN_BF16 = 0, /* bf16 in/out, fp32 accumulation (tcgen05 / decode kernels) */
  ATTN_FP32 = 1, /* fp32 in/out, fp32 SIMT path (head_dim <= 256) */
  ATTN_FP16 = 2  /* fp16 in/out, fp32 accumulation: the paper's precision */
} attn_dtype;

/* A [B][H][S][D] view. Strides are in ELEMENTS of the tensor's dtype. */
typedef struct {
  void* ptr;
  int64_t stride_b, stride_h, stride_s;
} attn_tensor;

/* Problem description shared by every call (Fig. 8 arguments + Table 1 variants). */
typedef struct {
  int32_t batch, heads_q, heads_kv;   /* heads_q % heads_kv == 0 (GQA group G) */
  int32_t seqlen_q, seqlen_kv;        /* local extents of q and of k/v         */
  int32_t head_dim;                   /* D: bf16/fp16 {64, 128}; fp32 1..256     */
  attn_dtype dtype;
  float scale;                        /* > 0, finite; configs use 1/sqrt(D)      */
  float softcap;                      /* 0 = off; else > 0, finite               */
  const float* alibi_slopes;          /* DEVICE fp32 [heads_q] or NULL           */
  int32_t causal;                     /* 0/1                                     */
  int32_t window_left, window_right;  /* -1 = unbounded, else >= 0               */
  int64_t seqlen_kv_total;            /* 0 => seqlen_kv; else >= kv_pos_offset + seqlen_kv */
  int64_t q_pos_offset;               /* INT64_MIN => seqlen_kv_total - seqlen_q (bottom-right) */
  int64_t kv_pos_offset;              /* absolute position of local key 0 (KV shard start) */
} attn_problem;

#define ATTN_Q_POS_DEFAULT INT64_MIN

/* Partial (m, l, O) triples of Split-K Update (Fig. 5 max_l / sum_l and the
 * local PV).  fp32, DEVICE memory, caller-owned.  For part p, batch b,
 * query head h:
 *   m[p*m_stride_part + b*m_stride_b + h*m_stride_h]  = max_j x over the part (exact max;
 *                                                        -inf if the part has no allowed key)
 *   l[same index]                                     = sum_j exp(x - m)
 *   o[p*o_stride_part + b*o_stride_b + h*o_stride_h + d] = sum_j exp(x - m) v_j[d]  (UN-normalised)
 * m and l share strides.  Natural-log units (x as defined above). */
typedef struct {
  float* m;
  float* l;
  float* o;
  int32_t num_parts;
  int64_t m_stride_part, m_stride_b, m_stride_h;
  int64_t o_stride_part, o_stride_b, o_stride_h;
} attn_parts;

/* ---------------------------------------------------------------------
 * attn_fused_fwd -- Rolling Update forward / prefill (Alg. 1, Fig. 19).
 *
 * One pass over KV tiles per (b, hq, 128-row q tile): S_j = Q K_j^T on
 * tcgen05 tensor cores into TMEM, score_mod/mask, running max, repair
 * alpha = exp(m_old - m_new) applied to l and to the TMEM O accumulator
 * (Eq. 7), O += P V_j, then O / l.
 *   q [B][Hq][Sq][D], k/v [B][Hkv][Skv][D], o [B][Hq][Sq][D] (q's dtype).
 *   lse: nullable DEVICE fp32 [B][Hq][Sq] contiguous.
 * Errors: INVALID_ARGUMENT (extents < 1, heads_q % heads_kv, bad scale /
 * softcap / window, offsets), ALIGNMENT, UNSUPPORTED (bf16/fp16 D not in {64,128};
 * fp32 D > 256), CUDA.
 * ------------------------------------------------------------------- */
ATTN_API attn_status attn_fused_fwd(const attn_problem* prob, attn_tensor q, attn_tensor k, attn_tensor v,
                           attn_tensor o, float* lse, attn_stream_t stream);

/* ---------------------------------------------------------------------
 * Rolling Update with the KV axis also split across CTAs (NEXT-2: small
 * grids such as chunked prefill / multi-token decode, s_q << s_kv, where
 * B * Hq * ceil(s_q / 256) CTAs would leave most SMs idle).  Split s runs the
 * same rolling loop over a contiguous run of 128-key tiles and writes a
 * NORMALISED partial (O_s, lse_s) -- the repaired triple (m = lse_s, l = 1,
 * O_s) of Thm. 2 -- into the workspace; Eq. 8 then merges the
 * splits into o / lse.  Exact in real arithmetic for any split (Eq. 4); the
 * partials stay fp32, so the output is rounded once (by the merge).
 *
 * attn_fused_fwd_default_splits: min(sm_count / units, n_kv_tiles / 4, 16)
 *   with units = B * Hq * ceil(s_q / 256) and 128-key tiles, or 1 when that is
 *   below 4 (a split pays for its merge launch only then -- measured).  Always
 *   1 for fp32.
 * attn_fused_fwd_workspace_bytes: DEVICE workspace (256-byte aligned) for
 *   num_splits (0 = default); 0 when no split is used.
 * attn_fused_fwd_splitkv: num_splits 0 = default, 1 = attn_fused_fwd.  Two
 *   launches when split (prefill kernel + merge).  Errors: those of
 *   attn_fused_fwd, WORKSPACE_TOO_SMALL, ALIGNMENT (workspace), UNSUPPORTED
 *   (fp32 with num_splits > 1).
 * ------------------------------------------------------------------- */
ATTN_API int32_t attn_fused_fwd_default_splits(const attn_problem* prob, int32_t sm_count);
ATTN_API size_t attn_fused_fwd_workspace_bytes(const attn_problem* prob, int32_t num_splits);
ATTN_API attn_status attn_fused_fwd_splitkv(const attn_problem* prob, attn_tensor q, attn_tensor k, attn_tensor v,
                                            attn_tensor o, float* lse, int32_t num_splits, void* workspace,
                                            size_t workspace_bytes, attn_stream_t stream);

/* ---------------------------------------------------------------------
 * attn_fused_fwd_partial -- Rolling Update over a KV SHARD with the result kept
 * as an fp32 normalised partial, for context-parallel prefill (each GPU holds
 * keys [kv_pos_offset, kv_pos_offset + seqlen_kv) of a longer sequence; the
 * per-GPU partials are merged with attn_merge_partials, Eq. 8).
 * A normalised partial (O_r, lse_r) is the repaired triple (m = lse_r, l = 1,
 * O_r) of Thm. 2, so keeping O_r in fp32 leaves one rounding (the merge's) in
 * the final output.
 *   q/k/v as attn_fused_fwd (bf16 or fp16, D in {64, 128});
 *   o_part: DEVICE fp32 [B][Hq][Sq][D] contiguous, 16-byte aligned (required);
 *   lse   : DEVICE fp32 [B][Hq][Sq] contiguous (required).
 * One launch.  Errors: those of attn_fused_fwd; UNSUPPORTED for fp32 inputs.
 * ------------------------------------------------------------------- */
ATTN_API attn_status attn_fused_fwd_partial(const attn_problem* prob, attn_tensor q, attn_tensor k, attn_tensor v,
                                            float* o_part, float* lse, attn_stream_t stream);

/* ---------------------------------------------------------------------
 * Split-K Update decode (Alg. 2, Fig. 5): dtype bf16 or fp16, D in {64, 128},
 * seqlen_q = 1 -- or a few query tokens (multi-token / speculative decode,
 * NEXT-2) with G * seqlen_q <= 16, G = heads_q / heads_kv: the G * seqlen_q
 * (head, query) rows of a KV group share one 16-row tensor-core tile, each
 * with its own causal / window mask (bottom-right positions as everywhere).
 * seqlen_q > 1 needs parts_out == NULL (the fused combine), o != NULL, and
 * writes lse as [B][Hq][Sq].  The KV axis of every (b, hkv) is cut into num_splits
 * contiguous parts (PrivatizeReduce); each CTA streams its part
 * of K and V once from HBM for all G query heads of the group and emits one
 * partial triple per (part, b, hq).  Then the global section (Eq. 8)
 * combines them (attn_combine).
 *
 * attn_splitkv_default_splits: split count used when num_splits == 0: the
 *   largest count with at most one (b, hkv, split) CTA per SM (>= 1; sm_count
 *   <= 0 means the current device's).
 * attn_splitkv_workspace_bytes: DEVICE workspace needed to hold the
 *   partials when parts_out == NULL (pure host function).  Its FIRST
 *   256-byte-rounded [B][Hkv] uint32 block holds the arrival tickets of the
 *   fused global section and MUST be zero before the call (e.g. cudaMemset
 *   once); every completed call leaves it zero, so a workspace reused for the
 *   same or a smaller B*Hkv needs no further clearing.  One workspace serves
 *   one stream at a time.
 * Part s covers local keys [s*L, min((s+1)*L, seqlen_kv)) with
 *   L = 64 * ceil(ceil(seqlen_kv / num_splits) / 64)   (trailing parts may be
 *   empty: m = -inf, l = 0, O = 0).
 * attn_splitkv_decode: if parts_out != NULL the raw partials go there
 *   (parts_out->num_parts must equal the split count) and no workspace is
 *   needed; if o != NULL the normalised output (q's dtype) and lse (nullable)
 *   are written after the combine.  At least one of parts_out / o must be set.
 *   With parts_out == NULL and o != NULL the global section runs INSIDE the
 *   split kernel: each CTA publishes its triples and takes a ticket; the last
 *   CTA of the (b, hkv) group combines all splits (Eq. 8) -- one launch.
 *   (If num_splits is too large for the kernel to stage the per-split
 *   weights, or parts_out is given, a separate combine launch is used.)
 * ------------------------------------------------------------------- */
ATTN_API int32_t attn_splitkv_default_splits(const attn_problem* prob, int32_t sm_count);
ATTN_API size_t attn_splitkv_workspace_bytes(const attn_problem* prob, int32_t num_splits);
ATTN_API attn_status attn_splitkv_decode(const attn_problem* prob, attn_tensor q, attn_tensor k, attn_tensor v,
                                int32_t num_splits, void* workspace, size_t workspace_bytes,
                                const attn_parts* parts_out, attn_tensor o, float* lse,
                                attn_stream_t stream);

/* attn_splitkv_decode_packed: the same local section with the fused global
 * section (Eq. 8 over the splits, last CTA per (b, hkv)) writing the UN-normalised
 * merged triple of every (b, hq) instead of O / lse:
 *   packed[(b*Hq + hq)*(D+2) + d] = sum_s w_s O_s[d]   (d < D),
 *   packed[... + D] = M (natural log; -inf if no key),  packed[... + D + 1] = L,
 * with M = max_s m_s, w_s = exp(m_s - M), L = sum_s w_s l_s -- the send buffer of
 * a KV-sharded decode (one launch).  seqlen_q must be 1; workspace as for
 * attn_splitkv_decode (ticket block zero); num_splits must not exceed the
 * kernel's staging limit (UNSUPPORTED otherwise; 0 = default, always within).
 * packed: DEVICE fp32 [B][Hq][D+2] contiguous. */
ATTN_API attn_status attn_splitkv_decode_packed(const attn_problem* prob, attn_tensor q, attn_tensor k,
                                                attn_tensor v, int32_t num_splits, void* workspace,
                                                size_t workspace_bytes, float* packed, attn_stream_t stream);

/* ---------------------------------------------------------------------
 * attn_combine -- the Split-K global section (Fig. 5 s_max_global /
 * s_sum_global, Eq. 8) over in->num_parts partial triples per
 * (b, h):  M = max_p m_p;  w_p = exp(m_p - M) (0 if m_p = -inf);
 *          L = sum_p w_p l_p;  O = sum_p w_p O_p.
 * Outputs (each nullable, at least one set):
 *   o     : O / L in out_dtype ([B][H][1][D] view; 0 where L = 0)
 *   lse   : M + ln L, fp32 [B][H] contiguous (-inf where L = 0)
 *   acc_out: the UN-normalised merged triple (num_parts must be 1), used to
 *            merge hierarchically (splits within a GPU, then GPUs).
 * Valid because h commutes with the reducer (Eq. 4).
 * ------------------------------------------------------------------- */
ATTN_API attn_status attn_combine(int32_t batch, int32_t heads, int32_t head_dim, const attn_parts* in,
                         attn_dtype out_dtype, attn_tensor o, float* lse, const attn_parts* acc_out,
                         attn_stream_t stream);

/* ---------------------------------------------------------------------
 * attn_merge_partials -- Eq. 8 over num_parts NORMALISED partial
 * results of the same query rows, e.g. the per-GPU outputs of a KV-sharded
 * (context-parallel) Rolling Update prefill.  A normalised partial (O_p,
 * lse_p) is the repaired triple (m = lse_p, l = 1, O_p) (Thm. 2: h
 * tag-updates to any reference), so for every row:
 *   M = max_p lse_p,  w_p = exp(lse_p - M) (0 if lse_p = -inf),
 *   L = sum_p w_p,    O = sum_p w_p O_p / L,   lse = M + ln L
 * (O = 0, lse = -inf if every part is empty).
 *   o_in : DEVICE, element type in_dtype; row r of part p at
 *          o_in + p*o_stride_part + r*o_stride_row (elements), head_dim contiguous.
 *   lse_in: DEVICE fp32, lse_in[p*lse_stride_part + r].
 *   o_out: DEVICE, element type out_dtype, row r at o_out + r*o_out_stride_row
 *          (nullable);  lse_out: DEVICE fp32 [rows] (nullable).
 * head_dim <= 256.  Errors: INVALID_ARGUMENT, UNSUPPORTED, CUDA.
 * ------------------------------------------------------------------- */
ATTN_API attn_status attn_merge_partials(int32_t num_parts, int64_t rows, int32_t head_dim, attn_dtype in_dtype,
                                         const void* o_in, int64_t o_stride_part, int64_t o_stride_row,
                                         const float* lse_in, int64_t lse_stride_part, attn_dtype out_dtype,
                                         void* o_out, int64_t o_out_stride_row, float* lse_out,
                                         attn_stream_t stream);

/* ---------------------------------------------------------------------
 * attn_softmax_rows -- the paper's motivating reduction chain (Fig. 2,
 * P:164-215) on a [rows][cols] matrix, fused into one pass with both repairs
 * (privatised local reductions rolled across chunks, Fig. 19 / Fig. 2c, then
 * the Eq. 8 merge across threads):
 *   row_max[r] = max_j x[r][j]                (natural units; -inf if empty)
 *   row_sum[r] = sum_j exp(x[r][j] - row_max[r])   (Fig. 2a's xsum; 0 if empty)
 *   y[r][j]    = exp(x[r][j] - row_max[r]) / row_sum[r]   (0 for an empty row)
 * x, y: DEVICE, element type dtype, row stride in elements, contiguous rows;
 * base 16-byte aligned and stride a multiple of 16 bytes.  y, row_max,
 * row_sum are each nullable (at least one set).  Errors: INVALID_ARGUMENT,
 * ALIGNMENT, CUDA.
 * ------------------------------------------------------------------- */
ATTN_API attn_status attn_softmax_rows(int64_t rows, int32_t cols, attn_dtype dtype, const void* x,
                                       int64_t x_stride_row, void* y, int64_t y_stride_row, float* row_max,
                                       float* row_sum, attn_stream_t stream);

/* ---------------------------------------------------------------------
 * Multi-GPU Split-K decode over a KV-SEQUENCE-sharded cache (
 * the same Eq. 8 algebra one level up, valid by Eq. 4).  One
 * process per GPU; NCCL is loaded at run time (dlopen "libnccl.so.2", so a
 * process that already loaded torch's NCCL shares it).
 *
 * attn_nccl_get_unique_id: writes the 128-byte ncclUniqueId (rank 0 calls it
 *   and ships the bytes to the other ranks out of band).
 * attn_nccl_comm_init: *comm = a new communicator handle (host memory) over
 *   nranks processes; this process is `rank`; the CURRENT CUDA device is
 *   used.  Blocks until all ranks joined (ncclCommInitRank).
 * attn_nccl_comm_destroy: frees the handle (NULL is a no-op).
 * attn_decode_kv_sharded_workspace_bytes: DEVICE workspace for the call below
 *   (256-byte aligned).  Its first 256-byte-rounded [B][Hkv] uint32 block holds
 *   the decode kernel's arrival tickets and MUST be zero before the first call
 *   (every call leaves it zero, as for attn_splitkv_decode).
 * attn_decode_kv_sharded: `local` describes THIS rank's shard: seqlen_kv =
 *   shard length, kv_pos_offset = absolute position of the shard's first key,
 *   seqlen_kv_total = global KV length; q is replicated on every rank.  Steps,
 *   all enqueued on `stream` (CUDA-graph capturable):
 *     1. attn_splitkv_decode_packed over the shard: the split kernel's fused
 *        global section merges this rank's splits into one UN-normalised
 *        triple per (b, hq), packed as [B][Hq][D+2] fp32 (O at 0..D-1, m at D,
 *        l at D+1) -- one launch (a separate merge launch only when the split
 *        count exceeds what the kernel can stage);
 *     2. ncclAllGather -> [nranks][B][Hq][D+2];
 *     3. attn_combine over the nranks parts -> o (q's dtype), lse (nullable,
 *        fp32 [B][Hq]) -- identical on every rank.
 *   Errors: those of attn_splitkv_decode / attn_combine, WORKSPACE_TOO_SMALL,
 *   ALIGNMENT, NCCL.
 * ------------------------------------------------------------------- */
ATTN_API attn_status attn_nccl_get_unique_id(void* id_out);
ATTN_API attn_status attn_nccl_comm_init(void** comm, int32_t nranks, int32_t rank, const void* nccl_unique_id);
ATTN_API attn_status attn_nccl_comm_destroy(void* comm);
ATTN_API size_t attn_decode_kv_sharded_workspace_bytes(const attn_problem* local, int32_t nranks);
ATTN_API attn_status attn_decode_kv_sharded(void* comm, const attn_problem* local, attn_tensor q,
                                            attn_tensor k_shard, attn_tensor v_shard, void* workspace,
                                            size_t workspace_bytes, attn_tensor o, float* lse,
                                            attn_stream_t stream);

/* ---------------------------------------------------------------------
 * Seeded synthetic inputs are produced by a separate library (datagen/);
 * nothing here generates data.  Introspection:
 * ------------------------------------------------------------------- */
ATTN_API const char* attn_status_string(attn_status s);
ATTN_API const char* attn_last_error(void);   /* thread-local detail of the last non-OK status */
ATTN_API int attn_abi_version(void);
/* Number of kernels the last successful call on this thread enqueued (for
 * launch accounting in bench.py). */
ATTN_API int attn_last_launch_count(void);

/* Repair-event counters (test instrumentation; proves that the Eq. 7 O-rescale,
 * P:604-607, h = exp(r - r') t of Fig. 18d, runs in a given kernel).
 * counters: DEVICE uint32 [ATTN_REPAIR_SLOTS], caller-owned, or NULL (off, the
 * default).  The setting is thread-local and applies to every later call on the
 * calling thread: each warp that rescales its O accumulator by a factor < 1
 * adds 1 to counters[slot] once per KV step, slot = the kernel that ran:
 *   ATTN_REPAIR_FWD128  prefill grid kernel, D = 128   (fwd_tc_kernel)
 *   ATTN_REPAIR_FWD64   prefill grid kernel, D = 64    (fwd_tc_kernel, 2 CTAs/SM)
 *   ATTN_REPAIR_PERSIST persistent causal prefill kernel (fwd_tc_persist_kernel)
 *   ATTN_REPAIR_DECODE  split-KV decode local section  (decode_split_kernel)
 * Off, it costs nothing; on, one atomic per warp inside the rescale branch. */
#define ATTN_REPAIR_FWD128 0
#define ATTN_REPAIR_FWD64 1
#define ATTN_REPAIR_PERSIST 2
#define ATTN_REPAIR_DECODE 3
#define ATTN_REPAIR_SLOTS 4
ATTN_API void attn_debug_repair_counters(unsigned int* counters);

#ifdef __cplusplus
}
#endif
#endif /* ATTN_H_ */
