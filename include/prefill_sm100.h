/*
 * prefill_sm100.h — C-ABI of libprefill_sm100.so, the B200 (sm_100a) hot path of prefill-only
 * shared-prefix relevance scoring (arxiv 2510.22101, reference package `prefrank`).
 *
 * The reference ships no code for this path: its interface is specified in
 * /root/reference/SPEC.md (model :172-238, prefixcache :240-309, scoring :311-343).  Each entry
 * point below cites the reference operation it replaces.  All pointers are DEVICE pointers unless
 * a function name ends in `_host`; all buffers are caller-owned (the library never cudaMallocs).
 * Return value: 0 on success, negative on error; the message is in pf_last_error().
 *
 * Error codes:  -1 bad handle/argument, -2 unsupported shape, -3 TMA descriptor encode failed,
 *               -4 CUDA launch/runtime error, -5 workspace too small, -6 non-finite logits
 *               ("non-finite logits" error of relevance_score).
 */
#ifndef PREFILL_SM100_H
#define PREFILL_SM100_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define PF_API __attribute__((visibility("default")))
#else
#define PF_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* pf_stream_t; /* == cudaStream_t */
typedef struct pf_model pf_model;        /* opaque: config + cached weight TMA descriptors */

/*
 * Model description — SPEC.md:177-184 ModelConfig/Weights, with the explicit d_head and padded
 * FFN width the B200 layout needs.  Weights are device tensors in the
 * K-major ("[out x in]") layout the tcgen05 GEMMs read:
 *   embedding  bf16 [vocab_size x d_model]
 *   w_qkv[l]   bf16 [(n_heads + 2 n_kv_heads) d_head x d_model]   rows: q heads | k heads | v heads
 *   w_o[l]     bf16 [d_model x n_heads d_head]
 *   w_gu[l]    bf16 [2 d_ff_pad x d_model]   per 128-neuron block j: 128 gate rows then 128 up rows
 *   w_down[l]  bf16 [d_model x d_ff_pad]     columns >= d_ff are zero (pruned/padded neurons)
 *   The per-layer RMSNorm gains are FOLDED into the GEMM input rows (RMSNorm is fused into the
 *   GEMM epilogues): w_qkv[l] = (diag(g_attn[l]) W_qkv)^T and w_gu[l] = (diag(g_mlp[l]) W_gu)^T.
 *   ln_final : fp32 [d_model] final RMSNorm scale (applied in the head kernel)
 *   w_yes, w_no: fp32 [d_model] — columns yes_id / no_id of the [d_model x vocab] output head
 *   rope_cos, rope_sin: fp32 [max_seq x d_head/2]  (theta^(-2i/d_head) * pos, rotate-half)
 *   d_head: 64 or 128.
 */
typedef struct pf_model_desc {
  int n_layers, d_model, n_heads, n_kv_heads, d_head, d_ff, d_ff_pad, vocab_size, max_seq;
  float rms_eps;
  const void* embedding;
  const void* const* w_qkv;
  const void* const* w_o;
  const void* const* w_gu;
  const void* const* w_down;
  const float* ln_final;
  const float* w_yes;
  const float* w_no;
  const float* rope_cos;
  const float* rope_sin;
} pf_model_desc;

/* Packed request batch (SPEC.md:245-263 SharedBatch, laid out flat):
 *   ids[T], pos[T]           token ids and absolute RoPE positions (prefix 0..P-1, each suffix P..)
 *   segs[n_seg][4]           {kv_off, kv_len, q_off, q_len}: query rows [q_off, q_off+q_len) attend
 *                            densely to rows [kv_off, kv_off+kv_len) (the shared prefix) and
 *                            causally to themselves.  A request's prefix is {q_off, 0, q_off, P}.
 *                            Segments are ordered by q_off with non-overlapping q ranges (as
 *                            pf_pack_requests emits them; the validators reject anything else).
 *   work[n_work][4]          {seg, q_tile, 0, 0}: one entry per 128-row query tile of a segment
 *   last_idx[n_items]        packed row of each item's last token
 */

/* Lifecycle.  Replaces: init_weights/Weights as the device-resident form. */
PF_API int pf_model_create(const pf_model_desc* desc, pf_model** out);
PF_API int pf_model_destroy(pf_model* model);

/* Bytes of device workspace pf_score needs for T packed tokens and n_items items. */
PF_API size_t pf_workspace_bytes(const pf_model* model, int T, int n_items);

/* The whole packed forward: embed -> L x [RMSNorm, QKV+RoPE, shared-prefix attention,
 * O+residual, RMSNorm, gate/up+SwiGLU, down+residual] -> last-token RMSNorm -> yes/no head ->
 * sigmoid.  Replaces score_shared_batch + relevance_score;
 * logits2[n_items][2] = (logit_yes, logit_no), p_yes[n_items].  Device pointers throughout;
 * asynchronous on `stream`.  bad_flag (device int) is OR-ed with 1 on non-finite logits. */
PF_API int pf_score(pf_model* model, const int32_t* ids, const int32_t* pos, const int32_t* segs,
             int n_seg, const int32_t* work, int n_work, const int32_t* last_idx, int n_items,
             int T, void* workspace, size_t ws_bytes, float* logits2, float* p_yes,
             int* bad_flag, pf_stream_t stream);

/* Same, with HOST input/output buffers: H2D copies of the packed batch and D2H copy of the
 * scores are inside the call, which returns after the stream synchronises (-6 on non-finite).
 * The host batch is validated first (ids < vocab, positions < max_seq, segments, work tiles and
 * last_idx inside [0, T)); violations return -1 before any device work. */
PF_API int pf_score_host(pf_model* model, const int32_t* ids, const int32_t* pos, const int32_t* segs,
                  int n_seg, const int32_t* work, int n_work, const int32_t* last_idx,
                  int n_items, int T, void* workspace, size_t ws_bytes, float* logits2_host,
                  float* p_yes_host, pf_stream_t stream);

/* Device-side bounds check of a packed batch already resident on the device (the pf_score inputs).
 * Asynchronous on `stream`: err (device int[2]) receives {code, index} of a violation, {0, 0} when
 * the batch is valid; code 1 token id outside [0, vocab), 2 position outside [0, max_seq), 3 segment
 * outside [0, T), 4 work tile naming a missing segment or tile, 5 last_idx outside [0, T).
 * pf_score / pf_score_capture run the same check (and wait for it, failing with -1 before any
 * forward work) when the environment sets PF_VALIDATE=1.  No reference counterpart: the spec's
 * shape-discipline diagnostics for a device-resident batch. */
PF_API int pf_validate_packed(const pf_model* model, const int32_t* ids, const int32_t* pos, const int32_t* segs,
                              int n_seg, const int32_t* work, int n_work, const int32_t* last_idx, int n_items,
                              int T, int* err, pf_stream_t stream);

/* Calibration capture: the reference forward_prefill's `capture` flag
 * records each layer's MLP input for the pruning module.
 * pf_score_capture runs pf_score and, for every layer l, writes
 *   out[l][i][:] = rmsnorm(x_l[rows[i]]) * gains[l]     (fp32, d_model columns, rows dense)
 * where x_l is the residual entering layer l's MLP block, for the packed rows `rows`
 * (device int32[n_rows], each in [0, T)).  gains = the MLP RMSNorm scales [n_layers x d_model]
 * (fp32, device; the product folds them into w_gu, so capture needs them separately).
 * Last-layer row compaction is disabled while capturing (every row runs every layer). */
typedef struct pf_capture {
  const int32_t* rows;
  int n_rows;
  const float* gains;
  float* out;
  long long out_layer_stride;   /* elements between out[l] and out[l+1]; 0 = n_rows * d_model */
} pf_capture;

PF_API int pf_score_capture(pf_model* model, const int32_t* ids, const int32_t* pos, const int32_t* segs,
                            int n_seg, const int32_t* work, int n_work, const int32_t* last_idx, int n_items,
                            int T, void* workspace, size_t ws_bytes, float* logits2, float* p_yes,
                            int* bad_flag, const pf_capture* capture, pf_stream_t stream);

/* Per-op entry points (unit parity tests). */
/* C = A[MxK] . B[NxK]^T (RoPE heads 128 wide here; pf_gemm_bf16_ex takes rope_dh 64/128)
 * with epilogue 0 bf16, 1 bf16+RoPE, 2 SwiGLU(bf16, N/2 cols),
 * 3 fp32 C += (residual add), 4 residual stream x = hi + lo with hi = xb (bf16, = bf16(x)) and
 * lo = C (uint8 b, x - hi = (b - 128) * 2^(E - 142), E = the biased fp32 exponent of hi; ldc in bytes),
 * updated in place to x + acc, and ss_out[nb * ss_ld + row] = sum over n-tile nb (256 columns)
 * of (x + acc)^2 (pf_gemm_bf16_ex). */
PF_API int pf_gemm_bf16(const void* A, int lda, const void* B, int ldb, void* C, int ldc, int M, int N,
                 int K, int epilogue, const int32_t* pos, const float* rope_cos,
                 const float* rope_sin, int rope_heads, pf_stream_t stream);
/* Full-option GEMM (fused RMSNorm): row_ss != NULL scales accumulator row r by
 * rsqrt(S_r * inv_d + eps), S_r = sum over p < ceil(K/256) of row_ss[p * ss_ld + r] (summed in
 * order: the forward is bit-reproducible).  ss_ld = row stride of row_ss / ss_out (0 -> M). */
typedef struct pf_gemm_args {
  const void* A; int lda; const void* B; int ldb; void* C; int ldc;
  int M, N, K, epilogue;
  const int32_t* pos; const float* rope_cos; const float* rope_sin; int rope_heads; int rope_dh;
  const float* row_ss; long long ss_ld; float* ss_out; void* xb; int ldxb; float inv_d, eps;
  const float* rope_cs;  /* optional: per-row cos/sin pre-gathered in the QKV epilogue's coalesced layout */
} pf_gemm_args;
PF_API int pf_gemm_bf16_ex(const pf_gemm_args* args, pf_stream_t stream);
/* Embedding gather; every output is optional (NULL skips it): resid = float(E[ids]) (fp32),
 * hi = E[ids] and lo = 0x80 bytes (zero; the bf16 hi + 8-bit lo residual the forward keeps), ss = per-row sum of squares
 * in the GEMMs' partial layout: ss[t] = sum, ss[p*T + t] = 0 for 1 <= p < ceil(d/256). */
PF_API int pf_embed(const int32_t* ids, const void* emb, float* resid, void* hi, void* lo, float* ss, int T,
             int d, pf_stream_t stream);
/* y = bf16(x * rsqrt(mean(x^2) + eps) * gamma); gamma may be NULL (all ones). */
PF_API int pf_rmsnorm(const float* x, const float* gamma, void* y_bf16, int T, int d, float eps,
               pf_stream_t stream);
PF_API int pf_prefix_attention(const void* qkv, void* out, int T, int n_heads, int n_kv_heads,
                        int d_head, const int32_t* segs, const int32_t* work, int n_work,
                        pf_stream_t stream);
/* Last layer, last-token rows (replaces the tile attention there; pf_score uses it):
 * out[i, h*dh:(h+1)*dh] = softmax(q_rows[i,h] . K^T / sqrt(dh)) V over row last_idx[i]'s keys (its
 * segment's shared prefix and its own tokens up to last_idx[i]); K, V = the k/v columns of qkv
 * ([T x (H+2Hkv)*dh], RoPE applied).  segs ordered by q_off as pf_pack_* emits them.  fp32 math.
 * max_keys bounds a row's key count (shared memory); a row past it is written as NaN. */
PF_API int pf_attention_last_rows(const void* q_rows, const void* qkv, int n_heads, int n_kv_heads, int d_head,
                                  const int32_t* segs, int n_seg, const int32_t* last_idx, int n_items,
                                  int max_keys, void* out, pf_stream_t stream);
PF_API int pf_head_last_token(const float* resid, const int32_t* last_idx, int n_items, int d,
                       const float* final_gamma, const float* w_yes, const float* w_no,
                       float eps, float* logits2, float* p_yes, int* bad_flag,
                       pf_stream_t stream);

/* ---- Host ingest (C++, no GPU needed) ------------------------------
 * FNV-1a-64 word-hash tokenizer, bit-identical to prefrank tokenizer.encode
 * (/root/reference/pkg/src/prefrank/tokenizer.py:119-134).  UTF-8 input; ids written to out_ids
 * (at most cap; *n_out = total count, -5 if it exceeded cap).  vocab_size/reserved as Vocab. */
PF_API int pf_tokenize(const char* text, size_t len, int vocab_size, int reserved, int32_t* out_ids,
                       int64_t cap, int64_t* n_out);
/* Same, plus the end of each token's span in the lowercased text, in Python str units (the span
 * end tokenizer.encode_with_spans reports, tokenizer.py:104-116; used by truncate_description). */
PF_API int pf_tokenize_spans(const char* text, size_t len, int vocab_size, int reserved, int32_t* out_ids,
                             int64_t* out_ends, int64_t cap, int64_t* n_out);
/* Batched (tokenizer.py:137-161 encode_batch): texts are data[text_offsets[i]..text_offsets[i+1]);
 * cap must be >= total input bytes; out_offsets[n_texts+1] delimits each text's ids.
 * n_threads <= 0 uses all hardware threads. */
PF_API int pf_tokenize_batch(const char* data, const int64_t* text_offsets, int n_texts, int vocab_size,
                             int reserved, int32_t* out_ids, int64_t cap, int64_t* out_offsets,
                             int n_threads);
/* split_shared_prefix + flat packing, bit-identical to prefixcache.pack_requests.
 * Request r owns token lists [list_begin[r], list_begin[r+1]) of the flat list set
 * ids[list_offsets[k]..list_offsets[k+1]).  pf_pack_sizes gives buffer upper bounds. */
PF_API int pf_pack_sizes(const int64_t* list_offsets, const int32_t* list_begin, int n_requests,
                         int64_t* T, int64_t* n_seg, int64_t* n_items);
PF_API int pf_pack_requests(const int32_t* ids, const int64_t* list_offsets, const int32_t* list_begin,
                            int n_requests, int max_seq, int32_t* out_ids, int32_t* out_pos,
                            int32_t* out_segs, int32_t* out_last, int32_t* out_prefix_lens,
                            int64_t* out_T, int64_t* out_n_seg);

/* The fused layer tail of layer `layer` (mlp.cu) on caller buffers: residual (xb bf16 hi, rlo uint8 lo,
 * [T x d_model], updated in place) += attn[T x H*dh] . W_o^T, writing the MLP RMSNorm partials ss_mlp
 * ([d_model/256][T] fp32); hbuf[T x d_ff_pad] = SwiGLU of the normalised residual; residual += hbuf .
 * W_down^T, writing ss_attn.  The same arithmetic as EPI_RESID_ADD_NORM -> EPI_SWIGLU (row_ss =
 * ss_mlp) -> EPI_RESID_ADD_NORM through pf_gemm_bf16_ex, in one launch.  counters: device scratch of
 * >= 8 * ceil(T / 256) bytes (zeroed by the call). */
PF_API int pf_layer_tail(pf_model* model, int layer, const void* attn, void* xb, void* rlo, void* hbuf,
                         float* ss_mlp, float* ss_attn, int T, void* counters, size_t counter_bytes,
                         pf_stream_t stream);

/* In-step kernel timing (measurement only).  pf_profile_enable(1) makes every eager pf_score /
 * pf_score_host / pf_score_capture call bracket each launch with CUDA events on its stream, tagged
 * by kernel class (PF_PROF_*); launches recorded while the stream is capturing a graph are skipped.
 * pf_profile_read waits for the events, writes the summed ms and launch count per class and resets.
 * Process-global, not thread-safe: one measuring thread.  An event record between two kernels ends
 * the programmatic-dependent-launch overlap there, so the per-class sums slightly exceed a graph
 * replay's step time. */
enum {
  PF_PROF_ELEMENTWISE = 0, /* embed, rope cos/sin gather, head */
  PF_PROF_QKV = 1,         /* QKV GEMM + RoPE epilogue */
  PF_PROF_ATTENTION = 2,
  PF_PROF_O_PROJ = 3,      /* O GEMM + residual + RMSNorm statistic */
  PF_PROF_GATE_UP = 4,     /* gate/up GEMM + SwiGLU epilogue */
  PF_PROF_DOWN = 5,        /* down GEMM + residual + RMSNorm statistic */
  PF_PROF_LAST_LAYER = 6,  /* last layer's row gather + O/gate-up/down on the n_items last rows */
  PF_PROF_MLP_FUSED = 7,   /* fused O + gate/up + down layer tail (one launch per layer, mlp.cu) */
  PF_PROF_CLASSES = 8
};
PF_API int pf_profile_enable(int on);
PF_API int pf_profile_read(double* ms, int* launches, int n_classes);
PF_API const char* pf_profile_class_name(int cls);

/* Debug hook: CTA 0 of the attention kernel appends {event, role, unit, block, globaltimer}
 * records (uint64) to device_buf (NULL disables).  Used by tools/attn_trace.py. */
PF_API int pf_debug_set_trace(void* device_buf, unsigned int capacity);
/* Debug: the fused layer tail accumulates ns / counts per wait site into device_buf (u64[16]); null
 * disables. */
PF_API int pf_debug_set_mlp_stats(void* device_buf);

PF_API const char* pf_last_error(void);
PF_API const char* pf_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PREFILL_SM100_H */
