// Internal declarations shared by the CUDA translation units of libprefill_sm100.so.
#pragma once
#include <cstdint>
#include <cstddef>
#include <cuda.h>
#include <cuda_runtime.h>

namespace pf {

enum Epilogue : int {
  EPI_BF16 = 0,
  EPI_ROPE_BF16 = 1,
  EPI_SWIGLU = 2,
  EPI_RESID_ADD = 3,
  EPI_RESID_ADD_NORM = 4,   // (hi=xb bf16, lo=C uint8) residual += acc in place, ss_out[nb][row] = tile sum(new^2)
};

// ---- programmatic dependent launch switch (PF_NO_PDL=1 disables)
bool pdl_enabled();

// ---- error state (thread-local message, negative return codes; see include/prefill_sm100.h)
void set_error(const char* fmt, ...);
int fail(int code, const char* fmt, ...);

// ---- per-device launch state.  CUDA function attributes (max dynamic smem) and SM counts belong
// to a device context, so launchers key them by the calling thread's current device (the engine
// makes the model's device current around every call).
constexpr int kMaxDevices = 64;
int current_device();          // cudaGetDevice, clamped to [0, kMaxDevices)
int device_sm_count(int dev);  // cached per device

// ---- tensor maps (host)
// 2-D row-major tensor [rows x cols] of `elem_bytes`-sized elements, `ld` elements per row,
// box = [box_rows x box_cols], 128-byte swizzle when box_cols*elem_bytes == 128.
bool make_tmap_2d(CUtensorMap* out, const void* base, int elem_bytes, uint64_t rows, uint64_t cols,
                  uint64_t ld, uint32_t box_rows, uint32_t box_cols, bool swizzle128);
bool make_tmap_2d_u8_sw64(CUtensorMap* out, const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                          uint32_t box_rows, uint32_t box_cols);

// ---- launchers (return 0 or negative error code)
struct GemmDesc {
  const void* A;     // [M x K] bf16, leading dim lda
  int lda;
  const void* B;     // [N x K] bf16, leading dim ldb
  int ldb;
  void* C;           // bf16 [M x ldc] (fp32 for EPI_RESID_ADD)
  int ldc;
  int M, N, K;
  int epilogue;
  const int32_t* pos;
  const float* rope_cos;
  const float* rope_sin;
  // optional: cos/sin pre-gathered per packed row in the coalesced layout of launch_rope_gather
  // (the forward builds it once per pass); null -> the epilogue reads the tables per row
  const float* rope_cs;
  int rope_heads;
  int rope_dh;     // head width for the RoPE epilogue (64 or 128; 0 -> 128)
  int max_seq;
  // 1: process M blocks last-to-first.  The forward alternates directions along producer/consumer
  // pairs so each GEMM first reads the rows its producer wrote last (L2-resident).
  int m_rev;
  // fused RMSNorm (see gemm.cu): A rows are bf16(residual); the epilogue multiplies row r by
  // rsqrt(sum_p row_ss[p*ss_ld + r] / d + eps) over the ceil(K/256) partial sums the producing
  // epilogue stored (fixed order: deterministic).  EPI_RESID_ADD_NORM stores its n-tile nb's
  // row partial sum(new^2) to ss_out[nb*ss_ld + r] (no atomics).  ss_ld 0 -> M.
  const float* row_ss;
  long long ss_ld;
  float* ss_out;
  void* xb;
  int ldxb;
  float inv_d, eps;
};
int launch_gemm(const GemmDesc& d, const CUtensorMap* cached_b, cudaStream_t stream);
// Per-row sum-of-squares statistics are kept as ss_parts(d) partial sums, one per 256-column
// n-tile of the producing GEMM (GEMM_BN), stored [part][row] with a row stride.
__host__ __device__ inline int ss_parts(int d_model) { return (d_model + 255) / 256; }
int gemm_smem_bytes();
int gemm_cta_group();   // 2 (default) or 1 via PF_GEMM_CTAS=1
bool make_weight_tmap(CUtensorMap* out, const void* B, int N, int K, int ldb);

int launch_embed(const int32_t* ids, const void* emb_bf16, float* resid, void* hi, void* lo, float* ss, int T,
                 int d, cudaStream_t stream);
int launch_rmsnorm(const float* resid, const float* gamma, void* out_bf16, int T, int d, float eps,
                   cudaStream_t stream);
// Per-row RoPE cos/sin gathered for the QKV epilogue: for row group g (32 rows), table t (0 cos,
// 1 sin), quad q (4 frequencies), lane l:  out[(((g*2 + t)*(half/4) + q)*32 + l)*4 + e] =
// tab_t[pos[32 g + l]][4 q + e].  A warp's float4 load of one quad is then 512 contiguous bytes.
int launch_rope_gather(const int32_t* pos, const float* cos_tab, const float* sin_tab, int half, int T,
                       float* out, cudaStream_t stream);
inline size_t rope_gather_floats(int T, int half) { return (size_t)((T + 31) / 32) * 32 * 2 * half; }
int launch_capture_rows(const int32_t* rows, int n, const void* hi, const void* lo, const float* ss, int ss_ld,
                        const float* g, int d, float eps, float* out, cudaStream_t stream);
int launch_gather_q_rows(const int32_t* last_idx, int n, const void* hi, int d, const float* ss, int T,
                         const int32_t* pos, void* hi_c, float* ss_c, int32_t* pos_c, cudaStream_t stream);
int launch_attention_last_rows(const void* q_c, const void* qkv, int qkv_n, const int32_t* segs, int n_seg,
                               const int32_t* last_idx, int n_items, int H, int Hkv, int dh, int l_max,
                               void* out, cudaStream_t stream);
int launch_gather_rows(const int32_t* last_idx, int n, const void* attn, int attn_cols, const void* hi,
                       const void* lo, int d, void* attn_c, void* hi_c, void* lo_c, cudaStream_t stream);
// resid (fp32) or, when resid == nullptr, the bf16 (hi, lo) pair
int launch_head(const float* resid, const void* rhi, const void* rlo, const int32_t* last_idx, int n_items, int d,
                const float* final_gamma, const float* w_yes, const float* w_no, float eps,
                float* logits2, float* p_yes, int* bad_flag, cudaStream_t stream);

// Packed-batch bounds check on the device (elementwise.cu).  err[0] = first violation's PF_BAD_*
// code (0 = valid), err[1] = its index inside that array.
enum PackedFault : int { PF_BAD_ID = 1, PF_BAD_POS = 2, PF_BAD_SEG = 3, PF_BAD_WORK = 4, PF_BAD_LAST = 5 };
int launch_validate_packed(const int32_t* ids, const int32_t* pos, const int32_t* segs, int n_seg,
                           const int32_t* work, int n_work, const int32_t* last_idx, int n_items, int T, int vocab,
                           int max_seq, int* err, cudaStream_t stream);

// Fused post-attention layer tail (mlp.cu): O projection + residual, gate/up + SwiGLU, down +
// residual in one persistent launch with per-row-block completion counters.
struct MlpDesc {
  const void* attn;     // [M x kq] bf16 attention output
  void* xb;             // [M x d] bf16 residual hi (updated in place)
  void* rlo;            // [M x d] uint8 residual lo (updated in place)
  void* hbuf;           // [M x fp] bf16 SwiGLU output
  int M, d, kq, fp;
  uint32_t* counters;   // mlp_counter_words(M) zeroed words
  float* ss_mlp;        // [d/256][ss_ld] written by O, read by gate/up
  float* ss_attn;       // [d/256][ss_ld] written by down (next layer's QKV reads it)
  int ss_ld;
  float inv_d, eps;
};
int launch_mlp_fused(const MlpDesc& d, const CUtensorMap* b_o, const CUtensorMap* b_gu, const CUtensorMap* b_dn,
                     cudaStream_t stream);
size_t mlp_counter_words(int M);
// debug: ns / counts per wait site of the fused tail, summed over CTAs (null disables)
int debug_set_mlp_stats(unsigned long long* buf);

struct AttnDesc {
  const void* qkv;        // [T x (H+2Hkv)*dh] bf16 (RoPE already applied to q, k)
  void* out;              // [T x H*dh] bf16
  int T, H, Hkv, dh;
  const int32_t* work;    // [n_work x 4] : {seg_kind|qtile, q_row0, q_rows, seg_index}
  int n_work;
  const int32_t* segs;    // [n_seg x 4] : {prefix_off, P, suffix_off, S}  (prefix segment: S=0)
  float scale;
  unsigned long long* trace;   // debug event trace (pf_debug_set_trace), normally null
  unsigned int trace_cap;
};
int launch_attention(const AttnDesc& d, cudaStream_t stream);
int debug_set_attention_trace(unsigned long long* buf, unsigned int cap);

}  // namespace pf
