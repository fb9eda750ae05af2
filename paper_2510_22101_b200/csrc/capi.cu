// C-ABI of libprefill_sm100.so (include/prefill_sm100.h): model handle, workspace layout,
// the packed forward (pf_score), the host-buffer variant and per-op entry points.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>
#include <cudaTypedefs.h>
#include "pf_internal.h"
#include "../../include/prefill_sm100.h"

namespace pf {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PF_NO_PDL");
    v = (e && e[0] == '1') ? 0 : 1;
  }
  return v == 1;
}

int current_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDevices) d = 0;
  return d;
}

int device_sm_count(int dev) {
  static int sms[kMaxDevices] = {};
  if (sms[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1) n = 148;
    sms[dev] = n;
  }
  return sms[dev];
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool make_tmap_2d(CUtensorMap* out, const void* base, int elem_bytes, uint64_t rows, uint64_t cols,
                  uint64_t ld, uint32_t box_rows, uint32_t box_cols, bool swizzle128) {
  auto enc = get_encode();
  if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return false; }
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0 || (ld * elem_bytes) % 16 != 0) {
    set_error("tensor map: base %p / row stride %llu B not 16-byte aligned", base,
              (unsigned long long)(ld * elem_bytes));
    return false;
  }
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * (uint64_t)elem_bytes};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUtensorMapDataType dt = elem_bytes == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  CUresult r = enc(out, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): rows=%llu cols=%llu ld=%llu box=%ux%u", (int)r,
              (unsigned long long)rows, (unsigned long long)cols, (unsigned long long)ld, box_rows,
              box_cols);
    return false;
  }
  return true;
}

bool make_tmap_2d_u8_sw64(CUtensorMap* out, const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                          uint32_t box_rows, uint32_t box_cols) {
  auto enc = get_encode();
  if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return false; }
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0 || ld % 16 != 0) {
    set_error("tensor map: base %p / row stride %llu B not 16-byte aligned", base, (unsigned long long)ld);
    return false;
  }
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (u8) failed (%d): rows=%llu cols=%llu ld=%llu", (int)r,
              (unsigned long long)rows, (unsigned long long)cols, (unsigned long long)ld);
    return false;
  }
  return true;
}

}  // namespace pf

using namespace pf;

struct pf_model {
  pf_model_desc d;
  std::vector<const void*> w_qkv, w_o, w_gu, w_down;
  std::vector<CUtensorMap> tm_qkv, tm_o, tm_gu, tm_down;  // cached weight (B operand) maps
  CUtensorMap tm_q_last, tm_kv_last;                        // last layer: q rows / k,v rows of W_qkv
  bool last_rows_attention;  // last layer: Q and attention on the last-token rows only (PF_LAST_ROWS_ATTN=0 disables)
  int qkv_n, attn_k;
  bool last_layer_compact;   // PF_NO_LAST_LAYER_COMPACT=1 disables (for tests/benchmarks)
};

namespace {

constexpr size_t kAlign = 1024;
size_t align_up(size_t x) { return (x + kAlign - 1) & ~(kAlign - 1); }

struct Workspace {
  // residual stream x = hi + lo: hi = bf16(x) is the A operand of the QKV and gate/up GEMMs (their
  // epilogues apply the fused RMSNorm), lo = byte b with x - hi = (b - 128) * 2^(E(hi) - 142)
  void* xb;          // hi
  void* rlo;         // lo: uint8 b, x - hi = (b - 128) * 2^(E(hi) - 142) (ptx.cuh resid_decode)
  float* ss_attn;    // per-row partial sums of squares of the residual feeding the attention block
  float* ss_mlp;     // ... feeding the MLP block ([ss_parts(d)][T], see pf_internal.h)
  float* rope_cs;    // per-row cos/sin gathered for the QKV epilogue (launch_rope_gather layout)
  void* qkv;
  void* attn;
  void* hbuf;
  void* attn_c;      // [n_items x H*dh] bf16  last-layer compacted rows
  void* hi_c;        // [n_items x d] bf16
  void* lo_c;        // [n_items x d] uint8
  void* q_c;         // [n_items x H*dh] bf16  last layer: q of the last-token rows (RoPE applied)
  float* ss_c;       // [ss_parts(d) x n_items] their fused-RMSNorm partial sums
  int32_t* pos_c;    // [n_items] their positions
  // device copies of host inputs/outputs (pf_score_host)
  int32_t *ids, *pos, *segs, *work, *last_idx;
  float *logits2, *p_yes;
  int* bad;
  int* verr;         // pf_score under PF_VALIDATE=1: device bounds-check result (launch_validate_packed)
  uint32_t* mlp_ctr; // [n_layers][mlp_counter_words(T)] row-block completion counters of the fused tail
  size_t mlp_ctr_bytes;
  size_t total;
};

Workspace layout(const pf_model* m, int T, int n_items, int n_seg, int n_work, uint8_t* base) {
  const pf_model_desc& d = m->d;
  Workspace w{};
  size_t off = 0;
  auto take = [&](size_t bytes) { uint8_t* p = base + off; off = align_up(off + bytes); return p; };
  w.xb = take((size_t)T * d.d_model * 2);
  w.rlo = take((size_t)T * d.d_model);
  w.ss_attn = reinterpret_cast<float*>(take((size_t)ss_parts(d.d_model) * T * 4));   // [part][T]
  w.ss_mlp = reinterpret_cast<float*>(take((size_t)ss_parts(d.d_model) * T * 4));
  w.rope_cs = reinterpret_cast<float*>(take(rope_gather_floats(T, d.d_head / 2) * 4));
  w.qkv = take((size_t)T * m->qkv_n * 2);
  w.attn = take((size_t)T * m->attn_k * 2);
  w.hbuf = take((size_t)T * d.d_ff_pad * 2);
  w.attn_c = take((size_t)n_items * m->attn_k * 2);
  w.hi_c = take((size_t)n_items * d.d_model * 2);
  w.lo_c = take((size_t)n_items * d.d_model);
  w.q_c = take((size_t)n_items * d.n_heads * d.d_head * 2);
  w.ss_c = reinterpret_cast<float*>(take((size_t)ss_parts(d.d_model) * n_items * 4));
  w.pos_c = reinterpret_cast<int32_t*>(take((size_t)n_items * 4));
  w.ids = reinterpret_cast<int32_t*>(take((size_t)T * 4));
  w.pos = reinterpret_cast<int32_t*>(take((size_t)T * 4));
  w.segs = reinterpret_cast<int32_t*>(take((size_t)n_seg * 16));
  w.work = reinterpret_cast<int32_t*>(take((size_t)n_work * 16));
  w.last_idx = reinterpret_cast<int32_t*>(take((size_t)n_items * 4));
  w.logits2 = reinterpret_cast<float*>(take((size_t)n_items * 8));
  w.p_yes = reinterpret_cast<float*>(take((size_t)n_items * 4));
  w.bad = reinterpret_cast<int*>(take(16));
  w.verr = reinterpret_cast<int*>(take(16));
  w.mlp_ctr_bytes = (size_t)d.n_layers * mlp_counter_words(T) * 4;
  w.mlp_ctr = reinterpret_cast<uint32_t*>(take(w.mlp_ctr_bytes));
  w.total = off;
  return w;
}

}  // namespace

extern "C" {

const char* pf_last_error(void) { return g_err; }
int pf_debug_set_mlp_stats(void* device_buf) {
  return debug_set_mlp_stats(reinterpret_cast<unsigned long long*>(device_buf));
}
int pf_debug_set_trace(void* device_buf, unsigned int capacity) {
  return debug_set_attention_trace(reinterpret_cast<unsigned long long*>(device_buf), capacity);
}

const char* pf_version(void) { return "prefill_sm100 0.1 (tcgen05 bf16, sm_100a)"; }

int pf_model_create(const pf_model_desc* desc, pf_model** out) {
  if (!desc || !out) return fail(-1, "pf_model_create: null argument");
  const pf_model_desc& d = *desc;
  if (d.n_layers < 1 || d.d_model % 128 != 0 || d.n_heads < 1 || d.n_kv_heads < 1 ||
      d.n_heads % d.n_kv_heads != 0)
    return fail(-2, "pf_model_create: invalid dims (L=%d d=%d H=%d Hkv=%d)", d.n_layers, d.d_model,
                d.n_heads, d.n_kv_heads);
  if (d.d_head != 128 && d.d_head != 64)
    return fail(-2, "pf_model_create: d_head must be 64 or 128 (got %d)", d.d_head);
  if (d.d_ff_pad % 128 != 0 || d.d_ff_pad < d.d_ff)
    return fail(-2, "pf_model_create: d_ff_pad=%d must be a multiple of 128 >= d_ff=%d", d.d_ff_pad, d.d_ff);
  pf_model* m = new (std::nothrow) pf_model();
  if (!m) return fail(-1, "pf_model_create: out of host memory");
  m->d = d;
  m->qkv_n = (d.n_heads + 2 * d.n_kv_heads) * d.d_head;
  m->attn_k = d.n_heads * d.d_head;
  {
    const char* e = getenv("PF_NO_LAST_LAYER_COMPACT");
    m->last_layer_compact = !(e && e[0] == '1');
  }
  const int L = d.n_layers;
  m->w_qkv.assign(d.w_qkv, d.w_qkv + L);
  m->w_o.assign(d.w_o, d.w_o + L);
  m->w_gu.assign(d.w_gu, d.w_gu + L);
  m->w_down.assign(d.w_down, d.w_down + L);
  m->d.w_qkv = m->w_qkv.data();
  m->d.w_o = m->w_o.data();
  m->d.w_gu = m->w_gu.data();
  m->d.w_down = m->w_down.data();
  m->tm_qkv.resize(L);
  m->tm_o.resize(L);
  m->tm_gu.resize(L);
  m->tm_down.resize(L);
  for (int l = 0; l < L; ++l) {
    bool ok = make_weight_tmap(&m->tm_qkv[l], m->w_qkv[l], m->qkv_n, d.d_model, d.d_model) &&
              make_weight_tmap(&m->tm_o[l], m->w_o[l], d.d_model, m->attn_k, m->attn_k) &&
              make_weight_tmap(&m->tm_gu[l], m->w_gu[l], 2 * d.d_ff_pad, d.d_model, d.d_model) &&
              make_weight_tmap(&m->tm_down[l], m->w_down[l], d.d_model, d.d_ff_pad, d.d_ff_pad);
    if (!ok) { delete m; return -3; }
  }
  {
    // the split needs the q and k,v widths to be GEMM N multiples (128); otherwise the last layer
    // runs the full QKV GEMM and tile attention before compacting
    const int qn = d.n_heads * d.d_head, kvn = m->qkv_n - qn;
    const char* e = getenv("PF_LAST_ROWS_ATTN");
    m->last_rows_attention = !(e && e[0] == '0') && qn % 128 == 0 && kvn % 128 == 0 &&
                             d.n_heads / d.n_kv_heads <= 8;
    if (m->last_rows_attention &&
        !(make_weight_tmap(&m->tm_q_last, m->w_qkv[L - 1], qn, d.d_model, d.d_model) &&
          make_weight_tmap(&m->tm_kv_last, static_cast<const char*>(m->w_qkv[L - 1]) + (size_t)qn * d.d_model * 2,
                           kvn, d.d_model, d.d_model))) {
      delete m;
      return -3;
    }
  }
  *out = m;
  return 0;
}

int pf_model_destroy(pf_model* model) {
  delete model;
  return 0;
}

size_t pf_workspace_bytes(const pf_model* model, int T, int n_items) {
  if (!model) return 0;
  // segs/work are bounded by T (every segment and tile holds >= 1 token)
  return layout(model, T, n_items, T, T, nullptr).total + kAlign;
}

// ---------------------------------------------------------------- in-step kernel timing
// pf_profile_enable(1): every eager pf_score* call brackets each launch with a pair of CUDA events on
// its stream, tagged with the kernel class; pf_profile_read sums them per class.  Skipped while the
// stream is being captured into a graph.  Measurement only: an event record between two kernels
// also ends the programmatic-dependent-launch overlap at that point.
namespace {
struct Profiler {
  bool on = false;
  std::vector<cudaEvent_t> ev;   // 2 per slot
  std::vector<int> cls;
  size_t used = 0;
};
Profiler g_prof;

struct ProfScope {
  cudaStream_t st;
  long idx = -1;
  ProfScope(int c, cudaStream_t s) : st(s) {
    if (!g_prof.on) return;
    cudaStreamCaptureStatus cs;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return;
    if (g_prof.used == g_prof.cls.size()) {
      cudaEvent_t a, b;
      if (cudaEventCreate(&a) != cudaSuccess) return;
      if (cudaEventCreate(&b) != cudaSuccess) { cudaEventDestroy(a); return; }
      g_prof.ev.push_back(a);
      g_prof.ev.push_back(b);
      g_prof.cls.push_back(c);
    }
    idx = (long)g_prof.used++;
    g_prof.cls[idx] = c;
    cudaEventRecord(g_prof.ev[2 * idx], st);
  }
  ~ProfScope() {
    if (idx >= 0) cudaEventRecord(g_prof.ev[2 * idx + 1], st);
  }
};
const char* const kProfNames[PF_PROF_CLASSES] = {"elementwise", "qkv_rope", "attention",  "o_proj",
                                                 "gate_up",     "down",     "last_layer", "mlp_fused"};
}  // namespace

#define PF_PROF(c) ProfScope _pf_prof_scope_##__LINE__(c, st)

static int mrev_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PF_GEMM_MREV");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v;
}

// PF_MLP_FUSED=1: the layer tail as mlp.cu's one persistent launch instead of three GEMM launches
// (O, gate/up, down).  Off by default: bit-identical, but measured 7-20% slower per layer than the
// three specialised kernels.
static bool mlp_fused_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PF_MLP_FUSED");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1 && gemm_cta_group() == 2;
}

static int run_forward(pf_model* m, const int32_t* ids, const int32_t* pos, const int32_t* segs,
                       int n_seg, const int32_t* work, int n_work, const int32_t* last_idx,
                       int n_items, int T, const Workspace& w, float* logits2, float* p_yes,
                       int* bad, cudaStream_t st, const pf_capture* cap = nullptr) {

  const pf_model_desc& d = m->d;
  const float eps = d.rms_eps;
  const float inv_d = 1.0f / (float)d.d_model;
  // Fused RMSNorm: the residual-update epilogues keep xb = bf16(resid) and ss = sum(resid^2) as
  // per-n-tile partials; the next GEMM sums them in order and scales its accumulator rows by
  // rsqrt(ss/d + eps): no atomics, so a pass is bit-reproducible (norm gains are folded into
  // w_qkv / w_gu by the caller, include/prefill_sm100.h).
  int rc;
  const bool fused = mlp_fused_enabled() && cap == nullptr;
  if (fused) {
    cudaError_t e = cudaMemsetAsync(w.mlp_ctr, 0, w.mlp_ctr_bytes, st);
    if (e != cudaSuccess) return fail(-4, "counter memset: %s", cudaGetErrorString(e));
  }
  {
    PF_PROF(PF_PROF_ELEMENTWISE);
    if ((rc = launch_embed(ids, d.embedding, nullptr, w.xb, w.rlo, w.ss_attn, T, d.d_model, st))) return rc;
    // positions are fixed for the pass: gather each row's cos/sin once into the coalesced layout
    if ((rc = launch_rope_gather(pos, d.rope_cos, d.rope_sin, d.d_head / 2, T, w.rope_cs, st))) return rc;
  }
  for (int l = 0; l < d.n_layers; ++l) {
    // Last layer: only the n_items last-token rows reach the head.  K and V are still needed for every
    // row, but Q, attention, the O projection and the MLP only for those rows (the per-row arithmetic
    // of the GEMMs is unchanged; their attention runs in attn_last_rows_kernel, fp32).
    const bool last = l == d.n_layers - 1 && n_items < T && m->last_layer_compact && cap == nullptr;
    const bool split_qkv = last && m->last_rows_attention;
    GemmDesc g{};
    g.A = w.xb; g.lda = d.d_model; g.B = d.w_qkv[l]; g.ldb = d.d_model;
    g.C = w.qkv; g.ldc = m->qkv_n; g.M = T; g.N = m->qkv_n; g.K = d.d_model;
    g.epilogue = EPI_ROPE_BF16; g.pos = pos; g.rope_cos = d.rope_cos; g.rope_sin = d.rope_sin;
    g.rope_heads = d.n_heads + d.n_kv_heads; g.rope_dh = d.d_head; g.max_seq = d.max_seq;
    g.rope_cs = w.rope_cs;
    g.row_ss = w.ss_attn; g.ss_ld = T; g.inv_d = inv_d; g.eps = eps;
    if (split_qkv) {
      const int qn = d.n_heads * d.d_head;
      {
        PF_PROF(PF_PROF_QKV);
        // K and V of every row: the weight rows after the q heads, written into the qkv buffer's k/v columns
        GemmDesc kv = g;
        kv.B = static_cast<const char*>(d.w_qkv[l]) + (size_t)qn * d.d_model * 2;
        kv.C = static_cast<char*>(w.qkv) + (size_t)qn * 2;
        kv.N = m->qkv_n - qn;
        kv.rope_heads = d.n_kv_heads;
        if ((rc = launch_gemm(kv, &m->tm_kv_last, st))) return rc;
        // q of the last-token rows
        if ((rc = launch_gather_q_rows(last_idx, n_items, w.xb, d.d_model, w.ss_attn, T, pos, w.hi_c, w.ss_c,
                                       w.pos_c, st)))
          return rc;
        GemmDesc q = g;
        q.A = w.hi_c; q.M = n_items; q.N = qn; q.C = w.q_c; q.ldc = qn;
        q.pos = w.pos_c; q.rope_cs = nullptr; q.rope_heads = d.n_heads;
        q.row_ss = w.ss_c; q.ss_ld = n_items;
        if ((rc = launch_gemm(q, &m->tm_q_last, st))) return rc;
      }
      PF_PROF(PF_PROF_ATTENTION);
      if ((rc = launch_attention_last_rows(w.q_c, w.qkv, m->qkv_n, segs, n_seg, last_idx, n_items, d.n_heads,
                                           d.n_kv_heads, d.d_head, d.max_seq, w.attn_c, st)))
        return rc;
    } else {
      {
        PF_PROF(PF_PROF_QKV);
        if ((rc = launch_gemm(g, &m->tm_qkv[l], st))) return rc;
      }
      AttnDesc a{};
      a.qkv = w.qkv; a.out = w.attn; a.T = T; a.H = d.n_heads; a.Hkv = d.n_kv_heads; a.dh = d.d_head;
      a.work = work; a.n_work = n_work; a.segs = segs; a.scale = 1.0f / sqrtf((float)d.d_head);
      PF_PROF(PF_PROF_ATTENTION);
      if ((rc = launch_attention(a, st))) return rc;
    }
    if (last) {
      // O-projection and MLP on the n_items last-token rows alone
      PF_PROF(PF_PROF_LAST_LAYER);
      if ((rc = launch_gather_rows(last_idx, n_items, split_qkv ? nullptr : w.attn, split_qkv ? 0 : m->attn_k,
                                   w.xb, w.rlo, d.d_model, w.attn_c, w.hi_c, w.lo_c, st)))
        return rc;
      GemmDesc o{};
      o.A = w.attn_c; o.lda = m->attn_k; o.B = d.w_o[l]; o.ldb = m->attn_k;
      o.C = w.lo_c; o.ldc = d.d_model; o.M = n_items; o.N = d.d_model; o.K = m->attn_k;
      o.epilogue = EPI_RESID_ADD_NORM; o.xb = w.hi_c; o.ldxb = d.d_model; o.ss_out = w.ss_mlp; o.ss_ld = T;
      if ((rc = launch_gemm(o, &m->tm_o[l], st))) return rc;
      GemmDesc gu{};
      gu.A = w.hi_c; gu.lda = d.d_model; gu.B = d.w_gu[l]; gu.ldb = d.d_model;
      gu.C = w.hbuf; gu.ldc = d.d_ff_pad; gu.M = n_items; gu.N = 2 * d.d_ff_pad; gu.K = d.d_model;
      gu.epilogue = EPI_SWIGLU; gu.row_ss = w.ss_mlp; gu.ss_ld = T; gu.inv_d = inv_d; gu.eps = eps;
      if ((rc = launch_gemm(gu, &m->tm_gu[l], st))) return rc;
      GemmDesc dn{};
      dn.A = w.hbuf; dn.lda = d.d_ff_pad; dn.B = d.w_down[l]; dn.ldb = d.d_ff_pad;
      dn.C = w.lo_c; dn.ldc = d.d_model; dn.M = n_items; dn.N = d.d_model; dn.K = d.d_ff_pad;
      dn.epilogue = EPI_RESID_ADD_NORM; dn.xb = w.hi_c; dn.ldxb = d.d_model; dn.ss_out = w.ss_attn; dn.ss_ld = T;
      if ((rc = launch_gemm(dn, &m->tm_down[l], st))) return rc;
      return launch_head(nullptr, w.hi_c, w.lo_c, nullptr, n_items, d.d_model, d.ln_final, d.w_yes, d.w_no,
                         eps, logits2, p_yes, bad, st);
    }
    if (fused) {
      MlpDesc md{};
      md.attn = w.attn; md.xb = w.xb; md.rlo = w.rlo; md.hbuf = w.hbuf;
      md.M = T; md.d = d.d_model; md.kq = m->attn_k; md.fp = d.d_ff_pad;
      md.counters = w.mlp_ctr + (size_t)l * mlp_counter_words(T);
      md.ss_mlp = w.ss_mlp; md.ss_attn = w.ss_attn; md.ss_ld = T; md.inv_d = inv_d; md.eps = eps;
      PF_PROF(PF_PROF_MLP_FUSED);
      if ((rc = launch_mlp_fused(md, &m->tm_o[l], &m->tm_gu[l], &m->tm_down[l], st))) return rc;
      continue;
    }
    GemmDesc o{};
    o.A = w.attn; o.lda = m->attn_k; o.B = d.w_o[l]; o.ldb = m->attn_k;
    o.C = w.rlo; o.ldc = d.d_model; o.M = T; o.N = d.d_model; o.K = m->attn_k;
    o.epilogue = EPI_RESID_ADD_NORM; o.xb = w.xb; o.ldxb = d.d_model; o.ss_out = w.ss_mlp; o.ss_ld = T;
    // M-order per GEMM (QKV ascending, attention last segments first, O descending, gate/up ascending,
    // down descending): gate/up starts on the residual rows O wrote last, down on the h rows gate/up
    // wrote last, the next QKV on the rows down wrote last
    o.m_rev = mrev_enabled();
    {
      PF_PROF(PF_PROF_O_PROJ);
      if ((rc = launch_gemm(o, &m->tm_o[l], st))) return rc;
    }
    if (cap != nullptr &&
        (rc = launch_capture_rows(cap->rows, cap->n_rows, w.xb, w.rlo, w.ss_mlp, T, cap->gains + (size_t)l * d.d_model,
                                  d.d_model, eps,
                                  cap->out + (size_t)l * (cap->out_layer_stride ? (size_t)cap->out_layer_stride
                                                                                 : (size_t)cap->n_rows * d.d_model),
                                  st)))
      return rc;
    GemmDesc gu{};
    gu.A = w.xb; gu.lda = d.d_model; gu.B = d.w_gu[l]; gu.ldb = d.d_model;
    gu.C = w.hbuf; gu.ldc = d.d_ff_pad; gu.M = T; gu.N = 2 * d.d_ff_pad; gu.K = d.d_model;
    gu.epilogue = EPI_SWIGLU; gu.row_ss = w.ss_mlp; gu.ss_ld = T; gu.inv_d = inv_d; gu.eps = eps;
    {
      PF_PROF(PF_PROF_GATE_UP);
      if ((rc = launch_gemm(gu, &m->tm_gu[l], st))) return rc;
    }
    GemmDesc dn{};
    dn.A = w.hbuf; dn.lda = d.d_ff_pad; dn.B = d.w_down[l]; dn.ldb = d.d_ff_pad;
    dn.C = w.rlo; dn.ldc = d.d_model; dn.M = T; dn.N = d.d_model; dn.K = d.d_ff_pad;
    dn.epilogue = EPI_RESID_ADD_NORM; dn.xb = w.xb; dn.ldxb = d.d_model; dn.ss_out = w.ss_attn; dn.ss_ld = T;
    dn.m_rev = mrev_enabled();
    {
      PF_PROF(PF_PROF_DOWN);
      if ((rc = launch_gemm(dn, &m->tm_down[l], st))) return rc;
    }
  }
  PF_PROF(PF_PROF_ELEMENTWISE);
  return launch_head(nullptr, w.xb, w.rlo, last_idx, n_items, d.d_model, d.ln_final, d.w_yes, d.w_no, eps,
                     logits2, p_yes, bad, st);
}

static int check_args(pf_model* m, int T, int n_items, int n_seg, int n_work, void* ws, size_t ws_bytes,
                      size_t* need) {
  if (!m) return fail(-1, "null model handle");
  if (T < 1 || n_items < 1 || n_seg < 1 || n_work < 1 || n_seg > T || n_work > T)
    return fail(-1, "bad batch sizes T=%d items=%d segs=%d work=%d", T, n_items, n_seg, n_work);
  *need = layout(m, T, n_items, T, T, nullptr).total;
  if (!ws || ws_bytes < *need)
    return fail(-5, "workspace too small: %zu < %zu bytes", ws_bytes, *need);
  if ((reinterpret_cast<uintptr_t>(ws) & (kAlign - 1)) != 0)
    return fail(-1, "workspace must be %zu-byte aligned", kAlign);
  return 0;
}

static const char* const kFaultNames[] = {"", "token id", "position", "segment", "work tile", "last_idx"};

// Runs the device bounds check into `err` and waits for it; 0 when the batch is valid.
static int validate_device_sync(const pf_model* m, const int32_t* ids, const int32_t* pos, const int32_t* segs,
                                int n_seg, const int32_t* work, int n_work, const int32_t* last_idx, int n_items,
                                int T, int* err, cudaStream_t st) {
  cudaStreamCaptureStatus cs;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
    return fail(-1, "PF_VALIDATE=1 cannot be used while the stream is captured into a graph");
  int rc = launch_validate_packed(ids, pos, segs, n_seg, work, n_work, last_idx, n_items, T, m->d.vocab_size,
                                  m->d.max_seq, err, st);
  if (rc) return rc;
  int h[2] = {0, 0};
  cudaError_t e = cudaMemcpyAsync(h, err, sizeof(h), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return fail(-4, "validate: %s", cudaGetErrorString(e));
  if (h[0] != 0)
    return fail(-1, "packed batch invalid: %s at index %d", kFaultNames[h[0] >= 1 && h[0] <= 5 ? h[0] : 0], h[1]);
  return 0;
}

static bool validate_env() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PF_VALIDATE");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

int pf_validate_packed(const pf_model* m, const int32_t* ids, const int32_t* pos, const int32_t* segs, int n_seg,
                       const int32_t* work, int n_work, const int32_t* last_idx, int n_items, int T, int* err,
                       pf_stream_t stream) {
  if (!m) return fail(-1, "null model handle");
  if (T < 1 || n_items < 1 || n_seg < 1 || n_work < 1 || n_seg > T || n_work > T)
    return fail(-1, "bad batch sizes T=%d items=%d segs=%d work=%d", T, n_items, n_seg, n_work);
  if (!ids || !pos || !segs || !work || !last_idx || !err) return fail(-1, "pf_validate_packed: null buffer");
  return launch_validate_packed(ids, pos, segs, n_seg, work, n_work, last_idx, n_items, T, m->d.vocab_size,
                                m->d.max_seq, err, reinterpret_cast<cudaStream_t>(stream));
}

int pf_score(pf_model* m, const int32_t* ids, const int32_t* pos, const int32_t* segs, int n_seg,
             const int32_t* work, int n_work, const int32_t* last_idx, int n_items, int T,
             void* workspace, size_t ws_bytes, float* logits2, float* p_yes, int* bad_flag,
             pf_stream_t stream) {
  size_t need = 0;
  int rc = check_args(m, T, n_items, n_seg, n_work, workspace, ws_bytes, &need);
  if (rc) return rc;
  Workspace w = layout(m, T, n_items, T, T, static_cast<uint8_t*>(workspace));
  if (validate_env() &&
      (rc = validate_device_sync(m, ids, pos, segs, n_seg, work, n_work, last_idx, n_items, T, w.verr,
                                 reinterpret_cast<cudaStream_t>(stream))))
    return rc;
  return run_forward(m, ids, pos, segs, n_seg, work, n_work, last_idx, n_items, T, w, logits2,
                     p_yes, bad_flag, reinterpret_cast<cudaStream_t>(stream));
}

int pf_score_capture(pf_model* m, const int32_t* ids, const int32_t* pos, const int32_t* segs, int n_seg,
                     const int32_t* work, int n_work, const int32_t* last_idx, int n_items, int T,
                     void* workspace, size_t ws_bytes, float* logits2, float* p_yes, int* bad_flag,
                     const pf_capture* cap, pf_stream_t stream) {
  size_t need = 0;
  int rc = check_args(m, T, n_items, n_seg, n_work, workspace, ws_bytes, &need);
  if (rc) return rc;
  if (!cap || cap->n_rows < 0 || (cap->n_rows > 0 && (!cap->rows || !cap->gains || !cap->out)) ||
      (cap->out_layer_stride != 0 && cap->out_layer_stride < (long long)cap->n_rows * m->d.d_model))
    return fail(-1, "pf_score_capture: bad capture descriptor");
  Workspace w = layout(m, T, n_items, T, T, static_cast<uint8_t*>(workspace));
  if (validate_env() &&
      (rc = validate_device_sync(m, ids, pos, segs, n_seg, work, n_work, last_idx, n_items, T, w.verr,
                                 reinterpret_cast<cudaStream_t>(stream))))
    return rc;
  return run_forward(m, ids, pos, segs, n_seg, work, n_work, last_idx, n_items, T, w, logits2, p_yes, bad_flag,
                     reinterpret_cast<cudaStream_t>(stream), cap);
}

// Host-side validation of a packed batch (pf_score_host only: the inputs are host memory).
static int validate_packed(const pf_model* m, const int32_t* ids, const int32_t* pos, const int32_t* segs,
                           int n_seg, const int32_t* work, int n_work, const int32_t* last_idx, int n_items,
                           int T) {
  const pf_model_desc& d = m->d;
  for (int t = 0; t < T; ++t) {
    if (ids[t] < 0 || ids[t] >= d.vocab_size) return fail(-1, "token id %d at row %d outside vocab", ids[t], t);
    if (pos[t] < 0 || pos[t] >= d.max_seq) return fail(-1, "position %d at row %d outside max_seq", pos[t], t);
  }
  for (int s = 0; s < n_seg; ++s) {
    const int32_t* g = segs + 4 * s;
    const int64_t kv_end = (int64_t)g[0] + g[1], q_end = (int64_t)g[2] + g[3];
    if (g[0] < 0 || g[1] < 0 || g[2] < 0 || g[3] < 1 || kv_end > T || q_end > T)
      return fail(-1, "segment %d {%d,%d,%d,%d} outside [0,%d)", s, g[0], g[1], g[2], g[3], T);
    if (s > 0 && g[2] < (int64_t)g[-2] + g[-1])   // q ranges increase (the last-row attention relies on it)
      return fail(-1, "segment %d q range [%d,+%d) overlaps or precedes segment %d", s, g[2], g[3], s - 1);
  }
  for (int w = 0; w < n_work; ++w) {
    const int32_t* k = work + 4 * w;
    if (k[0] < 0 || k[0] >= n_seg || k[1] < 0 || (int64_t)k[1] * 128 >= segs[4 * k[0] + 3])
      return fail(-1, "work tile %d {%d,%d} invalid", w, k[0], k[1]);
  }
  for (int i = 0; i < n_items; ++i)
    if (last_idx[i] < 0 || last_idx[i] >= T) return fail(-1, "last_idx[%d]=%d outside [0,%d)", i, last_idx[i], T);
  return 0;
}

int pf_score_host(pf_model* m, const int32_t* ids, const int32_t* pos, const int32_t* segs,
                  int n_seg, const int32_t* work, int n_work, const int32_t* last_idx, int n_items,
                  int T, void* workspace, size_t ws_bytes, float* logits2_host, float* p_yes_host,
                  pf_stream_t stream) {
  size_t need = 0;
  int rc = check_args(m, T, n_items, n_seg, n_work, workspace, ws_bytes, &need);
  if (rc) return rc;
  if (!ids || !pos || !segs || !work || !last_idx || !logits2_host || !p_yes_host)
    return fail(-1, "pf_score_host: null buffer");
  if ((rc = validate_packed(m, ids, pos, segs, n_seg, work, n_work, last_idx, n_items, T))) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Workspace w = layout(m, T, n_items, T, T, static_cast<uint8_t*>(workspace));
  cudaMemcpyAsync(w.ids, ids, (size_t)T * 4, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(w.pos, pos, (size_t)T * 4, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(w.segs, segs, (size_t)n_seg * 16, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(w.work, work, (size_t)n_work * 16, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(w.last_idx, last_idx, (size_t)n_items * 4, cudaMemcpyHostToDevice, st);
  cudaMemsetAsync(w.bad, 0, 4, st);
  rc = run_forward(m, w.ids, w.pos, w.segs, n_seg, w.work, n_work, w.last_idx, n_items, T, w,
                   w.logits2, w.p_yes, w.bad, st);
  if (rc) return rc;
  int bad = 0;
  cudaMemcpyAsync(logits2_host, w.logits2, (size_t)n_items * 8, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(p_yes_host, w.p_yes, (size_t)n_items * 4, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&bad, w.bad, 4, cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return fail(-4, "pf_score_host: %s", cudaGetErrorString(e));
  if (bad) return fail(-6, "non-finite logits");
  return 0;
}

int pf_gemm_bf16(const void* A, int lda, const void* B, int ldb, void* C, int ldc, int M, int N,
                 int K, int epilogue, const int32_t* pos, const float* rope_cos,
                 const float* rope_sin, int rope_heads, pf_stream_t stream) {
  GemmDesc g{};
  g.A = A; g.lda = lda; g.B = B; g.ldb = ldb; g.C = C; g.ldc = ldc; g.M = M; g.N = N; g.K = K;
  g.epilogue = epilogue; g.pos = pos; g.rope_cos = rope_cos; g.rope_sin = rope_sin;
  g.rope_heads = rope_heads;
  return launch_gemm(g, nullptr, reinterpret_cast<cudaStream_t>(stream));
}

int pf_embed(const int32_t* ids, const void* emb, float* resid, void* hi, void* lo, float* ss, int T, int d,
             pf_stream_t stream) {
  return launch_embed(ids, emb, resid, hi, lo, ss, T, d, reinterpret_cast<cudaStream_t>(stream));
}

int pf_gemm_bf16_ex(const pf_gemm_args* a, pf_stream_t stream) {
  if (!a) return fail(-1, "pf_gemm_bf16_ex: null args");
  GemmDesc g{};
  g.A = a->A; g.lda = a->lda; g.B = a->B; g.ldb = a->ldb; g.C = a->C; g.ldc = a->ldc;
  g.M = a->M; g.N = a->N; g.K = a->K; g.epilogue = a->epilogue;
  g.pos = a->pos; g.rope_cos = a->rope_cos; g.rope_sin = a->rope_sin; g.rope_heads = a->rope_heads;
  g.rope_dh = a->rope_dh;
  g.row_ss = a->row_ss; g.ss_ld = a->ss_ld; g.ss_out = a->ss_out; g.xb = a->xb; g.ldxb = a->ldxb;
  g.inv_d = a->inv_d; g.eps = a->eps;
  g.rope_cs = a->rope_cs;
  return launch_gemm(g, nullptr, reinterpret_cast<cudaStream_t>(stream));
}

int pf_layer_tail(pf_model* m, int layer, const void* attn, void* xb, void* rlo, void* hbuf, float* ss_mlp,
                  float* ss_attn, int T, void* counters, size_t counter_bytes, pf_stream_t stream) {
  if (!m) return fail(-1, "null model handle");
  if (layer < 0 || layer >= m->d.n_layers || T < 1) return fail(-1, "pf_layer_tail: layer %d / T %d", layer, T);
  if (!attn || !xb || !rlo || !hbuf || !ss_mlp || !ss_attn || !counters) return fail(-1, "pf_layer_tail: null buffer");
  const size_t need = mlp_counter_words(T) * 4;
  if (counter_bytes < need) return fail(-5, "pf_layer_tail: counters need %zu bytes", need);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(counters, 0, need, st);
  if (e != cudaSuccess) return fail(-4, "pf_layer_tail memset: %s", cudaGetErrorString(e));
  MlpDesc md{};
  md.attn = attn; md.xb = xb; md.rlo = rlo; md.hbuf = hbuf;
  md.M = T; md.d = m->d.d_model; md.kq = m->attn_k; md.fp = m->d.d_ff_pad;
  md.counters = static_cast<uint32_t*>(counters);
  md.ss_mlp = ss_mlp; md.ss_attn = ss_attn; md.ss_ld = T;
  md.inv_d = 1.0f / (float)m->d.d_model; md.eps = m->d.rms_eps;
  return launch_mlp_fused(md, &m->tm_o[layer], &m->tm_gu[layer], &m->tm_down[layer], st);
}

int pf_rmsnorm(const float* x, const float* gamma, void* y, int T, int d, float eps, pf_stream_t stream) {
  return launch_rmsnorm(x, gamma, y, T, d, eps, reinterpret_cast<cudaStream_t>(stream));
}

int pf_prefix_attention(const void* qkv, void* out, int T, int n_heads, int n_kv_heads, int d_head,
                        const int32_t* segs, const int32_t* work, int n_work, pf_stream_t stream) {
  AttnDesc a{};
  a.qkv = qkv; a.out = out; a.T = T; a.H = n_heads; a.Hkv = n_kv_heads; a.dh = d_head;
  a.segs = segs; a.work = work; a.n_work = n_work; a.scale = 1.0f / sqrtf((float)d_head);
  return launch_attention(a, reinterpret_cast<cudaStream_t>(stream));
}

int pf_attention_last_rows(const void* q_rows, const void* qkv, int n_heads, int n_kv_heads, int d_head,
                           const int32_t* segs, int n_seg, const int32_t* last_idx, int n_items, int max_keys,
                           void* out, pf_stream_t stream) {
  if (!q_rows || !qkv || !segs || !last_idx || !out) return fail(-1, "pf_attention_last_rows: null buffer");
  if (n_heads < 1 || n_kv_heads < 1) return fail(-2, "pf_attention_last_rows: bad head counts");
  return launch_attention_last_rows(q_rows, qkv, (n_heads + 2 * n_kv_heads) * d_head, segs, n_seg, last_idx,
                                    n_items, n_heads, n_kv_heads, d_head, max_keys, out,
                                    reinterpret_cast<cudaStream_t>(stream));
}

int pf_head_last_token(const float* resid, const int32_t* last_idx, int n_items, int d,
                       const float* g, const float* w_yes, const float* w_no, float eps,
                       float* logits2, float* p_yes, int* bad, pf_stream_t stream) {
  return launch_head(resid, nullptr, nullptr, last_idx, n_items, d, g, w_yes, w_no, eps, logits2, p_yes, bad,
                     reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"

int pf_profile_enable(int on) {
  g_prof.on = on != 0;
  g_prof.used = 0;
  return 0;
}

int pf_profile_read(double* ms, int* launches, int n_classes) {
  if (!ms || !launches || n_classes < 1) return fail(-1, "pf_profile_read: bad arguments");
  for (int c = 0; c < n_classes; ++c) { ms[c] = 0.0; launches[c] = 0; }
  for (size_t i = 0; i < g_prof.used; ++i) {
    cudaError_t e = cudaEventSynchronize(g_prof.ev[2 * i + 1]);
    float t = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&t, g_prof.ev[2 * i], g_prof.ev[2 * i + 1]);
    if (e != cudaSuccess) return fail(-4, "pf_profile_read: %s", cudaGetErrorString(e));
    const int c = g_prof.cls[i];
    if (c < n_classes) { ms[c] += t; launches[c] += 1; }
  }
  g_prof.used = 0;
  return 0;
}

const char* pf_profile_class_name(int cls) {
  return (cls >= 0 && cls < PF_PROF_CLASSES) ? kProfNames[cls] : "";
}
