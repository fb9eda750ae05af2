// Shared-prefix varlen attention.
//
// Packed layout: per request, prefix rows then item-suffix rows (no padding).  Each "segment"
// is a run of query rows whose keys are
//     dense  : rows [kv_off, kv_off + kv_len)        (the shared query prefix; may be empty)
//     causal : rows [q_off, q_off + 1 + local index) (the segment's own tokens)
// The prefix segment itself is {kv_len = 0, q = prefix rows}.  The prefix K/V are computed once
// per request by the QKV GEMM and read by every item's work unit; nothing is retained after the
// call.  Online softmax over the concatenated key blocks is algebraically the LSE merge of the
// prefix and suffix partials.
//
// Persistent kernel, one CTA per SM.  Work unit = (128-row query tile, GQA kv-head g, pair of
// query heads sharing g): both heads reuse every K/V block loaded.  64-key blocks (a 64-token
// prefix is one block; a 100-token item two).  Warp roles (384 threads):
//   WG0 / WG1   softmax for query head 0 / 1 of the pair: thread i owns row i (TMEM lane i);
//               tcgen05.ld S -> mask -> exp2 -> bf16 P written back to TMEM (tcgen05.st).
//               O is accumulated by the tensor core in TMEM; the running max is only raised
//               (and O rescaled in TMEM) when it grows by > 2^8 (lazy rescale).
//   warp 8      TMA producer: Q pair per unit (double-buffered); K/V 64-key blocks, 3-stage ring
//   warp 9      TMEM owner + tcgen05.mma issuer: S_j = Q_j K^T (SS, M128 N64 K128),
//               O_j += P_j V (TS: P from TMEM, V MN-major from smem, M128 N128 K64)
//   warps 10-11 fill a shared-memory table with this CTA's unit descriptors at kernel start
// TMEM columns: S_{j,buf} at 64 (2 j + buf) [0,256), O_j at 256 + DH j.  S is double-buffered per
// head and P_j(b) (bf16 pairs, 32 columns) overwrites the first half of its own S buffer, so the
// issuer runs S(b+1) while softmax(b) is still working: the softmax never waits for an MMA
// (ncu: the single-buffered version spent ~30% of softmax time in the s_full wait).
#include <cuda_runtime.h>
#include "ptx.cuh"
#include "pf_internal.h"

namespace pf {

constexpr int AT_THREADS = 384;
constexpr int AT_KB = 64;                       // keys per block
constexpr int AT_STAGES = 3;
constexpr int AT_QBOX = 128 * 64 * 2;           // [128 rows x 64 cols] bf16 = 16 KB
constexpr int AT_KBOX = 64 * 64 * 2;            // [64 rows x 64 cols] bf16 = 8 KB
constexpr int AT_TAB = 32;                      // unit descriptors cached per CTA
constexpr float AT_RESCALE_THRESH = 8.0f;       // log2 units

// Layout for head width DH (64 or 128): tiles are built from 64-column SW128 boxes.
template <int DH>
struct AtCfg {
  static constexpr int NBX = DH / 64;                           // boxes per head row
  static constexpr int Q_HEAD = NBX * AT_QBOX;                  // one head's 128-row Q tile
  static constexpr int Q_BUF = 2 * Q_HEAD;                      // a head pair (single-buffered)
  static constexpr int KV_STAGE = 2 * NBX * AT_KBOX;            // K boxes then V boxes
  static constexpr int OFF_KV = Q_BUF;
  static constexpr int OFF_OST = OFF_KV + AT_STAGES * KV_STAGE; // O staging [head][warp][NBX x 4 KB]
  static constexpr int OST_WARP = NBX * 32 * 128;
  static constexpr int OFF_TAB = OFF_OST + 8 * OST_WARP;
  static constexpr int OFF_BAR = OFF_TAB + AT_TAB * 48;
  static constexpr int SMEM = 1024 + OFF_BAR + 192;
  // TMEM columns: S_{j,buf} (and P_j over it) at 64 (2 j + buf), O_j at 256 + DH j
  static constexpr uint32_t TS = 0, TO = 256;
};

// ---- debug trace (pf_debug_set_trace): CTA 0 appends {event, unit, block, ns} records.  The
// buffer pointer travels in the kernel parameters (a global-memory flag cost ~5% of the warp-stall
// samples in the disabled state: one long-scoreboard load per call site).
static unsigned long long* g_trace_buf = nullptr;
static unsigned int g_trace_cap = 0;
enum AttEvt { EV_QFULL = 1, EV_KVFULL, EV_S_ISSUED, EV_PREADY, EV_PV_ISSUED, EV_SFULL, EV_PARRIVE, EV_ODONE, EV_EPI_DONE,
              EV_UNIT_START, EV_END };
PF_DEVICE void att_trace(const AttnDesc& d, int ev, int unit, int blk, int who) {
  // atomic-free: fixed slot per (role, unit, block, event) so tracing adds no round trips
  if (d.trace == nullptr || blockIdx.x != 0 || (threadIdx.x & 31) != 0) return;
  const int role = who == 8 ? 0 : (who == 9 || who == 25) ? 1 : 2 + (who & 1);
  if (unit >= 64 || blk >= 8) return;
  const unsigned int i = ((role * 64 + unit) * 8 + blk) * 16 + ev + (who == 25 ? 11 : 0);
  if (i >= d.trace_cap) return;
  d.trace[i] = ((unsigned long long)ev << 56) | ((unsigned long long)(who & 0xff) << 48) |
                   ((unsigned long long)(unit & 0xff) << 40) | ((unsigned long long)(blk & 0xff) << 32) |
                   (globaltimer_ns() & 0xffffffffull);
}

// Cycle accounting of the softmax warps (debug, with the trace buffer): per-phase clock64 sums,
// accumulated by lane 0 of every softmax warp into the last 64 slots of the trace buffer:
// [0] s_full wait, [1] softmax math (S load -> P store issued), [2] pv_done wait, [3] rescale,
// [4] P store wait + p_ready, [5] o_done/pv_done wait before the epilogue, [6] epilogue, [7] units.
enum AttPhase { PH_SWAIT, PH_MATH, PH_PVWAIT, PH_RESCALE, PH_ARRIVE, PH_ODONE, PH_EPI, PH_UNITS,
                PH_EPI_WAIT, PH_EPI_LD, PH_EPI_CVT, PH_N };
#ifdef PF_ATT_PHASES   // A/B builds only (tools/build_variant.sh NAME -DPF_ATT_PHASES)
struct PhaseClock {
  long long acc[PH_N];
  long long t;
  bool on;
  PF_DEVICE void start(bool enable) {
    on = enable;
    for (int i = 0; i < PH_N; ++i) acc[i] = 0;
    t = clock64();
  }
  PF_DEVICE void lap(int ph) {
    if (!on) return;
    const long long n = clock64();
    acc[ph] += n - t;
    t = n;
  }
  PF_DEVICE void flush(const AttnDesc& d) {
    if (!on || (threadIdx.x & 31) != 0) return;
    for (int i = 0; i < PH_N; ++i)
      atomicAdd(reinterpret_cast<unsigned long long*>(d.trace + d.trace_cap - 64 + i), (unsigned long long)acc[i]);
  }
};
#else
struct PhaseClock {
  long long acc[PH_N];
  static constexpr bool on = false;
  PF_DEVICE void start(bool) {}
  PF_DEVICE void lap(int) {}
  PF_DEVICE void flush(const AttnDesc&) {}
};
#endif

struct UnitInfo {
  int q_row0, q_len, q_local0, kv_off, kv_len, q_off, n_pre, n_blk, h0, nh, g, pad;
};

PF_DEVICE UnitInfo decode_unit(const AttnDesc& d, int u, int r, int n_pairs) {
  UnitInfo ui;
  const int per_w = d.Hkv * n_pairs;
  const int w = u / per_w;
  const int rem = u - w * per_w;
  ui.g = rem / n_pairs;
  const int p = rem - ui.g * n_pairs;
  const int4 wk = reinterpret_cast<const int4*>(d.work)[w];
  const int4 sg = reinterpret_cast<const int4*>(d.segs)[wk.x];
  const int qt = wk.y;
  ui.kv_off = sg.x; ui.kv_len = sg.y; ui.q_off = sg.z; ui.q_len = sg.w;
  ui.q_local0 = qt * 128;
  ui.q_row0 = sg.z + qt * 128;
  ui.n_pre = (sg.y + AT_KB - 1) / AT_KB;
  const int q_end = min(qt * 128 + 128, sg.w);
  ui.n_blk = ui.n_pre + (q_end + AT_KB - 1) / AT_KB;
  ui.h0 = ui.g * r + 2 * p;
  ui.nh = min(2, r - 2 * p);
  ui.pad = 0;
  return ui;
}

template <int DH>
__global__ void __launch_bounds__(AT_THREADS, 1)
    attn_prefix_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKV,
                       const __grid_constant__ CUtensorMap tmO, const AttnDesc d, int n_units) {
  using C = AtCfg<DH>;
  constexpr int AT_Q_HEAD = C::Q_HEAD, AT_Q_BUF = C::Q_BUF, AT_KV_STAGE = C::KV_STAGE;
  constexpr int AT_OFF_KV = C::OFF_KV, AT_OFF_OST = C::OFF_OST, AT_OST_WARP = C::OST_WARP;
  constexpr int AT_OFF_TAB = C::OFF_TAB, AT_OFF_BAR = C::OFF_BAR;
  constexpr uint32_t AT_TS = C::TS, AT_TO = C::TO;
  constexpr int NBX = C::NBX;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = smem + AT_OFF_KV;
  UnitInfo* tab = reinterpret_cast<UnitInfo*>(smem + AT_OFF_TAB);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + AT_OFF_BAR);
  uint64_t* q_full = bars + 0;             // [2]
  uint64_t* q_empty = bars + 2;            // [2]
  uint64_t* kv_full = bars + 4;            // [3]
  uint64_t* kv_empty = bars + 7;           // [3]
  uint64_t* s_full = bars + 10;            // [4]  [head j][S buffer]
  uint64_t* p_ready = bars + 14;           // [2]
  uint64_t* o_done = bars + 16;            // [2]
  uint64_t* pv_done = bars + 18;           // [2]  one phase per PV_j
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 20);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int r = d.H / d.Hkv;
  const int n_pairs = (r + 1) / 2;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmKV);
    tma_prefetch_desc(&tmO);
    for (int i = 0; i < 2; ++i) { mbar_init(&q_full[i], 1); mbar_init(&q_empty[i], 1); }
    for (int s = 0; s < AT_STAGES; ++s) { mbar_init(&kv_full[s], 1); mbar_init(&kv_empty[s], 1); }
    for (int j = 0; j < 4; ++j) mbar_init(&s_full[j], 1);
    for (int j = 0; j < 2; ++j) { mbar_init(&p_ready[j], 4); mbar_init(&o_done[j], 1); mbar_init(&pv_done[j], 1); }
    fence_barrier_init();
  }
  if (warp >= 10) {   // unit-descriptor table: one global round trip per CTA instead of per unit
    for (int i = threadIdx.x - 320; i < AT_TAB; i += 64) {
      const int u = blockIdx.x + i * gridDim.x;
      if (u < n_units) tab[i] = decode_unit(d, u, r, n_pairs);
    }
  }
  if (warp == 9) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_launch_dependents();
  pdl_wait();   // q/k/v come from the QKV GEMM
  auto unit = [&](int u, int k) { return k < AT_TAB ? tab[k] : decode_unit(d, u, r, n_pairs); };

  if (warp == 8) {
    // ---------------------------------------------------------------------- TMA producer
    uint32_t kv_it = 0, q_it = 0;
    int k = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++k) {
      const UnitInfo ui = unit(u, k);
      const int qb = 0;
      att_trace(d, EV_UNIT_START, k, ui.n_blk, 8);
      mbar_wait(&q_empty[qb], (q_it & 1) ^ 1);
      if (elect_one()) {
        mbar_arrive_expect_tx(&q_full[qb], ui.nh * AT_Q_HEAD);
        for (int j = 0; j < ui.nh; ++j) {
          const int qc = (ui.h0 + j) * d.dh;
          uint8_t* dst = sQ + qb * AT_Q_BUF + j * AT_Q_HEAD;
          for (int x = 0; x < NBX; ++x)
            tma_load_2d(dst + x * AT_QBOX, &tmQ, &q_full[qb], qc + 64 * x, ui.q_row0, kEvictFirst);
        }
      }
      __syncwarp();
      ++q_it;
      const int kc = (d.H + ui.g) * d.dh;
      const int vc = (d.H + d.Hkv + ui.g) * d.dh;
      for (int b = 0; b < ui.n_blk; ++b, ++kv_it) {
        const int st = kv_it % AT_STAGES;
        mbar_wait(&kv_empty[st], ((kv_it / AT_STAGES) & 1) ^ 1);
        const int krow = b < ui.n_pre ? ui.kv_off + b * AT_KB : ui.q_off + (b - ui.n_pre) * AT_KB;
        uint8_t* dst = sKV + st * AT_KV_STAGE;
        if (elect_one()) {
          mbar_arrive_expect_tx(&kv_full[st], AT_KV_STAGE);
          for (int x = 0; x < NBX; ++x) {
            tma_load_2d(dst + x * AT_KBOX, &tmKV, &kv_full[st], kc + 64 * x, krow, kEvictLast);
            tma_load_2d(dst + (NBX + x) * AT_KBOX, &tmKV, &kv_full[st], vc + 64 * x, krow, kEvictLast);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 9) {
    // ---------------------------------------------------------------------- MMA issuer
    // Warp-converged loop (uniform descriptors in uniform registers); one elected lane issues.
    // Per head j, S blocks are numbered globally (sc[j]) and alternate between two TMEM buffers;
    // S_j(g) overwrites buffer g&1, whose P_j(g-2) the PV issued just before it reads.  tcgen05.mma
    // ops of one thread execute in issue order, so S_j(b+2) follows PV_j(b) with no completion wait
    // (as CUTLASS's sm100 FMHA does).  Both heads' S(b+2) go out together after both PV(b): issuing
    // per head as soon as its own PV is out was 6% slower at C3 (the heads drift and the 3-stage
    // K/V ring is released by the slower one).
    constexpr uint32_t idesc_s = make_idesc_bf16(128, AT_KB, false, false);
    constexpr uint32_t idesc_o = make_idesc_bf16(128, DH, false, true);    // V is MN-major
    uint32_t kv_it = 0, q_it = 0;
    uint32_t sc[2] = {0u, 0u}, pc[2] = {0u, 0u};   // S blocks / PVs issued per head (global)
    const uint64_t q_desc = kmajor_desc(smem_u32(sQ));
    int k = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++k) {
      const UnitInfo ui = unit(u, k);
      mbar_wait(&q_full[0], q_it & 1);
      att_trace(d, EV_QFULL, k, 0, 9);
      auto wait_kv = [&](int b) {   // K/V block b resident in its ring stage
        const uint32_t st = (kv_it + b) % AT_STAGES;
        mbar_wait(&kv_full[st], ((kv_it + b) / AT_STAGES) & 1);
        att_trace(d, EV_KVFULL, k, b, 9);
        tc_fence_after();
      };
      auto issue_s = [&](int b, int j) {   // S_j(b) = Q_j K(b)^T into S buffer sc[j] & 1
        const uint32_t st = (kv_it + b) % AT_STAGES;
        if (elect_one()) {
          const uint64_t k_desc = kmajor_desc(smem_u32(sKV + st * AT_KV_STAGE));
          const uint32_t buf = sc[j] & 1;
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk) {   // descriptor start field is in 16-byte units
            const uint32_t qo = (j * AT_Q_HEAD + (kk >> 2) * AT_QBOX + (kk & 3) * 32) >> 4;
            const uint32_t ko = ((kk >> 2) * AT_KBOX + (kk & 3) * 32) >> 4;
            umma_bf16_ss(tmem_base + AT_TS + 64 * (2 * j + buf), q_desc + qo, k_desc + ko, idesc_s, kk != 0);
          }
          umma_commit(&s_full[2 * j + buf]);
          if (b == ui.n_blk - 1 && j == ui.nh - 1) umma_commit(&q_empty[0]);   // the unit's last S has read Q
        }
        __syncwarp();
        ++sc[j];
      };
      for (int b = 0; b < min(2, ui.n_blk); ++b) {
        wait_kv(b);
#pragma unroll
        for (int j = 0; j < 2; ++j)
          if (j < ui.nh) issue_s(b, j);
      }
      for (int b = 0; b < ui.n_blk; ++b) {
        const uint32_t st_b = (kv_it + b) % AT_STAGES;
        const uint32_t v_addr = smem_u32(sKV + st_b * AT_KV_STAGE) + NBX * AT_KBOX;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          if (j >= ui.nh) break;
          mbar_wait(&p_ready[j], pc[j] & 1);
          att_trace(d, EV_PREADY, k, b, 9 + 16 * j);
          tc_fence_after();
          const uint32_t tp = tmem_base + AT_TS + 64 * (2 * j + (pc[j] & 1));   // P_j(b) over S buffer
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < AT_KB / 16; ++kk) {
              umma_bf16_ts(tmem_base + AT_TO + j * DH, tp + kk * 8, sw128_desc(v_addr + kk * 2048, AT_KBOX, 1024),
                           idesc_o, (b | kk) != 0);
            }
            umma_commit(&pv_done[j]);
            if (b == ui.n_blk - 1) umma_commit(&o_done[j]);
            if (j == ui.nh - 1) umma_commit(&kv_empty[st_b]);   // S(b) and PV(b) of every head have read it
          }
          __syncwarp();
          ++pc[j];
        }
        if (b + 2 < ui.n_blk) {
          wait_kv(b + 2);
#pragma unroll
          for (int j = 0; j < 2; ++j)
            if (j < ui.nh) issue_s(b + 2, j);
        }
      }
      kv_it += ui.n_blk;
      ++q_it;
    }
  } else if (warp < 8) {
    // -------------------------------------------------------------------- softmax WG j
    const int j = warp >> 2;
    const uint32_t row = (warp & 3) * 32 + lane;
    const uint32_t lane_base = ((warp & 3) * 32) << 16;
    const uint32_t tS0 = tmem_base + lane_base + AT_TS + 64 * (2 * j);   // + 64 * buf
    const uint32_t tO = tmem_base + lane_base + AT_TO + j * DH;
    const float sl2 = d.scale * 1.4426950408889634f;
    uint32_t blk_it = 0, u_it = 0;
    PhaseClock pc;
    pc.start(d.trace != nullptr);
    int k = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++k) {
      const UnitInfo ui = unit(u, k);
      if (j >= ui.nh) continue;
      if (pc.on) pc.acc[PH_UNITS] += 1;
      const int q_local = ui.q_local0 + (int)row;
      float m_used = -INFINITY, l_run = 0.f;   // m_used in scaled (log2) units
      for (int b = 0; b < ui.n_blk; ++b, ++blk_it) {
        const bool is_pre = b < ui.n_pre;
        const int lim = is_pre ? (ui.kv_len - b * AT_KB) : (q_local - (b - ui.n_pre) * AT_KB + 1);
        const bool full = __all_sync(0xffffffffu, lim >= AT_KB);
        // 32-key halves masked for every row of this warp (causal diagonal): P = 0 there without
        // spending SFU work on exp(-inf)
        const int lim_max = __reduce_max_sync(0xffffffffu, lim);
        const uint32_t tS = tS0 + 64 * (blk_it & 1);
        pc.lap(PH_MATH);
        mbar_wait(&s_full[2 * j + (blk_it & 1)], (blk_it >> 1) & 1);
        pc.lap(PH_SWAIT);
        if (lane == 0 && (warp & 3) == 0) att_trace(d, EV_SFULL, k, b, j);
        tc_fence_after();
        uint32_t s[2][32];
        tmem_ld_32x32b_x32(tS, s[0]);
        tmem_ld_32x32b_x32(tS + 32, s[1]);
        tmem_ld_wait();
        if (!full) {
          // only a half that is partly visible to this warp needs per-key masking: on the causal
          // diagonal that is one 32x32 sub-block per warp (fully masked halves are skipped below)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            if (lim_max <= 32 * c || __all_sync(0xffffffffu, lim >= 32 * c + 32)) continue;
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (c * 32 + i >= lim) s[c][i] = __float_as_uint(-INFINITY);
          }
        }
        // row max with 3-input FMNMX (4 independent chains) over the halves this warp can see
        // (an unmasked, fully hidden half holds keys of later rows or of another segment)
        float mxv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) mxv[i] = fmaxf(__uint_as_float(s[0][2 * i]), __uint_as_float(s[0][2 * i + 1]));
#pragma unroll
        for (int i = 4; i < 16; ++i)
          mxv[i & 3] = fmax3(mxv[i & 3], __uint_as_float(s[0][2 * i]), __uint_as_float(s[0][2 * i + 1]));
        if (lim_max > 32) {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            mxv[i & 3] = fmax3(mxv[i & 3], __uint_as_float(s[1][2 * i]), __uint_as_float(s[1][2 * i + 1]));
        }
        const float mx = lim_max > 0 ? sl2 * fmax3(fmaxf(mxv[0], mxv[1]), mxv[2], mxv[3]) : -INFINITY;
        const bool need = mx > m_used + AT_RESCALE_THRESH;
        const bool rescale = __any_sync(0xffffffffu, need);
        const float m_old = m_used;
        if (rescale) m_used = fmaxf(m_used, mx);
        // P = exp2(s*scale - m_used) -> bf16 pairs -> TMEM (over S; PV(b-1) read the other buffer).
        // Key pairs go through FFMA2 / FADD2: ~3 issue slots per element instead of ~7.5.
        uint64_t sum2[2] = {0ull, 0ull};
        uint32_t w[32];
        const uint64_t scale2 = f2_pack(sl2, sl2), negm2 = f2_pack(-m_used, -m_used);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          if (lim_max <= 32 * c) {
#pragma unroll
            for (int i = 0; i < 16; ++i) w[c * 16 + i] = 0u;
            continue;
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const uint64_t x2 =
                ffma2(f2_pack(__uint_as_float(s[c][2 * i]), __uint_as_float(s[c][2 * i + 1])), scale2, negm2);
            float x0, x1;
            f2_unpack(x2, x0, x1);
            const float p0 = ex2_approx(x0), p1 = ex2_approx(x1);
            sum2[i & 1] = fadd2(sum2[i & 1], f2_pack(p0, p1));
            w[c * 16 + i] = pack_bf16x2(p0, p1);   // TMEM A operand: 2 keys per 32-bit column
          }
        }
        float sa, sb, sc2, sd;
        f2_unpack(sum2[0], sa, sb);
        f2_unpack(sum2[1], sc2, sd);
        const float bsum = (sa + sb) + (sc2 + sd);
        tmem_st_32x32b_x32(tS, w);   // P_j(b) over the first half of its own S buffer
        // Every PV phase is consumed in order: PV of this head's previous block (issued right
        // after this block's S) has finished by now, so this wait is ~free; it also guards O.
        // (A unit's last PV phase is consumed in its epilogue.)
        pc.lap(PH_MATH);
        if (b > 0) mbar_wait(&pv_done[j], (blk_it - 1) & 1);
        pc.lap(PH_PVWAIT);
        if (rescale && b > 0) {
          tc_fence_after();
          const float alpha = exp2f(m_old - m_used);
          l_run *= alpha;
#pragma unroll 1
          for (int c = 0; c < DH / 32; ++c) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(tO + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st_32x32b_x32(tO + c * 32, o);
          }
        }
        l_run += bsum;
        pc.lap(PH_RESCALE);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_ready[j]);
        pc.lap(PH_ARRIVE);
        if (lane == 0 && (warp & 3) == 0) att_trace(d, EV_PARRIVE, k, b, j);
      }
      // ---- unit epilogue: O / l -> bf16 -> global
      pc.lap(PH_MATH);
      mbar_wait(&o_done[j], u_it & 1);
      mbar_wait(&pv_done[j], (blk_it - 1) & 1);
      pc.lap(PH_ODONE);
      if (lane == 0 && (warp & 3) == 0) att_trace(d, EV_ODONE, k, 0, j);
      ++u_it;
      tc_fence_after();
      const float inv = 1.f / l_run;
      const bool valid = q_local < ui.q_len;
      // rows of this warp: [q_row0 + 32*(warp&3), +32); TMA-store them when all 32 belong to the
      // segment, else write the valid rows directly (never touch the next segment's rows)
      const bool warp_full = ui.q_local0 + (int)(warp & 3) * 32 + 31 < ui.q_len;
      uint8_t* ost = smem + AT_OFF_OST + (j * 4 + (warp & 3)) * AT_OST_WARP;
      if (warp_full) {
        if (lane == 0) tma_store_wait_read<0>();   // previous unit's store has left the buffer
        __syncwarp();
      }
      pc.lap(PH_EPI_WAIT);
      uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(d.out) +
                                            (size_t)(ui.q_row0 + row) * (d.H * d.dh) + (ui.h0 + j) * d.dh);
#pragma unroll 1
      for (int c2 = 0; c2 < DH / 64; ++c2) {
        uint32_t o2[2][32];   // two 32-column loads in flight per wait
        tmem_ld_32x32b_x32(tO + c2 * 64, o2[0]);
        tmem_ld_32x32b_x32(tO + c2 * 64 + 32, o2[1]);
        tmem_ld_wait();
        pc.lap(PH_EPI_LD);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = 2 * c2 + h;
          const uint32_t (&o)[32] = o2[h];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 v;
            v.x = pack_bf16x2(__uint_as_float(o[8 * q + 0]) * inv, __uint_as_float(o[8 * q + 1]) * inv);
            v.y = pack_bf16x2(__uint_as_float(o[8 * q + 2]) * inv, __uint_as_float(o[8 * q + 3]) * inv);
            v.z = pack_bf16x2(__uint_as_float(o[8 * q + 4]) * inv, __uint_as_float(o[8 * q + 5]) * inv);
            v.w = pack_bf16x2(__uint_as_float(o[8 * q + 6]) * inv, __uint_as_float(o[8 * q + 7]) * inv);
            if (warp_full) {
              // 64-column SW128 box (c >> 1); 16 B chunk (c & 1) * 4 + q of this row
              const uint32_t chunk = (c & 1) * 4 + q;
              st_shared_v4(smem_u32(ost + (c >> 1) * 4096) + lane * 128 + ((chunk ^ (lane & 7)) << 4), v.x, v.y,
                           v.z, v.w);
            } else if (valid) {
              dst[c * 4 + q] = v;
            }
          }
        }
      }
      pc.lap(PH_EPI_CVT);
      if (warp_full) {
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          const int r0 = ui.q_row0 + (warp & 3) * 32;
          const int c0 = (ui.h0 + j) * d.dh;
          for (int x = 0; x < NBX; ++x) tma_store_2d(&tmO, ost + x * 4096, c0 + 64 * x, r0);
          tma_store_commit();
        }
      }
      if (lane == 0 && (warp & 3) == 0) att_trace(d, EV_EPI_DONE, k, 0, j);
      tc_fence_before();
      pc.lap(PH_EPI);
    }
    pc.flush(d);
  }

  if (warp < 8 && lane == 0) tma_store_wait_all<0>();
  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

int debug_set_attention_trace(unsigned long long* buf, unsigned int cap) {
  g_trace_buf = buf;
  g_trace_cap = buf == nullptr ? 0 : cap;
  return 0;
}

template <int DH>
static int launch_attention_t(const AttnDesc& d, cudaStream_t stream) {
  const int ldq = (d.H + 2 * d.Hkv) * d.dh;
  CUtensorMap tq, tkv, to;
  if (!make_tmap_2d(&tq, d.qkv, 2, (uint64_t)d.T, (uint64_t)ldq, (uint64_t)ldq, 128, 64, true)) return -3;
  if (!make_tmap_2d(&tkv, d.qkv, 2, (uint64_t)d.T, (uint64_t)ldq, (uint64_t)ldq, AT_KB, 64, true)) return -3;
  const int ldo = d.H * d.dh;
  if (!make_tmap_2d(&to, d.out, 2, (uint64_t)d.T, (uint64_t)ldo, (uint64_t)ldo, 32, 64, true)) return -3;
  const int dev = current_device();
  static bool attr_set[kMaxDevices] = {};
  if (!attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(attn_prefix_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         AtCfg<DH>::SMEM);
    if (e != cudaSuccess) return fail(-4, "attention smem attr (device %d): %s", dev, cudaGetErrorString(e));
    attr_set[dev] = true;
  }
  const int sms = device_sm_count(dev);
  const int r = d.H / d.Hkv;
  const int n_units = d.n_work * d.Hkv * ((r + 1) / 2);
  const int grid = n_units < sms ? n_units : sms;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(AT_THREADS);
  cfg.dynamicSmemBytes = AtCfg<DH>::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  AttnDesc dd = d;
  dd.trace = g_trace_buf;
  dd.trace_cap = g_trace_cap;
  cudaError_t e = cudaLaunchKernelEx(&cfg, attn_prefix_kernel<DH>, tq, tkv, to, dd, n_units);
  if (e != cudaSuccess) return fail(-4, "attention launch: %s", cudaGetErrorString(e));
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(-4, "attention launch: %s", cudaGetErrorString(e));
  return 0;
}

int launch_attention(const AttnDesc& d, cudaStream_t stream) {
#ifdef PF_DEBUG_SKIP_ATTENTION   // A/B builds only (tools/build_variant.sh): the step without attention
  return 0;
#endif
  if (d.dh != 128 && d.dh != 64) return fail(-2, "attention: d_head must be 64 or 128 (got %d)", d.dh);
  if (d.H % d.Hkv != 0) return fail(-2, "attention: n_heads %% n_kv_heads != 0");
  if (d.n_work == 0) return 0;
  return d.dh == 128 ? launch_attention_t<128>(d, stream) : launch_attention_t<64>(d, stream);
}

}  // namespace pf
