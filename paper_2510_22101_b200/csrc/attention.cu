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
//               tcgen05.ld S -> mask -> exp2 -> bf16 P (swizzled smem).  O is accumulated by
//               the tensor core in TMEM; the running max is only raised (and O rescaled in
//               TMEM) when it grows by > 2^8 (lazy rescale), so most blocks never touch O.
//   warp 8      TMA producer: Q pair per unit; K/V 64-key blocks through a 3-stage ring
//   warp 9      TMEM owner + tcgen05.mma issuer: S_j = Q_j K^T (M128 N64 K128),
//               O_j += P_j V (M128 N128 K64, V MN-major), ping-ponging the two heads
#include <cuda_runtime.h>
#include "ptx.cuh"
#include "pf_internal.h"

namespace pf {

constexpr int AT_THREADS = 384;
constexpr int AT_KB = 64;                       // keys per block
constexpr int AT_STAGES = 3;
constexpr int AT_QBOX = 128 * 64 * 2;           // [128 rows x 64 cols] bf16 = 16 KB
constexpr int AT_KBOX = 64 * 64 * 2;            // [64 rows x 64 cols] bf16 = 8 KB
constexpr int AT_Q_HEAD = 2 * AT_QBOX;          // one head's Q tile (dh = 128)
constexpr int AT_KV_STAGE = 4 * AT_KBOX;        // K (2 boxes) + V (2 boxes)
constexpr int AT_P_HEAD = 128 * 128;            // [128 rows x 64 keys] bf16
constexpr int AT_OFF_KV = 2 * AT_Q_HEAD;
constexpr int AT_OFF_P = AT_OFF_KV + AT_STAGES * AT_KV_STAGE;
constexpr int AT_OFF_BAR = AT_OFF_P + 2 * AT_P_HEAD;
constexpr int AT_SMEM = 1024 + AT_OFF_BAR + 256;
constexpr float AT_RESCALE_THRESH = 8.0f;       // log2 units

struct UnitInfo {
  int q_row0, q_len, q_local0, kv_off, kv_len, q_off, n_pre, n_blk, h0, nh, g;
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
  return ui;
}

__global__ void __launch_bounds__(AT_THREADS, 1)
    attn_prefix_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKV,
                       const AttnDesc d, int n_units) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = smem + AT_OFF_KV;
  uint8_t* sP = smem + AT_OFF_P;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + AT_OFF_BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* kv_full = bars + 2;            // [3]
  uint64_t* kv_empty = bars + 5;           // [3]
  uint64_t* s_full = bars + 8;             // [2]
  uint64_t* p_ready = bars + 10;           // [2]
  uint64_t* o_done = bars + 12;            // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int r = d.H / d.Hkv;
  const int n_pairs = (r + 1) / 2;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmKV);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < AT_STAGES; ++s) { mbar_init(&kv_full[s], 1); mbar_init(&kv_empty[s], 1); }
    for (int j = 0; j < 2; ++j) { mbar_init(&s_full[j], 1); mbar_init(&p_ready[j], 4); mbar_init(&o_done[j], 1); }
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 8) {
    if (lane == 0) {
      // ------------------------------------------------------------------ TMA producer
      uint32_t kv_it = 0, q_it = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const UnitInfo ui = decode_unit(d, u, r, n_pairs);
        mbar_wait(q_empty, (q_it & 1) ^ 1);
        mbar_arrive_expect_tx(q_full, ui.nh * AT_Q_HEAD);
        for (int j = 0; j < ui.nh; ++j) {
          const int qc = (ui.h0 + j) * d.dh;
          tma_load_2d(sQ + j * AT_Q_HEAD, &tmQ, q_full, qc, ui.q_row0, kEvictFirst);
          tma_load_2d(sQ + j * AT_Q_HEAD + AT_QBOX, &tmQ, q_full, qc + 64, ui.q_row0, kEvictFirst);
        }
        ++q_it;
        const int kc = (d.H + ui.g) * d.dh;
        const int vc = (d.H + d.Hkv + ui.g) * d.dh;
        for (int b = 0; b < ui.n_blk; ++b, ++kv_it) {
          const int st = kv_it % AT_STAGES;
          mbar_wait(&kv_empty[st], ((kv_it / AT_STAGES) & 1) ^ 1);
          const int krow = b < ui.n_pre ? ui.kv_off + b * AT_KB : ui.q_off + (b - ui.n_pre) * AT_KB;
          uint8_t* dst = sKV + st * AT_KV_STAGE;
          mbar_arrive_expect_tx(&kv_full[st], AT_KV_STAGE);
          tma_load_2d(dst, &tmKV, &kv_full[st], kc, krow, kEvictLast);
          tma_load_2d(dst + AT_KBOX, &tmKV, &kv_full[st], kc + 64, krow, kEvictLast);
          tma_load_2d(dst + 2 * AT_KBOX, &tmKV, &kv_full[st], vc, krow, kEvictLast);
          tma_load_2d(dst + 3 * AT_KBOX, &tmKV, &kv_full[st], vc + 64, krow, kEvictLast);
        }
      }
    }
  } else if (warp == 9) {
    if (lane == 0) {
      // ------------------------------------------------------------------ MMA issuer
      constexpr uint32_t idesc_s = make_idesc_bf16(128, AT_KB, false, false);
      constexpr uint32_t idesc_o = make_idesc_bf16(128, 128, false, true);   // V is MN-major
      uint32_t kv_it = 0, q_it = 0;
      uint32_t blk_it[2] = {0, 0};
      const uint32_t q_addr = smem_u32(sQ);
      const uint32_t p_addr = smem_u32(sP);
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const UnitInfo ui = decode_unit(d, u, r, n_pairs);
        mbar_wait(q_full, q_it & 1);
        tc_fence_after();
        for (int b = 0; b < ui.n_blk; ++b, ++kv_it) {
          const int st = kv_it % AT_STAGES;
          mbar_wait(&kv_full[st], (kv_it / AT_STAGES) & 1);
          tc_fence_after();
          const uint32_t k_addr = smem_u32(sKV + st * AT_KV_STAGE);
          const uint32_t v_addr = k_addr + 2 * AT_KBOX;
          for (int j = 0; j < ui.nh; ++j) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              umma_bf16_ss(tmem_base + j * AT_KB,
                           kmajor_desc(q_addr + j * AT_Q_HEAD + (k >> 2) * AT_QBOX + (k & 3) * 32),
                           kmajor_desc(k_addr + (k >> 2) * AT_KBOX + (k & 3) * 32), idesc_s, k != 0);
            }
            umma_commit(&s_full[j]);
          }
          if (b == ui.n_blk - 1) umma_commit(q_empty);
          for (int j = 0; j < ui.nh; ++j) {
            mbar_wait(&p_ready[j], blk_it[j] & 1);
            ++blk_it[j];
            tc_fence_after();
#pragma unroll
            for (int k = 0; k < AT_KB / 16; ++k) {
              umma_bf16_ss(tmem_base + 128 + j * 128, kmajor_desc(p_addr + j * AT_P_HEAD + k * 32),
                           sw128_desc(v_addr + k * 2048, AT_KBOX, 1024), idesc_o, (b | k) != 0);
            }
            if (b == ui.n_blk - 1) umma_commit(&o_done[j]);
          }
          umma_commit(&kv_empty[st]);
        }
        ++q_it;
      }
    }
  } else if (warp < 8) {
    // -------------------------------------------------------------------- softmax WG j
    const int j = warp >> 2;
    const uint32_t row = (warp & 3) * 32 + lane;
    const uint32_t lane_base = ((warp & 3) * 32) << 16;
    const uint32_t tS = tmem_base + lane_base + j * AT_KB;
    const uint32_t tO = tmem_base + lane_base + 128 + j * 128;
    const uint32_t p_row = smem_u32(sP + j * AT_P_HEAD) + row * 128;
    const float sl2 = d.scale * 1.4426950408889634f;
    uint32_t blk_it = 0, u_it = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const UnitInfo ui = decode_unit(d, u, r, n_pairs);
      if (j >= ui.nh) continue;
      const int q_local = ui.q_local0 + (int)row;
      float m_used = -INFINITY, l_run = 0.f;
      for (int b = 0; b < ui.n_blk; ++b, ++blk_it) {
        const bool is_pre = b < ui.n_pre;
        const int lim = is_pre ? (ui.kv_len - b * AT_KB) : (q_local - (b - ui.n_pre) * AT_KB + 1);
        mbar_wait(&s_full[j], blk_it & 1);
        tc_fence_after();
        uint32_t s[2][32];
        tmem_ld_32x32b_x32(tS, s[0]);
        tmem_ld_32x32b_x32(tS + 32, s[1]);
        tmem_ld_wait();
        float mx = -INFINITY;
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float x = (c * 32 + i < lim) ? __uint_as_float(s[c][i]) * sl2 : -INFINITY;
            s[c][i] = __float_as_uint(x);
            mx = fmaxf(mx, x);
          }
        const bool need = mx > m_used + AT_RESCALE_THRESH;
        bool rescaled = false;
        if (__any_sync(0xffffffffu, need)) {
          const float m_new = fmaxf(m_used, mx);
          if (b > 0) {
            const float alpha = exp2f(m_used - m_new);
            l_run *= alpha;
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
              uint32_t o[32];
              tmem_ld_32x32b_x32(tO + c * 32, o);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
              tmem_st_32x32b_x32(tO + c * 32, o);
            }
            rescaled = true;
          }
          m_used = m_new;
        }
        float sum = 0.f;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t w[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float p0 = exp2f(__uint_as_float(s[c][2 * i]) - m_used);
            const float p1 = exp2f(__uint_as_float(s[c][2 * i + 1]) - m_used);
            sum += p0 + p1;
            w[i] = pack_bf16x2(p0, p1);
          }
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const uint32_t chunk = c * 4 + q4;
            st_shared_v4(p_row + ((chunk ^ (row & 7)) << 4), w[4 * q4], w[4 * q4 + 1], w[4 * q4 + 2],
                         w[4 * q4 + 3]);
          }
        }
        l_run += sum;
        if (rescaled) tmem_st_wait();
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_ready[j]);
      }
      // ---- unit epilogue: O / l -> bf16 -> global
      mbar_wait(&o_done[j], u_it & 1);
      ++u_it;
      tc_fence_after();
      const float inv = 1.f / l_run;
      const bool valid = q_local < ui.q_len;
      uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(d.out) +
                                            (size_t)(ui.q_row0 + row) * (d.H * d.dh) + (ui.h0 + j) * d.dh);
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t o[32];
        tmem_ld_32x32b_x32(tO + c * 32, o);
        tmem_ld_wait();
        if (valid) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 v;
            v.x = pack_bf16x2(__uint_as_float(o[8 * q + 0]) * inv, __uint_as_float(o[8 * q + 1]) * inv);
            v.y = pack_bf16x2(__uint_as_float(o[8 * q + 2]) * inv, __uint_as_float(o[8 * q + 3]) * inv);
            v.z = pack_bf16x2(__uint_as_float(o[8 * q + 4]) * inv, __uint_as_float(o[8 * q + 5]) * inv);
            v.w = pack_bf16x2(__uint_as_float(o[8 * q + 6]) * inv, __uint_as_float(o[8 * q + 7]) * inv);
            dst[c * 4 + q] = v;
          }
        }
      }
      tc_fence_before();
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

static int g_att_sms = 0;

int launch_attention(const AttnDesc& d, cudaStream_t stream) {
  if (d.dh != 128) return fail(-2, "attention: d_head must be 128 (got %d)", d.dh);
  if (d.H % d.Hkv != 0) return fail(-2, "attention: n_heads %% n_kv_heads != 0");
  if (d.n_work == 0) return 0;
  const int ldq = (d.H + 2 * d.Hkv) * d.dh;
  CUtensorMap tq, tkv;
  if (!make_tmap_2d(&tq, d.qkv, 2, (uint64_t)d.T, (uint64_t)ldq, (uint64_t)ldq, 128, 64, true)) return -3;
  if (!make_tmap_2d(&tkv, d.qkv, 2, (uint64_t)d.T, (uint64_t)ldq, (uint64_t)ldq, AT_KB, 64, true)) return -3;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(attn_prefix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, AT_SMEM);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_att_sms, cudaDevAttrMultiProcessorCount, dev);
    attr_set = true;
  }
  const int r = d.H / d.Hkv;
  const int n_units = d.n_work * d.Hkv * ((r + 1) / 2);
  const int grid = n_units < g_att_sms ? n_units : g_att_sms;
  attn_prefix_kernel<<<grid, AT_THREADS, AT_SMEM, stream>>>(tq, tkv, d, n_units);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(-4, "attention launch: %s", cudaGetErrorString(e));
  return 0;
}

}  // namespace pf
