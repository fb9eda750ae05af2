// Shared-prefix varlen attention.
//
// Packed layout: per request, prefix rows then item-suffix rows (no padding).  Each "segment"
// is a run of query rows whose keys are
//     dense  : rows [kv_off, kv_off + kv_len)        (the shared query prefix; may be empty)
//     causal : rows [q_off, q_off + 1 + local index) (the segment's own tokens)
// The prefix segment itself is {kv_len = 0, q = prefix rows}.  The prefix K/V are computed once
// per request by the QKV GEMM and read by every item's CTA; nothing is retained afterwards.
// Online softmax over the concatenated key blocks is algebraically the LSE merge of the
// prefix and suffix partials.
//
// One CTA = (128-row query tile of one segment, one query head).  Warp roles:
//   warps 0..3  softmax: thread i owns query row i (TMEM lane i) — tcgen05.ld S, mask, online
//               max/sum, P -> bf16 swizzled smem, O accumulated in registers from TMEM O_blk
//   warp 4      TMA producer: Q once, K/V 128-key blocks double-buffered
//   warp 5      tcgen05.mma issuer: S = Q.K^T (M128 N128 K128), O_blk = P.V (V MN-major)
#include <cuda_runtime.h>
#include "ptx.cuh"
#include "pf_internal.h"

namespace pf {

constexpr int ATT_THREADS = 192;
constexpr int ATT_TILE = 16384;                 // 128 rows x 64 bf16 (one SW128 box)
constexpr int ATT_OPER = 2 * ATT_TILE;          // 128 x 128 bf16 operand = 32 KB
constexpr int ATT_SMEM = 1024 + 6 * ATT_OPER + 256;   // Q, K[2], V[2], P

__global__ void __launch_bounds__(ATT_THREADS, 1)
    attn_prefix_kernel(const __grid_constant__ CUtensorMap tmQKV, const AttnDesc d) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = smem + ATT_OPER;           // 2 stages
  uint8_t* sV = smem + 3 * ATT_OPER;       // 2 stages
  uint8_t* sP = smem + 5 * ATT_OPER;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 6 * ATT_OPER);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;   // [2]
  uint64_t* kv_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;
  uint64_t* p_ready = bars + 6;
  uint64_t* o_full = bars + 7;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();

  const int4 wk = reinterpret_cast<const int4*>(d.work)[blockIdx.x];
  const int seg = wk.x, qt = wk.y;
  const int4 sg = reinterpret_cast<const int4*>(d.segs)[seg];
  const int kv_off = sg.x, kv_len = sg.y, q_off = sg.z, q_len = sg.w;
  const int h = blockIdx.y;
  const int g = h / (d.H / d.Hkv);
  const int q_row0 = q_off + qt * 128;
  const int n_pre = (kv_len + 127) / 128;
  const int n_blk = n_pre + qt + 1;
  const int q_col = h * d.dh;
  const int k_col = (d.H + g) * d.dh;
  const int v_col = (d.H + d.Hkv + g) * d.dh;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmQKV);
    mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) { mbar_init(&kv_full[s], 1); mbar_init(&kv_empty[s], 1); }
    mbar_init(s_full, 1);
    mbar_init(p_ready, 4);
    mbar_init(o_full, 1);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t tS = tmem_base;         // cols [0,128)
  const uint32_t tO = tmem_base + 128;   // cols [128,256)

  if (warp == 4) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, ATT_OPER);
      tma_load_2d(sQ, &tmQKV, q_full, q_col, q_row0, kEvictFirst);
      tma_load_2d(sQ + ATT_TILE, &tmQKV, q_full, q_col + 64, q_row0, kEvictFirst);
      for (int b = 0; b < n_blk; ++b) {
        const int s = b & 1;
        mbar_wait(&kv_empty[s], ((b >> 1) & 1) ^ 1);
        const int krow = (b < n_pre) ? (kv_off + b * 128) : (q_off + (b - n_pre) * 128);
        mbar_arrive_expect_tx(&kv_full[s], 2 * ATT_OPER);
        uint8_t* k_dst = sK + s * ATT_OPER;
        uint8_t* v_dst = sV + s * ATT_OPER;
        tma_load_2d(k_dst, &tmQKV, &kv_full[s], k_col, krow, kEvictLast);
        tma_load_2d(k_dst + ATT_TILE, &tmQKV, &kv_full[s], k_col + 64, krow, kEvictLast);
        tma_load_2d(v_dst, &tmQKV, &kv_full[s], v_col, krow, kEvictLast);
        tma_load_2d(v_dst + ATT_TILE, &tmQKV, &kv_full[s], v_col + 64, krow, kEvictLast);
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, false, false);
      constexpr uint32_t idesc_o = make_idesc_bf16(128, 128, false, true);   // V is MN-major
      mbar_wait(q_full, 0);
      const uint32_t q_addr = smem_u32(sQ);
      const uint32_t p_addr = smem_u32(sP);
      for (int b = 0; b < n_blk; ++b) {
        const int s = b & 1;
        mbar_wait(&kv_full[s], (b >> 1) & 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sK + s * ATT_OPER);
        const uint32_t v_addr = smem_u32(sV + s * ATT_OPER);
        // S = Q . K^T over dh = 128 (8 x K16 steps; 64-col boxes at +16 KB)
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t off = (k >> 2) * ATT_TILE + (k & 3) * 32;
          umma_bf16_ss(tS, kmajor_desc(q_addr + off), kmajor_desc(k_addr + off), idesc_s, k != 0);
        }
        umma_commit(s_full);
        mbar_wait(p_ready, b & 1);
        tc_fence_after();
        // O_blk = P . V over 128 keys: P K-major (keys contiguous), V MN-major (dh contiguous;
        // the two 64-wide dh boxes sit 16 KB apart = LBO, 8-key groups 1 KB apart = SBO).
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t poff = (k >> 2) * ATT_TILE + (k & 3) * 32;
          umma_bf16_ss(tO, kmajor_desc(p_addr + poff), sw128_desc(v_addr + k * 2048, ATT_TILE, 1024),
                       idesc_o, k != 0);
        }
        umma_commit(o_full);
        umma_commit(&kv_empty[s]);
      }
    }
  } else {
    // ---------------------------------------------------------------- softmax warps 0..3
    const uint32_t row = warp * 32 + lane;
    const int q_local = qt * 128 + (int)row;            // index within the segment
    const float sl2 = d.scale * 1.4426950408889634f;   // scale * log2(e)
    const uint32_t lane_base = (warp * 32) << 16;
    float o_acc[128];
#pragma unroll
    for (int j = 0; j < 128; ++j) o_acc[j] = 0.f;
    float m_run = -INFINITY, l_run = 0.f, alpha_prev = 1.f;
    const uint32_t p_base = smem_u32(sP);

    for (int b = 0; b < n_blk; ++b) {
      const bool is_pre = b < n_pre;
      // valid keys in this block: dense part -> j < kv_len - b*128 ; causal -> j <= q_local - kb0
      const int lim = is_pre ? (kv_len - b * 128) : (q_local - (b - n_pre) * 128 + 1);
      mbar_wait(s_full, b & 1);
      tc_fence_after();
      // pass 1: row max
      float mx = -INFINITY;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tS + lane_base + c * 32, v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float x = (c * 32 + j < lim) ? __uint_as_float(v[j]) * sl2 : -INFINITY;
          mx = fmaxf(mx, x);
        }
      }
      const float m_new = fmaxf(m_run, mx);
      const float alpha = exp2f(m_run - m_new);   // m_run = -inf on the first block -> 0
      // pass 2: P = exp2(s - m_new) -> bf16 smem (SW128, K-major over keys), row sum
      float sum = 0.f;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tS + lane_base + c * 32, v);
        tmem_ld_wait();
        uint32_t w[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int j0 = c * 32 + 2 * j;
          const float p0 = (j0 < lim) ? exp2f(__uint_as_float(v[2 * j]) * sl2 - m_new) : 0.f;
          const float p1 = (j0 + 1 < lim) ? exp2f(__uint_as_float(v[2 * j + 1]) * sl2 - m_new) : 0.f;
          sum += p0 + p1;
          w[j] = pack_bf16x2(p0, p1);
        }
        // 32 keys = 64 B = four 16 B chunks; box (c >> 1), chunk index within the 128 B row
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const uint32_t chunk = (c & 1) * 4 + q4;
          const uint32_t addr = p_base + (c >> 1) * ATT_TILE + row * 128 + ((chunk ^ (row & 7)) << 4);
          st_shared_v4(addr, w[4 * q4], w[4 * q4 + 1], w[4 * q4 + 2], w[4 * q4 + 3]);
        }
      }
      // fold in the previous block's P.V before the next PV MMA overwrites it
      if (b > 0) {
        mbar_wait(o_full, (b - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(tO + lane_base + c * 32, v);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) o_acc[c * 32 + j] = o_acc[c * 32 + j] * alpha_prev + __uint_as_float(v[j]);
        }
      }
      l_run = l_run * alpha + sum;
      m_run = m_new;
      alpha_prev = alpha;
      fence_proxy_async_smem();   // P visible to the tensor core (async proxy)
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_ready);
    }
    mbar_wait(o_full, (n_blk - 1) & 1);
    tc_fence_after();
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tO + lane_base + c * 32, v);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) o_acc[c * 32 + j] = o_acc[c * 32 + j] * alpha_prev + __uint_as_float(v[j]);
    }
    if (q_local < q_len) {
      const float inv = 1.f / l_run;
      uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(d.out) +
                                            (size_t)(q_row0 + row) * (d.H * d.dh) + h * d.dh);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        uint4 u;
        u.x = pack_bf16x2(o_acc[8 * j + 0] * inv, o_acc[8 * j + 1] * inv);
        u.y = pack_bf16x2(o_acc[8 * j + 2] * inv, o_acc[8 * j + 3] * inv);
        u.z = pack_bf16x2(o_acc[8 * j + 4] * inv, o_acc[8 * j + 5] * inv);
        u.w = pack_bf16x2(o_acc[8 * j + 6] * inv, o_acc[8 * j + 7] * inv);
        dst[j] = u;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc<256>(tmem_base);
  }
}

int launch_attention(const AttnDesc& d, cudaStream_t stream) {
  if (d.dh != 128) return fail(-2, "attention: d_head must be 128 (got %d)", d.dh);
  if (d.H % d.Hkv != 0) return fail(-2, "attention: n_heads %% n_kv_heads != 0");
  if (d.n_work == 0) return 0;
  const int ldq = (d.H + 2 * d.Hkv) * d.dh;
  CUtensorMap tm;
  if (!make_tmap_2d(&tm, d.qkv, 2, (uint64_t)d.T, (uint64_t)ldq, (uint64_t)ldq, 128, 64, true))
    return -3;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(attn_prefix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, ATT_SMEM);
    attr_set = true;
  }
  dim3 grid(d.n_work, d.H);
  attn_prefix_kernel<<<grid, ATT_THREADS, ATT_SMEM, stream>>>(tm, d);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(-4, "attention launch: %s", cudaGetErrorString(e));
  return 0;
}

}  // namespace pf
