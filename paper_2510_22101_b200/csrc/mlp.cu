// Fused post-attention half of a decoder block: ONE persistent tcgen05 launch per layer for
//   O   x1 = x0 + attn . W_o^T                (residual epilogue; writes the MLP RMSNorm partials)
//   GU  h  = silu(g) * u,  [g|u] = rmsnorm(x1) . W_gu^T   (SwiGLU epilogue)
//   DN  x2 = x1 + h . W_down^T                (residual epilogue; writes the attention RMSNorm partials)
// (SURVEY.md §8a K6/K7.)  The three GEMMs of gemm.cu, one launch instead of three:
// tiles of all three run on the same persistent CTA pairs, ordered by 256-row block with the GU tiles
// of a row block lagging its O tiles, and the DN tiles lagging its GU tiles, by a couple of schedule
// steps.  A row block's GU tiles start once its O tiles have stored x1, its DN tiles once its GU tiles
// have stored h (per-row-block completion counters, release/acquire at gpu scope).  Compared with three
// launches:
//   * x1 and h of a row block are consumed while they are still in L2 (the working set at any time is
//     a few row blocks, not the whole [T x 2 d_ff] intermediate), so h never makes a DRAM round trip;
//   * two kernel boundaries per layer disappear (each drains a grid and refills the pipeline), and the
//     tile tails of the three GEMMs merge into one.
// Everything else is the gemm.cu design: CTA pair (cta_group::2) on 256 x 256 tiles, 5-stage TMA ring,
// double-buffered TMEM accumulators, 4 epilogue warps; the residual is bf16 hi + 8-bit lo, updated in
// place through a per-warp TMA ring (gemm.cu EPI_RESID_ADD_NORM), the SwiGLU epilogue is gemm.cu's.
// Per-row arithmetic is identical to the three-launch path, so scores are bit-identical to it.
//
// Status: opt-in (PF_MLP_FUSED=1), not the default.  Measured on B200 at C4 (tools/mlp_probe.py,
// profiles/r02/mlp_fused.txt): 0.96-1.15 ms per layer against 0.89 ms for the three gemm.cu launches.
// Each tile kind alone runs 3-14% slower here than in its specialised kernel, and with all three
// weight matrices live (50 MB at C4) plus the lagged activations the weights no longer stay in L2
// (ncu: 1.33 GB DRAM reads per launch vs 0.78 GB for the three kernels).
#include <cuda_runtime.h>
#include "ptx.cuh"
#include "pf_internal.h"

namespace pf {

namespace {

constexpr int BM = 128, BN = 256, BK = 64;
constexpr int A_BYTES = BM * BK * 2;              // 16 KB
constexpr int B_ROWS = BN / 2;                    // per CTA of the pair
constexpr int B_BYTES = B_ROWS * BK * 2;          // 16 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int STAGES = 5;
constexpr int STG_BYTES = 32 * 128;               // 32 rows x 128 B staging box
constexpr int LO_BYTES = 32 * 64;                 // 32 rows x 64 B uint8 box
constexpr int SLOT = STG_BYTES + LO_BYTES;        // one residual ring slot (hi + lo of 64 columns)
constexpr int RBD = 2;                            // residual ring depth per warp
constexpr int WARP_EPI_BYTES = RBD * SLOT;        // 12 KB: ring slots, or two SwiGLU staging boxes
constexpr int EPI_BYTES = 4 * WARP_EPI_BYTES;
constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + EPI_BYTES + 512;
constexpr int THREADS = 192;
constexpr int EPI_ARRIVALS = 8;                   // 4 epilogue warps x 2 CTAs signal each tile

enum TileKind : int { T_O = 0, T_GU = 1, T_DN = 2 };

struct Tile {
  int kind, m, n;
};

PF_DEVICE float silu(float g) { return __fdividef(g, 1.0f + __expf(-g)); }

PF_DEVICE void stage_row_128B(uint32_t stg, uint32_t row, const uint32_t (&w)[32]) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    uint32_t addr = stg + row * 128 + ((c ^ (row & 7)) << 4);
    st_shared_v4(addr, w[4 * c], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]);
  }
}

PF_DEVICE uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
PF_DEVICE void red_release_gpu_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
PF_DEVICE void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// Spin until *ctr >= target (acquire).  A dependency that never completes traps after ~10 s (a CUDA
// error in the caller) instead of hanging the GPU.
PF_DEVICE void wait_counter(const uint32_t* ctr, uint32_t target, unsigned long long* stat = nullptr) {
  if (ld_acquire_gpu(ctr) >= target) return;
  const uint64_t t0 = globaltimer_ns();
  while (ld_acquire_gpu(ctr) < target) {
    __nanosleep(128);
    if (globaltimer_ns() - t0 > 10000000000ull) __trap();
  }
  if (stat != nullptr) {
    atomicAdd(stat, (unsigned long long)(globaltimer_ns() - t0));
    atomicAdd(stat + 1, 1ull);
  }
}

}  // namespace

struct MlpArgs {
  int M;          // packed rows
  int d;          // d_model (N of O and DN, K of GU)
  int kq;         // attention width H*dh (K of O)
  int fp;         // d_ff_pad (K of DN; GU N = 2 fp)
  int nm;         // 256-row blocks
  int n_o, n_gu, n_dn;
  int lag_gu, lag_dn;            // schedule lags in steps
  int rows_per_step;             // row blocks per schedule step
  uint32_t* ctr_o;               // [nm] O tiles finished (x EPI_ARRIVALS)
  uint32_t* ctr_gu;              // [nm] GU tiles finished
  float* ss_mlp;                 // [d/256][ss_ld] MLP RMSNorm partials (written by O, read by GU)
  float* ss_attn;                // [d/256][ss_ld] next layer's attention RMSNorm partials (written by DN)
  int ss_ld;
  float inv_d, eps;
  int nodep;                     // debug (PF_MLP_NODEP=1): skip dependency waits/signals (wrong results)
  unsigned long long* stats;     // debug (pf_debug_set_mlp_stats): ns spent per wait site, CTA-summed
};

// Schedule: step s covers R = rows_per_step row blocks; it holds the O tiles of row blocks
// [sR, sR+R), the GU tiles of the row blocks of step s - lag_gu and the DN tiles of the row blocks of
// step s - lag_gu - lag_dn.  Inside a step a kind's tiles run row-block-fastest, so the R row blocks
// share each weight tile while it is in L2.  C(s) = tiles before step s; tile t -> (kind, m, n) by
// binary search on s.
PF_DEVICE int rows_before(const MlpArgs& a, int s) {
  const int r = s * a.rows_per_step;
  return r < 0 ? 0 : (r > a.nm ? a.nm : r);
}

PF_DEVICE int tiles_before(const MlpArgs& a, int s) {
  return a.n_o * rows_before(a, s) + a.n_gu * rows_before(a, s - a.lag_gu) +
         a.n_dn * rows_before(a, s - a.lag_gu - a.lag_dn);
}

PF_DEVICE Tile decode_tile(const MlpArgs& a, int t) {
  const int steps = (a.nm + a.rows_per_step - 1) / a.rows_per_step;
  int lo = 0, hi = steps + a.lag_gu + a.lag_dn;   // invariant: C(lo) <= t < C(hi)
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (tiles_before(a, mid) <= t) lo = mid; else hi = mid;
  }
  const int s = lo;
  int r = t - tiles_before(a, s);
  const int kinds_s[3] = {s, s - a.lag_gu, s - a.lag_gu - a.lag_dn};
  const int n_k[3] = {a.n_o, a.n_gu, a.n_dn};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int m0 = rows_before(a, kinds_s[k]);
    const int rows = rows_before(a, kinds_s[k] + 1) - m0;
    if (r < rows * n_k[k]) return {k, m0 + r % rows, r / rows};
    r -= rows * n_k[k];
  }
  return {T_DN, 0, 0};   // unreachable for t < num_tiles
}

// Tensor maps: A/B operands per kind, residual hi (bf16 32x64 boxes) and lo (u8 32x64, 64B swizzle),
// h store (bf16 32x64 boxes).
struct MlpMaps {
  CUtensorMap a_o, b_o, a_gu, b_gu, a_dn, b_dn, hi, lo, h;
};

__global__ void __launch_bounds__(THREADS, 1)
    mlp_fused_kernel(const __grid_constant__ MlpMaps maps, const MlpArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint8_t* sEpi = smem + STAGES * STAGE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sEpi + EPI_BYTES);
  uint64_t* full_bar = bars;
  uint64_t* empty_bar = bars + STAGES;
  uint64_t* tfull_bar = bars + 2 * STAGES;
  uint64_t* tempty_bar = bars + 2 * STAGES + 2;
  uint64_t* rbar = bars + 2 * STAGES + 4;                 // [4 warps][RBD]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4 + 4 * RBD);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int num_tiles = args.nm * (args.n_o + args.n_gu + args.n_dn);
  const uint32_t rank = cluster_ctarank();
  const int grp = (int)cluster_id_x();
  const int ngrp = (int)nclusters_x();
  const bool leader = rank == 0;
  const int kb_o = args.kq / BK, kb_gu = args.d / BK, kb_dn = args.fp / BK;
  auto num_kb = [&](int kind) { return kind == T_O ? kb_o : kind == T_GU ? kb_gu : kb_dn; };

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&maps.a_o);
    tma_prefetch_desc(&maps.b_o);
    tma_prefetch_desc(&maps.a_gu);
    tma_prefetch_desc(&maps.b_gu);
    tma_prefetch_desc(&maps.a_dn);
    tma_prefetch_desc(&maps.b_dn);
    tma_prefetch_desc(&maps.hi);
    tma_prefetch_desc(&maps.lo);
    tma_prefetch_desc(&maps.h);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 4 * 2);
    }
    for (int i = 0; i < 4 * RBD; ++i) mbar_init(&rbar[i], 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_launch_dependents();
  if (warp != 0) pdl_wait();

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer (each CTA)
    auto amap = [&](int kind) { return kind == T_O ? &maps.a_o : kind == T_GU ? &maps.a_gu : &maps.a_dn; };
    auto bmap = [&](int kind) { return kind == T_O ? &maps.b_o : kind == T_GU ? &maps.b_gu : &maps.b_dn; };
    // the first tile's first weight boxes go out before griddepcontrol.wait (weights do not depend on
    // the previous kernel)
    int pre = 0;
    Tile t0{};
    if (grp < num_tiles) {
      t0 = decode_tile(args, grp);
      pre = min(STAGES, num_kb(t0.kind));
      const int n0 = t0.n * BN + rank * B_ROWS;
      if (elect_one()) {
        for (int kb = 0; kb < pre; ++kb) {
          const uint32_t lbar = mapa_shared(smem_u32(&full_bar[kb]), 0);
          if (leader) mbar_arrive_expect_tx(&full_bar[kb], 2 * STAGE_BYTES);
          tma_load_2d_pair(sB + kb * B_BYTES, bmap(t0.kind), lbar, kb * BK, n0, kEvictLast);
        }
      }
      __syncwarp();
    }
    pdl_wait();
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = grp; tile < num_tiles; tile += ngrp) {
      const Tile tl = tile == grp ? t0 : decode_tile(args, tile);
      const int m0 = tl.m * 2 * BM + rank * BM;
      const int n0 = tl.n * BN + rank * B_ROWS;
      const int nkb = num_kb(tl.kind);
      // A of a GU tile is x1 (all O tiles of its row block), of a DN tile h (all GU tiles)
      if ((tl.kind == T_GU || tl.kind == T_DN) && !args.nodep) {
        if (lane == 0) {
          if (tl.kind == T_GU) wait_counter(args.ctr_o + tl.m, args.n_o * EPI_ARRIVALS, args.stats ? args.stats + 0 : nullptr);
          else wait_counter(args.ctr_gu + tl.m, args.n_gu * EPI_ARRIVALS, args.stats ? args.stats + 2 : nullptr);
          fence_proxy_async_global();
        }
        __syncwarp();
      }
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        const uint32_t lbar = mapa_shared(smem_u32(&full_bar[stage]), 0);
        if (tile == grp && kb < pre) {   // B already requested, barrier armed: A only
          if (elect_one())
            tma_load_2d_pair(sA + stage * A_BYTES, amap(tl.kind), lbar, kb * BK, m0, kEvictNormal);
        } else if (elect_one()) {
          if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * STAGE_BYTES);
          tma_load_2d_pair(sA + stage * A_BYTES, amap(tl.kind), lbar, kb * BK, m0, kEvictNormal);
          tma_load_2d_pair(sB + stage * B_BYTES, bmap(tl.kind), lbar, kb * BK, n0, kEvictLast);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ---------------------------------------------------------------- MMA issuer (leader CTA)
      constexpr uint32_t idesc = make_idesc_bf16(2 * BM, BN, false, false);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB);
      for (int tile = grp; tile < num_tiles; tile += ngrp) {
        const int nkb = num_kb(decode_tile(args, tile).kind);
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint64_t a_desc = kmajor_desc(a_base + stage * A_BYTES);
          const uint64_t b_desc = kmajor_desc(b_base + stage * B_BYTES);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              umma_bf16_ss_pair(d_tmem, a_desc + 2 * k, b_desc + 2 * k, idesc, (kb | k) != 0 ? 1u : 0u);
            umma_commit_pair(&empty_bar[stage], 0x3);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) umma_commit_pair(&tfull_bar[acc], 0x3);
        __syncwarp();
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue (warps 2..5)
    const uint32_t quad = warp & 3;
    const uint32_t row = quad * 32 + lane;
    uint8_t* my = sEpi + (warp - 2) * WARP_EPI_BYTES;
    uint64_t* my_rbar = rbar + (warp - 2) * RBD;
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t ring_issued = 0, ring_used = 0;
    int stg_idx = 0;
    // residual chunk c (64 columns: hi + lo) of tile tl's 32 rows of this warp -> ring slot
    auto ring_issue = [&](const Tile& tl, int c) {
      const int mm = tl.m * 2 * BM + rank * BM + quad * 32;
      const int nn = tl.n * BN + c * 64;
      const uint32_t b = ring_issued % RBD;
      if (lane == 0) {
        mbar_arrive_expect_tx(&my_rbar[b], SLOT);
        tma_load_2d(my + b * SLOT, &maps.hi, &my_rbar[b], nn, mm, kEvictFirst);
        tma_load_2d(my + b * SLOT + STG_BYTES, &maps.lo, &my_rbar[b], nn, mm, kEvictFirst);
      }
      ++ring_issued;
    };
    // 64-column chunks of a residual tile (the last n-tile is partial when d % 256 == 128)
    auto ring_chunks = [&](const Tile& tl) { return min(BN / 64, (args.d - tl.n * BN) / 64); };
    // the residual a DN tile reads is x1: written by its row block's O tiles in this launch
    auto ring_start = [&](const Tile& tl) {
      if (tl.kind == T_GU) return;
      if (tl.kind == T_DN && !args.nodep) {
        if (lane == 0) {
          wait_counter(args.ctr_o + tl.m, args.n_o * EPI_ARRIVALS, args.stats ? args.stats + 4 : nullptr);
          fence_proxy_async_global();
        }
        __syncwarp();
      }
      for (int c = 0; c < min(RBD, ring_chunks(tl)); ++c) ring_issue(tl, c);
    };
    if (grp < num_tiles) ring_start(decode_tile(args, grp));

    for (int tile = grp; tile < num_tiles; tile += ngrp) {
      const Tile tl = decode_tile(args, tile);
      const int m0 = tl.m * 2 * BM + rank * BM;
      const int n0 = tl.n * BN;
      const int r0 = m0 + quad * 32;
      const int grow = m0 + (int)row;
      const bool rvalid = grow < args.M;
      float rs = 1.f;
      if (tl.kind == T_GU) {
        // fused RMSNorm of x1: partial sums stored by this row block's O tiles (this launch)
        if (lane == 0 && !args.nodep)
          wait_counter(args.ctr_o + tl.m, args.n_o * EPI_ARRIVALS, args.stats ? args.stats + 6 : nullptr);
        __syncwarp();
        if (rvalid) {
          float ssum = 0.f;
          const int parts = (args.d + 255) / 256;
#pragma unroll 8
          for (int p = 0; p < parts; ++p) ssum += __ldcg(args.ss_mlp + (size_t)p * args.ss_ld + grow);
          rs = rsqrtf(ssum * args.inv_d + args.eps);
        }
      }
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t t_row = tmem_base + ((quad * 32) << 16) + acc * BN;

      if (tl.kind == T_GU) {
        // staging boxes overlap the residual ring slots: the previous tile's stores must have left
        if (lane == 0) tma_store_wait_read<0>();
        __syncwarp();
        uint32_t gA[32], uA[32], gB[32], uB[32], w[32];
        tmem_ld_32x32b_x32(t_row, gA);
        tmem_ld_32x32b_x32(t_row + 128, uA);
#pragma unroll 1
        for (int cq = 0; cq < 2; ++cq) {
          tmem_ld_wait();
          tmem_ld_32x32b_x32(t_row + cq * 64 + 32, gB);
          tmem_ld_32x32b_x32(t_row + 128 + cq * 64 + 32, uB);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float a0 = silu(__uint_as_float(gA[2 * i]) * rs) * (__uint_as_float(uA[2 * i]) * rs);
            const float a1 = silu(__uint_as_float(gA[2 * i + 1]) * rs) * (__uint_as_float(uA[2 * i + 1]) * rs);
            w[i] = pack_bf16x2(a0, a1);
          }
          tmem_ld_wait();
          if (cq == 0) {
            tmem_ld_32x32b_x32(t_row + 64, gA);
            tmem_ld_32x32b_x32(t_row + 128 + 64, uA);
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float a0 = silu(__uint_as_float(gB[2 * i]) * rs) * (__uint_as_float(uB[2 * i]) * rs);
            const float a1 = silu(__uint_as_float(gB[2 * i + 1]) * rs) * (__uint_as_float(uB[2 * i + 1]) * rs);
            w[16 + i] = pack_bf16x2(a0, a1);
          }
          if (cq == 1) {   // last TMEM read of this accumulator
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster_relaxed(mapa_shared(smem_u32(&tempty_bar[acc]), 0));
          }
          if (lane == 0) tma_store_wait_read<1>();
          __syncwarp();
          const uint32_t stg = smem_u32(my + stg_idx * STG_BYTES);
          stage_row_128B(stg, lane, w);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&maps.h, my + stg_idx * STG_BYTES, n0 / 2 + cq * 64, r0);
            tma_store_commit();
          }
          stg_idx ^= 1;
        }
      } else {
        // residual x = hi + lo (+ acc), updated in place (gemm.cu EPI_RESID_ADD_NORM)
        float ssq = 0.f;
        const int n_chunks = ring_chunks(tl);
#pragma unroll 1
        for (int c = 0; c < n_chunks; ++c) {
          const uint32_t k = ring_used;
          const uint32_t b = k % RBD;
          if (c >= 2) {
            if (lane == 0) tma_store_wait_read<1>();
            __syncwarp();
            if (c + RBD - 2 < n_chunks) ring_issue(tl, c + RBD - 2);
          }
          mbar_wait(&my_rbar[b], (k / RBD) & 1);
          ++ring_used;
          uint32_t v0[32], v1[32];
          tmem_ld_32x32b_x32(t_row + c * 64, v0);
          tmem_ld_32x32b_x32(t_row + c * 64 + 32, v1);
          const uint32_t hrow = smem_u32(my + b * SLOT) + lane * 128;
          const uint32_t lrow = smem_u32(my + b * SLOT + STG_BYTES) + lane * 64;
          tmem_ld_wait();
          if (c == n_chunks - 1) {   // last TMEM read of this accumulator
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster_relaxed(mapa_shared(smem_u32(&tempty_bar[acc]), 0));
          }
          uint32_t l[4];
          float qn[16];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t off = (j ^ (lane & 7)) << 4;
            const uint32_t loff = ((j >> 1) ^ ((lane >> 1) & 3)) << 4;
            uint32_t h[4];
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(h[0]), "=r"(h[1]), "=r"(h[2]), "=r"(h[3]) : "r"(hrow + off));
            if ((j & 1) == 0)
              asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(l[0]), "=r"(l[1]), "=r"(l[2]), "=r"(l[3]) : "r"(lrow + loff));
            uint32_t nh[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int col = 8 * j + 2 * e;
              const int kq = (j & 1) * 8 + 2 * e;
              const float a0 = (col < 32) ? __uint_as_float(v0[col]) : __uint_as_float(v1[col - 32]);
              const float a1 = (col + 1 < 32) ? __uint_as_float(v0[col + 1]) : __uint_as_float(v1[col + 1 - 32]);
              const float x0 = resid_decode(__uint_as_float(h[e] << 16), l[kq >> 2], kq & 3) + a0;
              const float x1 = resid_decode(__uint_as_float(h[e] & 0xffff0000u), l[kq >> 2], (kq + 1) & 3) + a1;
              ssq += x0 * x0 + x1 * x1;
              const __nv_bfloat162 h2 = __floats2bfloat162_rn(x0, x1);
              const uint32_t hw = *reinterpret_cast<const uint32_t*>(&h2);
              qn[kq] = resid_lo_encode(x0, __uint_as_float(hw << 16));
              qn[kq + 1] = resid_lo_encode(x1, __uint_as_float(hw & 0xffff0000u));
              nh[e] = hw;
            }
            st_shared_v4(hrow + off, nh[0], nh[1], nh[2], nh[3]);
            if (j & 1)
              st_shared_v4(lrow + loff, pack_lo4(qn[0], qn[1], qn[2], qn[3]), pack_lo4(qn[4], qn[5], qn[6], qn[7]),
                           pack_lo4(qn[8], qn[9], qn[10], qn[11]), pack_lo4(qn[12], qn[13], qn[14], qn[15]));
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&maps.hi, my + b * SLOT, n0 + c * 64, r0);
            tma_store_2d(&maps.lo, my + b * SLOT + STG_BYTES, n0 + c * 64, r0);
            tma_store_commit();
          }
        }
        float* ss_out = tl.kind == T_O ? args.ss_mlp : args.ss_attn;
        if (rvalid) ss_out[(size_t)tl.n * args.ss_ld + grow] = ssq;
      }
      // O and GU tiles feed later tiles of this launch: publish once this warp's stores have landed
      if (tl.kind != T_DN && !args.nodep) {
        __syncwarp();
        if (lane == 0) {
          const uint64_t ts = args.stats ? globaltimer_ns() : 0;
          tma_store_wait_all<0>();
          fence_proxy_async_global();
          __threadfence();
          red_release_gpu_add((tl.kind == T_O ? args.ctr_o : args.ctr_gu) + tl.m, 1u);
          if (args.stats) {
            atomicAdd(args.stats + 8, (unsigned long long)(globaltimer_ns() - ts));
            atomicAdd(args.stats + 9, 1ull);
          }
        }
        __syncwarp();
      }
      // the next tile's residual loads start now; they land while its MMAs run
      const int nt = tile + ngrp;
      if (nt < num_tiles) {
        const Tile tn = decode_tile(args, nt);
        if (tn.kind != T_GU) {
          if (lane == 0) tma_store_wait_read<0>();
          __syncwarp();
          ring_start(tn);
        }
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0) tma_store_wait_all<0>();
    __syncwarp();
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair<512>(tmem_base);
  }
}

static unsigned long long* g_mlp_stats = nullptr;

int debug_set_mlp_stats(unsigned long long* buf) {
  g_mlp_stats = buf;
  return 0;
}

static int mlp_lag(const char* name, int dflt) {
  const char* e = getenv(name);
  return (e && e[0] >= '0' && e[0] <= '9') ? atoi(e) : dflt;
}

int launch_mlp_fused(const MlpDesc& d, const CUtensorMap* b_o, const CUtensorMap* b_gu, const CUtensorMap* b_dn,
                     cudaStream_t stream) {
  if (d.M == 0) return 0;
  if (d.d % 128 != 0 || d.kq % 64 != 0 || d.fp % 128 != 0)
    return fail(-2, "mlp: d=%d must be a multiple of 128, attn width %d of 64, d_ff_pad %d of 128", d.d, d.kq, d.fp);
  if (gemm_cta_group() != 2) return fail(-2, "mlp: the fused layer tail needs CTA pairs (PF_GEMM_CTAS=2)");
  MlpMaps maps;
  if (!make_tmap_2d(&maps.a_o, d.attn, 2, d.M, d.kq, d.kq, BM, BK, true)) return -3;
  if (!make_tmap_2d(&maps.a_gu, d.xb, 2, d.M, d.d, d.d, BM, BK, true)) return -3;
  if (!make_tmap_2d(&maps.a_dn, d.hbuf, 2, d.M, d.fp, d.fp, BM, BK, true)) return -3;
  maps.b_o = *b_o;
  maps.b_gu = *b_gu;
  maps.b_dn = *b_dn;
  if (!make_tmap_2d(&maps.hi, d.xb, 2, d.M, d.d, d.d, 32, 64, true)) return -3;
  if (!make_tmap_2d_u8_sw64(&maps.lo, d.rlo, d.M, d.d, d.d, 32, 64)) return -3;
  if (!make_tmap_2d(&maps.h, d.hbuf, 2, d.M, d.fp, d.fp, 32, 64, true)) return -3;
  MlpArgs a{};
  a.M = d.M; a.d = d.d; a.kq = d.kq; a.fp = d.fp;
  a.nm = (d.M + 2 * BM - 1) / (2 * BM);
  a.n_o = (d.d + BN - 1) / BN;
  a.n_gu = 2 * d.fp / BN;
  a.n_dn = (d.d + BN - 1) / BN;
  {   // debug (PF_MLP_KINDS bitmask 1 O | 2 GU | 4 DN, with PF_MLP_NODEP=1): time a subset of the tiles
    const int kinds = mlp_lag("PF_MLP_KINDS", 7);
    if (!(kinds & 1)) a.n_o = 0;
    if (!(kinds & 2)) a.n_gu = 0;
    if (!(kinds & 4)) a.n_dn = 0;
  }
  a.lag_gu = mlp_lag("PF_MLP_LAG_GU", 2);
  a.lag_dn = mlp_lag("PF_MLP_LAG_DN", 2);
  a.rows_per_step = max(1, mlp_lag("PF_MLP_ROWS", 1));
  a.ctr_o = d.counters;
  a.ctr_gu = d.counters + a.nm;
  a.ss_mlp = d.ss_mlp; a.ss_attn = d.ss_attn; a.ss_ld = d.ss_ld;
  a.inv_d = d.inv_d; a.eps = d.eps;
  a.nodep = mlp_lag("PF_MLP_NODEP", 0);
  a.stats = g_mlp_stats;
  if (2 * d.fp % BN != 0) return fail(-2, "mlp: 2*d_ff_pad=%d must be a multiple of %d", 2 * d.fp, BN);
  const int dev = current_device();
  static bool attr_set[kMaxDevices] = {};
  if (!attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(mlp_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return fail(-4, "mlp smem attr (device %d): %s", dev, cudaGetErrorString(e));
    attr_set[dev] = true;
  }
  const int tiles = a.nm * (a.n_o + a.n_gu + a.n_dn);
  const int groups = device_sm_count(dev) / 2;
  const int grid = (tiles < groups ? tiles : groups) * 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, mlp_fused_kernel, maps, a);
  if (e != cudaSuccess) return fail(-4, "mlp launch: %s", cudaGetErrorString(e));
  e = cudaGetLastError();
  return e == cudaSuccess ? 0 : fail(-4, "mlp launch: %s", cudaGetErrorString(e));
}

size_t mlp_counter_words(int M) { return 2 * (size_t)((M + 2 * BM - 1) / (2 * BM)); }

}  // namespace pf
