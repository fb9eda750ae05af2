// tcgen05 bf16 GEMM for the packed prefill:  C[M x N] = A[M x K] . B[N x K]^T
//
// A = activations (T packed tokens x K, row-major), B = weights stored K-major ([out x in], i.e.
// the spec's x.W weights transposed at load).  Persistent, warp-specialised, 1 CTA per SM:
//   warp 0      TMA producer (A 128x64 + B 256x64 bf16 boxes, 128B swizzle, STAGES-deep ring)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=256, K=16 per op)
//   warps 2..5  epilogue: tcgen05.ld -> fused op -> swizzled smem -> TMA store / TMA reduce-add
// The accumulator is double-buffered in TMEM (2 x 256 fp32 columns) so the epilogue of tile i
// overlaps the main loop of tile i+1.
//
// Fused epilogues:
//   EPI_BF16       plain bf16 store
//   EPI_ROPE_BF16  QKV projection: rotate-half RoPE on the first `rope_heads` 128-wide heads
//   EPI_SWIGLU     gate/up projection with B rows interleaved per 128-neuron block
//                  ([gate_j | up_j] per 256-row tile); writes silu(gate)*up as bf16 (N/2 cols)
//   EPI_RESID_ADD  O / down projection: fp32 residual stream += acc via TMA reduce-add
#include <cstdlib>
#include <cuda_runtime.h>
#include "ptx.cuh"
#include "pf_internal.h"

namespace pf {

constexpr int GEMM_BM = 128;                          // rows per CTA (TMEM lanes)
constexpr int GEMM_BN = 256;                          // output columns per tile (both CG modes)
constexpr int GEMM_BK = 64;

constexpr int GEMM_A_BYTES = GEMM_BM * GEMM_BK * 2;   // 16 KB
constexpr int GEMM_STG_BYTES = 32 * 128;              // one 32-row x 128 B staging box

// CG = CTAs per MMA (cta_group).  CG=2: a CTA pair computes a 256 x 256 tile with
// tcgen05.mma.cta_group::2 (M=256); each CTA loads its own 128 A rows and half (128) of the
// B rows, so per-CTA operand bytes per MMA drop from 48 KB to 32 KB per k-block.
// EPI_RESID_ADD_NORM reads the old residual (bf16 hi + 8-bit lo, 3 B/elem) through a per-warp ring of
// RBD TMA-loaded 64-column chunks (hi box 4 KB + lo box 2 KB), updating it in place; it trades
// mainloop stages for that ring (PF_RING_STAGES / PF_RB_DEPTH override for A/B builds).  5 stages +
// depth 2 beat 4 + 3 by 2-8 us at the C4 shapes (tools/epi_sweep.py, profiles/r01/epi_sweep.txt):
// the epilogue math is free (hidden under the MMAs); its residual traffic is not, it competes with
// the mainloop's operand loads in L2 / HBM.  An 8-bit low word (6 B/elem read + write) instead of a
// bf16 one (8 B/elem) took C4 from 35.5 to ~34.6 ms/step at unchanged parity margins.
#ifndef PF_RB_DEPTH
#define PF_RB_DEPTH 2
#endif
#ifndef PF_RING_STAGES
#define PF_RING_STAGES 5
#endif
// Epilogue warps of the RoPE (QKV) GEMM: 4 (one per TMEM lane quadrant) or 8 (two per quadrant, each
// taking one 128-column half of the tile).
#ifndef PF_ROPE_EPI_WARPS
#define PF_ROPE_EPI_WARPS 4
#endif
// Mainloop stages of the plain / SwiGLU epilogues at CG = 2 (A/B builds: -DPF_PLAIN_STAGES=5)
#ifndef PF_PLAIN_STAGES
#define PF_PLAIN_STAGES 6
#endif
// Internal variant of EPI_RESID_ADD_NORM for short K (the C4 O projection, K = 1280): 4 mainloop stages
// and a 4-deep ring, so a tile's whole residual (4 chunks) is requested while its MMAs run.  At K >= 2048
// the fifth mainloop stage is worth more (tools/gemm_bench.py: C4 O 127.5 -> 123.4 us, C2 O 113 -> 116).
constexpr int EPI_RESID_ADD_NORM_DEEP = 100;
// (A/B knobs; at the C4 O shape 4 + 4 beats 5 + 2: 118 vs 122.5 us alone, tools/gemm_bench.py)
// A tile's residual chunks are requested once its accumulator is ready, not while its MMAs run: the
// residual TMA traffic then no longer competes with the mainloop's operand loads (round 2,
// tools/gemm_bench.py: C4 O + norm 118.0 -> 115.9 us, C2 O 108.6 -> 107.9, down unchanged; the
// epilogue warps had slack, ncu shows them waiting for the accumulator 22% of the time).
// PF_RING_LATE=0 restores the prefetch during the previous tile's epilogue.
#ifndef PF_RING_LATE
#define PF_RING_LATE 1
#endif
#ifndef PF_DEEP_STAGES
#define PF_DEEP_STAGES 4
#endif
#ifndef PF_DEEP_RBD
#define PF_DEEP_RBD 4
#endif
#ifndef PF_DEEP_RING_MAX_K
#define PF_DEEP_RING_MAX_K 1536
#endif
constexpr int RB_LO_BYTES = 32 * 64;                 // one 32-row x 64 B uint8 box (64B swizzle)
constexpr int RB_SLOT = GEMM_STG_BYTES + RB_LO_BYTES; // hi + lo boxes of one 64-column chunk (1 KB multiple)
template <int CG, int EPI>
struct GemmCfg {
  static constexpr int B_ROWS = GEMM_BN / CG;                // B rows loaded per CTA
  static constexpr int B_BYTES = B_ROWS * GEMM_BK * 2;
  static constexpr int STAGE_BYTES = GEMM_A_BYTES + B_BYTES;
  static constexpr bool DEEP = EPI == EPI_RESID_ADD_NORM_DEEP;
  static constexpr bool RING = EPI == EPI_RESID_ADD_NORM || DEEP;
  static constexpr int RBD = DEEP ? PF_DEEP_RBD : PF_RB_DEPTH;   // ring depth (chunks in flight per warp)
  static_assert(!RING || RBD >= 2, "the residual ring recycles slot k-2: depth >= 2");
  static constexpr bool ROPE = EPI == EPI_ROPE_BF16;
  // the RoPE epilogue stages a whole 256-column tile (4 boxes per warp) and gives up a stage for it
  static constexpr int STAGES = DEEP ? PF_DEEP_STAGES : RING ? PF_RING_STAGES : ROPE ? (CG == 2 ? 5 : 3) : (CG == 2 ? PF_PLAIN_STAGES : 4);
  // ring: RBD (hi, lo) chunk slots per epilogue warp; otherwise 2 (RoPE: 4) staging boxes per warp
  static constexpr int EPI_BYTES = RING ? 4 * RBD * RB_SLOT : 4 * (ROPE ? 4 : 2) * GEMM_STG_BYTES;
  static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + EPI_BYTES + 512;
  static constexpr int TILE_M = GEMM_BM * CG;
  static constexpr int EPI_WARPS = ROPE ? PF_ROPE_EPI_WARPS : 4;
  static constexpr int THREADS = 64 + 32 * EPI_WARPS;
};

struct GemmArgs {
  int M, N, K;
  int num_m_blk, num_n_blk;
  const int32_t* pos;      // EPI_ROPE: position per row
  const float* rope_cos;   // [max_seq x dh/2]
  const float* rope_sin;
  const float* rope_cs;    // gathered per-row cos/sin (launch_rope_gather layout) or null
  int rope_heads;          // heads (of rope_dh cols) that receive RoPE
  int rope_dh;             // head width: 64 or 128
  const float* row_ss;     // fused RMSNorm: per-row partial sums of squares [ss_parts_in][ss_ld] (or null)
  int ss_parts_in;         // = ceil(K / 256): partials written by the producing epilogue
  int ss_ld;               // row stride of row_ss / ss_out partial arrays
  float* ss_out;           // EPI_RESID_ADD_NORM: this n-tile's partial sum of squares per row
  const float* resid;      // EPI_RESID_ADD_NORM: residual base pointer (== C)
  int ldr;
  void* xb_out;            // EPI_RESID_ADD_NORM: bf16 copy of the new residual
  int ldxb;
  float inv_d, eps;
  int m_rev;               // walk the M blocks last-to-first (see GemmDesc::m_rev)
};

// M block of tile t: tiles run n-fastest; m_rev reverses the M order so that a consumer GEMM starts
// on the rows its producer wrote last (still in L2)
PF_DEVICE int m_block(const GemmArgs& a, int t) {
  const int mb = t / a.num_n_blk;
  return a.m_rev ? a.num_m_blk - 1 - mb : mb;
}

PF_DEVICE float4 ldg_cg_f4(const float* p) {
  float4 v;
  asm volatile("ld.global.cg.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

// silu(g) = g * sigmoid(g) with MUFU ex2/rcp (fast-math; the result is rounded to bf16 anyway)
PF_DEVICE float silu(float g) { return __fdividef(g, 1.0f + __expf(-g)); }

// Write 32 packed words (one 128-byte row) into a 32x128B swizzled staging box.
PF_DEVICE void stage_row_128B(uint32_t stg, uint32_t row, const uint32_t (&w)[32]) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    uint32_t addr = stg + row * 128 + ((c ^ (row & 7)) << 4);
    st_shared_v4(addr, w[4 * c], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]);
  }
}

template <int EPI, int CG>
__global__ void __launch_bounds__(GemmCfg<CG, EPI>::THREADS, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmD,
                     const GemmArgs args) {
  using Cfg = GemmCfg<CG, EPI>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + Cfg::STAGES * GEMM_A_BYTES;
  uint8_t* sStg = smem + Cfg::STAGES * Cfg::STAGE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sStg + Cfg::EPI_BYTES);
  uint64_t* full_bar = bars;
  uint64_t* empty_bar = bars + Cfg::STAGES;
  uint64_t* tfull_bar = bars + 2 * Cfg::STAGES;
  uint64_t* tempty_bar = bars + 2 * Cfg::STAGES + 2;
  uint64_t* rbar = bars + 2 * Cfg::STAGES + 4;            // [4 warps][RBD] (ring epilogue)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * Cfg::STAGES + 4 + 4 * Cfg::RBD);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int num_tiles = args.num_m_blk * args.num_n_blk;   // num_m_blk counts TILE_M rows
  const int num_kb = (args.K + GEMM_BK - 1) / GEMM_BK;
  // persistent schedule over CTA groups (a pair shares one tile)
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
  const int grp = CG == 2 ? (int)cluster_id_x() : (int)blockIdx.x;
  const int ngrp = CG == 2 ? (int)nclusters_x() : (int)gridDim.x;
  const bool leader = rank == 0;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmC);
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], Cfg::EPI_WARPS * CG);   // every epilogue warp of the group arrives
    }
    if constexpr (Cfg::RING)
      for (int i = 0; i < 4 * Cfg::RBD; ++i) mbar_init(&rbar[i], 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    if constexpr (CG == 2) tmem_alloc_pair<512>(tmem_slot);
    else tmem_alloc<512>(tmem_slot);
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_launch_dependents();
  // activations / residual / row statistics come from the previous kernel (the producer waits below,
  // after requesting the weights, which do not)
  if (warp != 0) pdl_wait();

  if (warp == 0) {
    // -------------------------------------------------------------- TMA producer (each CTA)
    // The first tile's first B (weight) boxes are requested before griddepcontrol.wait, so they
    // arrive while the previous kernel drains; their stages are armed for the full A + B bytes.
    const int pre = grp < num_tiles ? min(Cfg::STAGES, num_kb) : 0;
    if (pre > 0) {
      const int n0 = (grp % args.num_n_blk) * GEMM_BN + rank * Cfg::B_ROWS;
      if (elect_one()) {
        for (int kb = 0; kb < pre; ++kb) {
          if constexpr (CG == 2) {
            const uint32_t lbar = mapa_shared(smem_u32(&full_bar[kb]), 0);
            if (leader) mbar_arrive_expect_tx(&full_bar[kb], CG * Cfg::STAGE_BYTES);
            tma_load_2d_pair(sB + kb * Cfg::B_BYTES, &tmB, lbar, kb * GEMM_BK, n0, kEvictLast);
          } else {
            mbar_arrive_expect_tx(&full_bar[kb], Cfg::STAGE_BYTES);
            tma_load_2d(sB + kb * Cfg::B_BYTES, &tmB, &full_bar[kb], kb * GEMM_BK, n0, kEvictLast);
          }
        }
      }
      __syncwarp();
    }
    pdl_wait();
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = grp; tile < num_tiles; tile += ngrp) {
      const int m0 = m_block(args, tile) * Cfg::TILE_M + rank * GEMM_BM;
      const int n0 = (tile % args.num_n_blk) * GEMM_BN + rank * Cfg::B_ROWS;
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        if (tile == grp && kb < pre) {   // B already requested, barrier armed: A only
          if (elect_one()) {
            if constexpr (CG == 2)
              tma_load_2d_pair(sA + stage * GEMM_A_BYTES, &tmA, mapa_shared(smem_u32(&full_bar[stage]), 0),
                               kb * GEMM_BK, m0, kEvictNormal);
            else
              tma_load_2d(sA + stage * GEMM_A_BYTES, &tmA, &full_bar[stage], kb * GEMM_BK, m0);
          }
        } else if (elect_one()) {
          if constexpr (CG == 2) {
            // both CTAs' bytes complete on the leader's barrier; only the leader arms it
            const uint32_t lbar = mapa_shared(smem_u32(&full_bar[stage]), 0);
            if (leader) mbar_arrive_expect_tx(&full_bar[stage], CG * Cfg::STAGE_BYTES);
            tma_load_2d_pair(sA + stage * GEMM_A_BYTES, &tmA, lbar, kb * GEMM_BK, m0, kEvictNormal);
            tma_load_2d_pair(sB + stage * Cfg::B_BYTES, &tmB, lbar, kb * GEMM_BK, n0, kEvictLast);
          } else {
            mbar_arrive_expect_tx(&full_bar[stage], Cfg::STAGE_BYTES);
            tma_load_2d(sA + stage * GEMM_A_BYTES, &tmA, &full_bar[stage], kb * GEMM_BK, m0);
            tma_load_2d(sB + stage * Cfg::B_BYTES, &tmB, &full_bar[stage], kb * GEMM_BK, n0, kEvictLast);
          }
        }
        __syncwarp();
        if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ------------------------------------------------------------ MMA issuer (leader CTA)
      // The whole warp runs the loop (warp-uniform control flow and descriptors, so they live in
      // uniform registers); one elected lane issues the tcgen05 instructions.
      constexpr uint32_t idesc = make_idesc_bf16(Cfg::TILE_M, GEMM_BN, false, false);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB);
      for (int tile = grp; tile < num_tiles; tile += ngrp) {
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * GEMM_BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint64_t a_desc = kmajor_desc(a_base + stage * GEMM_A_BYTES);
          const uint64_t b_desc = kmajor_desc(b_base + stage * Cfg::B_BYTES);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < GEMM_BK / 16; ++k) {
              // +32 B along K inside the 128 B swizzle row = +2 in the descriptor's start field
              if constexpr (CG == 2)
                umma_bf16_ss_pair(d_tmem, a_desc + 2 * k, b_desc + 2 * k, idesc, (kb | k) != 0 ? 1u : 0u);
              else
                umma_bf16_ss(d_tmem, a_desc + 2 * k, b_desc + 2 * k, idesc, (kb | k) != 0 ? 1u : 0u);
            }
            if constexpr (CG == 2) umma_commit_pair(&empty_bar[stage], 0x3);
            else umma_commit(&empty_bar[stage]);
          }
          __syncwarp();
          if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) {
          if constexpr (CG == 2) umma_commit_pair(&tfull_bar[acc], 0x3);
          else umma_commit(&tfull_bar[acc]);
        }
        __syncwarp();
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // -------------------------------------------------------------- epilogue (warps 2..)
    const uint32_t quad = warp & 3;          // TMEM lane quadrant this warp may access
    const uint32_t row = quad * 32 + lane;   // row within the 128-row tile
    uint8_t* my_stg = sStg + (warp - 2) * (Cfg::EPI_BYTES / Cfg::EPI_WARPS);
    int stg_idx = 0;
    int acc = 0;
    uint32_t acc_phase = 0;

    // Stage one 32x128B box and launch its TMA store / reduce. Buffers alternate; the wait
    // keeps at most one store per warp in flight against the buffer being overwritten.
    auto emit_to = [&](const uint32_t (&w)[32], int c0, int r0, const CUtensorMap* map, bool reduce) {
      if (lane == 0) tma_store_wait_read<1>();
      __syncwarp();
      const uint32_t stg = smem_u32(my_stg + stg_idx * GEMM_STG_BYTES);
      stage_row_128B(stg, lane, w);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        if (reduce) tma_reduce_add_2d(map, my_stg + stg_idx * GEMM_STG_BYTES, c0, r0);
        else tma_store_2d(map, my_stg + stg_idx * GEMM_STG_BYTES, c0, r0);
        tma_store_commit();
      }
      stg_idx ^= 1;
    };
    auto emit = [&](const uint32_t (&w)[32], int c0, int r0) {
      emit_to(w, c0, r0, &tmC, EPI == EPI_RESID_ADD);
    };

    // ---- EPI_RESID_ADD_NORM residual ring: chunk k of this warp lives in buffer k % RBD
    uint64_t* my_rbar = rbar + (warp - 2) * Cfg::RBD;
    uint32_t ring_issued = 0, ring_used = 0;
    auto ring_issue = [&](int t, int c) {   // TMA-load chunk c (64 cols, hi + lo) of tile t's 32 rows
      const int mm = m_block(args, t) * Cfg::TILE_M + rank * GEMM_BM + quad * 32;
      const int nn = (t % args.num_n_blk) * GEMM_BN + c * 64;
      const uint32_t b = ring_issued % Cfg::RBD;
      if (lane == 0) {
        mbar_arrive_expect_tx(&my_rbar[b], RB_SLOT);
        tma_load_2d(my_stg + b * RB_SLOT, &tmD, &my_rbar[b], nn, mm, kEvictFirst);                    // hi
        tma_load_2d(my_stg + b * RB_SLOT + GEMM_STG_BYTES, &tmC, &my_rbar[b], nn, mm, kEvictFirst);   // lo (uint8)
      }
      ++ring_issued;
    };
    auto ring_chunks = [&](int t) { return min(GEMM_BN / 64, (args.N - (t % args.num_n_blk) * GEMM_BN) / 64); };
    // tile t's first RBD chunks go straight into the ring (once its accumulator is ready, PF_RING_LATE;
    // else while its MMAs run).  An extra L2 prefetch of the remaining chunks made no difference.
    auto ring_start = [&](int t) {
      for (int c = 0; c < min(Cfg::RBD, ring_chunks(t)); ++c) ring_issue(t, c);
    };
    if constexpr (Cfg::RING && !PF_RING_LATE) {
      if (grp < num_tiles) ring_start(grp);
    }
    for (int tile = grp; tile < num_tiles; tile += ngrp) {
      const int m0 = m_block(args, tile) * Cfg::TILE_M + rank * GEMM_BM;
      const int n0 = (tile % args.num_n_blk) * GEMM_BN;
      const int r0 = m0 + quad * 32;
      const int grow = m0 + (int)row;
      const bool rvalid = grow < args.M;
      // Global loads that do not depend on the accumulator are issued before waiting for it, so
      // their latency hides behind the mainloop: the fused-RMSNorm row statistics and (RoPE) the
      // first cos/sin block of this row.
      float rs = 1.f;
      if (args.row_ss != nullptr && rvalid) {
        // the A rows were bf16(residual): scale the accumulator row by rstd.  Partials summed in a
        // fixed order: bit-reproducible (no atomics anywhere on the path)
        float ssum = 0.f;
#pragma unroll 8
        for (int p = 0; p < args.ss_parts_in; ++p) ssum += __ldg(args.row_ss + (size_t)p * args.ss_ld + grow);
        rs = rsqrtf(ssum * args.inv_d + args.eps);
      }
      [[maybe_unused]] float4 cv[8], sv[8];
      [[maybe_unused]] const float4* cs4 = nullptr;
      [[maybe_unused]] const float4* sn4 = nullptr;
      [[maybe_unused]] int qstride = 1;
      if constexpr (EPI == EPI_ROPE_BF16) {
        // cos/sin of this row: gathered layout (coalesced: quad q of the warp's 32 rows is 512
        // contiguous bytes, stride 32 float4) or the tables' row p (32 lines per warp load)
        const int half = args.rope_dh / 2;
        const int qn = half / 4;
        if (args.rope_cs != nullptr) {
          cs4 = reinterpret_cast<const float4*>(args.rope_cs) + (size_t)(r0 / 32) * 2 * qn * 32 + lane;
          sn4 = cs4 + (size_t)qn * 32;
          qstride = 32;
        } else {
          const int p = rvalid ? __ldg(args.pos + grow) : 0;
          cs4 = reinterpret_cast<const float4*>(args.rope_cos + (size_t)p * half);
          sn4 = reinterpret_cast<const float4*>(args.rope_sin + (size_t)p * half);
        }
#ifdef PF_DEBUG_ROPE_NO_TABLE   // A/B timing only (wrong results): the RoPE epilogue without table reads
        const bool row_rot = false;
#else
        const bool row_rot = r0 < args.M;   // rows past M are padding (the gathered table ends there)
#endif
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          cv[j4] = row_rot ? __ldg(cs4 + j4 * qstride) : make_float4(1.f, 1.f, 1.f, 1.f);
          sv[j4] = row_rot ? __ldg(sn4 + j4 * qstride) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      if constexpr (Cfg::RING && PF_RING_LATE) {   // residual loads once the tile's MMAs are done
        mbar_wait(&tfull_bar[acc], acc_phase);
        if (lane == 0) tma_store_wait_read<0>();
        __syncwarp();
        ring_start(tile);
      }
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t t_row = tmem_base + ((quad * 32) << 16) + acc * GEMM_BN;
      // Hand the accumulator buffer back to the MMA issuer (its tcgen05.ld reads are complete).
      auto release_acc = [&]() {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          // the MMA issuer waits on the leader CTA's tmem-empty barrier
          if constexpr (CG == 2) mbar_arrive_cluster_relaxed(mapa_shared(smem_u32(&tempty_bar[acc]), 0));
          else mbar_arrive_relaxed(&tempty_bar[acc]);
        }
      };

      if constexpr (EPI == EPI_BF16) {
#pragma unroll 1
        for (int c = 0; c < GEMM_BN / 64; ++c) {
          uint32_t v0[32], v1[32], w[32];
          tmem_ld_32x32b_x32(t_row + c * 64, v0);
          tmem_ld_32x32b_x32(t_row + c * 64 + 32, v1);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            w[i] = pack_bf16x2(__uint_as_float(v0[2 * i]) * rs, __uint_as_float(v0[2 * i + 1]) * rs);
            w[16 + i] = pack_bf16x2(__uint_as_float(v1[2 * i]) * rs, __uint_as_float(v1[2 * i + 1]) * rs);
          }
          emit(w, n0 + c * 64, r0);
        }
      } else if constexpr (EPI == EPI_RESID_ADD) {
#pragma unroll 1
        for (int c = 0; c < GEMM_BN / 32; ++c) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(t_row + c * 32, v);
          tmem_ld_wait();
          emit(v, n0 + c * 32, r0);
        }
      } else if constexpr (Cfg::RING) {
        // Residual stream x = hi + lo: hi = bf16(x) (the next GEMM's A operand), lo = byte b with
        // x - hi = (b - 128) * 2^(E(hi) - 142) (resid_decode, ptx.cuh; ~16 significant bits together).
        // new = hi + lo + acc in fp32; hi/lo are rewritten in place in the ring slot and leave by TMA
        // store; ss_out[nb][row] = sum(new^2) (next RMSNorm).  Old chunks arrive through the TMA ring
        // (the first RBD issued while this tile's MMAs ran).  Bulk groups: one per chunk.
        const int n_chunks = ring_chunks(tile);
        float ssq = 0.f;
#pragma unroll 1
        for (int c = 0; c < n_chunks; ++c) {
          const uint32_t k = ring_used;
          const uint32_t b = k % Cfg::RBD;
          // G(k-2) has exactly one later group: once read, its slot takes chunk c + RBD - 2
          if (c >= 2) {
            if (lane == 0) tma_store_wait_read<1>();
            __syncwarp();
            if (c + Cfg::RBD - 2 < n_chunks) ring_issue(tile, c + Cfg::RBD - 2);
          }
          mbar_wait(&my_rbar[b], (k / Cfg::RBD) & 1);
          ++ring_used;
          uint32_t v0[32], v1[32];
          tmem_ld_32x32b_x32(t_row + c * 64, v0);
          tmem_ld_32x32b_x32(t_row + c * 64 + 32, v1);
          const uint32_t hrow = smem_u32(my_stg + b * RB_SLOT) + lane * 128;
          const uint32_t lrow = smem_u32(my_stg + b * RB_SLOT + GEMM_STG_BYTES) + lane * 64;
          tmem_ld_wait();
          uint32_t l[4];
          float qn[16];
#pragma unroll
          for (int j = 0; j < 8; ++j) {      // 16 B chunk j = columns [8j, 8j+8) of this 64-col chunk
            const uint32_t off = (j ^ (lane & 7)) << 4;
            // lo row: 64 B, 64B swizzle (16 B unit u of row r sits at u ^ ((r >> 1) & 3)); unit j/2
            // holds columns [16(j/2), 16(j/2)+16)
            const uint32_t loff = ((j >> 1) ^ ((lane >> 1) & 3)) << 4;
            uint32_t h[4];
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(h[0]), "=r"(h[1]), "=r"(h[2]), "=r"(h[3]) : "r"(hrow + off));
            if ((j & 1) == 0)
              asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(l[0]), "=r"(l[1]), "=r"(l[2]), "=r"(l[3]) : "r"(lrow + loff));
            uint32_t nh[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int col = 8 * j + 2 * e;      // within the 64-col chunk
              const int kq = (j & 1) * 8 + 2 * e; // byte within the 16-col lo unit
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
            tma_store_2d(&tmD, my_stg + b * RB_SLOT, n0 + c * 64, r0);
            tma_store_2d(&tmC, my_stg + b * RB_SLOT + GEMM_STG_BYTES, n0 + c * 64, r0);
            tma_store_commit();
          }
        }
        if (rvalid) args.ss_out[(size_t)(tile % args.num_n_blk) * args.ss_ld + grow] = ssq;
        // start the next tile's residual loads now; they land while its MMAs run
        const int nt = tile + ngrp;
        if (!PF_RING_LATE && nt < num_tiles) {
          if (lane == 0) tma_store_wait_read<0>();
          __syncwarp();
          ring_start(nt);
        }
      } else if constexpr (EPI == EPI_SWIGLU) {
        // B tile rows [0,128) = gate neurons, [128,256) = matching up neurons.  The four 32-column
        // halves are software-pipelined: the next half's tcgen05.ld is in flight during this half's
        // math (TMEM -> registers is asynchronous until tcgen05.wait::ld).
        uint32_t gA[32], uA[32], gB[32], uB[32], w[32];
        tmem_ld_32x32b_x32(t_row, gA);
        tmem_ld_32x32b_x32(t_row + 128, uA);
#pragma unroll 1
        for (int cq = 0; cq < 2; ++cq) {       // output chunk cq = cols [64cq, 64cq+64)
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
          emit(w, n0 / 2 + cq * 64, r0);
        }
      } else {  // EPI_ROPE_BF16
        // Rotate-half RoPE on heads of width dh (64 or 128): head column e pairs with e + dh/2.
        // Work item = (32-column block c of the head half, head hd): x1 = cols [32c, 32c+32) and
        // x2 = cols [dh/2 + 32c, ...) of head hd.  c is the outer loop, so each row's cos/sin block
        // is loaded once and serves every head of the tile (dh=128: 2 heads, dh=64: 4).  Items are
        // software-pipelined (item i+1's tcgen05.ld in flight during item i's math); the whole
        // 256-column tile is staged in 4 SW128 boxes per warp and leaves by TMA after the last item,
        // so the only staging wait is for the previous tile's stores (issued a mainloop earlier).
        // With 8 epilogue warps, warp (2 + 4 h + q) takes the heads of column half h of the tile.
        constexpr int NH = Cfg::EPI_WARPS / 4;        // column halves: 1 or 2
        const int dh = args.rope_dh;
        const int half = dh / 2;
        const int cpb = half / 32;                    // 32-col blocks per head half (1 or 2)
        const int hpt = GEMM_BN / dh;                 // heads per tile (2 or 4)
        const int hpw = hpt / NH;                     // heads per warp
        const int hd0 = ((int)warp - 2) / 4 * hpw;    // first head of this warp
        const int box0 = hd0 * dh / 64;               // first 64-column staging box of this warp
        const int n_items = cpb * hpw;
#ifdef PF_DEBUG_ROPE_NO_TABLE
        const bool row_rot = false;
#else
        const bool row_rot = r0 < args.M;   // rows past M are padding (the gathered table ends there)
#endif
        const uint32_t stg0 = smem_u32(my_stg);
        uint32_t x1[32], x2[32];
        tmem_ld_32x32b_x32(t_row + hd0 * dh, x1);
        tmem_ld_32x32b_x32(t_row + hd0 * dh + half, x2);
#pragma unroll 1
        for (int it = 0; it < n_items; ++it) {
          const int c = it / hpw, hd = hd0 + it % hpw;
          if (hd == hd0 && c > 0) {   // block 0 was loaded before the accumulator wait
#pragma unroll
            for (int j4 = 0; j4 < 8; ++j4) {
              cv[j4] = row_rot ? __ldg(cs4 + (c * 8 + j4) * qstride) : make_float4(1.f, 1.f, 1.f, 1.f);
              sv[j4] = row_rot ? __ldg(sn4 + (c * 8 + j4) * qstride) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
          }
          const bool rot = ((n0 + hd * dh) / dh) < args.rope_heads;   // q and k heads; v passes through
          tmem_ld_wait();
          if (it == n_items - 1) release_acc();   // last TMEM read done: the MMA may reuse the buffer
          uint32_t w1[16], w2[16];
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
            const float cc[4] = {cv[j4].x, cv[j4].y, cv[j4].z, cv[j4].w};
            const float ss[4] = {sv[j4].x, sv[j4].y, sv[j4].z, sv[j4].w};
            float o1[4], o2[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float a = __uint_as_float(x1[j4 * 4 + e]) * rs;
              const float b = __uint_as_float(x2[j4 * 4 + e]) * rs;
              o1[e] = rot ? a * cc[e] - b * ss[e] : a;
              o2[e] = rot ? b * cc[e] + a * ss[e] : b;
            }
            w1[j4 * 2] = pack_bf16x2(o1[0], o1[1]);
            w1[j4 * 2 + 1] = pack_bf16x2(o1[2], o1[3]);
            w2[j4 * 2] = pack_bf16x2(o2[0], o2[1]);
            w2[j4 * 2 + 1] = pack_bf16x2(o2[2], o2[3]);
          }
          if (it + 1 < n_items) {
            const int cn = (it + 1) / hpw, hn = hd0 + (it + 1) % hpw;
            tmem_ld_32x32b_x32(t_row + hn * dh + cn * 32, x1);
            tmem_ld_32x32b_x32(t_row + hn * dh + half + cn * 32, x2);
          }
          if (it == 0) {   // previous tile's boxes have been read by their TMA stores
            if (lane == 0) tma_store_wait_read<0>();
            __syncwarp();
          }
          const int e1 = hd * dh + c * 32, e2 = hd * dh + half + c * 32;   // tile column of each part
          const uint32_t b1 = stg0 + (e1 / 64 - box0) * GEMM_STG_BYTES + lane * 128;
          const uint32_t b2 = stg0 + (e2 / 64 - box0) * GEMM_STG_BYTES + lane * 128;
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const uint32_t k1 = (e1 % 64) / 8 + q4, k2 = (e2 % 64) / 8 + q4;
            st_shared_v4(b1 + ((k1 ^ (lane & 7)) << 4), w1[4 * q4], w1[4 * q4 + 1], w1[4 * q4 + 2], w1[4 * q4 + 3]);
            st_shared_v4(b2 + ((k2 ^ (lane & 7)) << 4), w2[4 * q4], w2[4 * q4 + 1], w2[4 * q4 + 2], w2[4 * q4 + 3]);
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          for (int x = 0; x < GEMM_BN / 64 / NH; ++x)
            if (n0 + 64 * (box0 + x) < args.N)
              tma_store_2d(&tmC, my_stg + x * GEMM_STG_BYTES, n0 + 64 * (box0 + x), r0);
          tma_store_commit();
        }
      }
      // All TMEM reads of this accumulator are complete (tcgen05.wait::ld above).
      if constexpr (EPI != EPI_ROPE_BF16) release_acc();
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0) tma_store_wait_all<0>();
    __syncwarp();
  }

  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (CG == 2) tmem_dealloc_pair<512>(tmem_base);
    else tmem_dealloc<512>(tmem_base);
  }
}


int gemm_smem_bytes() { return GemmCfg<2, EPI_BF16>::SMEM; }

static int g_gemm_cg = 0;

int gemm_cta_group() {
  if (g_gemm_cg == 0) {
    const char* e = getenv("PF_GEMM_CTAS");
    g_gemm_cg = (e && e[0] == '1') ? 1 : 2;
  }
  return g_gemm_cg;
}

template <int EPI, int CG>
static int launch_gemm_t(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc,
                         const CUtensorMap& td, const GemmArgs& a, cudaStream_t stream) {
  using Cfg = GemmCfg<CG, EPI>;
  const int dev = current_device();
  static bool attr_set[kMaxDevices] = {};
  if (!attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(gemm_bf16_kernel<EPI, CG>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return fail(-4, "gemm smem attr (device %d): %s", dev, cudaGetErrorString(e));
    attr_set[dev] = true;
  }
  const int tiles = a.num_m_blk * a.num_n_blk;
  const int groups = device_sm_count(dev) / CG;
  const int grid = (tiles < groups ? tiles : groups) * CG;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(Cfg::THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, gemm_bf16_kernel<EPI, CG>, ta, tb, tc, td, a);
  if (e != cudaSuccess) return fail(-4, "gemm launch: %s", cudaGetErrorString(e));
  e = cudaGetLastError();
  return e == cudaSuccess ? 0 : fail(-4, "gemm launch: %s", cudaGetErrorString(e));
}

template <int CG>
static int dispatch_gemm(const GemmDesc& d, const CUtensorMap& ta, const CUtensorMap& tb,
                         const CUtensorMap& tc, const CUtensorMap& td, GemmArgs a, cudaStream_t stream) {
  a.num_m_blk = (d.M + GemmCfg<CG, EPI_BF16>::TILE_M - 1) / GemmCfg<CG, EPI_BF16>::TILE_M;
  switch (d.epilogue) {
    case EPI_BF16: return launch_gemm_t<EPI_BF16, CG>(ta, tb, tc, td, a, stream);
    case EPI_ROPE_BF16: return launch_gemm_t<EPI_ROPE_BF16, CG>(ta, tb, tc, td, a, stream);
    case EPI_SWIGLU: return launch_gemm_t<EPI_SWIGLU, CG>(ta, tb, tc, td, a, stream);
    case EPI_RESID_ADD: return launch_gemm_t<EPI_RESID_ADD, CG>(ta, tb, tc, td, a, stream);
    case EPI_RESID_ADD_NORM:
      if (CG == 2 && d.K <= PF_DEEP_RING_MAX_K)
        return launch_gemm_t<EPI_RESID_ADD_NORM_DEEP, CG>(ta, tb, tc, td, a, stream);
      return launch_gemm_t<EPI_RESID_ADD_NORM, CG>(ta, tb, tc, td, a, stream);
    default: return fail(-2, "gemm: unknown epilogue %d", d.epilogue);
  }
}

bool make_weight_tmap(CUtensorMap* out, const void* B, int N, int K, int ldb) {
  return make_tmap_2d(out, B, 2, N, K, ldb, GEMM_BN / gemm_cta_group(), GEMM_BK, true);
}

int launch_gemm(const GemmDesc& d, const CUtensorMap* cached_b, cudaStream_t stream) {
  if (d.M == 0) return 0;
  if (d.K % 64 != 0) return fail(-2, "gemm: K=%d must be a multiple of 64", d.K);
  if (d.N % 128 != 0) return fail(-2, "gemm: N=%d must be a multiple of 128", d.N);
  if (d.epilogue == EPI_SWIGLU && d.N % GEMM_BN != 0)
    return fail(-2, "gemm: SwiGLU N=%d must be a multiple of %d", d.N, GEMM_BN);
  if (d.epilogue == EPI_ROPE_BF16 && (d.pos == nullptr || d.rope_cos == nullptr))
    return fail(-2, "gemm: RoPE epilogue needs positions and tables");
  const int cg = gemm_cta_group();
  CUtensorMap ta, tb, tc, td;
  if (!make_tmap_2d(&ta, d.A, 2, d.M, d.K, d.lda, GEMM_BM, GEMM_BK, true)) return -3;
  if (cached_b) tb = *cached_b;
  else if (!make_weight_tmap(&tb, d.B, d.N, d.K, d.ldb)) return -3;
  const int out_cols = d.epilogue == EPI_SWIGLU ? d.N / 2 : d.N;
  if (d.epilogue == EPI_RESID_ADD) {
    if (!make_tmap_2d(&tc, d.C, 4, d.M, out_cols, d.ldc, 32, 32, true)) return -3;
  } else if (d.epilogue == EPI_RESID_ADD_NORM) {   // 8-bit low word of the residual, 64B swizzle
    if (!make_tmap_2d_u8_sw64(&tc, d.C, d.M, out_cols, d.ldc, 32, 64)) return -3;
  } else {
    if (!make_tmap_2d(&tc, d.C, 2, d.M, out_cols, d.ldc, 32, 64, true)) return -3;
  }
  if (d.epilogue == EPI_RESID_ADD_NORM) {
    if (d.xb == nullptr || d.ss_out == nullptr) return fail(-2, "gemm: RESID_ADD_NORM needs xb and ss_out");
    if (!make_tmap_2d(&td, d.xb, 2, d.M, out_cols, d.ldxb, 32, 64, true)) return -3;
  } else {
    td = tc;
  }
  GemmArgs a;
  a.M = d.M; a.N = d.N; a.K = d.K;
  a.num_n_blk = (d.N + GEMM_BN - 1) / GEMM_BN;
  a.pos = d.pos; a.rope_cos = d.rope_cos; a.rope_sin = d.rope_sin; a.rope_heads = d.rope_heads;
  a.rope_cs = d.rope_cs;
  a.rope_dh = d.rope_dh == 64 ? 64 : 128;
  a.row_ss = d.row_ss; a.ss_out = d.ss_out;
  a.ss_parts_in = ss_parts(d.K);
  a.ss_ld = d.ss_ld > 0 ? (int)d.ss_ld : d.M;
  a.resid = reinterpret_cast<const float*>(d.C); a.ldr = d.ldc;
  a.xb_out = d.xb; a.ldxb = d.ldxb;
  a.inv_d = d.inv_d; a.eps = d.eps;
  a.m_rev = d.m_rev;
  return cg == 2 ? dispatch_gemm<2>(d, ta, tb, tc, td, a, stream)
                 : dispatch_gemm<1>(d, ta, tb, tc, td, a, stream);
}

}  // namespace pf
