// HBM-bound kernels of the packed prefill:
//   embed_kernel    x[t] = float(E[id[t]])                  (bf16 table -> fp32 residual stream)
//   rmsnorm_kernel  y = bf16(x * rsqrt(mean(x^2) + eps) * g) (fp32 residual -> bf16 GEMM operand)
//   head_kernel     last-token gather -> final RMSNorm -> 2-row yes/no head -> sigmoid
// One warp per row, 16-byte vector loads/stores, row kept in registers (single HBM read).
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "ptx.cuh"
#include "pf_internal.h"

namespace pf {

PF_DEVICE float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------- embedding gather
// x[t] = float(E[id[t]]) (fp32 residual stream); optionally also xb[t] = E[id[t]] (the bf16 A
// operand of layer 0's QKV GEMM) and ss = sum(x^2) (its fused RMSNorm statistic) in the
// partial-sum layout the GEMMs read: ss[0*T + t] = sum, ss[p*T + t] = 0 for p = 1..parts-1.
__global__ void __launch_bounds__(256) embed_kernel(const int32_t* __restrict__ ids,
                                                    const __nv_bfloat16* __restrict__ emb,
                                                    float* __restrict__ resid, uint4* __restrict__ hi,
                                                    uint4* __restrict__ lo, float* __restrict__ ss, int T, int d) {
  // lo: low byte of the residual (16 per uint4); embedding rows are bf16, so lo = 0 (byte 0x80)
  pdl_launch_dependents();
  pdl_wait();
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  const int id = __ldg(ids + t);
  const uint4* src = reinterpret_cast<const uint4*>(emb + (size_t)id * d);
  float4* dst = resid ? reinterpret_cast<float4*>(resid + (size_t)t * d) : nullptr;
  float acc = 0.f;
  for (int i = lane; i < d / 8; i += 32) {
    const uint4 u = __ldg(src + i);
    const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&u);
    const float2 a = __bfloat1622float2(p[0]), b = __bfloat1622float2(p[1]);
    const float2 c = __bfloat1622float2(p[2]), f = __bfloat1622float2(p[3]);
    if (dst) {
      dst[2 * i] = make_float4(a.x, a.y, b.x, b.y);
      dst[2 * i + 1] = make_float4(c.x, c.y, f.x, f.y);
    }
    if (hi) hi[(size_t)t * (d / 8) + i] = u;
    if (lo && (i & 1) == 0) lo[(size_t)t * (d / 16) + i / 2] = make_uint4(0x80808080u, 0x80808080u, 0x80808080u, 0x80808080u);
    acc += a.x * a.x + a.y * a.y + b.x * b.x + b.y * b.y + c.x * c.x + c.y * c.y + f.x * f.x + f.y * f.y;
  }
  if (ss) {
    acc = warp_sum(acc);
    const int parts = ss_parts(d);
    for (int p = lane; p < parts; p += 32) ss[(size_t)p * T + t] = p == 0 ? acc : 0.f;
  }
}

// ---------------------------------------------------------------- RMSNorm
// NV = float4 per lane (d = 128 * NV).  Row held in registers: one read of the fp32 row,
// one write of the bf16 row.
template <int NV>
__global__ void __launch_bounds__(256) rmsnorm_kernel(const float* __restrict__ x,
                                                      const float* __restrict__ g,
                                                      __nv_bfloat16* __restrict__ y, int T,
                                                      float eps) {
  constexpr int d = NV * 128;
  pdl_launch_dependents();
  pdl_wait();
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  const float4* src = reinterpret_cast<const float4*>(x + (size_t)t * d);
  float4 v[NV];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    v[i] = __ldcs(src + lane + 32 * i);
    ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
  }
  ss = warp_sum(ss);
  const float r = rsqrtf(ss / (float)d + eps);
  const float4* g4 = reinterpret_cast<const float4*>(g);
  uint2* dst = reinterpret_cast<uint2*>(y + (size_t)t * d);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const float4 gg = g4 ? __ldg(g4 + lane + 32 * i) : make_float4(1.f, 1.f, 1.f, 1.f);
    uint2 o;
    o.x = pack_bf16x2(v[i].x * r * gg.x, v[i].y * r * gg.y);
    o.y = pack_bf16x2(v[i].z * r * gg.z, v[i].w * r * gg.w);
    dst[lane + 32 * i] = o;
  }
}

// ---------------------------------------------------------------- last-token head
// One warp per item: never forms [N x V] logits — only the yes/no columns of W_head are read.
__global__ void __launch_bounds__(256) head_kernel(const float* __restrict__ resid,
                                                   const __nv_bfloat16* __restrict__ rhi,
                                                   const uint8_t* __restrict__ rlo,
                                                   const int32_t* __restrict__ last_idx,
                                                   int n_items, int d,
                                                   const float* __restrict__ g,
                                                   const float* __restrict__ w_yes,
                                                   const float* __restrict__ w_no, float eps,
                                                   float* __restrict__ logits2,
                                                   float* __restrict__ p_yes, int* bad) {
  pdl_launch_dependents();
  pdl_wait();
  const int i = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n_items) return;
  const size_t r = (size_t)(last_idx ? __ldg(last_idx + i) : i) * d;
  auto X = [&](int j) -> float {   // residual value: fp32, or hi (bf16) + lo (byte; resid_decode)
    if (resid) return resid[r + j];
    return resid_decode(__bfloat162float(rhi[r + j]), rlo[r + j], 0);
  };
  float ss = 0.f;
  for (int j = lane; j < d; j += 32) { const float v = X(j); ss += v * v; }
  ss = warp_sum(ss);
  const float rs = rsqrtf(ss / (float)d + eps);
  float ly = 0.f, ln = 0.f;
  for (int j = lane; j < d; j += 32) {
    const float hn = X(j) * rs * __ldg(g + j);
    ly += hn * __ldg(w_yes + j);
    ln += hn * __ldg(w_no + j);
  }
  ly = warp_sum(ly);
  ln = warp_sum(ln);
  if (lane == 0) {
    logits2[2 * i] = ly;
    logits2[2 * i + 1] = ln;
    p_yes[i] = 1.f / (1.f + expf(-(ly - ln)));
    if (!isfinite(ly) || !isfinite(ln)) atomicOr(bad, 1);
  }
}

// ---------------------------------------------------------------- last-row gather
// Compacts the rows the head needs (one per item) before the last layer's O-projection + MLP:
// attn_c[i] = attn[last_idx[i]] (bf16), hi_c/lo_c[i] = the residual row (bf16 hi, uint8 lo).
__global__ void __launch_bounds__(256) gather_rows_kernel(const int32_t* __restrict__ last_idx, int n,
                                                          const uint4* __restrict__ attn, int attn_v4,
                                                          const uint4* __restrict__ hi, const uint4* __restrict__ lo,
                                                          int resid_v4, uint4* __restrict__ attn_c,
                                                          uint4* __restrict__ hi_c, uint4* __restrict__ lo_c) {
  pdl_launch_dependents();
  pdl_wait();
  const int i = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const size_t r = (size_t)__ldg(last_idx + i);
  for (int j = lane; j < attn_v4; j += 32) attn_c[(size_t)i * attn_v4 + j] = __ldg(attn + r * attn_v4 + j);
  for (int j = lane; j < resid_v4; j += 32) hi_c[(size_t)i * resid_v4 + j] = __ldg(hi + r * resid_v4 + j);
  for (int j = lane; j < resid_v4 / 2; j += 32) lo_c[(size_t)i * resid_v4 / 2 + j] = __ldg(lo + r * resid_v4 / 2 + j);
}

// ---------------------------------------------------------------- last layer, last-token rows
// Only the n_items last-token rows of the last layer reach the head, so that layer needs K and V for
// every packed row but Q, attention, O and the MLP only for those rows.  gather_q_rows collects the
// Q GEMM's inputs for them: the residual hi row, its fused-RMSNorm partial sums ([parts][T] ->
// [parts][n]) and its position (RoPE).
__global__ void __launch_bounds__(256) gather_q_rows_kernel(const int32_t* __restrict__ last_idx, int n,
                                                            const uint4* __restrict__ hi, int resid_v4,
                                                            const float* __restrict__ ss, int parts, int T,
                                                            const int32_t* __restrict__ pos,
                                                            uint4* __restrict__ hi_c, float* __restrict__ ss_c,
                                                            int32_t* __restrict__ pos_c) {
  pdl_launch_dependents();
  pdl_wait();
  const int i = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const size_t r = (size_t)__ldg(last_idx + i);
  for (int j = lane; j < resid_v4; j += 32) hi_c[(size_t)i * resid_v4 + j] = __ldg(hi + r * resid_v4 + j);
  for (int p = lane; p < parts; p += 32) ss_c[(size_t)p * n + i] = __ldg(ss + (size_t)p * T + r);
  if (lane == 0) pos_c[i] = __ldg(pos + r);
}

int launch_gather_q_rows(const int32_t* last_idx, int n, const void* hi, int d, const float* ss, int T,
                         const int32_t* pos, void* hi_c, float* ss_c, int32_t* pos_c, cudaStream_t stream) {
  if (n == 0) return 0;
  gather_q_rows_kernel<<<(n + 7) / 8, 256, 0, stream>>>(last_idx, n, reinterpret_cast<const uint4*>(hi), d / 8, ss,
                                                        ss_parts(d), T, pos, reinterpret_cast<uint4*>(hi_c), ss_c,
                                                        pos_c);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : fail(-4, "gather_q launch: %s", cudaGetErrorString(e));
}

// Attention of one query row per item (its last token) against the item's keys: the shared prefix
// [kv_off, kv_off + kv_len) and its own tokens up to the row (SPEC.md:249-272 at the rows that reach
// the head).  One CTA per (item, kv head): the r = H / Hkv query heads of the GQA group share every
// K/V row loaded.  fp32 scores, exact expf, fp32 P and accumulation (the tile kernel's P is bf16).
// The row's segment is the last one with q_off <= row (segs are ordered by q_off, as the packer emits
// them): counted by the whole CTA, one load per thread per 256 segments (a binary search would be a
// chain of dependent global loads).  HBM-bound at long items: each CTA streams its item's K and V once,
// 8 keys in flight per thread in the P.V loop.
// A key count above l_max (max_seq, the smem bound) writes NaN: the head's non-finite flag reports it.
constexpr int LR_THREADS = 256;
constexpr int LR_WARPS = LR_THREADS / 32;
constexpr int LR_MAX_R = 8;
template <int DH>
__global__ void __launch_bounds__(LR_THREADS) attn_last_rows_kernel(const __nv_bfloat16* __restrict__ q_c,
                                                                   const __nv_bfloat16* __restrict__ qkv, int qkv_n,
                                                                   const int4* __restrict__ segs, int n_seg,
                                                                   const int32_t* __restrict__ last_idx, int H,
                                                                   int Hkv, float scale, int l_max,
                                                                   __nv_bfloat16* __restrict__ out) {
  extern __shared__ float lr_sm[];   // q [r][4][DH/4 + 4] (pre-scaled), p [r][l_max], PV partials [8][r][DH]
  __shared__ float red[LR_MAX_R][LR_WARPS];
  __shared__ float inv[LR_MAX_R];
  pdl_launch_dependents();
  pdl_wait();
  const int i = blockIdx.x, g = blockIdx.y, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int r = H / Hkv;
  const int row = __ldg(last_idx + i);
  int cnt = 0;
  for (int k0 = 0; k0 < n_seg; k0 += LR_THREADS) {
    const int k = k0 + tid;
    cnt += __syncthreads_count(k < n_seg && __ldg(&segs[k].z) <= row);
  }
  const int4 sg = segs[max(cnt - 1, 0)];
  const int kv_len = sg.y;
  const int L = kv_len + (row - sg.z + 1);
  __nv_bfloat16* orow = out + (size_t)i * H * DH + (size_t)g * r * DH;
  if (L < 1 || L > l_max) {
    for (int e = tid; e < r * DH; e += LR_THREADS) orow[e] = __float2bfloat16(__int_as_float(0x7fc00000));
    return;
  }
  float* qs = lr_sm;
  float* ps = lr_sm + r * (DH + 16);
  const __nv_bfloat16* qrow = q_c + (size_t)i * H * DH + (size_t)g * r * DH;
  for (int e = tid; e < r * DH; e += LR_THREADS) {   // [h][quarter][DH/4 + 4 pad]
    const int h = e / DH, c = e % DH;
    qs[h * (DH + 16) + (c / (DH / 4)) * (DH / 4 + 4) + c % (DH / 4)] = __bfloat162float(qrow[e]) * scale;
  }
  __syncthreads();
  const size_t kcol = (size_t)(H + g) * DH, vcol = (size_t)(H + Hkv + g) * DH;
  auto key_row = [&](int j) { return (size_t)(j < kv_len ? sg.x + j : sg.z + (j - kv_len)); };
  // scores: four lanes per key, eight keys per warp step; lane (k, sub) reads DH/4 columns of key k's
  // K row (64 contiguous bytes: a warp load touches 8 rows, not 32) against the same q columns, kept
  // in smem with a 4-float pad per quarter so the four quarters hit different banks
  constexpr int VPL = DH / 32;
  constexpr int QD = DH / 4;
  auto load_row = [&](const __nv_bfloat16* p, float (&v)[VPL]) {
    if constexpr (VPL == 4) {
      const uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
      const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
      const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
      v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    } else {
      const float2 a = __bfloat1622float2(__ldg(reinterpret_cast<const __nv_bfloat162*>(p)));
      v[0] = a.x; v[1] = a.y;
    }
  };
  {
    const int sub = lane & 3;
    const float* qsub = qs + sub * (QD + 4);
#pragma unroll 2
    for (int j0 = wid * 8; j0 < L; j0 += LR_WARPS * 8) {
      const int j = j0 + (lane >> 2);
      float acc[LR_MAX_R];
#pragma unroll
      for (int h = 0; h < LR_MAX_R; ++h) acc[h] = 0.f;
      if (j < L) {
        const uint4* kp = reinterpret_cast<const uint4*>(qkv + key_row(j) * qkv_n + kcol + sub * QD);
        uint4 ku[QD / 8];
#pragma unroll
        for (int c = 0; c < QD / 8; ++c) ku[c] = __ldg(kp + c);
#pragma unroll
        for (int c = 0; c < QD / 8; ++c) {
          const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&ku[c]);
          float kf[8];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = __bfloat1622float2(b2[e]);
            kf[2 * e] = f.x;
            kf[2 * e + 1] = f.y;
          }
#pragma unroll
          for (int h = 0; h < LR_MAX_R; ++h) {
            if (h >= r) break;
            const float4 qa = *reinterpret_cast<const float4*>(qsub + h * 4 * (QD + 4) + 8 * c);
            const float4 qb = *reinterpret_cast<const float4*>(qsub + h * 4 * (QD + 4) + 8 * c + 4);
            acc[h] += qa.x * kf[0] + qa.y * kf[1] + qa.z * kf[2] + qa.w * kf[3] + qb.x * kf[4] + qb.y * kf[5] +
                      qb.z * kf[6] + qb.w * kf[7];
          }
        }
      }
#pragma unroll
      for (int h = 0; h < LR_MAX_R; ++h) {
        if (h >= r) break;
        acc[h] += __shfl_xor_sync(0xffffffffu, acc[h], 1);
        acc[h] += __shfl_xor_sync(0xffffffffu, acc[h], 2);
        if (sub == 0 && j < L) ps[h * l_max + j] = acc[h];
      }
    }
  }
  __syncthreads();
  // softmax per head (block reductions through red[][])
#pragma unroll
  for (int h = 0; h < LR_MAX_R; ++h) {
    if (h >= r) break;
    float m = -INFINITY;
    for (int j = tid; j < L; j += LR_THREADS) m = fmaxf(m, ps[h * l_max + j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) red[h][wid] = m;
    __syncthreads();
    m = red[h][0];
#pragma unroll
    for (int w = 1; w < LR_WARPS; ++w) m = fmaxf(m, red[h][w]);
    __syncthreads();
    float sum = 0.f;
    for (int j = tid; j < L; j += LR_THREADS) {
      const float p = expf(ps[h * l_max + j] - m);
      ps[h * l_max + j] = p;
      sum += p;
    }
    sum = warp_sum(sum);
    if (lane == 0) red[h][wid] = sum;
    __syncthreads();
    if (tid == 0) {
      float t = 0.f;
#pragma unroll
      for (int w = 0; w < LR_WARPS; ++w) t += red[h][w];
      inv[h] = 1.f / t;
    }
  }
  // O = P V / l: warp w takes keys w, w + 8, ...; lane l holds DH/32 consecutive columns (one 8- or
  // 4-byte load per key, a warp reads the whole V row); the eight warps' partial sums meet in smem
  float o[LR_MAX_R][VPL];
#pragma unroll
  for (int h = 0; h < LR_MAX_R; ++h)
#pragma unroll
    for (int e = 0; e < VPL; ++e) o[h][e] = 0.f;
#pragma unroll 8
  for (int j = wid; j < L; j += LR_WARPS) {
    float v[VPL];
    load_row(qkv + key_row(j) * qkv_n + vcol + lane * VPL, v);
#pragma unroll
    for (int h = 0; h < LR_MAX_R; ++h) {
      if (h >= r) break;
      const float p = ps[h * l_max + j];
#pragma unroll
      for (int e = 0; e < VPL; ++e) o[h][e] = fmaf(p, v[e], o[h][e]);
    }
  }
  float* part = ps + r * l_max;   // [LR_WARPS][r][DH]
#pragma unroll
  for (int h = 0; h < LR_MAX_R; ++h) {
    if (h >= r) break;
#pragma unroll
    for (int e = 0; e < VPL; ++e) part[(wid * r + h) * DH + lane * VPL + e] = o[h][e];
  }
  __syncthreads();
  for (int e = tid; e < r * DH; e += LR_THREADS) {
    const int h = e / DH;
    float sum = 0.f;
#pragma unroll
    for (int w = 0; w < LR_WARPS; ++w) sum += part[w * r * DH + e];
    orow[e] = __float2bfloat16(sum * inv[h]);
  }
}

int launch_attention_last_rows(const void* q_c, const void* qkv, int qkv_n, const int32_t* segs, int n_seg,
                               const int32_t* last_idx, int n_items, int H, int Hkv, int dh, int l_max,
                               void* out, cudaStream_t stream) {
  if (n_items == 0) return 0;
  if (dh != 128 && dh != 64) return fail(-2, "last-row attention: d_head must be 64 or 128 (got %d)", dh);
  if (H % Hkv != 0 || H / Hkv > LR_MAX_R)
    return fail(-2, "last-row attention: n_heads / n_kv_heads must divide and be <= %d", LR_MAX_R);
  if (n_seg < 1 || l_max < 1) return fail(-2, "last-row attention: empty segment table or l_max");
  const int r = H / Hkv;
  const size_t smem = (size_t)r * ((1 + LR_WARPS) * dh + 16 + l_max) * sizeof(float);
  if (smem > 200 * 1024) return fail(-2, "last-row attention: %zu B of shared memory (l_max %d)", smem, l_max);
  const int dev = current_device();
  static size_t attr_bytes[kMaxDevices][2] = {};
  const int ti = dh == 128 ? 0 : 1;
  if (smem > 48 * 1024 && attr_bytes[dev][ti] < smem) {
    cudaError_t e = dh == 128 ? cudaFuncSetAttribute(attn_last_rows_kernel<128>,
                                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                              : cudaFuncSetAttribute(attn_last_rows_kernel<64>,
                                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return fail(-4, "last-row attention smem attr: %s", cudaGetErrorString(e));
    attr_bytes[dev][ti] = smem;
  }
  const dim3 grid(n_items, Hkv);
  const float scale = 1.0f / sqrtf((float)dh);
  const auto* qc = reinterpret_cast<const __nv_bfloat16*>(q_c);
  const auto* kv = reinterpret_cast<const __nv_bfloat16*>(qkv);
  const auto* sg = reinterpret_cast<const int4*>(segs);
  auto* o = reinterpret_cast<__nv_bfloat16*>(out);
  if (dh == 128)
    attn_last_rows_kernel<128><<<grid, LR_THREADS, smem, stream>>>(qc, kv, qkv_n, sg, n_seg, last_idx, H, Hkv, scale,
                                                                   l_max, o);
  else
    attn_last_rows_kernel<64><<<grid, LR_THREADS, smem, stream>>>(qc, kv, qkv_n, sg, n_seg, last_idx, H, Hkv, scale,
                                                                  l_max, o);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : fail(-4, "last-row attention launch: %s", cudaGetErrorString(e));
}

int launch_gather_rows(const int32_t* last_idx, int n, const void* attn, int attn_cols, const void* hi,
                       const void* lo, int d, void* attn_c, void* hi_c, void* lo_c, cudaStream_t stream) {
  if (n == 0) return 0;
  gather_rows_kernel<<<(n + 7) / 8, 256, 0, stream>>>(
      last_idx, n, reinterpret_cast<const uint4*>(attn), attn_cols / 8, reinterpret_cast<const uint4*>(hi),
      reinterpret_cast<const uint4*>(lo), d / 8, reinterpret_cast<uint4*>(attn_c), reinterpret_cast<uint4*>(hi_c),
      reinterpret_cast<uint4*>(lo_c));
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : fail(-4, "gather launch: %s", cudaGetErrorString(e));
}

// Calibration capture ("capture flag records MLP inputs for the pruning module"):
// out[i, :] = rmsnorm(x[rows[i]]) * g, the MLP block's input, for the sampled packed rows.  x is the
// residual hi (bf16) + lo (uint8 byte) after the O-projection and ss its per-row partial sums of squares
// ([ss_parts(d)][ss_ld], summed in order; final once the preceding GEMM completes).  One warp per
// captured row, 8 columns per lane step.
__global__ void __launch_bounds__(256) capture_rows_kernel(const int32_t* __restrict__ rows, int n,
                                                           const uint4* __restrict__ hi,
                                                           const uint2* __restrict__ lo,
                                                           const float* __restrict__ ss, int ss_ld,
                                                           const float* __restrict__ g, int d_v8, float inv_d,
                                                           float eps, float* __restrict__ out) {
  pdl_launch_dependents();
  pdl_wait();
  const int i = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const size_t r = (size_t)__ldg(rows + i);
  float ssum = 0.f;
  for (int p = 0; p < ss_parts(d_v8 * 8); ++p) ssum += __ldg(ss + (size_t)p * ss_ld + r);
  const float rs = rsqrtf(ssum * inv_d + eps);
  float4* o = reinterpret_cast<float4*>(out + (size_t)i * d_v8 * 8);
  const float4* g4 = reinterpret_cast<const float4*>(g);
  for (int j = lane; j < d_v8; j += 32) {
    const uint4 h = __ldg(hi + r * d_v8 + j);
    const uint2 l = __ldg(lo + r * d_v8 + j);
    const uint32_t hw[4] = {h.x, h.y, h.z, h.w}, lw[2] = {l.x, l.y};
    float x[8];
#pragma unroll
    for (int e = 0; e < 8; ++e)
      x[e] = resid_decode(__uint_as_float((e & 1) ? hw[e / 2] & 0xffff0000u : hw[e / 2] << 16), lw[e / 4], e & 3);
    const float4 ga = __ldg(g4 + 2 * j), gb = __ldg(g4 + 2 * j + 1);
    o[2 * j] = make_float4(x[0] * rs * ga.x, x[1] * rs * ga.y, x[2] * rs * ga.z, x[3] * rs * ga.w);
    o[2 * j + 1] = make_float4(x[4] * rs * gb.x, x[5] * rs * gb.y, x[6] * rs * gb.z, x[7] * rs * gb.w);
  }
}

// RoPE cos/sin gathered per packed row (layout in pf_internal.h): warp = (32-row group, quad),
// lane = row, so every store is 512 contiguous bytes; rows past T use position 0.
__global__ void __launch_bounds__(256) rope_gather_kernel(const int32_t* __restrict__ pos,
                                                          const float4* __restrict__ cos_tab,
                                                          const float4* __restrict__ sin_tab, int qn, int T,
                                                          int n_groups, float4* __restrict__ out) {
  pdl_launch_dependents();
  pdl_wait();
  const int w = blockIdx.x * 8 + (threadIdx.x >> 5);   // (group, quad) pair
  const int lane = threadIdx.x & 31;
  if (w >= n_groups * qn) return;
  const int g = w / qn, q = w - (w / qn) * qn;
  const int row = g * 32 + lane;
  const size_t p = row < T ? (size_t)__ldg(pos + row) : 0;
  out[((size_t)(g * 2 + 0) * qn + q) * 32 + lane] = __ldg(cos_tab + p * qn + q);
  out[((size_t)(g * 2 + 1) * qn + q) * 32 + lane] = __ldg(sin_tab + p * qn + q);
}

int launch_rope_gather(const int32_t* pos, const float* cos_tab, const float* sin_tab, int half, int T,
                       float* out, cudaStream_t stream) {
  if (T == 0) return 0;
  if (half % 4 != 0) return fail(-2, "rope_gather: d_head/2 must be a multiple of 4");
  const int qn = half / 4, n_groups = (T + 31) / 32;
  rope_gather_kernel<<<(n_groups * qn + 7) / 8, 256, 0, stream>>>(
      pos, reinterpret_cast<const float4*>(cos_tab), reinterpret_cast<const float4*>(sin_tab), qn, T, n_groups,
      reinterpret_cast<float4*>(out));
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : fail(-4, "rope_gather launch: %s", cudaGetErrorString(e));
}

// ---------------------------------------------------------------- packed-batch bounds check
// Device-side twin of capi.cu validate_packed for batches that are already resident on the device
// (pf_validate_packed, and pf_score under PF_VALIDATE=1).  One thread per checked element over the
// concatenated index space [ids | pos | segs | work | last_idx]; the first violation found wins
// err[0] (code, PF_BAD_* in pf_internal.h) via atomicCAS and records its index in err[1].
__global__ void __launch_bounds__(256) validate_packed_kernel(
    const int32_t* __restrict__ ids, const int32_t* __restrict__ pos, const int4* __restrict__ segs, int n_seg,
    const int4* __restrict__ work, int n_work, const int32_t* __restrict__ last_idx, int n_items, int T,
    int vocab, int max_seq, int* __restrict__ err) {
  const long long total = 2LL * T + n_seg + n_work + n_items;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    int code = 0;
    long long idx = i;
    if (idx < T) {
      const int v = __ldg(ids + idx);
      if (v < 0 || v >= vocab) code = PF_BAD_ID;
    } else if ((idx -= T) < T) {
      const int v = __ldg(pos + idx);
      if (v < 0 || v >= max_seq) code = PF_BAD_POS;
    } else if ((idx -= T) < n_seg) {
      const int4 g = __ldg(segs + idx);
      if (g.x < 0 || g.y < 0 || g.z < 0 || g.w < 1 || (long long)g.x + g.y > T || (long long)g.z + g.w > T)
        code = PF_BAD_SEG;
      if (idx > 0) {   // q ranges increase and do not overlap (the packer's order)
        const int4 p = __ldg(segs + idx - 1);
        if ((long long)g.z < (long long)p.z + p.w) code = PF_BAD_SEG;
      }
    } else if ((idx -= n_seg) < n_work) {
      const int4 k = __ldg(work + idx);
      if (k.x < 0 || k.x >= n_seg || k.y < 0 || (long long)k.y * 128 >= __ldg(segs + k.x).w) code = PF_BAD_WORK;
    } else {
      idx -= n_work;
      const int v = __ldg(last_idx + idx);
      if (v < 0 || v >= T) code = PF_BAD_LAST;
    }
    if (code != 0 && atomicCAS(err, 0, code) == 0) err[1] = (int)idx;
  }
}

int launch_validate_packed(const int32_t* ids, const int32_t* pos, const int32_t* segs, int n_seg,
                           const int32_t* work, int n_work, const int32_t* last_idx, int n_items, int T, int vocab,
                           int max_seq, int* err, cudaStream_t stream) {
  if (((reinterpret_cast<uintptr_t>(segs) | reinterpret_cast<uintptr_t>(work)) & 15) != 0)
    return fail(-1, "validate: segs/work must be 16-byte aligned");
  cudaError_t e = cudaMemsetAsync(err, 0, 2 * sizeof(int), stream);
  if (e != cudaSuccess) return fail(-4, "validate memset: %s", cudaGetErrorString(e));
  const long long total = 2LL * T + n_seg + n_work + n_items;
  const long long blocks = (total + 255) / 256;
  validate_packed_kernel<<<(unsigned)(blocks < 1184 ? blocks : 1184), 256, 0, stream>>>(
      ids, pos, reinterpret_cast<const int4*>(segs), n_seg, reinterpret_cast<const int4*>(work), n_work, last_idx,
      n_items, T, vocab, max_seq, err);
  e = cudaGetLastError();
  return e == cudaSuccess ? 0 : fail(-4, "validate launch: %s", cudaGetErrorString(e));
}

int launch_capture_rows(const int32_t* rows, int n, const void* hi, const void* lo, const float* ss, int ss_ld,
                        const float* g, int d, float eps, float* out, cudaStream_t stream) {
  if (n == 0) return 0;
  if (d % 8 != 0) return fail(-2, "capture: d_model must be a multiple of 8");
  capture_rows_kernel<<<(n + 7) / 8, 256, 0, stream>>>(rows, n, reinterpret_cast<const uint4*>(hi),
                                                        reinterpret_cast<const uint2*>(lo), ss, ss_ld, g, d / 8,
                                                        1.0f / (float)d, eps, out);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : fail(-4, "capture launch: %s", cudaGetErrorString(e));
}

int launch_embed(const int32_t* ids, const void* emb, float* resid, void* hi, void* lo, float* ss, int T,
                 int d, cudaStream_t stream) {
  if (d % 16 != 0) return fail(-2, "embed: d_model must be a multiple of 16");
  if (T == 0) return 0;
  embed_kernel<<<(T + 7) / 8, 256, 0, stream>>>(ids, reinterpret_cast<const __nv_bfloat16*>(emb), resid,
                                                reinterpret_cast<uint4*>(hi), reinterpret_cast<uint4*>(lo), ss,
                                                T, d);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : fail(-4, "embed launch: %s", cudaGetErrorString(e));
}

int launch_rmsnorm(const float* x, const float* g, void* y, int T, int d, float eps,
                   cudaStream_t stream) {
  if (T == 0) return 0;
  const dim3 grid((T + 7) / 8);
  auto* yb = reinterpret_cast<__nv_bfloat16*>(y);
  if (d % 128 != 0 || d < 128 || d > 4096) return fail(-2, "rmsnorm: unsupported d_model %d", d);
  switch (d / 128) {
#define PF_RMS_CASE(n) case n: rmsnorm_kernel<n><<<grid, 256, 0, stream>>>(x, g, yb, T, eps); break;
    PF_RMS_CASE(1) PF_RMS_CASE(2) PF_RMS_CASE(3) PF_RMS_CASE(4) PF_RMS_CASE(5) PF_RMS_CASE(6)
    PF_RMS_CASE(7) PF_RMS_CASE(8) PF_RMS_CASE(9) PF_RMS_CASE(10) PF_RMS_CASE(11) PF_RMS_CASE(12)
    PF_RMS_CASE(13) PF_RMS_CASE(14) PF_RMS_CASE(15) PF_RMS_CASE(16) PF_RMS_CASE(18) PF_RMS_CASE(20)
    PF_RMS_CASE(24) PF_RMS_CASE(28) PF_RMS_CASE(32)
#undef PF_RMS_CASE
    default: return fail(-2, "rmsnorm: unsupported d_model %d", d);
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : fail(-4, "rmsnorm launch: %s", cudaGetErrorString(e));
}

int launch_head(const float* resid, const void* rhi, const void* rlo, const int32_t* last_idx, int n_items,
                int d, const float* g, const float* w_yes, const float* w_no, float eps, float* logits2,
                float* p_yes, int* bad, cudaStream_t stream) {
  if (n_items == 0) return 0;
  head_kernel<<<(n_items + 7) / 8, 256, 0, stream>>>(resid, reinterpret_cast<const __nv_bfloat16*>(rhi),
                                                     reinterpret_cast<const uint8_t*>(rlo), last_idx,
                                                     n_items, d, g, w_yes, w_no, eps, logits2, p_yes, bad);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : fail(-4, "head launch: %s", cudaGetErrorString(e));
}

}  // namespace pf
