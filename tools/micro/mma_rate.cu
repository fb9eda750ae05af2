// Microbenchmark: tcgen05.mma issue rate per SM for the attention shapes, SS (A and B from smem)
// vs TS (A from TMEM), M128 x N x K16 bf16, back-to-back accumulate into one TMEM tile.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2510_22101_b200/csrc mma_rate.cu -o mma_rate -lcuda
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace pf;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) mma_kernel(int reps, unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  // zero A (128 x 64 bf16 = 16 KB) and B (N x 64 bf16)
  for (int i = threadIdx.x; i < (16384 + N * 128) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0) {
    const uint32_t idesc = make_idesc_bf16(128, N, false, false);
    const uint64_t a = kmajor_desc(smem_u32(smem));
    const uint64_t b = kmajor_desc(smem_u32(smem + 16384));
    long long t0 = clock64();
    if (elect_one()) {
      for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          if (TS) umma_bf16_ts(tmem, tmem + 256 + kk * 8, b + ((kk * 32) >> 4), idesc, 1);
          else umma_bf16_ss(tmem, a + ((kk * 32) >> 4), b + ((kk * 32) >> 4), idesc, 1);
        }
      }
      umma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

// The attention block mix: per iteration S_0, S_1 (SS M128 N64, 8 K-steps each) and PV_0, PV_1
// (TS M128 N128, 4 K-steps each), every op into its own TMEM tile; optionally with background
// warps loading the SM (bg: 1 TMEM ld/st, 2 bulk smem writes, 4 FFMA streams, 12 MUFU streams).
__global__ void __launch_bounds__(384, 1) mix_kernel(int reps, unsigned long long* out, int mode, int bg,
                                                     const uint8_t* gsrc) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  __shared__ uint64_t bar2;
  __shared__ uint64_t cbar[5];
  __shared__ volatile int stop;
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&bar2, 1); for (int i = 0; i < 5; ++i) mbar_init(&cbar[i], 1); fence_barrier_init(); stop = 0; }
  const int iw = (bg & 16) ? 11 : 0;   // issuer warp
  if (warp == iw) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == iw) {
    const int jlo = 0, jhi = 2;
    const uint32_t idesc_s = make_idesc_bf16(128, 64, false, false);
    const uint32_t idesc_o = make_idesc_bf16(128, 128, false, true);
    const uint64_t q = kmajor_desc(smem_u32(smem));            // Q pair: 2 x 32 KB
    const uint64_t kd = kmajor_desc(smem_u32(smem + 65536 - 16384));
    long long t0 = clock64();
    if (elect_one()) {
      for (int r = 0; r < reps; ++r) {
        for (int j = jlo; j < jhi; ++j) {
          if (mode == 1 || mode == 4) continue;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16_ss(tmem + 64 * j, q + ((j * 32768 + (kk >> 2) * 16384 + (kk & 3) * 32) >> 4),
                         kd + (((kk >> 2) * 8192 + (kk & 3) * 32) >> 4), idesc_s, kk != 0);
          if (mode == 3) umma_commit(&cbar[j]);
        }
        for (int j = jlo; j < jhi; ++j) {
          if (mode == 2) continue;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_bf16_ts(tmem + 256 + 128 * j, tmem + 128 + 64 * j + kk * 8,
                         sw128_desc(smem_u32(smem + 65536 - 16384) + kk * 2048, 8192, 1024), idesc_o, 1);
          if (mode == 3) { umma_commit(&cbar[2 + j]); if (j == 1) umma_commit(&cbar[4]); }
        }
      }
      umma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if ((threadIdx.x & 31) == 0 && warp == iw) { out[blockIdx.x] = (unsigned long long)(t1 - t0); stop = 1; }
  } else if (warp >= 4 && (bg & 1)) {
    // softmax-like TMEM traffic on the S columns: load 64 columns, store 32 (P) per iteration
    const uint32_t t = tmem + (((warp & 3) * 32) << 16) + 64 * ((warp >> 2) & 1);
    uint32_t acc = 0;
    while (!stop) {
      uint32_t a[32], b2[32];
      tmem_ld_32x32b_x32(t, a); tmem_ld_32x32b_x32(t + 32, b2);
      tmem_ld_wait();
      for (int i = 0; i < 32; ++i) a[i] ^= b2[i];
      tmem_st_32x32b_x32(tmem + (((warp & 3) * 32) << 16) + 128 + 64 * ((warp >> 2) & 1), a);
      tmem_st_wait();
      acc += a[3];
    }
    if (acc == 12345) out[200] = acc;
  } else if (((bg & 16) ? (warp < 8) : (warp >= 4)) && (bg & 4)) {
    // softmax-like issue pressure: 8 warps of independent FFMA2 / MUFU streams
    float x[8];
    for (int i = 0; i < 8; ++i) x[i] = 0.001f * (threadIdx.x + i);
    while (!stop) {
#pragma unroll
      for (int r = 0; r < 16; ++r)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = (bg & 8) ? ex2_approx(x[i]) * 0.5f : fmaf(x[i], 1.0001f, 0.0001f);
    }
    float acc = 0; for (int i = 0; i < 8; ++i) acc += x[i];
    if (acc == 12345.f) out[200] = 1;
  } else if (warp == 1 && (bg & 2)) {
    // K/V-like smem writes: 32 KB bulk copies from global into the upper smem (not the MMA operands)
    uint32_t ph = 0;
    while (!stop) {
      if (elect_one()) {
        mbar_arrive_expect_tx(&bar2, 32768);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(smem_u32(smem + 65536)), "l"(gsrc + (blockIdx.x % 64) * 32768), "r"(32768), "r"(smem_u32(&bar2)) : "memory");
      }
      __syncwarp();
      mbar_wait(&bar2, ph);
      ph ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == iw) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

template <int N, bool TS>
void run(const char* name, unsigned long long* d_out, int grid) {
  const int reps = 4096;
  const int smem = 1024 + 16384 + N * 128;
  cudaFuncSetAttribute(mma_kernel<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_kernel<N, TS><<<grid, 128, smem>>>(reps, d_out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mma_kernel<N, TS><<<grid, 128, smem>>>(reps, d_out);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148];
  cudaMemcpy(h, d_out, sizeof(unsigned long long) * grid, cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < grid; ++i) avg += h[i]; avg /= grid;
  const double n_mma = 4.0 * reps;
  const double flops = 2.0 * 128 * N * 16 * n_mma * grid;
  printf("%-10s N=%3d grid=%3d: %6.1f cyc/MMA (floor %d)  %7.1f TFLOP/s  err=%s\n", name, N, grid, avg / n_mma,
         128 * N / 256, flops / (ms * 1e-3) / 1e12, cudaGetErrorString(e));
}

int main() {
  unsigned long long* d_out;
  cudaMalloc(&d_out, 148 * sizeof(unsigned long long));
  cudaFuncSetAttribute(mix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 32768 + 1024);
  uint8_t* gsrc; cudaMalloc(&gsrc, 64 * 32768); cudaMemset(gsrc, 0, 64 * 32768);
  for (int bg : {1, 2, 4, 12}) {
    mix_kernel<<<148, 384, 65536 + 32768 + 1024>>>(1024, d_out, 0, bg, gsrc);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h; cudaMemcpy(&h, d_out, 8, cudaMemcpyDeviceToHost);
    printf("attention MMA mix S+PV with background %s: %.0f cyc per block (alone 1259) %s\n",
           bg == 1 ? "8 warps of TMEM ld/st" : bg == 2 ? "32 KB bulk smem writes" : bg == 4 ? "8 FFMA warps" : "8 MUFU warps", h / 1024.0, cudaGetErrorString(e));
  }
  for (int mode = 0; mode < 4; ++mode) {
    mix_kernel<<<148, 384, 65536 + 32768 + 1024>>>(1024, d_out, mode, 0, gsrc);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h; cudaMemcpy(&h, d_out, 8, cudaMemcpyDeviceToHost);
    printf("attention MMA mix mode %d (0 S+PV, 1 PV only, 2 S only, 3 S+PV with per-group commits): %.0f cyc per block (ideal %d) %s\n", mode, h / 1024.0,
           mode == 0 || mode == 3 ? 1280 : mode == 1 ? 512 : 768, cudaGetErrorString(e));
  }
  for (int grid : {1, 148}) {
    run<64, false>("SS", d_out, grid);
    run<64, true>("TS", d_out, grid);
    run<128, false>("SS", d_out, grid);
    run<128, true>("TS", d_out, grid);
    run<256, false>("SS", d_out, grid);
    run<256, true>("TS", d_out, grid);
  }
  return 0;
}
