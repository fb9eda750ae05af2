// Microbenchmark: tcgen05.ld / tcgen05.st throughput per SM (32x32b.x32 by 4 or 8 warps).
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace pf;
PF_DEVICE void ld_16x256b_x8(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x8.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
PF_DEVICE void ld_16x128b_x16(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x128b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
template <int MODE>
__global__ void __launch_bounds__(256, 1) tmem_ld_kernel(int reps, unsigned long long* cyc, float* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = slot + (((warp & 3) * 32) << 16) + (warp >> 2) * 128;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < reps; ++it) {
    uint32_t a[32], b[32];
    if (MODE == 0) { tmem_ld_32x32b_x32(t, a); tmem_ld_32x32b_x32(t + 32, b); }
    if (MODE == 1) { ld_16x256b_x8(t, a); ld_16x256b_x8(t + 64, b); }
    if (MODE == 2) { ld_16x128b_x16(t, a); ld_16x128b_x16(t + 64, b); }
    if (MODE == 3) { tmem_ld_32x32b_x32(t, a); tmem_ld_32x32b_x32(t + 32, b); tmem_ld_wait(); uint32_t c[32], e[32]; tmem_ld_32x32b_x32(t + 64, c); tmem_ld_32x32b_x32(t + 96, e); tmem_ld_wait(); acc += c[1] ^ e[3]; }
    tmem_ld_wait();
    acc += a[0] ^ b[5] ^ a[31];
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(slot); }
}
template <bool ST>
__global__ void __launch_bounds__(256, 1) tmem_kernel(int reps, unsigned long long* cyc, float* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = slot + (((warp & 3) * 32) << 16) + (warp >> 2) * 128;
  uint32_t acc = 0;
  uint32_t r[32];
  for (int i = 0; i < 32; ++i) r[i] = i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < reps; ++it) {
    if (ST) {
      tmem_st_32x32b_x32(t, r);
      tmem_st_32x32b_x32(t + 32, r);
      tmem_st_wait();
    } else {
      uint32_t a[32], b[32];
      tmem_ld_32x32b_x32(t, a);
      tmem_ld_32x32b_x32(t + 32, b);
      tmem_ld_wait();
      acc += a[0] ^ b[5] ^ a[31];
    }
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(slot); }
}
int main() {
  unsigned long long* cyc; float* out;
  cudaMalloc(&cyc, 148 * 8); cudaMalloc(&out, 148 * 256 * 4);
  const int reps = 2048;
  for (int threads : {128, 256}) {
    for (int m = 0; m < 4; ++m) {
      if (m == 0) tmem_ld_kernel<0><<<148, threads>>>(reps, cyc, out);
      if (m == 1) tmem_ld_kernel<1><<<148, threads>>>(reps, cyc, out);
      if (m == 2) tmem_ld_kernel<2><<<148, threads>>>(reps, cyc, out);
      if (m == 3) tmem_ld_kernel<3><<<148, threads>>>(reps, cyc, out);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      const double bytes = (double)threads * reps * 64 * 4 * (m == 3 ? 2 : 1);
      printf("ld mode %d (0: 32x32b.x32, 1: 16x256b.x8, 2: 16x128b.x16, 3: 4 x32 in 2 waits) warps=%d: %.1f B/clk/SM (%s)\n", m, threads / 32, bytes / h, cudaGetErrorString(e));
    }
    for (int st = 0; st < 2; ++st) {
      if (st) tmem_kernel<true><<<148, threads>>>(reps, cyc, out); else tmem_kernel<false><<<148, threads>>>(reps, cyc, out);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      const double bytes = (double)threads * reps * 64 * 4;
      printf("%s warps=%d: %.1f B/clk/SM (%s)\n", st ? "tcgen05.st" : "tcgen05.ld", threads / 32, bytes / h, cudaGetErrorString(e));
    }
  }
}
