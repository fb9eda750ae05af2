// Microbenchmark: tcgen05.ld throughput of 4 warps while one thread keeps the tensor pipe busy
// with M128 N128 K16 MMAs (SS or TS) into other TMEM columns.
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace pf;
template <int MODE>   // 0: no MMA, 1: SS MMA, 2: TS MMA
__global__ void __launch_bounds__(192, 1) k(int reps, unsigned long long* cyc, float* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  __shared__ volatile int stop;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 32768 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); stop = 0; }
  if (warp == 4) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = slot;
  if (warp == 4) {
    if (MODE > 0) {
      const uint32_t idesc = make_idesc_bf16(128, 128, false, false);
      const uint64_t a = kmajor_desc(smem_u32(smem)), b = kmajor_desc(smem_u32(smem + 16384));
      int n = 0;
      while (!stop && n < 200000) {
        if (elect_one()) {
          for (int kk = 0; kk < 8; ++kk) {
            if (MODE == 1) umma_bf16_ss(tb + 256, a + ((kk & 3) * 2), b + ((kk & 3) * 2), idesc, 1);
            else umma_bf16_ts(tb + 256, tb + 384 + kk * 8, b + ((kk & 3) * 2), idesc, 1);
          }
        }
        __syncwarp();
        n += 8;
      }
      if (elect_one()) umma_commit(&bar);
      __syncwarp();
      mbar_wait(&bar, 0);
    }
  } else {
    const uint32_t t = tb + ((warp * 32) << 16);
    uint32_t acc = 0;
    long long t0 = clock64();
    for (int it = 0; it < reps; ++it) {
      uint32_t a[32], b[32], c[32], e[32];
      tmem_ld_32x32b_x32(t, a); tmem_ld_32x32b_x32(t + 32, b); tmem_ld_32x32b_x32(t + 64, c); tmem_ld_32x32b_x32(t + 96, e);
      tmem_ld_wait();
      acc += a[0] ^ b[5] ^ c[7] ^ e[31];
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
    if (threadIdx.x == 0) { cyc[blockIdx.x] = t1 - t0; stop = 1; }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) { tc_fence_after(); tmem_dealloc<512>(tb); }
}
int main() {
  unsigned long long* cyc; float* out;
  cudaMalloc(&cyc, 148 * 8); cudaMalloc(&out, 148 * 256 * 4);
  const int reps = 4096;
  for (int m = 0; m < 3; ++m) {
    auto f = m == 0 ? k<0> : m == 1 ? k<1> : k<2>;
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    f<<<148, 192, 40000>>>(reps, cyc, out);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("mode %d (0 none, 1 SS MMA, 2 TS MMA running): 4 warps x 4 LDTM.x32 + wait: %.0f cyc/iter = %.1f B/clk/SM (%s)\n",
           m, (double)h / reps, 128.0 * 128 * 4 * reps / h, cudaGetErrorString(e));
  }
}
