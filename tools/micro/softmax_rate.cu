// Microbenchmark: the attention softmax of one 64-key block per thread (row), as attention.cu runs it
// (TMEM load of S, row max, exp2 on MUFU, bf16 P pairs, row sum, TMEM store of P), with 1 or 2 warps
// per SM sub-partition and no other work on the SM: cycles per block per warp.
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace pf;

template <bool TMEM_IO>
__global__ void __launch_bounds__(256, 1) softmax_kernel(int reps, int nwarps, unsigned long long* cyc, float* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tS = slot + (((warp & 3) * 32) << 16) + 64 * (warp >> 2);
  float m_used = -INFINITY, l_run = 0.f;
  const float sl2 = 0.12f;
  uint32_t s[2][32];
  for (int c = 0; c < 2; ++c)
    for (int i = 0; i < 32; ++i) s[c][i] = __float_as_uint(0.01f * (lane + i + 32 * c));
  if (TMEM_IO && warp < nwarps) { tmem_st_32x32b_x32(tS, s[0]); tmem_st_32x32b_x32(tS + 32, s[1]); tmem_st_wait(); }
  __syncthreads();
  long long t0 = clock64();
  if (warp < nwarps) {
    for (int it = 0; it < reps; ++it) {
      if (TMEM_IO) {
        tmem_ld_32x32b_x32(tS, s[0]);
        tmem_ld_32x32b_x32(tS + 32, s[1]);
        tmem_ld_wait();
      }
      float mxv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) mxv[i] = fmaxf(__uint_as_float(s[0][2 * i]), __uint_as_float(s[0][2 * i + 1]));
#pragma unroll
      for (int i = 4; i < 16; ++i) mxv[i & 3] = fmax3(mxv[i & 3], __uint_as_float(s[0][2 * i]), __uint_as_float(s[0][2 * i + 1]));
#pragma unroll
      for (int i = 0; i < 16; ++i) mxv[i & 3] = fmax3(mxv[i & 3], __uint_as_float(s[1][2 * i]), __uint_as_float(s[1][2 * i + 1]));
      const float mx = sl2 * fmax3(fmaxf(mxv[0], mxv[1]), mxv[2], mxv[3]);
      const bool rescale = __any_sync(0xffffffffu, mx > m_used + 8.f);
      if (rescale) m_used = fmaxf(m_used, mx);
      uint64_t sum2[2] = {0ull, 0ull};
      uint32_t w[32];
      const uint64_t scale2 = f2_pack(sl2, sl2), negm2 = f2_pack(-m_used, -m_used);
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const uint64_t x2 = ffma2(f2_pack(__uint_as_float(s[c][2 * i]), __uint_as_float(s[c][2 * i + 1])), scale2, negm2);
          float x0, x1;
          f2_unpack(x2, x0, x1);
          const float p0 = ex2_approx(x0), p1 = ex2_approx(x1);
          sum2[i & 1] = fadd2(sum2[i & 1], f2_pack(p0, p1));
          w[c * 16 + i] = pack_bf16x2(p0, p1);
        }
      float a, b, c2, d2;
      f2_unpack(sum2[0], a, b);
      f2_unpack(sum2[1], c2, d2);
      l_run += (a + b) + (c2 + d2);
      if (TMEM_IO) {
        tmem_st_32x32b_x32(tS + 128, w);
        tmem_st_wait();
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) s[i >> 4][i & 15] ^= w[i] & 1u;   // keep the dependency
      }
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = l_run;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(slot); }
}

int main() {
  unsigned long long* cyc; float* out;
  cudaMalloc(&cyc, 148 * 8); cudaMalloc(&out, 148 * 256 * 4);
  const int reps = 2000;
  for (int io = 0; io < 2; ++io)
    for (int nw : {4, 8}) {
      if (io) softmax_kernel<true><<<148, 256>>>(reps, nw, cyc, out); else softmax_kernel<false><<<148, 256>>>(reps, nw, cyc, out);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      printf("softmax 64-key block, %s, %d warps (%d per SMSP): %.0f cycles per block per warp (%s)\n",
             io ? "S/P through TMEM" : "registers only", nw, nw / 4, (double)h / reps, cudaGetErrorString(e));
    }
}
