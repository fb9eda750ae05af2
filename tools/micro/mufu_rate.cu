// Microbenchmark: MUFU.EX2 and FFMA2 throughput per SM (cycles per warp instruction).
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include "ptx.cuh"
using namespace pf;
// 2^x for a pair on the FMA pipe (FA4-style): clamp, floor by the 1.5*2^23 round-down trick, minimax
// cubic for 2^frac (max rel. error 8.8e-5), exponent add.
__device__ __forceinline__ uint64_t ex2_emu2(uint64_t x2) {
  constexpr float kMagic = 12582912.0f;
  float x0, x1;
  f2_unpack(x2, x0, x1);
  const uint64_t xc = f2_pack(fmaxf(x0, -127.f), fmaxf(x1, -127.f));
  uint64_t t, jf, f, p;
  asm("add.rm.f32x2 %0, %1, %2;" : "=l"(t) : "l"(xc), "l"(f2_pack(kMagic, kMagic)));
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(jf) : "l"(t), "l"(f2_pack(-kMagic, -kMagic)));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(f) : "l"(jf), "l"(f2_pack(-1.f, -1.f)), "l"(xc));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(p) : "l"(f), "l"(f2_pack(0.0771190897f, 0.0771190897f)), "l"(f2_pack(0.2275643945f, 0.2275643945f)));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(p) : "l"(p), "l"(f), "l"(f2_pack(0.6951461434f, 0.6951461434f)));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(p) : "l"(p), "l"(f), "l"(f2_pack(1.f, 1.f)));
  float t0, t1, p0, p1;
  f2_unpack(t, t0, t1);
  f2_unpack(p, p0, p1);
  return f2_pack(__uint_as_float((__float_as_uint(t0) << 23) + __float_as_uint(p0)),
                 __uint_as_float((__float_as_uint(t1) << 23) + __float_as_uint(p1)));
}
__global__ void ex2_kernel(int reps, float* out, unsigned long long* cyc) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = -0.001f * (threadIdx.x + i);
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = ex2_approx(x[i]) - 1.0f;
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void emu_kernel(int reps, float* out, unsigned long long* cyc) {
  uint64_t x[4];
  for (int i = 0; i < 4; ++i) x[i] = f2_pack(-0.001f * (threadIdx.x + i), -0.002f * i);
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = fadd2(ex2_emu2(x[i]), f2_pack(-1.f, -1.f));
  }
  long long t1 = clock64();
  float s = 0, a, b; for (int i = 0; i < 4; ++i) { f2_unpack(x[i], a, b); s += a + b; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void ex2h_kernel(int reps, float* out, unsigned long long* cyc) {
  uint32_t x[8];
  for (int i = 0; i < 8; ++i) { __half2 h = __floats2half2_rn(-0.001f * (threadIdx.x + i), -0.002f * i); x[i] = *reinterpret_cast<uint32_t*>(&h); }
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { uint32_t y; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x[i])); x[i] = y ^ 0x80008000u; }
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += __half2float(*reinterpret_cast<__half*>(&x[i]));
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int OP>
__global__ void op_kernel(int reps, float* out, unsigned long long* cyc) {
  float x[8]; uint32_t u[8];
  for (int i = 0; i < 8; ++i) { x[i] = 0.001f * (threadIdx.x + i); u[i] = threadIdx.x * 7 + i; }
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) { u[i] = pack_bf16x2(x[i], __uint_as_float(u[i])); }                        // F2FP
      if (OP == 1) { x[i] = fmax3(x[i], __uint_as_float(u[i]), x[(i + 1) & 7]); }               // FMNMX3
      if (OP == 2) { u[i] = __byte_perm(u[i], __float_as_uint(x[i]), 0x7632); }                // PRMT
      if (OP == 3) { float a, b; f2_unpack(ffma2(f2_pack(x[i], x[i]), f2_pack(1.0001f, 1.0001f), f2_pack(0.1f, 0.1f)), a, b); x[i] = a + 0.f * b; }  // FFMA2
    }
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i] + __uint_as_float(u[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; unsigned long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const int reps = 4096;
  for (int threads : {128, 256, 512}) {
    ex2_kernel<<<148, threads>>>(reps, out, cyc);
    cudaDeviceSynchronize();
    unsigned long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    const double warp_instr = (threads / 32.0) * reps * 8;
    printf("ex2  threads=%d: %.2f cyc per warp-MUFU per SM (%.1f ex2/clk/SM)\n", threads, h / warp_instr, warp_instr * 32 / h);
    emu_kernel<<<148, threads>>>(reps, out, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    const double elems = threads * (double)reps * 8;
    printf("emu  threads=%d: %.1f exp2/clk/SM (FMA-pipe emulation)\n", threads, elems / h);
    ex2h_kernel<<<148, threads>>>(reps, out, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("ex2.f16x2 threads=%d: %.1f exp2/clk/SM\n", threads, threads * (double)reps * 16 / h);
  }
  const char* names[] = {"F2FP.BF16 pack", "FMNMX3", "PRMT", "FFMA2"};
  for (int op = 0; op < 4; ++op) {
    for (int threads : {256, 512}) {
      if (op == 0) op_kernel<0><<<148, threads>>>(reps, out, cyc);
      if (op == 1) op_kernel<1><<<148, threads>>>(reps, out, cyc);
      if (op == 2) op_kernel<2><<<148, threads>>>(reps, out, cyc);
      if (op == 3) op_kernel<3><<<148, threads>>>(reps, out, cyc);
      cudaDeviceSynchronize();
      unsigned long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      printf("%-16s threads=%d: %.1f warp-instr/clk/SM (%.0f lanes/clk)\n", names[op], threads, (threads / 32.0) * reps * 8 / h, threads * (double)reps * 8 / h);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
