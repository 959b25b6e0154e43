// XU-pipe calibration: MUFU.EX2 and F2FP (f32x2 -> f16x2) throughput per SM on this GPU,
// at full occupancy and at one warp per SMSP (the softmax-warp situation of the SSA kernels).
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ unsigned pk(float a, float b) { __half2 h = __floats2half2_rn(a, b); return *(unsigned*)&h; }

__device__ __forceinline__ unsigned ex2h2(unsigned x) { unsigned y; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ unsigned ex2bf2(unsigned x) { unsigned y; asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }

template <int MODE>
__global__ void k(float* out, int iters) {
  float a[8];
  unsigned u = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = -1e-3f * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] = ex2(a[i]) - 1.0f;                  // ex2 only (+1 FADD)
      if (MODE == 1) { u ^= pk(a[i], a[(i + 1) & 7]); a[i] += 1e-7f; }   // pack only
      if (MODE == 2) { float e = ex2(a[i]) - 1.0f; u ^= pk(e, a[(i + 1) & 7]); a[i] = e; }  // ex2 + pack per element pair
      if (MODE == 3) { unsigned h = ex2h2(__float_as_uint(a[i])); a[i] = __uint_as_float(h ^ 0x80008000u); }   // f16x2 ex2 (2 results)
      if (MODE == 4) { unsigned h = ex2bf2(__float_as_uint(a[i])); a[i] = __uint_as_float(h ^ 0x80008000u); }  // bf16x2 ex2 (2 results)
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + __uint_as_float(u);
}

template <int MODE>
void run(const char* name, int blocks, int threads, int iters) {
  float* o;
  cudaMalloc(&o, sizeof(float) * blocks * threads);
  k<MODE><<<blocks, threads>>>(o, 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MODE><<<blocks, threads>>>(o, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double ops = double(blocks) * threads * iters * 8;
  double cyc = ms * 1e-3 * clk * 1e3;
  printf("%-28s blocks %4d threads %4d: %.1f ops/clk/SM (%.3f ms)\n", name, blocks, threads, ops / cyc / 148, ms);
  cudaFree(o);
}

int main() {
  run<0>("ex2, full occupancy", 148 * 4, 512, 4000);
  run<0>("ex2, 1 warp/SMSP", 148, 128, 4000);
  run<0>("ex2, 2 warps/SMSP", 148, 256, 4000);
  run<1>("f16x2 pack, full occ", 148 * 4, 512, 4000);
  run<1>("f16x2 pack, 1 warp/SMSP", 148, 128, 4000);
  run<2>("ex2+pack, full occ", 148 * 4, 512, 4000);
  run<2>("ex2+pack, 1 warp/SMSP", 148, 128, 4000);
  run<2>("ex2+pack, 2 warps/SMSP", 148, 256, 4000);
  run<3>("ex2.f16x2 (x2 results)", 148 * 4, 512, 4000);
  run<3>("ex2.f16x2 1 warp/SMSP", 148, 128, 4000);
  run<4>("ex2.bf16x2 (x2 results)", 148 * 4, 512, 4000);
  return 0;
}
