// Softmax-turn calibration: the exponential loop of one MUFU turn of the tcgen05 kernels (per thread:
// p = exp2(s * c - m) over its S row, row sum, f16x2 pack), timed per 128 rows x 128 columns, with
//   * 1 warp per SMSP (128 threads x 128 columns: the current turn) or 2 warps per SMSP (256 threads x 64
//     columns: a row split across two warps of the same sub-partition),
//   * a fraction of the exponentials on the FMA pipe (Cody-Waite split by a round-down magic add, degree-3
//     minimax polynomial, exponent added with an integer shift; no F2I/FRND, which share the XU pipe).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/turn tools/turn_microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t pk(float a, float b) {
  uint32_t r; asm("cvt.rn.f16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(a), "f"(b)); return r;
}
// 2^x for x in [-127, 0]-ish: j = floor(x) by a round-down add of 1.5 * 2^23, f = x - j in [0, 1),
// 2^f by a degree-3 minimax polynomial (rel. err ~9e-5), exponent j added to the bits.
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -126.f);
  float j;
  asm("add.rm.f32 %0, %1, 0f4B400000;" : "=f"(j) : "f"(x));   // 12582912 + floor(x)
  const float jf = j - 12582912.f;
  const float f = x - jf;
  float p = fmaf(fmaf(fmaf(0.0790209f, f, 0.2249904f), f, 0.6957561f), f, 1.0000026f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(j) << 23));
}

template <int NCOL, int POLY_EVERY>   // POLY_EVERY: every k-th pair of columns by polynomial (0: none)
__global__ void __launch_bounds__(256, 1) k(float* out, int iters, float cl2) {
  float v[NCOL];
#pragma unroll
  for (int i = 0; i < NCOL; ++i) v[i] = -0.01f * ((threadIdx.x * 7 + i * 13) & 255);
  float l = 0.f;
  uint32_t x = 0;
  float m = 0.5f;
  for (int it = 0; it < iters; ++it) {
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < NCOL; i += 2) {
      float p0, p1;
      if (POLY_EVERY > 0 && ((i >> 1) % POLY_EVERY) == POLY_EVERY - 1) {
        p0 = ex2_poly(fmaf(v[i], cl2, -m));
        p1 = ex2_poly(fmaf(v[i + 1], cl2, -m));
      } else {
        p0 = ex2(fmaf(v[i], cl2, -m));
        p1 = ex2(fmaf(v[i + 1], cl2, -m));
      }
      acc[(i >> 1) & 3] += p0 + p1;
      x ^= pk(p0, p1);
    }
    l += (acc[0] + acc[1]) + (acc[2] + acc[3]);
    m += 1e-7f;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = l + __uint_as_float(x & 0x3fffu);
}

__global__ void chk(float* e) {
  float mx = 0.f;
  for (int i = 0; i < 1 << 16; ++i) {
    const float xx = -30.f * i / 65536.f;
    const float a = ex2_poly(xx), b = exp2f(xx);
    mx = fmaxf(mx, fabsf(a - b) / b);
  }
  e[0] = mx;
}

template <int NCOL, int PE>
void run(const char* name, int threads) {
  float* o;
  cudaMalloc(&o, sizeof(float) * 148 * 256);
  const int iters = 20000;
  k<NCOL, PE><<<148, threads>>>(o, 10, 0.18f);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<NCOL, PE><<<148, threads>>>(o, iters, 0.18f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double cyc = ms * 1e-3 * clk * 1e3;
  const double exps = double(threads) * NCOL * iters;   // per SM
  printf("%-40s %.2f exp/clk/SM, %.0f clk per 128x128 turn\n", name, exps / cyc, cyc / (exps / 16384.0));
  cudaFree(o);
}

int main() {
  float* e; cudaMalloc(&e, 4); chk<<<1, 1>>>(e); float he; cudaMemcpy(&he, e, 4, cudaMemcpyDeviceToHost);
  printf("poly max rel err on [-30, 0]: %.3g\n", he);
  run<128, 0>("1 warp/SMSP, MUFU only", 128);
  run<128, 8>("1 warp/SMSP, 1/8 poly", 128);
  run<128, 4>("1 warp/SMSP, 1/4 poly", 128);
  run<128, 3>("1 warp/SMSP, 1/3 poly", 128);
  run<128, 2>("1 warp/SMSP, 1/2 poly", 128);
  run<64, 0>("2 warps/SMSP (64 col), MUFU only", 256);
  run<64, 8>("2 warps/SMSP (64 col), 1/8 poly", 256);
  run<64, 4>("2 warps/SMSP (64 col), 1/4 poly", 256);
  run<64, 3>("2 warps/SMSP (64 col), 1/3 poly", 256);
  run<128, 0>("2 warps/SMSP (128 col), MUFU only", 256);
  run<128, 4>("2 warps/SMSP (128 col), 1/4 poly", 256);
  return 0;
}
