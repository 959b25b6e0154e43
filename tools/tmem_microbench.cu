// tcgen05.ld latency / throughput calibration (one CTA per SM, 4 warps reading their TMEM lanes).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
template <int X>
__device__ __forceinline__ void ld(uint32_t a, uint32_t* r);
template <> __device__ __forceinline__ void ld<16>(uint32_t a, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
                 "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]) : "r"(a));
}
__global__ void k(unsigned long long* out, int iters, int mode) {
  __shared__ uint32_t base;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = base + (uint32_t(warp * 32) << 16);
  uint32_t r[16], acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (mode == 0) {            // latency: load 16 cols, wait, use
      ld<16>(t + (i & 7) * 16, r);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      acc += r[0] ^ r[15];
    } else {                    // throughput: 8 loads, one wait
      for (int j = 0; j < 8; ++j) { ld<16>(t + j * 16, r); acc += r[j]; }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 12345) out[1000] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(base));
}
int main() {
  unsigned long long* o;
  cudaMalloc(&o, 8 * 2000);
  for (int mode = 0; mode < 2; ++mode)
    for (int warps : {4, 8}) {
      k<<<148, warps * 32>>>(o, 100, mode);
      k<<<148, warps * 32>>>(o, 2000, mode);
      unsigned long long h[148];
      cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
      printf("mode %d (%s) warps %d: %.1f clk per iteration\n", mode, mode ? "8 lds, 1 wait" : "ld+wait", warps, double(h[0]) / 2000);
    }
  return 0;
}
