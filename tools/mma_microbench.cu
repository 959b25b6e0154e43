// tcgen05.mma (kind::f16, cta_group::1, SS form) issue-to-completion cost per instruction for the shapes
// and operand majors the SSA kernels use. One CTA per SM; one thread issues R back-to-back MMAs into
// one TMEM accumulator, commits, waits; clocks per MMA vs the dense-peak ideal (M*N*K*2 / 8192 clk).
// Operand contents are irrelevant (zeros); the SW128 descriptors walk valid shared memory.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/mma_microbench tools/mma_microbench.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t((addr & 0x3FFFF) >> 4)) | (uint64_t((lbo & 0x3FFFF) >> 4) << 16) |
         (uint64_t((sbo & 0x3FFFF) >> 4) << 32) | (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4) | (uint32_t(a_mn) << 15) | (uint32_t(b_mn) << 16) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
               ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
               ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}

struct Shape { int M, N; bool a_mn, b_mn; const char* name; int nacc = 1; bool a_tmem = false; };

template <int NACC, bool TS>
__global__ void __launch_bounds__(128, 1) kbench(Shape sh, int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 155648 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0;
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (threadIdx.x == 0) {
    const uint32_t id = idesc_f16(sh.M, sh.N, sh.a_mn, sh.b_mn);
    const uint32_t a0 = smem_u32(base), b0 = smem_u32(base + 65536);
    // K-major: k-step 32 B inside the 128 B row (atoms of 64 K at +16 KB); MN-major: k-step 16 rows = 2 KB
    uint64_t da[8], db[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      da[k] = sh.a_mn ? desc_sw128(a0 + k * 2048, 16384, 1024) : desc_sw128(a0 + (k >> 2) * 16384 + (k & 3) * 32, 0, 1024);
      db[k] = sh.b_mn ? desc_sw128(b0 + k * 2048, 16384, 1024) : desc_sw128(b0 + (k >> 2) * 16384 + (k & 3) * 32, 0, 1024);
    }
    const uint32_t d0 = tmem_base, stride = sh.N;
    uint32_t ph = 0;
    unsigned long long t0 = 0;
    for (int pass = 0; pass < 2; ++pass) {
      if (pass == 1) t0 = clock64();
      for (int r = 0; r < reps; r += 8) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (TS) mma_ts(d0 + (k % NACC) * stride, d0 + 384 + k * 8, db[k], id, 1u);   // A: TMEM cols 384..447
          else mma(d0 + (k % NACC) * stride, da[k], db[k], id, 1u);
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)) : "memory");
      asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n"
                   ::"r"(smem_u32(&bar)), "r"(ph) : "memory");
      ph ^= 1u;
    }
    out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem_base));
}

int main() {
  const Shape shapes[] = {
      {128, 256, false, false, "128x256 A K  B K"}, {128, 128, false, false, "128x128 A K  B K"},
      {128, 64, false, false, "128x64  A K  B K"},  {128, 64, false, true, "128x64  A K  B MN"},
      {128, 64, true, true, "128x64  A MN B MN"},   {128, 128, true, false, "128x128 A MN B K"},
      {128, 32, true, false, "128x32  A MN B K"},   {128, 16, true, false, "128x16  A MN B K"},
      {128, 16, false, false, "128x16  A K  B K"},  {64, 128, false, true, "64x128  A K  B MN"},
      {64, 64, false, false, "64x64   A K  B K"},   {128, 112, false, false, "128x112 A K  B K"},
      {128, 128, false, false, "128x128 K K  2 acc", 2}, {128, 128, false, false, "128x128 K K  4 acc", 4},
      {128, 64, false, true, "128x64  K MN 2 acc", 2},  {128, 64, false, true, "128x64  K MN 4 acc", 4},
      {128, 64, false, true, "128x64  K MN 8 acc", 8},  {128, 16, true, false, "128x16  MN K 4 acc", 4},
      {128, 16, true, false, "128x16  MN K 8 acc", 8},
      {128, 64, false, true, "TS 128x64 B MN", 1, true}, {128, 128, false, false, "TS 128x128 B K", 1, true},
      {128, 64, false, true, "TS 128x64 B MN 2acc", 2, true}, {128, 256, false, false, "TS 128x256 B K", 1, true}, {128, 32, false, false, "128x32  K K  8 acc", 8},  {128, 256, false, false, "128x256 K K  2 acc", 2},
  };
  unsigned long long* d;
  cudaMalloc(&d, 148 * sizeof(unsigned long long));
  cudaFuncSetAttribute(kbench<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  cudaFuncSetAttribute(kbench<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  cudaFuncSetAttribute(kbench<4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  cudaFuncSetAttribute(kbench<8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  cudaFuncSetAttribute(kbench<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  cudaFuncSetAttribute(kbench<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  unsigned long long h[148];
  for (const Shape& s : shapes) {
    for (int reps : {64, 1024}) {
      if (s.nacc == 1 && !s.a_tmem) kbench<1, false><<<148, 128, 160 * 1024>>>(s, reps, d);
      if (s.nacc == 2 && !s.a_tmem) kbench<2, false><<<148, 128, 160 * 1024>>>(s, reps, d);
      if (s.nacc == 4 && !s.a_tmem) kbench<4, false><<<148, 128, 160 * 1024>>>(s, reps, d);
      if (s.nacc == 8 && !s.a_tmem) kbench<8, false><<<148, 128, 160 * 1024>>>(s, reps, d);
      if (s.nacc == 1 && s.a_tmem) kbench<1, true><<<148, 128, 160 * 1024>>>(s, reps, d);
      if (s.nacc == 2 && s.a_tmem) kbench<2, true><<<148, 128, 160 * 1024>>>(s, reps, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("%s: %s\n", s.name, cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += double(h[i]);
      avg /= 148.0 * reps;
      const double ideal = double(s.M) * s.N * 16 * 2 / 8192.0;
      printf("%-20s reps %5d: %7.1f clk/MMA  ideal %5.1f  -> %5.1f%% of peak\n", s.name, reps, avg, ideal, 100.0 * ideal / avg);
    }
  }
  return 0;
}
