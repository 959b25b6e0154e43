// tc_selftest.cu — tensor-map encoding (host) and a UMMA descriptor self-test kernel that checks every
// operand layout the SSA tcgen05 kernels use against a plain matmul (tests/test_gpu_umma.py).
#include <mutex>

#include "../../include/ssa_selftest.h"
#include "internal.h"
#include "tc_common.cuh"

namespace ssa {

namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}
}  // namespace

bool make_tmap_bf16_2d(CUtensorMap* m, const void* base, uint64_t rows, uint32_t box_rows) {
  EncodeFn enc = get_encode();
  if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return false; }
  cuuint64_t dims[2] = {64, rows};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { set_error("cuTensorMapEncodeTiled failed: " + std::to_string(int(r))); return false; }
  return true;
}

namespace {
using namespace tc;

// mode 0: D[128][N] = A[128][64] . B[N][64]^T     A, B K-major, both by TMA            (S = Q K^T)
// mode 1: D[128][64] = At[128][128]^T . B[128][64] A MN-major (manual), B MN-major TMA (O = P V, P^T stored)
// mode 2: D[128][64] = A[128][K] . B[K][64]       A K-major (manual), B MN-major TMA  (O = P V / dQ = dS K)
__global__ void __launch_bounds__(128) k_umma_selftest(int mode, int N, int K, const __nv_bfloat16* __restrict__ a,
                                                        __grid_constant__ const CUtensorMap tmA,
                                                        __grid_constant__ const CUtensorMap tmB, float* __restrict__ d) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = sm;                // up to 32 KB
  uint8_t* sB = sm + 32768;        // up to 32 KB
  __shared__ uint64_t bar_ld, bar_mma;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    mbar_init(&bar_ld, 1);
    mbar_init(&bar_mma, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<256>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  // manual operand writes
  if (mode == 1) {          // a = At [K=128][M=128]; MN-major: M block mb at mb*K*128 bytes, line = k
    for (int i = tid; i < 128 * 16; i += 128) {
      int k = i / 16, c = i % 16, mb = c / 8, ch = c % 8;
      const uint4 v = *reinterpret_cast<const uint4*>(a + k * 128 + c * 8);
      uint32_t off = mb * (K * 128) + sw128(k, ch);
      *reinterpret_cast<uint4*>(sA + off) = v;
    }
  } else if (mode == 2 || mode == 3) {   // a = A [M=128][K]; K-major: K block kb (64 wide) at kb*16384, line = m
    for (int i = tid; i < 128 * (K / 8); i += 128) {
      int m = i / (K / 8), c = i % (K / 8), kb = c / 8, ch = c % 8;
      const uint4 v = *reinterpret_cast<const uint4*>(a + m * K + c * 8);
      *reinterpret_cast<uint4*>(sA + kb * 16384 + sw128(m, ch)) = v;
    }
  }
  if (mode == 4 || mode == 5) {   // A [128][K] bf16 -> TMEM columns 128.., lane = row, two K per column
    uint32_t w[32];
    for (int c0 = 0; c0 < K / 2; c0 += 16) {
      for (int i = 0; i < 16; ++i) {
        const __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(a + tid * K + 2 * (c0 + i));
        w[i] = *reinterpret_cast<const uint32_t*>(&h);
      }
      tmem_st16(tmem + (uint32_t(warp * 32) << 16) + 128 + c0, w);
    }
    tmem_wait_st();
    tc_fence_before();
  }
  fence_proxy_async_smem();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    uint32_t bytes = 0;
    if (mode == 0) {
      tma_load_2d(sA, &tmA, &bar_ld, 0, 0);
      tma_load_2d(sB, &tmB, &bar_ld, 0, 0);
      bytes = 128 * 128 + N * 128;
    } else if (mode == 5) {
      tma_load_2d(sB, &tmB, &bar_ld, 0, 0);
      bytes = N * 128;
    } else {
      tma_load_2d(sB, &tmB, &bar_ld, 0, 0);
      bytes = K * 128;
    }
    mbar_expect_tx(&bar_ld, bytes);
    mbar_wait(&bar_ld, 0);
    tc_fence_after();
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    if (mode == 4) {          // A in TMEM, B MN-major [K][64] (TMA)
      const uint32_t id = idesc_bf16(128, 64, false, true);
      for (int s = 0; s < K / 16; ++s)
        umma_ts(tmem, tmem + 128 + s * 8, desc_sw128(b0 + s * 2048, 0, 1024), id, s > 0);
    } else if (mode == 5) {   // A in TMEM (K = 64), B K-major [N][64] (TMA)
      const uint32_t id = idesc_bf16(128, N, false, false);
      for (int s = 0; s < 4; ++s)
        umma_ts(tmem, tmem + 128 + s * 8, desc_sw128(b0 + s * 32, 0, 1024), id, s > 0);
    } else if (mode == 0) {
      const uint32_t id = idesc_bf16(128, N, false, false);
      for (int s = 0; s < 4; ++s)
        umma_bf16(tmem, desc_sw128(a0 + s * 32, 0, 1024), desc_sw128(b0 + s * 32, 0, 1024), id, s > 0);
    } else if (mode == 1) {
      const uint32_t id = idesc_bf16(128, 64, true, true);
      for (int s = 0; s < K / 16; ++s)
        umma_bf16(tmem, desc_sw128(a0 + s * 2048, K * 128, 1024), desc_sw128(b0 + s * 2048, 0, 1024), id, s > 0);
    } else {
      // mode 3: A and B fp16 (the P.V operand format)
      const uint32_t id = mode == 3 ? idesc_f16(128, 64, false, true) : idesc_bf16(128, 64, false, true);
      for (int s = 0; s < K / 16; ++s)
        umma_bf16(tmem, desc_sw128(a0 + (s / 4) * 16384 + (s % 4) * 32, 0, 1024),
                  desc_sw128(b0 + s * 2048, 0, 1024), id, s > 0);
    }
    umma_commit(&bar_mma);
  }
  __syncwarp();
  mbar_wait(&bar_mma, 0);
  tc_fence_after();
  const int ncol = (mode == 0 || mode == 5) ? N : 64;
  for (int c0 = 0; c0 < ncol; c0 += 16) {
    float v[16];
    tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + c0, v);
    tmem_wait_ld();
    for (int i = 0; i < 16; ++i) d[tid * ncol + c0 + i] = v[i];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tmem);
}
}  // namespace
}  // namespace ssa

using namespace ssa;

extern "C" ssa_status ssa_selftest_umma(int mode, int n, int k, const void* a, const void* b, float* d, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CUtensorMap tmA{}, tmB{};
  if (mode == 0) {
    if (!make_tmap_bf16_2d(&tmA, a, 128, 128) || !make_tmap_bf16_2d(&tmB, b, n, n)) return SSA_ERR_CUDA;
  } else if (mode == 5) {
    if (!make_tmap_bf16_2d(&tmA, b, n, n) || !make_tmap_bf16_2d(&tmB, b, n, n)) return SSA_ERR_CUDA;
  } else {
    if (!make_tmap_bf16_2d(&tmA, b, k, k) || !make_tmap_bf16_2d(&tmB, b, k, k)) return SSA_ERR_CUDA;
  }
  const int smem = 65536 + 1024;
  SSA_CUDA_TRY(cudaFuncSetAttribute(k_umma_selftest, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k_umma_selftest<<<1, 128, smem, st>>>(mode, n, k, static_cast<const __nv_bfloat16*>(a), tmA, tmB, d);
  SSA_LAUNCH_CHECK("k_umma_selftest");
  SSA_CUDA_TRY(cudaStreamSynchronize(st));
  return SSA_OK;
}
