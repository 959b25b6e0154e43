// scan.cu — device-wide exclusive prefix sum (int32), used by the block build (compaction of block
// starts, bitmap ranks) and by the inverse-selection CSR. Reduce-then-scan, recursive over block
// sums; 1024 threads x 4 items per CTA.
#include "internal.h"

namespace ssa {
namespace {
constexpr int kThreads = 1024;
constexpr int kItems = 4;
constexpr int kTile = kThreads * kItems;

__device__ __forceinline__ int32_t warp_incl(int32_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int32_t n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

// block-wide exclusive scan of one value per thread; returns exclusive prefix, *agg = block total
__device__ __forceinline__ int32_t block_excl(int32_t v, int32_t* smem, int32_t* agg) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t inc = warp_incl(v);
  if (lane == 31) smem[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int32_t s = smem[lane];
    int32_t si = warp_incl(s);
    smem[lane] = si - s;
    if (lane == 31) smem[32] = si;
  }
  __syncthreads();
  int32_t r = inc - v + smem[warp];
  *agg = smem[32];
  __syncthreads();
  return r;
}

__global__ void k_tile_sums(const int32_t* __restrict__ in, int64_t n, int32_t* __restrict__ sums) {
  __shared__ int32_t sm[33];
  int64_t base = int64_t(blockIdx.x) * kTile + int64_t(threadIdx.x) * kItems;
  int32_t s = 0;
#pragma unroll
  for (int i = 0; i < kItems; ++i)
    if (base + i < n) s += in[base + i];
  int32_t agg;
  block_excl(s, sm, &agg);
  if (threadIdx.x == 0) sums[blockIdx.x] = agg;
}

__global__ void k_tile_scan(const int32_t* in, int64_t n, int32_t* out, const int32_t* __restrict__ offs,
                            int32_t* total) {
  __shared__ int32_t sm[33];
  int64_t base = int64_t(blockIdx.x) * kTile + int64_t(threadIdx.x) * kItems;
  int32_t x[kItems];
  int32_t s = 0;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    x[i] = (base + i < n) ? in[base + i] : 0;
    s += x[i];
  }
  int32_t agg;
  int32_t pre = block_excl(s, sm, &agg) + (offs ? offs[blockIdx.x] : 0);
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    if (base + i < n) out[base + i] = pre;
    pre += x[i];
  }
  if (total && blockIdx.x == gridDim.x - 1 && threadIdx.x == kThreads - 1) *total = pre;
}
}  // namespace

size_t scan_ws_bytes(int64_t n) {
  size_t b = 0;
  while (n > kTile) {
    int64_t nb = (n + kTile - 1) / kTile;
    b += ((size_t(nb) * 4 + 255) & ~size_t(255));
    n = nb;
  }
  return b + 256;
}

ssa_status exclusive_scan(const int32_t* in, int32_t* out, int64_t n, int32_t* total, void* ws,
                          cudaStream_t st) {
  if (n <= 0) {
    if (total) SSA_CUDA_TRY(cudaMemsetAsync(total, 0, sizeof(int32_t), st));
    return SSA_OK;
  }
  if (n <= kTile) {
    k_tile_scan<<<1, kThreads, 0, st>>>(in, n, out, nullptr, total);
    SSA_LAUNCH_CHECK("k_tile_scan");
    return SSA_OK;
  }
  int64_t nb = (n + kTile - 1) / kTile;
  int32_t* sums = static_cast<int32_t*>(ws);
  void* rest = static_cast<char*>(ws) + ((size_t(nb) * 4 + 255) & ~size_t(255));
  k_tile_sums<<<unsigned(nb), kThreads, 0, st>>>(in, n, sums);
  SSA_LAUNCH_CHECK("k_tile_sums");
  ssa_status s = exclusive_scan(sums, sums, nb, nullptr, rest, st);
  if (s != SSA_OK) return s;
  k_tile_scan<<<unsigned(nb), kThreads, 0, st>>>(in, n, out, sums, total);
  SSA_LAUNCH_CHECK("k_tile_scan");
  return SSA_OK;
}

}  // namespace ssa
