// tc_bwd.cu — tcgen05/TMEM/TMA backward kernels of the bf16, d = 64 SSA path.
// Probabilities are recomputed from the forward's saved LSEs (flash-style); the block structure and
// the selected indices I are constants (hard routing, reading R15). With D_c = omega_c <dO, O_c>:
//   dS = P (omega_c dP - D_c),  dP = dO V^T,  dq = scale dS K,  dk = scale dS^T q,  dv = (P omega_c)^T dO.
//
//  k_tc_dq    Q-outer: CTA per (query block, kv group); for every 128-row tile, S = Q K^T and dP = dO V^T
//             over the compression keys, the selected blocks and the window (96-key tiles; selected
//             blocks packed in 8-row granules), dS -> smem, dQ += dS K accumulated in TMEM over all three branches,
//             written once to the caller's dq (no atomics, deterministic).
//  k_tc_dkdv  KV-outer: CTA per key tile; S^T = K Q^T and dP^T = V dO^T for 64-row tiles (keys on TMEM
//             lanes), (P omega)^T and dS^T -> smem as K-major A operands, dV += (P omega)^T dO and
//             dK += dS^T Q accumulated in TMEM. Raw keys (mode 1): the rows of every query block that
//             selected the key's block (inverse CSR, ascending) + the window's own rows. Compressed keys
//             (mode 0): a 1/n_chunk share of the batch item's rows -> per-chunk partials reduced in a
//             fixed order (deterministic).
#include <cfloat>
#include <cstdlib>
#include <mutex>

#include "internal.h"
#include "tc.h"
#include "tc_common.cuh"

namespace ssa {
namespace {
using namespace tc;

constexpr int kD = 64;
constexpr float kLog2e = 1.4426950408889634f;
constexpr int kStages = 3;

struct Ring {
  int idx = 0;
  uint32_t ph = 0;
  int n;
  __device__ explicit Ring(int n_) : n(n_) {}
  __device__ void next() {
    if (++idx == n) { idx = 0; ph ^= 1u; }
  }
};

// fp16 operand copies for the backward MMAs. bf16 inputs convert exactly while |x| < 65504
// (saturating beyond); dS and P*omega are then packed in fp16 (11-bit mantissa).
// (dO scaled by the row's gate of each branch feeds the KV-outer kernel: dV = P^T (w dO) and
// dP = V (w dO)^T, which removes two multiplies per score element there.)
__device__ float g_pos_inf = INFINITY;
__device__ float g_zero = 0.f;
// two floats -> f16x2 (saturating; element lo in the low half)
__device__ __forceinline__ uint32_t h2_sat(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ void bf16x8_to_f32(uint4 u, float* f) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    f[2 * j] = __uint_as_float(w[j] << 16);
    f[2 * j + 1] = __uint_as_float(w[j] & 0xFFFF0000u);
  }
}
__device__ __forceinline__ uint4 f32x8_to_h(const float* f, float s) {
  return make_uint4(h2_sat(f[0] * s, f[1] * s), h2_sat(f[2] * s, f[3] * s), h2_sat(f[4] * s, f[5] * s),
                    h2_sat(f[6] * s, f[7] * s));
}
// Power-of-two scale of the fp16 dO operands (a loss averaged over ~1e5 tokens gives dO of
// ~1e-6 and below, where an unscaled fp16 copy loses bits or flushes to zero). s = 2^(2 - e) for
// max|dO| in [2^e, 2^(e+1)) brings max|s dO| into [4, 8): every bf16 dO value with |x| >= 2^-20 max|dO|
// converts exactly, and dP = (s dO) V^T keeps the fp16 headroom of unit-variance data. dO, w dO and
// D_c are scaled by s in the row prologue; dq / dk / dv (and the compressed-key partials) are
// multiplied by 1/s where they leave TMEM. s = 1 for a zero or non-finite maximum.
__device__ __forceinline__ float do_pow2(const uint32_t* amax, bool inverse) {
  const uint32_t bits = *amax;
  const int e = int((bits >> 23) & 0xffu) - 127;
  if (bits == 0u || e > 120 || e < -120) return 1.f;
  const int k = inverse ? e - 2 : 2 - e;
  return __int_as_float((k + 127) << 23);
}
// max |dO| over the caller's dout (bf16, 8 elements per thread; non-negative floats order as uint32)
__global__ void k_do_absmax(const __nv_bfloat16* dout, int64_t n8, uint32_t* amax) {
  uint32_t m = 0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n8; i += int64_t(gridDim.x) * blockDim.x) {
    const uint4 u = reinterpret_cast<const uint4*>(dout)[i];
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) m = max(m, max((w[j] << 16) & 0x7fff0000u, w[j] & 0x7fff0000u));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(amax, m);
}
// one thread per 8 consecutive elements (16-byte loads and stores; every count is a multiple of 64)
// Row prologue of the backward, one pass over the query rows: 8 lanes per row (g, p, s) in plan order,
// 8 elements each. Gathers q and dO straight from the caller's order (bf16), writes the fp16 MMA
// operands q16, do16 and the gate-scaled dow[c] = omega_c dO, and reduces <dO, O_c> for the three
// branches (shuffles over the 8 lanes): D_c = omega_c <dO, O_c> and dgates_c = <dO, O_c> (Eq. 6
// backward). Replaces the separate row gathers, the SIMT prologue and the row part of the fp16 prep.
__global__ void k_tc_bwd_rows(Ctx c, __half* q16, __half* do16, __half* dow) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;     // 32-bit: N * H * 8 < 2^31
  const int nrows = c.N * c.H;
  const int row = t >> 3, sub = t & 7;
  const bool valid = row < nrows;
  const int rr = valid ? row : 0;
  const int s = rr % c.h_s, p = (rr / c.h_s) % c.N, g = rr / (c.h_s * c.N);
  const int h = g * c.h_s + s;
  const bool owned = valid && p >= c.row_lo && p < c.row_hi;   // rows of other shards are never touched
  const int src_p = c.sorted_input ? p : c.perm[p];
  const int64_t so = (int64_t(src_p) * c.H + h) * c.Dc + sub * 8, io = int64_t(rr) * kD + sub * 8;
  float fq[8] = {}, fd[8] = {};
  if (owned && sub * 8 < c.Dc) {                 // (Dc = 32: dims 32..63 are the zero padding)
    bf16x8_to_f32(*reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(c.q) + so), fq);
    bf16x8_to_f32(*reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(c.dout) + so), fd);
  }
  const float* w = c.gs + int64_t(rr) * 3;
  const float ds = do_pow2(c.do_amax, false);
  float acc[3];
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    const float4* o = reinterpret_cast<const float4*>(static_cast<const float*>(c.o[b]) + io);
    const float4 x = o[0], y = o[1];
    acc[b] = fd[0] * x.x + fd[1] * x.y + fd[2] * x.z + fd[3] * x.w + fd[4] * y.x + fd[5] * y.y + fd[6] * y.z + fd[7] * y.w;
  }
  if (valid) {   // rows of other shards: zeros (fq = fd = 0), so padded tile tails stay finite
    *reinterpret_cast<uint4*>(q16 + io) = f32x8_to_h(fq, 1.f);
    *reinterpret_cast<uint4*>(do16 + io) = f32x8_to_h(fd, ds);
#pragma unroll
    for (int b = 0; b < 3; ++b)
      *reinterpret_cast<uint4*>(dow + int64_t(b) * nrows * kD + io) = f32x8_to_h(fd, owned ? w[b] * ds : 0.f);
  }
#pragma unroll
  for (int o = 4; o; o >>= 1)
#pragma unroll
    for (int b = 0; b < 3; ++b) acc[b] += __shfl_xor_sync(0xffffffffu, acc[b], o);
  if (!owned || sub != 0) return;
  if (p < c.off[SSA_LEVEL_Q][c.q_begin] || p >= c.off[SSA_LEVEL_Q][c.q_end]) return;   // rows of other shards
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    if (c.dz) c.dz[int64_t(rr) * 3 + b] = acc[b] * w[b] * (1.f - w[b]);   // gate projection backward (R18)
    c.Dd[b][rr] = w[b] * acc[b] * ds;
    __nv_bfloat16* dg = static_cast<__nv_bfloat16*>(c.dgates) + (int64_t(src_p) * c.H + h) * 3 + b;
    *dg = __float2bfloat16_rn(c.accumulate ? acc[b] + __bfloat162float(*dg) : acc[b]);
  }
}

// fp16 copies of the keys (k, v in plan order) and of the pooled keys (fp32 -> fp16), 8 elements per thread
__global__ void k_tc_bwd_prep(Ctx c, __half* k16, __half* v16, __half* kc16, __half* vc16) {
  const int64_t i = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 8;
  const int64_t nk = int64_t(c.h_kv) * c.N * kD;
  const int64_t nc = int64_t(c.h_kv) * c.n_blk[SSA_LEVEL_CMP] * kD;
  float f[8];
  if (i < nk) {
    bf16x8_to_f32(*reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(c.ks) + i), f);
    *reinterpret_cast<uint4*>(k16 + i) = f32x8_to_h(f, 1.f);
    bf16x8_to_f32(*reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(c.vs) + i), f);
    *reinterpret_cast<uint4*>(v16 + i) = f32x8_to_h(f, 1.f);
  }
  if (i < nc) {
    const float4* kc = reinterpret_cast<const float4*>(static_cast<const float*>(c.kc) + i);
    const float4* vc = reinterpret_cast<const float4*>(static_cast<const float*>(c.vc) + i);
    const float4 a0 = kc[0], a1 = kc[1], b0 = vc[0], b1 = vc[1];
    const float fk[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
    const float fv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    *reinterpret_cast<uint4*>(kc16 + i) = f32x8_to_h(fk, 1.f);
    *reinterpret_cast<uint4*>(vc16 + i) = f32x8_to_h(fv, 1.f);
  }
}

// ================================================================================================
// dQ (Q-outer)
// ================================================================================================
// 352 threads: warps 0-3 / 4-7 = warpgroups 0 / 1, each owning one 128-row tile of a row-tile pair
// (thread i <-> TMEM lane i), warp 8 = TMA producer, warps 9 / 10 = MMA issuers of warpgroups 0 / 1
// (warp 9 owns TMEM). Both row tiles share every K/V tile load. TMEM per warpgroup w (256 columns
// at w * 256): S [0, 96) | dP [96, 192) | dQ [192, 256). The warpgroups take turns in their
// exponential loops (named barriers 4 / 5) so each runs at the full MUFU rate.
constexpr int kKT = 96;                  // keys per tile
constexpr int kDqThreads = 352;
constexpr int kMaxKT = 64 + 4 * 64 * 2 + 16;
constexpr int kMaxBlkDq = 4 * 64 + 8;    // >= top_k (tc_plan_ok)
constexpr int kMaxSegDq = kMaxKT + kMaxBlkDq + 8;
constexpr int kKVBytes = kKT * 128;      // one K or V tile (bf16/fp16, 64 wide)
#ifndef SSA_DQ_PINGPONG
#define SSA_DQ_PINGPONG 1
#endif
constexpr bool kDqPingPong = SSA_DQ_PINGPONG;
#ifndef SSA_DQ_DS_TMEM
#define SSA_DQ_DS_TMEM 0
#endif
constexpr bool kDqDsTmem = SSA_DQ_DS_TMEM;   // dS over S in TMEM (TS-form dQ): measured slower (7.7 vs 6.5 ms at C3), off
#ifdef SSA_TRACE
__device__ unsigned long long g_trace_dq[3][128];
__device__ int g_trace_dq_cnt[3];
#define TRACE_ON (blockIdx.x == 5 && blockIdx.y == 0 && (threadIdx.x & 31) == 0)
#define TRACE_R(role, ev, j)                                                                              \
  do {                                                                                                  \
    if (TRACE_ON && tr_n < 128) S->trace[role][tr_n++] = (clock64() << 16) | (unsigned long long)(((ev) << 12) | ((j) & 0xfff)); \
  } while (0)
#else
#define TRACE_R(role, ev, j) do { } while (0)
#endif
struct DqSmem {
  uint64_t q_full, q_empty, kv_full[kStages], kv_empty[kStages], s_full[2], s_empty[2], ds_full[2], ds_empty[2],
      dq_full[2], dq_empty[2];
  uint32_t tmem;
  int n_tiles;
  int tile_row[kMaxKT];                   // compressed-key tiles: first row (one 96-row box)
  uint32_t tile_mask[kMaxKT][3];          // valid keys of the tile
  int tile_seg[kMaxKT + 1];               // selection / window tiles: packed segments [tile_seg[j], tile_seg[j + 1])
  int seg_row[kMaxSegDq];                 // first key row of an 8-row-aligned run of one block's keys
  int seg_dst_len[kMaxSegDq];             // destination slot << 8 | rows
  int blk_a0[kMaxBlkDq], blk_a1[kMaxBlkDq];   // key ranges of the selected blocks
  int8_t tile_br[kMaxKT];
  uint8_t seg_slot[kMaxSegDq];            // selection slot of every segment (0xff: window)
#ifdef SSA_TRACE
  unsigned long long trace[3][128];
#endif
};

// kMask: per-row union-slot masks of small query blocks (pertoken.cu), a separate instantiation
template <bool kMask>
__global__ void __launch_bounds__(kDqThreads, 1)
k_tc_dq(Ctx c, __grid_constant__ const CUtensorMap tmQ, __grid_constant__ const CUtensorMap tmDO,
        __grid_constant__ const CUtensorMap tmKc, __grid_constant__ const CUtensorMap tmVc,
        __grid_constant__ const TmapSet4 tmK, __grid_constant__ const TmapSet4 tmV) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = sm;                       // 2 x 16 KB (row tiles of the pair)
  uint8_t* sDO = sm + 32768;              // 2 x 16 KB
  uint8_t* sKV = sm + 65536;              // kStages x {K, V} (kKVBytes each)
  uint8_t* sDS = sKV + kStages * 2 * kKVBytes;   // 2 x 32 KB: dS K-major, 2 key blocks x [128 rows][128 B]
  DqSmem* S = reinterpret_cast<DqSmem*>(sDS + 65536);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int Q = c.q_order[blockIdx.x], g = blockIdx.y;
  if (Q < c.q_begin || Q >= c.q_end) return;          // not owned by this shard (uniform per CTA)
  const int t0 = c.off[SSA_LEVEL_Q][Q], t1 = c.off[SSA_LEVEL_Q][Q + 1];
  if (t1 <= t0) return;                               // empty virtual query block (uniform per CTA)
  const int rows = (t1 - t0) * c.h_s;
  const int n_rt = (rows + 127) / 128;
  const int n_pair = (n_rt + 1) / 2;
  const int qrow0 = (g * c.N + t0) * c.h_s;

  if (warp == 0) {   // the selected blocks' key ranges, fetched by all lanes at once
    for (int j = lane; j < c.T; j += 32) {
      const int B = c.I[(int64_t(Q) * c.h_kv + g) * c.T + j];
      S->blk_a0[j] = B >= 0 ? c.off[SSA_LEVEL_SLC][B] : 0;
      S->blk_a1[j] = B >= 0 ? c.off[SSA_LEVEL_SLC][B + 1] : 0;
    }
    __syncwarp();
  }
  if (tid == 0) {
    mbar_init(&S->q_full, 1);
    mbar_init(&S->q_empty, 2);                        // one arrival per MMA issuer
    for (int i = 0; i < kStages; ++i) { mbar_init(&S->kv_full[i], 1); mbar_init(&S->kv_empty[i], 2); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&S->s_full[i], 1);
      mbar_init(&S->s_empty[i], 128);
      mbar_init(&S->ds_full[i], 128);
      mbar_init(&S->ds_empty[i], 1);
      mbar_init(&S->dq_full[i], 1);
      mbar_init(&S->dq_empty[i], 128);
    }
    fence_barrier_init();
    // compressed keys: contiguous 96-key tiles; selected blocks: keys packed back to back in 8-row
    // granules (a 96-key tile mixes blocks); window: packed from a fresh tile (tiles never mix branches)
    int n = 0, ns = 0, pos = kKT;
    uint32_t mk[3] = {0u, 0u, 0u};
    const int b = c.q_batch[Q];
    const int c0 = c.bb[SSA_LEVEL_CMP][b], c1 = c.bb[SSA_LEVEL_CMP][b + 1];
    const int ncmp = c.n_blk[SSA_LEVEL_CMP];
    auto set_bits = [&](int lo0, int hi0) {
#pragma unroll
      for (int w = 0; w < 3; ++w) {
        const int lo = max(lo0, 32 * w), hi = min(hi0, 32 * w + 32);
        if (hi > lo) mk[w] |= (hi - lo == 32 ? 0xffffffffu : ((1u << (hi - lo)) - 1u)) << (lo - 32 * w);
      }
    };
    for (int x = c0; x < c1 && n < kMaxKT && !c.win_only && !c.sel_partial; x += kKT) {   // (window-only / per-block pass: no compressed keys)
      mk[0] = mk[1] = mk[2] = 0u;
      set_bits(0, min(kKT, c1 - x));
      S->tile_row[n] = g * ncmp + x;
      S->tile_br[n] = 0;
      S->tile_seg[n] = ns;
      for (int w = 0; w < 3; ++w) S->tile_mask[n][w] = mk[w];
      ++n;
    }
    auto flush = [&]() { for (int w = 0; w < 3; ++w) S->tile_mask[n - 1][w] = mk[w]; };
    auto add_block = [&](int a0, int a1, int br, int slot) {
      const int len = a1 - a0, l8 = (len + 7) & ~7;
      for (int x = 0; x < l8 && n <= kMaxKT;) {
        if (pos == kKT) {
          if (n > 0 && S->tile_br[n - 1] != 0) flush();
          if (n == kMaxKT) { n = kMaxKT + 1; break; }
          S->tile_seg[n] = ns;
          S->tile_br[n] = int8_t(br);
          mk[0] = mk[1] = mk[2] = 0u;
          ++n;
          pos = 0;
        }
        const int take = min(l8 - x, kKT - pos), valid = max(0, min(take, len - x));
        if (ns < kMaxSegDq) {
          S->seg_row[ns] = g * c.N + a0 + x;
          S->seg_dst_len[ns] = (pos << 8) | take;
          S->seg_slot[ns] = uint8_t(slot);
          ++ns;
        }
        set_bits(pos, pos + valid);
        pos += take;
        x += take;
      }
    };
    for (int j = 0; j < c.T; ++j) add_block(S->blk_a0[j], S->blk_a1[j], 1, j);   // (unselected: empty range)
    if (n <= kMaxKT && n > 0 && S->tile_br[n - 1] != 0) flush();
    pos = kKT;                                    // the window starts a fresh tile
    if (!c.no_win) {                              // the window holding the query block (SSA_NO_WINDOW: none)
      const int wb = c.tok_block[SSA_LEVEL_WIN][t0];
      add_block(c.off[SSA_LEVEL_WIN][wb], c.off[SSA_LEVEL_WIN][wb + 1], 2, 0xff);
    }
    if (n <= kMaxKT && n > 0) flush();
    n = min(n, kMaxKT);
    S->tile_seg[n] = ns;
    S->n_tiles = n;
  }
  // zero the K/V stages once: slots a packed tile leaves unfilled must hold finite values (dS = 0 there)
  for (int i = tid; i < kStages * 2 * kKVBytes / 16; i += kDqThreads)
    *reinterpret_cast<uint4*>(sKV + 16 * i) = make_uint4(0u, 0u, 0u, 0u);
  fence_proxy_async_smem();
  if (warp == 8 && lane == 0) {
    tma_prefetch(&tmQ); tma_prefetch(&tmDO); tma_prefetch(&tmKc); tma_prefetch(&tmVc);
    for (int bx = 0; bx < 4; ++bx) { tma_prefetch(&tmK.m[bx]); tma_prefetch(&tmV.m[bx]); }
  }
  if (warp == 9) tmem_alloc<512>(&S->tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S->tmem;
  const int n_tiles = S->n_tiles;
#ifdef SSA_TRACE
  int tr_n = 0;
#endif

  if (warp == 8) {
    // ---------------------------------------------------------------- TMA producer
    Ring kv(kStages);
    uint32_t qph = 0;
    for (int pr = 0; pr < n_pair; ++pr) {
      const bool duo = 2 * pr + 1 < n_rt;
      mbar_wait(&S->q_empty, qph ^ 1u);
      qph ^= 1u;
      if (lane == 0) {
        mbar_expect_tx(&S->q_full, duo ? 65536u : 32768u);
        for (int w = 0; w < (duo ? 2 : 1); ++w) {
          tma_load_2d(sQ + w * 16384, &tmQ, &S->q_full, 0, qrow0 + (2 * pr + w) * 128);
          tma_load_2d(sDO + w * 16384, &tmDO, &S->q_full, 0, qrow0 + (2 * pr + w) * 128);
        }
      }
      for (int j = 0; j < n_tiles; ++j) {
        mbar_wait(&S->kv_empty[kv.idx], kv.ph ^ 1u);
        TRACE_R(0, 1, j);
        if (lane == 0) {
          uint8_t* st = sKV + kv.idx * 2 * kKVBytes;
          if (S->tile_br[j] == 0) {
            mbar_expect_tx(&S->kv_full[kv.idx], 2u * kKVBytes);
            tma_load_2d(st, &tmKc, &S->kv_full[kv.idx], 0, S->tile_row[j]);
            tma_load_2d(st + kKVBytes, &tmVc, &S->kv_full[kv.idx], 0, S->tile_row[j]);
          } else {
            const int s0 = S->tile_seg[j], s1 = S->tile_seg[j + 1];
            uint32_t rows_in = 0;
            for (int q = s0; q < s1; ++q) rows_in += uint32_t(S->seg_dst_len[q] & 0xff);
            mbar_expect_tx(&S->kv_full[kv.idx], rows_in * 256u);
            for (int q = s0; q < s1; ++q) {
              const int dst = S->seg_dst_len[q] >> 8, len = S->seg_dst_len[q] & 0xff, src = S->seg_row[q];
              for (int off = 0; off < len;) {   // boxes of 64 / 32 / 16 / 8 rows
                const int bx = len - off >= 64 ? 0 : (len - off >= 32 ? 1 : (len - off >= 16 ? 2 : 3));
                tma_load_2d(st + (dst + off) * 128, &tmK.m[bx], &S->kv_full[kv.idx], 0, src + off);
                tma_load_2d(st + kKVBytes + (dst + off) * 128, &tmV.m[bx], &S->kv_full[kv.idx], 0, src + off);
                off += 64 >> bx;
              }
            }
          }
        }
        __syncwarp();
        kv.next();
      }
    }
  } else if (warp >= 9) {
    // ---------------------------------------------------------------- MMA issuer of warpgroup w
    const int w = warp - 9;
    const uint32_t idS = idesc_f16(128, kKT, false, false);    // S = Q K^T, dP = dO V^T
    const uint32_t idQ = idesc_f16(128, 64, false, true);      // dQ += dS K (K as MN-major B)
    const uint32_t aQ = smem_u32(sQ + w * 16384), aDO = smem_u32(sDO + w * 16384);
    const uint32_t tS = tmem + w * 256, tQ = tS + 192;
    Ring kv(kStages), sb(1), db(1);
    uint32_t qph = 0, dqph = 0;
    for (int pr = 0; pr < n_pair; ++pr) {
      const bool mine = w == 0 || 2 * pr + 1 < n_rt;
      mbar_wait(&S->q_full, qph);
      qph ^= 1u;
      tc_fence_after();
      if (lane == 0) {
        if (!mine) {
          for (int j = 0; j < n_tiles; ++j) {   // keep the shared K/V ring moving
            mbar_wait(&S->kv_full[kv.idx], kv.ph);
            mbar_arrive(&S->kv_empty[kv.idx]);
            kv.next();
          }
          mbar_arrive(&S->q_empty);
        } else {
          Ring kv_q = kv;
          auto issue_s = [&]() {
            mbar_wait(&S->kv_full[kv.idx], kv.ph);
            if (!kDqDsTmem) mbar_wait(&S->s_empty[w], sb.ph ^ 1u);   // (TMEM dS: ordered after dQ instead)
            tc_fence_after();
            const uint32_t sk = smem_u32(sKV + kv.idx * 2 * kKVBytes);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_bf16(tS, desc_sw128(aQ + k * 32, 0, 1024), desc_sw128(sk + k * 32, 0, 1024), idS, k > 0);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_bf16(tS + kKT, desc_sw128(aDO + k * 32, 0, 1024), desc_sw128(sk + kKVBytes + k * 32, 0, 1024), idS,
                        k > 0);
            umma_commit(&S->s_full[w]);
            kv.next();
            sb.next();
          };
          issue_s();
          mbar_wait(&S->dq_empty[w], dqph ^ 1u);
          dqph ^= 1u;
          for (int j = 0; j < n_tiles; ++j) {
            if (!kDqDsTmem && j + 1 < n_tiles) issue_s();
            if (w == 0) TRACE_R(1, 3, j + 1);
            mbar_wait(&S->ds_full[w], db.ph);
            tc_fence_after();
            const uint32_t sk = smem_u32(sKV + kv_q.idx * 2 * kKVBytes);
            if (kDqDsTmem) {
              // dS (fp16, two keys per column) sits over S in TMEM: A from TMEM
#pragma unroll
              for (int k = 0; k < kKT / 16; ++k)
                umma_ts(tQ, tS + k * 8, desc_sw128(sk + k * 2048, 0, 1024), idQ, (j > 0 || k > 0) ? 1u : 0u);
            } else {
              const uint32_t ads = smem_u32(sDS + w * 32768);
#pragma unroll
              for (int k = 0; k < kKT / 16; ++k)
                umma_bf16(tQ, desc_sw128(ads + (k >> 2) * 16384 + (k & 3) * 32, 0, 1024),
                          desc_sw128(sk + k * 2048, 0, 1024), idQ, (j > 0 || k > 0) ? 1u : 0u);
            }
            umma_commit(&S->ds_empty[w]);
            umma_commit(&S->kv_empty[kv_q.idx]);
            if (w == 0) TRACE_R(1, 5, j);
            kv_q.next();
            db.next();
            // (TMEM dS) S(j+1) overwrites dS(j): issued after dQ(j) by the same thread, in pipe order
            if (kDqDsTmem && j + 1 < n_tiles) issue_s();
          }
          umma_commit(&S->dq_full[w]);
          umma_commit(&S->q_empty);
        }
      }
      __syncwarp();   // lanes 1-31 only track q_full; the ring cursors live in lane 0
    }
  } else {
    // ---------------------------------------------------------------- softmax / dS warpgroup wg
    const int wg = warp >> 2, t = tid & 127;
    const uint32_t lrow = uint32_t((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + lrow + wg * 256, tQ = tS + 192;
    const float cl2 = c.scale * kLog2e;
    Ring sb(1), db(1);
    uint32_t dqph = 0;
    if (kDqPingPong && wg == 1 && n_rt >= 2) named_bar_arrive(4, 256);   // warpgroup 0 takes the first turn
    for (int pr = 0; pr < n_pair; ++pr) {
      const int rt = 2 * pr + wg;
      if (rt >= n_rt) break;                          // warpgroup 1 sits out the last, odd pair
      const bool duo = 2 * pr + 1 < n_rt;
      const int r = rt * 128 + t;
      const bool rvalid = r < rows;
      const int64_t row = qrow0 + (rvalid ? r : 0);
      float lse2[3], wgt[3], Dv[3];
#pragma unroll
      for (int br = 0; br < 3; ++br) {
        lse2[br] = rvalid ? c.lse[br][row] : INFINITY;
        wgt[br] = c.gs[row * 3 + br];
        Dv[br] = c.Dd[br][row];
      }
      // small query blocks (virtual level): the selection slots this row's query block selected
      const int64_t mi = (int64_t(t0 + (rvalid ? r : 0) / c.h_s) * c.h_kv + g) * 2;
      const unsigned long long rm0 = (kMask && rvalid) ? c.umask[mi] : ~0ull, rm1 = (kMask && rvalid) ? c.umask[mi + 1] : ~0ull;
      for (int j = 0; j < n_tiles; ++j) {
        const int br = S->tile_br[j];
        const uint32_t mk0 = S->tile_mask[j][0], mk1 = S->tile_mask[j][1], mk2 = S->tile_mask[j][2];
        const bool full = (mk0 & mk1 & mk2) == 0xffffffffu;
        const float l2 = br == 0 ? lse2[0] : (br == 1 ? lse2[1] : lse2[2]);
        const float wb = br == 0 ? wgt[0] : (br == 1 ? wgt[1] : wgt[2]);
        const float Db = br == 0 ? Dv[0] : (br == 1 ? Dv[1] : Dv[2]);
        uint32_t umk = 0u;                             // virtual level: granules this row must not see
        if (kMask && br == 1)
          for (int q = S->tile_seg[j]; q < S->tile_seg[j + 1]; ++q) {
            const uint32_t slot = S->seg_slot[q];
            if (slot < 128u && !(((slot < 64u ? rm0 : rm1) >> (slot & 63u)) & 1ull)) {
              const int dst = S->seg_dst_len[q] >> 8, len = S->seg_dst_len[q] & 0xff;
              umk |= ((1u << (len / 8)) - 1u) << (dst / 8);
            }
          }
        mbar_wait(&S->s_full[wg], sb.ph);
        if (warp == 0) TRACE_R(2, 7, j);
        tc_fence_after();
        uint32_t pk[kKT / 2];
        if (kDqPingPong && duo) named_bar_sync(4 + wg, 256);
        if (warp == 0) TRACE_R(2, 8, j);
#pragma unroll
        for (int c0 = 0; c0 < kKT; c0 += 32) {
          float s[32], dp[32];
          tmem_ld32(tS + c0, s);
          tmem_ld32(tS + kKT + c0, dp);
          tmem_wait_ld();
          if (!kDqDsTmem && c0 + 32 == kKT) {
            tc_fence_before();
            mbar_arrive(&S->s_empty[wg]);
          }
          if (!full) {                               // unfilled slots / granule padding: p = 0
            const uint32_t mw = c0 == 0 ? mk0 : (c0 == 32 ? mk1 : mk2);
#pragma unroll
            for (int gr = 0; gr < 4; ++gr) {
              const uint32_t bits = (mw >> (8 * gr)) & 0xffu;
              if (bits != 0xffu) {
#pragma unroll
                for (int i = 0; i < 8; ++i) s[8 * gr + i] = (bits >> i) & 1u ? s[8 * gr + i] : -INFINITY;
              }
            }
          }
          if (kMask && umk) {                        // granules of blocks this row's query block did not select
#pragma unroll
            for (int gr = 0; gr < 4; ++gr)
              if ((umk >> (c0 / 8 + gr)) & 1u) {
#pragma unroll
                for (int i = 0; i < 8; ++i) s[8 * gr + i] = -INFINITY;
              }
          }
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const float p0 = ex2(fmaf(s[i], cl2, -l2)), p1 = ex2(fmaf(s[i + 1], cl2, -l2));
            pk[(c0 + i) / 2] = pack_f16(p0 * fmaf(wb, dp[i], -Db), p1 * fmaf(wb, dp[i + 1], -Db));
          }
          // (TMEM dS) columns [c0/2, c0/2 + 16) hold keys c0..c0+31; S columns below c0 + 32 are read
          if (kDqDsTmem) tmem_st16(tS + c0 / 2, pk + c0 / 2);
        }
        if (kDqPingPong && duo) named_bar_arrive(5 - wg, 256);
        if (warp == 0) TRACE_R(2, 9, j);
        sb.next();
        if (kDqDsTmem) {
          tmem_wait_st();
          tc_fence_before();
        } else {
          mbar_wait(&S->ds_empty[wg], db.ph ^ 1u);
          if (warp == 0) TRACE_R(2, 10, j);
          const uint32_t base = smem_u32(sDS + wg * 32768);
#pragma unroll
          for (int ch = 0; ch < kKT / 8; ++ch)
            st_shared_v4(base + (ch >> 3) * 16384 + sw128(t, ch & 7), pk[4 * ch], pk[4 * ch + 1], pk[4 * ch + 2],
                         pk[4 * ch + 3]);
          fence_proxy_async_smem();
        }
        mbar_arrive(&S->ds_full[wg]);
        if (warp == 0) TRACE_R(2, 11, j);
        db.next();
      }
      mbar_wait(&S->dq_full[wg], dqph);
      dqph ^= 1u;
      tc_fence_after();
      float v[64];
      tmem_ld32(tQ, v);
      tmem_ld32(tQ + 32, v + 32);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&S->dq_empty[wg]);
      if (rvalid && c.sel_partial) {   // per-block selection pass: fp32 partial of this (token, block) row
        const float osc = c.scale * do_pow2(c.do_amax, true);
        float* o = c.dq_part + (int64_t(qrow0) + r) * kD;
#pragma unroll
        for (int e = 0; e < kD; e += 4)
          *reinterpret_cast<float4*>(o + e) = make_float4(v[e] * osc, v[e + 1] * osc, v[e + 2] * osc, v[e + 3] * osc);
      } else if (rvalid) {
        const float osc = c.scale * do_pow2(c.do_amax, true);
        const int tok = t0 + r / c.h_s, hs = r % c.h_s;
        const float* xtra = c.dq_extra ? c.dq_extra + (int64_t(qrow0) + r) * kD : nullptr;
        const int dst = c.sorted_input ? tok : c.perm[tok];
        __nv_bfloat16* o = static_cast<__nv_bfloat16*>(c.dq) + (int64_t(dst) * c.H + g * c.h_s + hs) * c.Dc;
#pragma unroll
        for (int e = 0; e < kD; e += 8) {
          if (e >= c.Dc) break;                  // zero-padded head dims are not output
          float y[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) y[u] = v[e + u] * osc + (xtra ? xtra[e + u] : 0.f);
          if (c.accumulate) {   // SSA_ACCUMULATE: add to the caller's dq
            const uint4 old = *reinterpret_cast<const uint4*>(o + e);
            const uint32_t ow[4] = {old.x, old.y, old.z, old.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const float2 f = unpack_bf16(ow[u]);
              y[2 * u] += f.x;
              y[2 * u + 1] += f.y;
            }
          }
          *reinterpret_cast<uint4*>(o + e) = make_uint4(pack_bf16(y[0], y[1]), pack_bf16(y[2], y[3]),
                                                        pack_bf16(y[4], y[5]), pack_bf16(y[6], y[7]));
        }
      }
    }
  }
#ifdef SSA_TRACE
  if (TRACE_ON && (warp == 8 || warp == 9 || warp == 0)) {
    const int role = warp == 8 ? 0 : (warp == 9 ? 1 : 2);
    for (int i = 0; i < tr_n; ++i) g_trace_dq[role][i] = S->trace[role][i];
    g_trace_dq_cnt[role] = tr_n;
  }
#endif
  tc_fence_before();
  __syncthreads();
  if (warp == 9) tmem_dealloc<512>(tmem);
}
#undef TRACE_R
#undef TRACE_ON

// ================================================================================================
// dK / dV (KV-outer)
// ================================================================================================
constexpr int kRT = 64;                  // rows per tile: S^T 64 + dP^T 64 + dK 64 + dV 64 = 256 TMEM cols
#ifndef SSA_KV_RSTAGES
#define SSA_KV_RSTAGES 3
#endif
constexpr int kRStages = SSA_KV_RSTAGES;   // row-tile (Q, dO, stats) pipeline depth per warpgroup
#ifndef SSA_KV_PBUF
#define SSA_KV_PBUF 1
#endif
// (P w)^T / dS^T shared-memory buffers per warpgroup. Measured at C3: 2 buffers only fit
// with 2 row stages, and 3 row stages / 1 buffer (3.18 + 6.29 ms) beat 2 / 2 (3.88 + 7.02) and 2 / 1
// (4.15 + 7.62): the row-tile loads need the third stage more than the stores need a second buffer.
constexpr int kPBuf = SSA_KV_PBUF;
#ifndef SSA_KV_QB_PER_ITEM
#define SSA_KV_QB_PER_ITEM 8
#endif
constexpr int kQBlocksPerItem = SSA_KV_QB_PER_ITEM;       // raw keys: query blocks per work item (splits popular blocks)
#ifndef SSA_BWD_FORK
#define SSA_BWD_FORK 1
#endif
constexpr bool kBwdFork = SSA_BWD_FORK;   // dQ and the KV-outer launches on two streams (see tc_backward)
#ifndef SSA_KV_STATS_WAIT
#define SSA_KV_STATS_WAIT 0       // 1: cp.async + wait_all + plain arrive (synccheck unchanged, 0.8 ms slower at C3)
#endif
// One CTA per SM, 352 threads: warpgroups 0 / 1 (warps 0-3 / 4-7, thread = key = TMEM lane) split the
// row tiles of the item (even / odd), each with its own 256 TMEM columns (S^T 64 | dP^T 64 | dK 64 |
// dV 64), its own row-stage ring and its own MMA issuer (warps 9 / 10); warp 8 is the producer. The
// warpgroups share the K/V tile and take turns in their exponential loops (named barriers 4 / 5).
constexpr int kKvThreads = 352;
#ifndef SSA_KV_PINGPONG
#define SSA_KV_PINGPONG 0
#endif
constexpr bool kKvPingPong = SSA_KV_PINGPONG;
struct KvSmem {
  uint64_t k_full, k_empty, r_full[2][kRStages], r_empty[2][kRStages], s_full[2], s_empty[2], p_full[2][kPBuf],
      p_empty[2][kPBuf], pv_empty[2][kPBuf], acc_full[2], acc_empty[2];
  uint32_t tmem;
  alignas(16) float st_l2[2][kRStages][kRT];
  alignas(16) float st_D[2][kRStages][kRT];
#ifdef SSA_TRACE
  unsigned long long trace[3][128];
#endif
};
#ifdef SSA_TRACE
__device__ unsigned long long g_trace_kv[3][128];
__device__ int g_trace_kv_cnt[3];
#define TRACE_ON (blockIdx.x == 5 && blockIdx.y == 0 && blockIdx.z == 0 && (threadIdx.x & 31) == 0)
#define TRACE_R(role, ev, j)                                                                              \
  do {                                                                                                  \
    if (TRACE_ON && tr_n < 128) S->trace[role][tr_n++] = (clock64() << 16) | (unsigned long long)(((ev) << 12) | ((j) & 0xfff)); \
  } while (0)
#else
#define TRACE_R(role, ev, j) do { } while (0)
#endif

// Work item -> (key block, g, query-block range, window?) and the row-tile walker shared by the roles.
struct Item {
  int mode, g, kblock, b, chunk, li, le, with_win, part_slot, first;
  int64_t ra, re;       // mode 0 row range
};

__device__ __forceinline__ bool make_item(const Ctx& c, int mode, int id, Item* it) {
  it->mode = mode;
  if (mode == 0) {
    const int tile = blockIdx.x;
    it->g = blockIdx.y;
    it->b = c.cmp_tiles[2 * tile];
    it->kblock = c.cmp_tiles[2 * tile + 1];
    it->chunk = blockIdx.z;
    const int bt0 = max(c.batch_tokens[it->b], c.off[SSA_LEVEL_Q][c.q_begin]);
    const int bt1 = max(bt0, min(c.batch_tokens[it->b + 1], c.off[SSA_LEVEL_Q][c.q_end]));   // owned rows
    const int64_t rows = int64_t(bt1 - bt0) * c.h_s;
    const int64_t per = ((rows + c.n_chunk - 1) / c.n_chunk + kRT - 1) / kRT * kRT;
    const int64_t base = (int64_t(it->g) * c.N + bt0) * c.h_s;
    it->ra = base + min(rows, per * it->chunk);
    it->re = base + min(rows, per * (it->chunk + 1));
    it->li = it->le = 0;
    it->with_win = 0;
    it->first = 1;
    return true;
  }
  const int nkeys = c.n_blk[SSA_LEVEL_SLC] * c.h_kv;
  if (id >= c.kv_item_off[nkeys]) return false;
  int lo = 0, hi = nkeys;                 // largest key with item_off[key] <= id
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (c.kv_item_off[mid] <= id) lo = mid; else hi = mid;
  }
  const int key = lo;
  const int nch = c.kv_item_off[key + 1] - c.kv_item_off[key];
  it->chunk = id - c.kv_item_off[key];
  it->kblock = key / c.h_kv;
  it->g = key % c.h_kv;
  const int l0 = c.inv_off[key], l1 = c.inv_off[key + 1];
  it->li = min(l1, l0 + it->chunk * c.qb_per_item);
  it->le = min(l1, it->li + c.qb_per_item);
  it->with_win = !c.no_win && it->chunk == nch - 1 && it->kblock >= c.q_begin && it->kblock < c.q_end;  // window = block
  it->first = it->chunk == 0;
  it->part_slot = id;
  it->ra = it->re = 0;
  return true;
}

struct RowWalk {
  Item it;
  int li;
  int64_t cur, end;
  int br;
  int win_done;
  const Ctx* c;
  __device__ void init(const Ctx& cc, const Item& i) {
    c = &cc;
    it = i;
    li = i.li;
    win_done = !i.with_win;
    if (i.mode == 0) { cur = i.ra; end = i.re; br = 0; } else { cur = end = 0; br = 1; }
  }
  __device__ bool next_range() {
    if (it.mode == 0) return false;
    if (li < it.le) {
      int Qb = c->inv_list[li++];
      cur = (int64_t(it.g) * c->N + c->off[SSA_LEVEL_Q][Qb]) * c->h_s;
      // consecutive query blocks in the (ascending) list are contiguous rows: one range, so 64-row
      // tiles are not cut at every query block (small query blocks, e.g. per-token selection)
      while (li < it.le && c->inv_list[li] == Qb + 1) Qb = c->inv_list[li++];
      end = (int64_t(it.g) * c->N + c->off[SSA_LEVEL_Q][Qb + 1]) * c->h_s;
      br = 1;
      return true;
    }
    if (!win_done) {   // the window is the key block itself (m_win == m_slc)
      win_done = 1;
      cur = (int64_t(it.g) * c->N + c->off[SSA_LEVEL_SLC][it.kblock]) * c->h_s;
      end = (int64_t(it.g) * c->N + c->off[SSA_LEVEL_SLC][it.kblock + 1]) * c->h_s;
      br = 2;
      return true;
    }
    return false;
  }
  __device__ bool next_tile(int64_t* r0, int* nr, int* b) {
    while (cur >= end) {
      if (!next_range()) return false;
    }
    *r0 = cur;
    *nr = int((end - cur) < kRT ? (end - cur) : int64_t(kRT));
    *b = br;
    cur += kRT;
    return true;
  }
};

// Packed row tiles of the raw-key work items. The rows of an item (the rows of each selecting query block
// in list order, then the window's rows from a fresh tile) are laid back to back in 64-row tiles at 8-row
// granularity: a query block of n rows takes ceil(n / 8) granules and may continue in the next tile, so
// a tile mixes query blocks (short ones, e.g. one token of h_s rows at m_q = 1, would otherwise leave a
// tile mostly empty). Every granule is a slot of 8 rows at an 8-row (1024-B) aligned position, so a TMA
// box of 8k rows there lands in the 128-B swizzle pattern of one 64-row box. A pre-pass (one warp per
// item, the query blocks' slot offsets by a warp scan) writes, per tile and granule, int2 {first row,
// meta}: meta bits 0-3 = valid rows (slots past them get an LSE of +inf: p = 0), bits 4-5 = branch
// (1 selection, 2 window), bits 8-10 = TMA box starting at this granule (0 none, 1..4 = 64/32/16/8 rows).
constexpr int kGranMetaBoxShift = 8;
__device__ __forceinline__ int qb_rows(const Ctx& c, int Qb) {
  return (c.off[SSA_LEVEL_Q][Qb + 1] - c.off[SSA_LEVEL_Q][Qb]) * c.h_s;
}
__device__ __forceinline__ int64_t round8(int64_t x) { return (x + 7) & ~int64_t(7); }
// slots of the item's selection part and of the whole item (window from a fresh tile)
__device__ __forceinline__ void item_slots(const Ctx& c, const Item& it, int lane, int64_t* sel, int64_t* total) {
  int64_t s = 0;
  for (int i = it.li + lane; i < it.le; i += 32) s += round8(qb_rows(c, c.inv_list[i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  *sel = s;
  *total = s;
  if (it.with_win) {
    const int64_t w = int64_t(c.off[SSA_LEVEL_SLC][it.kblock + 1] - c.off[SSA_LEVEL_SLC][it.kblock]) * c.h_s;
    *total = (s + kRT - 1) / kRT * kRT + round8(w);
  }
}
__global__ void k_kv_tile_count(Ctx c, int32_t* __restrict__ cnt, int bound) {
  const int id = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (id >= bound) return;   // warp-uniform
  Item it;
  if (!make_item(c, 1, id, &it)) {
    if (lane == 0) cnt[id] = 0;
    return;
  }
  int64_t sel, total;
  item_slots(c, it, lane, &sel, &total);
  if (lane == 0) cnt[id] = int32_t((total + kRT - 1) / kRT);
}
// granules of one piece: rows [row0, row0 + rows) at item slot s0 (a multiple of 8), boxes cut at tiles
__device__ void write_piece(int2* __restrict__ desc, int64_t t0, int64_t s0, int64_t row0, int rows, int br) {
  const int l8 = int(round8(rows));
  for (int r = 0; r < l8;) {
    const int64_t s = s0 + r;
    const int in_tile = min(l8 - r, kRT - int(s % kRT));
    int2* dt = desc + (t0 + s / kRT) * 8 + (s % kRT) / 8;
    for (int o = 0; o < in_tile;) {
      const int b = in_tile - o >= 64 ? 0 : (in_tile - o >= 32 ? 1 : (in_tile - o >= 16 ? 2 : 3));
      for (int k = 0; k < (8 >> b); ++k) {
        const int rr = r + o + 8 * k, nv = rows - rr < 8 ? rows - rr : 8;
        dt[o / 8 + k] = make_int2(int(row0 + rr), nv | (br << 4) | (k == 0 ? (b + 1) << kGranMetaBoxShift : 0));
      }
      o += 64 >> b;
    }
    r += in_tile;
  }
}
__global__ void k_kv_tile_fill(Ctx c, const int32_t* __restrict__ off, int2* __restrict__ desc, int bound) {
  const int id = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (id >= bound) return;   // warp-uniform
  Item it;
  if (!make_item(c, 1, id, &it)) return;
  const int64_t t0 = off[id];
  int64_t sel, total;
  item_slots(c, it, lane, &sel, &total);
  int64_t base = 0;
  for (int i0 = it.li; i0 < it.le; i0 += 32) {   // selecting query blocks, list order
    const int i = i0 + lane;
    const int Qb = i < it.le ? c.inv_list[i] : 0;
    const int rows = i < it.le ? qb_rows(c, Qb) : 0;
    int64_t x = round8(rows);                      // inclusive warp scan of the slots
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (rows > 0)
      write_piece(desc, t0, base + x - round8(rows), (int64_t(it.g) * c.N + c.off[SSA_LEVEL_Q][Qb]) * c.h_s, rows, 1);
    base += __shfl_sync(0xffffffffu, x, 31);
  }
  int64_t pad0 = sel, pad1 = (sel + kRT - 1) / kRT * kRT;   // unused granules: selection tail, item tail
  if (it.with_win) {
    const int t_a = c.off[SSA_LEVEL_SLC][it.kblock], t_b = c.off[SSA_LEVEL_SLC][it.kblock + 1];
    if (lane == 0) write_piece(desc, t0, pad1, (int64_t(it.g) * c.N + t_a) * c.h_s, (t_b - t_a) * c.h_s, 2);
  }
  for (int64_t s = pad0 + 8 * lane; s < pad1; s += 256) desc[(t0 + s / kRT) * 8 + (s % kRT) / 8] = make_int2(0, 0);
  const int64_t tend = (total + kRT - 1) / kRT * kRT;
  for (int64_t s = round8(total) + 8 * lane; s < tend && total > pad1; s += 256)
    desc[(t0 + s / kRT) * 8 + (s % kRT) / 8] = make_int2(0, 0);
}

__global__ void __launch_bounds__(kKvThreads, 1)
k_tc_dkdv(Ctx c, int mode, __grid_constant__ const TmapSet4 tmQ, __grid_constant__ const TmapSet4 tmDO,
          __grid_constant__ const TmapSet4 tmDO2, __grid_constant__ const CUtensorMap tmK,
          __grid_constant__ const CUtensorMap tmV) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = sm;                       // 16 KB
  uint8_t* sV = sm + 16384;               // 16 KB
  uint8_t* sR = sm + 32768;               // [warpgroup][kRStages] x {Q 8 KB, (w) dO 8 KB}
  uint8_t* sP = sR + 2 * kRStages * 16384;  // [warpgroup][kPBuf] x {(P w)^T 16 KB, dS^T 16 KB}, K-major [128 keys][64 rows]
  KvSmem* S = reinterpret_cast<KvSmem*>(sP + 2 * kPBuf * 32768);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  Item it;
  const bool ok = make_item(c, mode, blockIdx.x, &it);
  if (!ok) return;                        // uniform for the whole CTA (grid is an upper bound)
  const int g = it.g;
  int kbase, nkeys_total;
  int64_t krow_g;
  if (mode == 0) {
    kbase = it.kblock;
    nkeys_total = min(128, c.bb[SSA_LEVEL_CMP][it.b + 1] - kbase);
    krow_g = int64_t(g) * c.n_blk[SSA_LEVEL_CMP];
  } else {
    kbase = c.off[SSA_LEVEL_SLC][it.kblock];
    nkeys_total = c.off[SSA_LEVEL_SLC][it.kblock + 1] - kbase;
    krow_g = int64_t(g) * c.N;
  }
  const int n_kt = (nkeys_total + 127) / 128;
  int n_tiles = 0;                        // row tiles of the item (the same for every key tile)
  const bool packed = mode == 1 && c.kv_desc != nullptr;   // raw keys, short query blocks: packed row tiles
  int64_t tile0 = 0;
  if (packed) {
    tile0 = c.kv_tile_off[blockIdx.x];
    n_tiles = int(c.kv_tile_off[blockIdx.x + 1] - tile0);
  } else {
    RowWalk w2;
    w2.init(c, it);
    int64_t r0;
    int nr, br;
    while (w2.next_tile(&r0, &nr, &br)) ++n_tiles;
  }
  const int n_own0 = (n_tiles + 1) / 2;   // warpgroup 0 takes row tiles 0, 2, 4 ..., warpgroup 1 1, 3, 5 ...

  if (tid == 0) {
    mbar_init(&S->k_full, 1);
    mbar_init(&S->k_empty, 2);            // one arrival per MMA issuer
    for (int w = 0; w < 2; ++w) {
      // r_full: 32 producer lanes' cp.async arrivals (row stats) + lane 0's expect_tx (Q/dO TMA)
      for (int i = 0; i < kRStages; ++i) { mbar_init(&S->r_full[w][i], 33); mbar_init(&S->r_empty[w][i], 1); }
      mbar_init(&S->s_full[w], 1);
      mbar_init(&S->s_empty[w], 128);
      for (int b = 0; b < kPBuf; ++b) {
        mbar_init(&S->p_full[w][b], 128);
        mbar_init(&S->p_empty[w][b], 1);    // dK MMAs done: dS^T may be rewritten
        mbar_init(&S->pv_empty[w][b], 1);   // dV MMAs done: (P w)^T may be rewritten
      }
      mbar_init(&S->acc_full[w], 1);
      mbar_init(&S->acc_empty[w], 256);   // both warpgroups read both accumulator sets
    }
    fence_barrier_init();
  }
  // packed row tiles may leave slots unwritten: the row stages must hold finite values from the start
  if (packed) {
    for (int i = tid; i < 2 * kRStages * 16384 / 16; i += kKvThreads)
      *reinterpret_cast<uint4*>(sR + 16 * i) = make_uint4(0u, 0u, 0u, 0u);
    fence_proxy_async_smem();
  }
  if (warp == 8 && lane == 0) {
    for (int b = 0; b < 4; ++b) { tma_prefetch(&tmQ.m[b]); tma_prefetch(&tmDO.m[b]); tma_prefetch(&tmDO2.m[b]); }
    tma_prefetch(&tmK); tma_prefetch(&tmV);
  }
  if (warp == 9) tmem_alloc<512>(&S->tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S->tmem;
#ifdef SSA_TRACE
  int tr_n = 0;
#endif

  if (warp == 8) {
    // ------------------------------------------------ producer: K/V tile, then row tiles + row stats
    Ring rs0(kRStages), rs1(kRStages);
    uint32_t kph = 0;
    for (int kt = 0; kt < n_kt; ++kt) {
      mbar_wait(&S->k_empty, kph ^ 1u);
      kph ^= 1u;
      if (lane == 0) {
        mbar_expect_tx(&S->k_full, 32768);
        tma_load_2d(sK, &tmK, &S->k_full, 0, int(krow_g + kbase + kt * 128));
        tma_load_2d(sV, &tmV, &S->k_full, 0, int(krow_g + kbase + kt * 128));
      }
      if (packed) {
        // lane j < 8 holds granule j of the tile; the next tile's descriptor is loaded one tile ahead
        int2 nxt = lane < 8 && n_tiles > 0 ? c.kv_desc[tile0 * 8 + lane] : make_int2(0, 0);
        for (int i = 0; i < n_tiles; ++i) {
          const int w = i & 1;
          Ring& rs = w ? rs1 : rs0;
          const int2 cd = nxt;
          if (lane < 8 && i + 1 < n_tiles) nxt = c.kv_desc[(tile0 + i + 1) * 8 + lane];
          mbar_wait(&S->r_empty[w][rs.idx], rs.ph ^ 1u);
          TRACE_R(0, 1, i);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int e = lane + 32 * h;
            const int gx = __shfl_sync(0xffffffffu, cd.x, e >> 3), gy = __shfl_sync(0xffffffffu, cd.y, e >> 3);
            const int nv = gy & 15, br = (gy >> 4) & 3;
            const int64_t row = int64_t(gx) + (e & 7);
            const bool valid = (e & 7) < nv;
            bool keep = valid;
            if (keep && br == 1 && c.umask) {   // virtual level: rows whose query block did not select the block
              const int tok = int(row / c.h_s) - it.g * c.N;
              const int32_t* sel = c.tok_I + (int64_t(c.tok_qb[tok]) * c.h_kv + it.g) * c.tok_T;
              bool hit = false;
              for (int jj = 0; jj < c.tok_T; ++jj) hit |= sel[jj] == it.kblock;
              keep = hit;
            }
            cp_async4(&S->st_l2[w][rs.idx][e], keep ? c.lse[br] + row : &g_pos_inf);
            cp_async4(&S->st_D[w][rs.idx][e], valid ? c.Dd[br] + row : &g_zero);
          }
#if SSA_KV_STATS_WAIT
          asm volatile("cp.async.wait_all;\n" ::: "memory");
          mbar_arrive(&S->r_full[w][rs.idx]);
#else
          cp_async_mbar_arrive_noinc(&S->r_full[w][rs.idx]);
#endif
          int2 gd[8];
#pragma unroll
          for (int gq = 0; gq < 8; ++gq) gd[gq] = make_int2(__shfl_sync(0xffffffffu, cd.x, gq), __shfl_sync(0xffffffffu, cd.y, gq));
          if (lane == 0) {
            uint8_t* st = sR + (w * kRStages + rs.idx) * 16384;
            uint32_t rows = 0;
#pragma unroll
            for (int gq = 0; gq < 8; ++gq) {
              const int bc = (gd[gq].y >> kGranMetaBoxShift) & 7;
              rows += bc ? (64u >> (bc - 1)) : 0u;
            }
            mbar_expect_tx(&S->r_full[w][rs.idx], rows * 256u);
#pragma unroll
            for (int gq = 0; gq < 8; ++gq) {
              const int bc = (gd[gq].y >> kGranMetaBoxShift) & 7;
              if (bc) {
                const TmapSet4& td = ((gd[gq].y >> 4) & 3) == 2 ? tmDO2 : tmDO;
                tma_load_2d(st + gq * 1024, &tmQ.m[bc - 1], &S->r_full[w][rs.idx], 0, gd[gq].x);
                tma_load_2d(st + 8192 + gq * 1024, &td.m[bc - 1], &S->r_full[w][rs.idx], 0, gd[gq].x);
              }
            }
          }
          __syncwarp();
          rs.next();
        }
        continue;
      }
      RowWalk wk;
      wk.init(c, it);
      int64_t r0;
      int nr, br;
      int i = 0;
      while (wk.next_tile(&r0, &nr, &br)) {
        const int w = i & 1;
        Ring& rs = w ? rs1 : rs0;
        mbar_wait(&S->r_empty[w][rs.idx], rs.ph ^ 1u);
        TRACE_R(0, 1, i);
        // row stats by cp.async (completion tracked by r_full); rows past the range read lse = +inf,
        // D = 0 -> p = 0 without per-element masking
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int e = lane + 32 * h;
          const int64_t row = r0 + e;
          bool keep = e < nr;
          if (keep && br == 1 && c.umask) {   // virtual level: rows whose query block did not select the key block
            const int tok = int(row / c.h_s) - it.g * c.N;
            const int32_t* sel = c.tok_I + (int64_t(c.tok_qb[tok]) * c.h_kv + it.g) * c.tok_T;
            bool hit = false;
            for (int jj = 0; jj < c.tok_T; ++jj) hit |= sel[jj] == it.kblock;
            keep = hit;
          }
          cp_async4(&S->st_l2[w][rs.idx][e], keep ? c.lse[br] + row : &g_pos_inf);
          cp_async4(&S->st_D[w][rs.idx][e], e < nr ? c.Dd[br] + row : &g_zero);
        }
#if SSA_KV_STATS_WAIT
        // wait for this lane's two copies, then a plain (release) arrival: the cp.async.mbarrier
        // arrive.noinc form is not modelled by compute-sanitizer synccheck ("missing init", r1f)
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        mbar_arrive(&S->r_full[w][rs.idx]);
#else
        cp_async_mbar_arrive_noinc(&S->r_full[w][rs.idx]);
#endif
        if (lane == 0) {
          uint8_t* st = sR + (w * kRStages + rs.idx) * 16384;
          mbar_expect_tx(&S->r_full[w][rs.idx], 16384);
          tma_load_2d(st, &tmQ.m[0], &S->r_full[w][rs.idx], 0, int(r0));
          tma_load_2d(st + 8192, br == 2 ? &tmDO2.m[0] : &tmDO.m[0], &S->r_full[w][rs.idx], 0, int(r0));
        }
        __syncwarp();
        rs.next();
        ++i;
      }
    }
  } else if (warp >= 9) {
    // ------------------------------------------------ MMA issuer of warpgroup w (lane 0)
    // Per own row tile: S^T(t+1), dP^T(t+1) as soon as the warpgroup has read S^T(t), dP^T(t) (they
    // overlap its softmax work), then dV += (P w)^T (w dO), dK += dS^T Q from the shared-memory P / dS.
    const int w = warp - 9;
    const uint32_t idS = idesc_f16(128, kRT, false, false);    // S^T = K Q^T, dP^T = V dO^T
    const uint32_t idA = idesc_f16(128, 64, false, true);      // dV += (P w)^T dO, dK += dS^T Q
    const uint32_t aK = smem_u32(sK), aV = smem_u32(sV);
    const uint32_t tS = tmem + w * 256, tDP = tS + 64, tK = tS + 128, tV = tS + 192;
    const uint32_t ap0 = smem_u32(sP + w * kPBuf * 32768);
    const int n_own = w == 0 ? n_own0 : n_tiles / 2;
    Ring rs(kRStages), sb(1), pb(kPBuf);
    uint32_t kph = 0, aph = 0;
    if (lane == 0) {
      for (int kt = 0; kt < n_kt; ++kt) {
        mbar_wait(&S->k_full, kph);
        kph ^= 1u;
        tc_fence_after();
        auto issue_s = [&]() {
          mbar_wait(&S->r_full[w][rs.idx], rs.ph);
          mbar_wait(&S->s_empty[w], sb.ph ^ 1u);
          tc_fence_after();
          const uint32_t aq = smem_u32(sR + (w * kRStages + rs.idx) * 16384), ado = aq + 8192;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16(tS, desc_sw128(aK + k * 32, 0, 1024), desc_sw128(aq + k * 32, 0, 1024), idS, k > 0);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16(tDP, desc_sw128(aV + k * 32, 0, 1024), desc_sw128(ado + k * 32, 0, 1024), idS, k > 0);
          umma_commit(&S->s_full[w]);
          if (w == 0) TRACE_R(1, 3, 0);
          rs.next();
          sb.next();
        };
        Ring rs_a = rs;
        if (n_own > 0) issue_s();
        mbar_wait(&S->acc_empty[w], aph ^ 1u);
        tc_fence_after();
        for (int q = 0; q < n_own; ++q) {
          if (q + 1 < n_own) issue_s();
          mbar_wait(&S->p_full[w][pb.idx], pb.ph);
          tc_fence_after();
          const uint32_t ap = ap0 + pb.idx * 32768, ads = ap + 16384;
          const uint32_t aq = smem_u32(sR + (w * kRStages + rs_a.idx) * 16384), ado = aq + 8192;
#pragma unroll
          for (int k = 0; k < kRT / 16; ++k)
            umma_bf16(tV, desc_sw128(ap + k * 32, 0, 1024), desc_sw128(ado + k * 2048, 0, 1024), idA,
                      (q > 0 || k > 0) ? 1u : 0u);
          umma_commit(&S->pv_empty[w][pb.idx]);
#pragma unroll
          for (int k = 0; k < kRT / 16; ++k)
            umma_bf16(tK, desc_sw128(ads + k * 32, 0, 1024), desc_sw128(aq + k * 2048, 0, 1024), idA,
                      (q > 0 || k > 0) ? 1u : 0u);
          umma_commit(&S->p_empty[w][pb.idx]);
          umma_commit(&S->r_empty[w][rs_a.idx]);
          if (w == 0) TRACE_R(1, 5, q);
          rs_a.next();
          pb.next();
        }
        umma_commit(&S->acc_full[w]);
        umma_commit(&S->k_empty);
        aph ^= 1u;
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------ softmax: thread = key (TMEM lane)
    const int wg = warp >> 2, t = tid & 127;
    const uint32_t lrow = uint32_t((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + lrow + wg * 256, tDP = tS + 64;
    const float cl2 = c.scale * kLog2e;
    const int n_own = wg == 0 ? n_own0 : n_tiles / 2;
    const uint32_t pbase0 = smem_u32(sP + wg * kPBuf * 32768);
    Ring rs(kRStages), pr(kPBuf);
    uint32_t sph = 0, aph = 0;
    // MUFU ping-pong (named barriers 4 / 5); warpgroup 1 runs a turn for every warpgroup-0 tile (an
    // empty one when it has no tile) so the turn counts always match
    if (kKvPingPong && wg == 1 && n_own0 > 0) named_bar_arrive(4, 256);
    for (int kt = 0; kt < n_kt; ++kt) {
      const int key = kt * 128 + t;
      const bool kvalid = key < nkeys_total;
      for (int q = 0; q < n_own0; ++q) {
        if (q >= n_own) {                        // warpgroup 1 without a tile: keep the turn order
          if (kKvPingPong) {
            named_bar_sync(5, 256);
            named_bar_arrive(4, 256);
          }
          continue;
        }
        mbar_wait(&S->r_full[wg][rs.idx], rs.ph);      // row stats of this stage are visible
        mbar_wait(&S->s_full[wg], sph);
        sph ^= 1u;
        if (warp == 0) TRACE_R(2, 7, q);
        tc_fence_after();
        const uint32_t sbase = smem_u32(&S->st_l2[wg][rs.idx][0]);
        const uint32_t dbase = smem_u32(&S->st_D[wg][rs.idx][0]);
        if (kKvPingPong) named_bar_sync(4 + wg, 256);
        if (warp == 0) TRACE_R(2, 8, q);
#pragma unroll
        for (int half = 0; half < 2; ++half) {   // 32 rows at a time keeps the register file in budget
          float s[32], dp[32];
          tmem_ld32(tS + half * 32, s);
          tmem_ld32(tDP + half * 32, dp);        // already (w dO) V^T
          tmem_wait_ld();
          if (half == 1) {
            tc_fence_before();
            mbar_arrive(&S->s_empty[wg]);        // S^T / dP^T fully read: the next tile's MMA may start
          }
          uint32_t pw[16], ds[16];
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const int rr = half * 32 + i;
            float4 l4, d4;
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(l4.x), "=f"(l4.y), "=f"(l4.z), "=f"(l4.w) : "r"(sbase + rr * 4));
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(d4.x), "=f"(d4.y), "=f"(d4.z), "=f"(d4.w) : "r"(dbase + rr * 4));
            const float p0 = ex2(fmaf(s[i], cl2, -l4.x)), p1 = ex2(fmaf(s[i + 1], cl2, -l4.y));
            const float p2 = ex2(fmaf(s[i + 2], cl2, -l4.z)), p3 = ex2(fmaf(s[i + 3], cl2, -l4.w));
            pw[i / 2] = pack_f16(p0, p1);
            pw[i / 2 + 1] = pack_f16(p2, p3);
            ds[i / 2] = pack_f16(p0 * (dp[i] - d4.x), p1 * (dp[i + 1] - d4.y));
            ds[i / 2 + 1] = pack_f16(p2 * (dp[i + 2] - d4.z), p3 * (dp[i + 3] - d4.w));
          }
          if (!kvalid) {
#pragma unroll
            for (int i = 0; i < 16; ++i) pw[i] = ds[i] = 0u;
          }
          const uint32_t pbase = pbase0 + pr.idx * 32768;
          // (P w)^T may be rewritten once the previous tile's dV MMAs are done, dS^T once its dK MMAs are
          if (half == 0) mbar_wait(&S->pv_empty[wg][pr.idx], pr.ph ^ 1u);
#pragma unroll
          for (int ch = 0; ch < 4; ++ch)
            st_shared_v4(pbase + sw128(t, half * 4 + ch), pw[4 * ch], pw[4 * ch + 1], pw[4 * ch + 2], pw[4 * ch + 3]);
          if (half == 0) mbar_wait(&S->p_empty[wg][pr.idx], pr.ph ^ 1u);
#pragma unroll
          for (int ch = 0; ch < 4; ++ch)
            st_shared_v4(pbase + 16384 + sw128(t, half * 4 + ch), ds[4 * ch], ds[4 * ch + 1], ds[4 * ch + 2],
                         ds[4 * ch + 3]);
        }
        if (kKvPingPong) named_bar_arrive(5 - wg, 256);
        if (warp == 0) TRACE_R(2, 9, q);
        fence_proxy_async_smem();
        mbar_arrive(&S->p_full[wg][pr.idx]);
        if (warp == 0) TRACE_R(2, 11, q);
        rs.next();
        pr.next();
      }
      // accumulators: dK at 128, dV at 192 of each warpgroup; warpgroup 0 writes dK = dK_0 + dK_1,
      // warpgroup 1 writes dV = dV_0 + dV_1 (fixed order: deterministic)
      const bool has1 = n_tiles > 1;
      mbar_wait(&S->acc_full[0], aph);
      if (has1) mbar_wait(&S->acc_full[1], aph);
      aph ^= 1u;
      tc_fence_after();
      const uint32_t col = wg == 0 ? 128u : 192u;
      float a0[64], a1[64];
      tmem_ld32(tmem + lrow + col, a0);
      tmem_ld32(tmem + lrow + col + 32, a0 + 32);
      if (has1) {
        tmem_ld32(tmem + lrow + 256 + col, a1);
        tmem_ld32(tmem + lrow + 256 + col + 32, a1 + 32);
      }
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&S->acc_empty[0]);
      mbar_arrive(&S->acc_empty[1]);
      if (kvalid) {
        float* o;
        if (mode == 0) {
          const int64_t idx = ((int64_t(it.chunk) * c.h_kv + g) * c.n_blk[SSA_LEVEL_CMP] + kbase + key) * kD;
          o = (wg == 0 ? c.dkc_part : c.dvc_part) + idx;
        } else if (it.first) {
          const int64_t idx = (int64_t(g) * c.N + kbase + key) * kD;
          o = (wg == 0 ? c.dk_acc : c.dv_acc) + idx;
        } else {
          const int64_t idx = (int64_t(it.part_slot) * c.max_fill[SSA_LEVEL_SLC] + key) * kD;
          o = (wg == 0 ? c.kv_part_k : c.kv_part_v) + idx;
        }
        const bool none = n_tiles == 0;
        const float sc = (wg == 0 ? c.scale : 1.f) * do_pow2(c.do_amax, true);
#pragma unroll
        for (int e = 0; e < kD; e += 4) {
          float4 v4;
          v4.x = none ? 0.f : (a0[e] + (has1 ? a1[e] : 0.f)) * sc;
          v4.y = none ? 0.f : (a0[e + 1] + (has1 ? a1[e + 1] : 0.f)) * sc;
          v4.z = none ? 0.f : (a0[e + 2] + (has1 ? a1[e + 2] : 0.f)) * sc;
          v4.w = none ? 0.f : (a0[e + 3] + (has1 ? a1[e + 3] : 0.f)) * sc;
          *reinterpret_cast<float4*>(o + e) = v4;
        }
      }
    }
  }
#ifdef SSA_TRACE
  if (TRACE_ON && (warp == 8 || warp == 9 || warp == 0)) {
    const int role = warp == 8 ? 0 : (warp == 9 ? 1 : 2);
    for (int i = 0; i < tr_n; ++i) g_trace_kv[role][i] = S->trace[role][i];
    g_trace_kv_cnt[role] = tr_n;
  }
#endif
  tc_fence_before();
  __syncthreads();
  if (warp == 9) tmem_dealloc<512>(tmem);
}

// raw-key work items: ceil(len / kQBlocksPerItem) (at least 1, for the window) per (block, g)
__global__ void k_kv_item_count(Ctx c, int32_t* cnt) {
  const int key = blockIdx.x * blockDim.x + threadIdx.x;
  if (key >= c.n_blk[SSA_LEVEL_SLC] * c.h_kv) return;
  const int len = c.inv_off[key + 1] - c.inv_off[key];
  cnt[key] = max(1, (len + c.qb_per_item - 1) / c.qb_per_item);
}
// fold the partials of items 1.. of every (block, g) into dk_acc / dv_acc, in item order
__global__ void k_kv_reduce(Ctx c) {
  // 4 consecutive elements per thread (float4), 32-bit index math
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= c.N * c.h_kv * (kD / 4)) return;
  const int e = (i % (kD / 4)) * 4;
  const int g = (i / (kD / 4)) % c.h_kv;
  const int p = i / ((kD / 4) * c.h_kv);
  const int B = c.tok_block[SSA_LEVEL_SLC][p];
  const int key = B * c.h_kv + g;
  const int i0 = c.kv_item_off[key], i1 = c.kv_item_off[key + 1];
  if (i1 - i0 <= 1) return;
  const int local = p - c.off[SSA_LEVEL_SLC][B];
  float4 sk = make_float4(0.f, 0.f, 0.f, 0.f), sv = sk;
#pragma unroll 4
  for (int s = i0 + 1; s < i1; ++s) {
    const int64_t idx = (int64_t(s) * c.max_fill[SSA_LEVEL_SLC] + local) * kD + e;
    const float4 a = *reinterpret_cast<const float4*>(c.kv_part_k + idx), b = *reinterpret_cast<const float4*>(c.kv_part_v + idx);
    sk.x += a.x; sk.y += a.y; sk.z += a.z; sk.w += a.w;
    sv.x += b.x; sv.y += b.y; sv.z += b.z; sv.w += b.w;
  }
  const int64_t o = (int64_t(g) * c.N + p) * kD + e;
  float4* dk = reinterpret_cast<float4*>(c.dk_acc + o);
  float4* dv = reinterpret_cast<float4*>(c.dv_acc + o);
  const float4 k0 = *dk, v0 = *dv;
  *dk = make_float4(k0.x + sk.x, k0.y + sk.y, k0.z + sk.z, k0.w + sk.w);
  *dv = make_float4(v0.x + sv.x, v0.y + sv.y, v0.z + sv.z, v0.w + sv.w);
}

}  // namespace

bool tc_bwd_available() { return true; }

static int64_t kv_items_bound(int n_slc, int n_q, int h_kv, int T, int qbpi) {
  return int64_t(n_slc) * h_kv + (int64_t(n_q) * h_kv * T + qbpi - 1) / qbpi + 1;
}

// packed row tiles of all raw-key items: every row of every range once ((T + 1) N H: the selections and
// the window), at most 7 padding rows per range (inverse-list entries + windows), and per item two partial
// tiles (the selection part's last tile: the window starts a fresh one; the item's last tile)
static int64_t kv_tiles_bound(int64_t N, int H, int h_kv, int n_slc, int n_q, int T, int64_t items) {
  const int64_t rows = N * H * (T + 1) + 7 * (int64_t(n_q) * h_kv * T + int64_t(n_slc) * h_kv);
  return rows / 64 + 2 * items + 1;
}

int tc_qb_per_item(int m_slc, int m_q) {
  const char* e = getenv("SSA_KV_QBPI");   // A/B knob: raw-key work item size in query blocks
  if (e && atoi(e) > 0) return atoi(e);
  const int r = m_q > 0 && m_slc % m_q == 0 ? m_slc / m_q : 1;
  return kQBlocksPerItem * r * r * r;
}

size_t tc_bwd_ws_bytes(int64_t N, int H, int h_kv, int D, int n_slc, int n_q, int T, int max_fill_slc, int qb_per_item) {
  // fp16 copies: q, dO, 3 x gate-scaled dO (rows), k, v (keys), K^cmp, V^cmp (n_cmp <= N)
  size_t b = (size_t(5) * size_t(N) * size_t(H) + size_t(4) * size_t(h_kv) * size_t(N)) * size_t(D) * 2 + 8 * 256;
  const int64_t nkeys = int64_t(n_slc) * h_kv;
  b += size_t(2 * nkeys + 2) * 4 + 512 + scan_ws_bytes(nkeys + 1);                  // item counts / offsets
  const int64_t items = kv_items_bound(n_slc, n_q, h_kv, T, qb_per_item);
  b += size_t(2) * items * max_fill_slc * D * 4 + 512;  // partials
  b += size_t(2 * items + 4) * 4 + 512 + scan_ws_bytes(items + 1);                    // packed tile counts / offsets
  b += size_t(kv_tiles_bound(N, H, h_kv, n_slc, n_q, T, items)) * 8 * sizeof(int2) + 1024;  // granule descriptors
  return b;
}

ssa_status tc_backward(const Ctx& c_in, const Ctx& ck_in, void* ws, cudaStream_t st) {
  Ctx c = c_in;     // row prologue, dQ, compressed-key KV-outer
  Ctx ck = ck_in;   // raw-key KV-outer (its own query level: inverse CSR, work items)
  const int n_cmp = c.n_blk[SSA_LEVEL_CMP];
  const int n_slc = c.n_blk[SSA_LEVEL_SLC];
  Carve cw(ws, tc_bwd_ws_bytes(c.N, c.H, c.h_kv, c.D, n_slc, ck.n_blk[SSA_LEVEL_Q], ck.T, c.max_fill[SSA_LEVEL_SLC], ck.qb_per_item));
  const uint64_t qrows = uint64_t(c.h_kv) * c.N * c.h_s, crows = uint64_t(c.h_kv) * n_cmp, krows = uint64_t(c.h_kv) * c.N;
  __half* q16 = cw.take<__half>(qrows * kD);
  __half* do16 = cw.take<__half>(qrows * kD);
  __half* dow = cw.take<__half>(3 * qrows * kD);   // dO * gate, one copy per branch
  __half* k16 = cw.take<__half>(krows * kD);
  __half* v16 = cw.take<__half>(krows * kD);
  __half* kc = cw.take<__half>(crows * kD);
  __half* vc = cw.take<__half>(crows * kD);
  const int64_t nkeys = int64_t(n_slc) * c.h_kv;
  int32_t* item_cnt = cw.take<int32_t>(nkeys + 1);
  ck.kv_item_off = cw.take<int32_t>(nkeys + 1);
  void* scan_ws = cw.take<char>(scan_ws_bytes(nkeys + 1));
  const int64_t bound = kv_items_bound(n_slc, ck.n_blk[SSA_LEVEL_Q], c.h_kv, ck.T, ck.qb_per_item);
  ck.kv_part_k = cw.take<float>(size_t(bound) * c.max_fill[SSA_LEVEL_SLC] * kD);
  ck.kv_part_v = cw.take<float>(size_t(bound) * c.max_fill[SSA_LEVEL_SLC] * kD);
  int32_t* tile_cnt = cw.take<int32_t>(bound + 1);
  ck.kv_tile_off = cw.take<int32_t>(bound + 1);
  void* tscan_ws = cw.take<char>(scan_ws_bytes(bound + 1));
  ck.kv_desc = cw.take<int2>(size_t(kv_tiles_bound(c.N, c.H, c.h_kv, n_slc, ck.n_blk[SSA_LEVEL_Q], ck.T, bound)) * 8);
  // packed row tiles only where query blocks are short (m_q < m_slc: a few rows each); long query blocks
  // fill their tiles contiguously and keep the cheaper arithmetic row walk (measured: C3 raw keys 3.2 ms
  // contiguous vs 4.0 ms packed)
  const bool pack = ck.n_blk[SSA_LEVEL_Q] > 0 && int64_t(ck.N) * ck.h_s < int64_t(256) * ck.n_blk[SSA_LEVEL_Q];
  if (!pack) ck.kv_desc = nullptr;
  uint32_t* amax = cw.take<uint32_t>(1);
  if (!cw.ok()) { set_error("tcgen05 backward: workspace carve exceeds tc_bwd_ws_bytes"); return SSA_ERR_WORKSPACE; }
  c.do_amax = amax;
  ck.do_amax = amax;
  SSA_CUDA_TRY(cudaMemsetAsync(amax, 0, 4, st));
  {  // over the rows this call may read (the owned range with a query-block range / SSA_LOCAL_ROWS)
    const int64_t n8 = int64_t(c.row_hi - c.row_lo) * c.H * c.Dc / 8;
    const __nv_bfloat16* d0 = static_cast<const __nv_bfloat16*>(c.dout) + int64_t(c.row_lo) * c.H * c.Dc;
    const unsigned blocks = unsigned(std::min<int64_t>((n8 + 255) / 256, 148 * 8));
    if (n8 > 0) {
      k_do_absmax<<<std::max(1u, blocks), 256, 0, st>>>(c.sorted_input ? d0 : static_cast<const __nv_bfloat16*>(c.dout),
                                                         c.sorted_input ? n8 : int64_t(c.N) * c.H * c.Dc / 8, amax);
      SSA_LAUNCH_CHECK("k_do_absmax");
    }
  }
  k_tc_bwd_rows<<<unsigned((int64_t(c.N) * c.H * 8 + 255) / 256), 256, 0, st>>>(c, q16, do16, dow);
  SSA_LAUNCH_CHECK("k_tc_bwd_rows");
  const int64_t n = int64_t(krows) * kD;   // >= h_kv * n_cmp * kD
  k_tc_bwd_prep<<<unsigned((n / 8 + 255) / 256), 256, 0, st>>>(c, k16, v16, kc, vc);
  SSA_LAUNCH_CHECK("k_tc_bwd_prep");
  CUtensorMap tmQ, tmDO, tmKc, tmVc, tmKc128, tmVc128, tmK128, tmV128;
  TmapSet4 tmK, tmV, tmQs, tmDWs[3];
  for (int br = 0; br < 3; ++br)
    if (!make_tmap_set4(&tmDWs[br], dow + size_t(br) * qrows * kD, qrows))
      return SSA_ERR_CUDA;
  if (!make_tmap_set4(&tmQs, q16, qrows)) return SSA_ERR_CUDA;
  if (!make_tmap_bf16_2d(&tmQ, q16, qrows, 128) || !make_tmap_bf16_2d(&tmDO, do16, qrows, 128) ||
      !make_tmap_bf16_2d(&tmKc, kc, crows, kKT) || !make_tmap_bf16_2d(&tmVc, vc, crows, kKT) ||
      !make_tmap_set4(&tmK, k16, krows) || !make_tmap_set4(&tmV, v16, krows) ||
      !make_tmap_bf16_2d(&tmKc128, kc, crows, 128) || !make_tmap_bf16_2d(&tmVc128, vc, crows, 128) ||
      !make_tmap_bf16_2d(&tmK128, k16, krows, 128) || !make_tmap_bf16_2d(&tmV128, v16, krows, 128))
    return SSA_ERR_CUDA;
  // The Q-outer dQ kernel and the KV-outer dK/dV kernels read the same operands and write disjoint
  // outputs: with SSA_BWD_FORK the KV-outer launches go to an internal stream forked from (and joined
  // back into) the caller's stream, so each kernel's last partial wave overlaps the other's work.
  cudaStream_t kst = st;
  cudaEvent_t ev_join = nullptr;
  if (kBwdFork) {
    static cudaStream_t side[16] = {};
    static std::mutex side_mu;
    int dev = 0;
    SSA_CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 16) {
      {
        std::lock_guard<std::mutex> lk(side_mu);   // one internal stream per device, created once
        if (!side[dev]) SSA_CUDA_TRY(cudaStreamCreateWithFlags(&side[dev], cudaStreamNonBlocking));
      }
      cudaEvent_t ev_fork;
      SSA_CUDA_TRY(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
      SSA_CUDA_TRY(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
      SSA_CUDA_TRY(cudaEventRecord(ev_fork, st));
      SSA_CUDA_TRY(cudaStreamWaitEvent(side[dev], ev_fork, 0));
      cudaEventDestroy(ev_fork);      // released once the recorded work completes
      kst = side[dev];
    }
  }
  {
    const size_t smem = 1024 + 65536 + kStages * 2 * kKVBytes + 65536 + sizeof(DqSmem);
    static_assert(1024 + 65536 + kStages * 2 * kKVBytes + 65536 + sizeof(DqSmem) <= 232448, "dQ shared memory");
    SSA_CUDA_TRY(cudaFuncSetAttribute(k_tc_dq<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    SSA_CUDA_TRY(cudaFuncSetAttribute(k_tc_dq<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    if (c.blk_ws) {
      // per-token selection (pertoken.cu): the selection branch's dQ per (token, selected block) pair on the
      // expanded rows (ck: the real level, whose inverse CSR lists the tokens selecting every block), summed
      // per row into dq_extra; the virtual level then runs the compressed keys + window and adds it
      ProfScope pb("tc_bwd_blk_dq", st);
      BlkPass bb;
      Ctx ce;
      float* dqx = nullptr;
      ssa_status s = blk_bwd_build(ck, q16, do16, c.blk_ws, st, &bb, &ce, &dqx);
      if (s != SSA_OK) return s;
      ce.do_amax = amax;
      const uint64_t erows = uint64_t(bb.n_exp) * c.h_s;
      CUtensorMap tmQe, tmDOe;
      if (!make_tmap_bf16_2d(&tmQe, ce.qs, erows, 128) || !make_tmap_bf16_2d(&tmDOe, ce.dos, erows, 128)) return SSA_ERR_CUDA;
      k_tc_dq<false><<<dim3(unsigned(bb.bound), 1), kDqThreads, smem, st>>>(ce, tmQe, tmDOe, tmKc, tmVc, tmK, tmV);
      SSA_LAUNCH_CHECK("k_tc_dq(blocks)");
      if ((s = blk_bwd_merge(ck, bb, dqx, st)) != SSA_OK) return s;
      c.dq_extra = dqx;   // (c: the plain virtual level, empty selection lists: compressed keys + window)
    }
    ProfScope ps("tc_bwd_dq", st);
    if (c.umask) k_tc_dq<true><<<dim3(c.n_blk[SSA_LEVEL_Q], c.h_kv), kDqThreads, smem, st>>>(c, tmQ, tmDO, tmKc, tmVc, tmK, tmV);
    else k_tc_dq<false><<<dim3(c.n_blk[SSA_LEVEL_Q], c.h_kv), kDqThreads, smem, st>>>(c, tmQ, tmDO, tmKc, tmVc, tmK, tmV);
    SSA_LAUNCH_CHECK("k_tc_dq");
  }
  const size_t smem = 1024 + 32768 + 2 * kRStages * 16384 + 2 * kPBuf * 32768 + sizeof(KvSmem);
  if (smem > 232448) { set_error("KV-outer shared memory exceeds 227 KB"); return SSA_ERR_UNSUPPORTED; }
  SSA_CUDA_TRY(cudaFuncSetAttribute(k_tc_dkdv, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  {
    k_kv_item_count<<<unsigned((nkeys + 255) / 256), 256, 0, kst>>>(ck, item_cnt);
    SSA_LAUNCH_CHECK("k_kv_item_count");
    ssa_status s = exclusive_scan(item_cnt, ck.kv_item_off, nkeys, ck.kv_item_off + nkeys, scan_ws, kst);
    if (s != SSA_OK) return s;
    if (ck.kv_desc) {
      k_kv_tile_count<<<unsigned((bound + 3) / 4), 128, 0, kst>>>(ck, tile_cnt, int(bound));
      SSA_LAUNCH_CHECK("k_kv_tile_count");
      s = exclusive_scan(tile_cnt, ck.kv_tile_off, bound, ck.kv_tile_off + bound, tscan_ws, kst);
      if (s != SSA_OK) return s;
      k_kv_tile_fill<<<unsigned((bound + 3) / 4), 128, 0, kst>>>(ck, ck.kv_tile_off, ck.kv_desc, int(bound));
      SSA_LAUNCH_CHECK("k_kv_tile_fill");
    }
    ProfScope ps("tc_bwd_kv", kst);
    k_tc_dkdv<<<dim3(unsigned(bound), 1, 1), kKvThreads, smem, kst>>>(ck, 1, tmQs, tmDWs[1], tmDWs[2], tmK128, tmV128);
    SSA_LAUNCH_CHECK("k_tc_dkdv(raw)");
  }
  {
    const int64_t nk = int64_t(c.N) * c.h_kv * (kD / 4);
    k_kv_reduce<<<unsigned((nk + 255) / 256), 256, 0, kst>>>(ck);
    SSA_LAUNCH_CHECK("k_kv_reduce");
  }
  if (!c.win_only) {
    ProfScope ps("tc_bwd_cmp_kv", kst);
    k_tc_dkdv<<<dim3(c.n_cmp_tiles, c.h_kv, c.n_chunk), kKvThreads, smem, kst>>>(c, 0, tmQs, tmDWs[0], tmDWs[0], tmKc128,
                                                                               tmVc128);
    SSA_LAUNCH_CHECK("k_tc_dkdv(cmp)");
  }
  if (ev_join) {   // join: the caller's stream continues after the KV-outer work
    SSA_CUDA_TRY(cudaEventRecord(ev_join, kst));
    SSA_CUDA_TRY(cudaStreamWaitEvent(st, ev_join, 0));
    cudaEventDestroy(ev_join);
  }
  return SSA_OK;
}

}  // namespace ssa

#ifdef SSA_TRACE
extern "C" int ssa_debug_trace_kv(unsigned long long* host, int cap) {
  int cnt[3];
  unsigned long long buf[3][128];
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(cnt, ssa::g_trace_kv_cnt, sizeof(cnt));
  cudaMemcpyFromSymbol(buf, ssa::g_trace_kv, sizeof(buf));
  int n = 0;
  for (int r = 0; r < 3; ++r)
    for (int i = 0; i < cnt[r] && n < cap; ++i) host[n++] = buf[r][i];
  return n;
}
extern "C" int ssa_debug_trace_dq(unsigned long long* host, int cap) {
  int cnt[3];
  unsigned long long buf[3][128];
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(cnt, ssa::g_trace_dq_cnt, sizeof(cnt));
  cudaMemcpyFromSymbol(buf, ssa::g_trace_dq, sizeof(buf));
  int n = 0;
  for (int r = 0; r < 3; ++r)
    for (int i = 0; i < cnt[r] && n < cap; ++i) host[n++] = buf[r][i];
  return n;
}
#endif
