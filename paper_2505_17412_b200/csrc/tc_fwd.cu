// tc_fwd.cu — tcgen05/TMEM/TMA forward kernels of the bf16, d = 64 SSA path.
//
//  k_tc_prep      fp32 pooled K/V (Eq. 7) -> bf16 operand copies: K^cmp as a hi/lo bf16 pair (so the
//                 compression scores that drive top-k keep ~16 mantissa bits), V^cmp in bf16.
//  k_tc_cmp_fwd   compression attention + Eq. 8 block scores + top-k, CTA per (query block, kv group):
//                 pass 1 S = Q K^T (rows on TMEM lanes) -> per-row LSE; pass 2 S^T = K Q^T (keys on TMEM
//                 lanes) -> P^T = exp(S^T - LSE) so the Eq. 8 column sums are exact fp32 per-thread
//                 sums, P^T goes to smem as the MN-major A operand of O += P V (accumulated in TMEM with
//                 fixed normalisation). Scores stay in smem; top-k runs in the same CTA.
//  k_tc_slcwin_fwd selection attention over the T selected blocks (Alg. 1 at query-block granularity)
//                 and window attention with online softmax, then the gated sum of Eq. 6 and
//                 the scatter to caller order. Key tiles pack the selected blocks' keys in 8-row
//                 granules (TMA boxes of 64/32/16/8 rows); a per-tile bit mask drops granule padding.
//
// Warp roles (192 threads): warps 0-3 softmax/epilogue (thread i <-> TMEM lane i), warp 4 TMA
// producer, warp 5 MMA issuer (one elected lane) + TMEM owner.
#include <cfloat>

#include <cstdlib>

#include "internal.h"
#include "tc.h"
#include "tc_common.cuh"

namespace ssa {
namespace {
using namespace tc;

constexpr int kD = 64;
constexpr int kTile = 128;
constexpr float kLog2e = 1.4426950408889634f;
#ifndef SSA_SW_EPI_HALF
#define SSA_SW_EPI_HALF 1   // epilogue staged 32 columns at a time (4 KB per warp): room for a 4th K/V stage
#endif
constexpr bool kEpiHalf = SSA_SW_EPI_HALF;
#ifndef SSA_SW_STAGES
#define SSA_SW_STAGES (SSA_SW_EPI_HALF ? 4 : 3)
#endif
constexpr int kStages = SSA_SW_STAGES;   // K/V stages of the selection+window kernel
constexpr int kEpiBytes = kEpiHalf ? 32768 : 65536;   // epilogue staging, all 8 softmax warps
#ifndef SSA_SW_PINGPONG
#define SSA_SW_PINGPONG 1
#endif
constexpr bool kSwPingPong = SSA_SW_PINGPONG;   // MUFU turns alternate between the two softmax warpgroups

#ifdef SSA_TRACE
// per-role shared-memory trace of one CTA (debug builds: -DSSA_TRACE); flushed at kernel end
__device__ unsigned long long g_trace[3][128];
__device__ int g_trace_cnt[3];
#define TRACE_ON (blockIdx.x == 5 && blockIdx.y == 0 && (threadIdx.x & 31) == 0)
#define TRACE_R(role, ev, j)                                                                              \
  do {                                                                                                  \
    if (TRACE_ON && tr_n < 128) S->trace[role][tr_n++] = (clock64() << 16) | (unsigned long long)(((ev) << 12) | ((j) & 0xfff)); \
  } while (0)
#else
#define TRACE_R(role, ev, j) do { } while (0)
#endif
#ifdef SSA_TRACE
// selection/window kernel event trace of CTA (5, 0), written straight to global memory (debug builds)
__device__ unsigned long long g_trace_sw[3][512];
__device__ int g_trace_sw_cnt[3];
#define TRACE_SW(role, ev, j)                                                                             \
  do {                                                                                                   \
    if (blockIdx.x == 5 && blockIdx.y == 0 && (threadIdx.x & 31) == 0 && sw_n < 512) {                   \
      g_trace_sw[role][sw_n++] = (clock64() << 16) | (unsigned long long)(((ev) << 12) | ((j) & 0xfff)); \
      g_trace_sw_cnt[role] = sw_n;                                                                       \
    }                                                                                                    \
  } while (0)
#else
#define TRACE_SW(role, ev, j) do { } while (0)
#endif
#ifdef SSA_TRACE
// per-CTA [start, end) globaltimer stamps + SM id of the selection/window kernel (debug builds)
__device__ unsigned long long g_cta_stamp[2 * 4096][3];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif

struct TcArgs {
  Ctx c;
  const __nv_bfloat16* kc_hi;   // [h_kv][n_cmp][64]
  const __nv_bfloat16* kc_lo;
  const __half* vc;
};

// K^cmp -> bf16 hi/lo pair, V^cmp -> fp16 (P.V runs in fp16), raw V -> fp16 copy (exact for bf16)
// part: 1 = pooled keys only (K^cmp hi/lo, V^cmp fp16), 2 = raw values only (V fp16), 3 = both
__global__ void k_tc_prep(Ctx c, __nv_bfloat16* kc_hi, __nv_bfloat16* kc_lo, __half* vc16, __half* vs16, int part) {
  // 4 elements per thread (every array is a multiple of 64 long and 256-B aligned)
  const int64_t i = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
  const int64_t n = int64_t(c.h_kv) * c.n_blk[SSA_LEVEL_CMP] * kD;
  const int64_t nv = int64_t(c.h_kv) * c.N * kD;
  if ((part & 1) && i < n) {
    const float4 k = *reinterpret_cast<const float4*>(static_cast<const float*>(c.kc) + i);
    const float4 v = *reinterpret_cast<const float4*>(static_cast<const float*>(c.vc) + i);
    const float kk[4] = {k.x, k.y, k.z, k.w};
    __nv_bfloat16 hi[4], lo[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      hi[u] = __float2bfloat16_rn(kk[u]);
      lo[u] = __float2bfloat16_rn(kk[u] - __bfloat162float(hi[u]));
    }
    *reinterpret_cast<uint2*>(kc_hi + i) = *reinterpret_cast<const uint2*>(hi);
    *reinterpret_cast<uint2*>(kc_lo + i) = *reinterpret_cast<const uint2*>(lo);
    const __half2 v01 = __floats2half2_rn(v.x, v.y), v23 = __floats2half2_rn(v.z, v.w);
    *reinterpret_cast<uint2*>(vc16 + i) = make_uint2(*reinterpret_cast<const uint32_t*>(&v01), *reinterpret_cast<const uint32_t*>(&v23));
  }
  if ((part & 2) && i < nv) {
    const uint2 b = *reinterpret_cast<const uint2*>(static_cast<const __nv_bfloat16*>(c.vs) + i);
    const __nv_bfloat162 b01 = *reinterpret_cast<const __nv_bfloat162*>(&b.x), b23 = *reinterpret_cast<const __nv_bfloat162*>(&b.y);
    const float2 f01 = __bfloat1622float2(b01), f23 = __bfloat1622float2(b23);
    const __half2 h01 = __floats2half2_rn(f01.x, f01.y), h23 = __floats2half2_rn(f23.x, f23.y);
    *reinterpret_cast<uint2*>(vs16 + i) = make_uint2(*reinterpret_cast<const uint32_t*>(&h01), *reinterpret_cast<const uint32_t*>(&h23));
  }
}

// simple (index, phase) ring cursor
struct Ring {
  int idx = 0;
  uint32_t ph = 0;
  int n;
  __device__ explicit Ring(int n_) : n(n_) {}
  __device__ void next() {
    if (++idx == n) { idx = 0; ph ^= 1u; }
  }
};

// ================================================================================================
// compression attention + scores + top-k (two softmax warpgroups)
// ================================================================================================
// 352 threads: warps 0-3 = softmax warpgroup 0, warps 4-7 = softmax warpgroup 1 (each owns one
// 128-row tile of a row-tile pair; thread i <-> TMEM lane i of its own S / O / P columns), warp 8 =
// TMA producer, warps 9 / 10 = MMA issuers of warpgroups 0 / 1 (warp 9 owns TMEM). Both row tiles
// share every K/V tile load.
//  pass 1 (rows on lanes): S = Q K^T -> online softmax with lazy rescaling (the reference max moves
//         only when a row max exceeds it by kRescale, log2 units); P (fp16) is written to TMEM and
//         O += P V runs with A from TMEM, so P never touches shared memory.
//  pass 2 (keys on lanes): S^T = K Q^T -> p = exp2(S^T c - LSE) with the final row LSEs; each thread
//         sums its key's column in fp32: the Eq. 8 column sums, exact per thread.
// TMEM columns: S_0 S_1 [0, 256) | O_0 O_1 [256, 384) | P_0 P_1 [384, 512).
constexpr int kCmpThreads = 352;
constexpr int kCmpStages = 2;
constexpr float kRescale = 8.f;
#ifndef SSA_CMP_P2_PINGPONG
#define SSA_CMP_P2_PINGPONG 0   // 1: pass 2 (Eq. 8 column sums) also alternates MUFU turns (measured slower: 7.16 vs 6.96 ms)
#endif
constexpr bool kCmpP2PingPong = SSA_CMP_P2_PINGPONG;
#ifndef SSA_CMP_P1_PINGPONG
#define SSA_CMP_P1_PINGPONG 1
#endif
constexpr bool kCmpP1PingPong = SSA_CMP_P1_PINGPONG;   // pass 1 (online softmax, P -> TMEM, P.V) alternates MUFU turns
struct CmpSmem {
  uint64_t q_full, q_empty, k_full[kCmpStages], k_empty[kCmpStages], v_full[kCmpStages], v_empty[kCmpStages];
  uint64_t s_full[2], s_empty[2], p_full[2], p_free[2], o_full[2], o_empty[2];
  uint32_t tmem;
  alignas(16) float lse[2][kTile];
#ifdef SSA_TRACE
  unsigned long long trace[3][128];
#endif
  float bv[8];
  int bi[8];
  int chosen[64];
};

__device__ __forceinline__ float4 ld_shared_f4(const float* p) {
  float4 r;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "r"(smem_u32(p)));
  return r;
}

// kTok = 0: CTA per query block (any m_q), Eq. 8 column sums and selection scores in shared memory.
// kTok = h_s (per-token selection, m_q = 1): CTA per group of 256 / h_s consecutive tokens of one batch
// item (tc_tok_groups), two full row tiles; pass 2 sums each key's column per token (h_s rows) and folds
// the sums into per-token selection-block scores tile by tile (fixed order: keys of a block in key
// order, then tile order) in an L2-resident per-SM scratch; top-k per token by one warp each.
template <int kTok>
__global__ void __launch_bounds__(kCmpThreads, 1)
k_tc_cmp_fwd(TcArgs a, __grid_constant__ const CUtensorMap tmQ, __grid_constant__ const CUtensorMap tmKh,
             __grid_constant__ const CUtensorMap tmKl, __grid_constant__ const CUtensorMap tmV) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = sm;                                  // 2 x 16 KB (row tiles a, b)
  uint8_t* sK = sm + 32768;                          // kCmpStages x {Khi, Klo} 32 KB
  uint8_t* sV = sK + kCmpStages * 32768;             // kCmpStages x V 16 KB (pass 1 only)
  CmpSmem* S = reinterpret_cast<CmpSmem*>(sV + kCmpStages * 16384);
  const Ctx& c = a.c;
  float* sc_cmp0 = reinterpret_cast<float*>(S + 1);  // [max_cmp_b] Eq. 8 column sums, per warpgroup
  float* sc_cmp1 = sc_cmp0 + c.max_cmp_b;
  float* sc_slc = sc_cmp1 + c.max_cmp_b;             // [max_slc_b]
  constexpr int kGT = kTok > 0 ? kTile / kTok : 1;   // tokens per row tile (per-token mode)
  float* tbuf = reinterpret_cast<float*>(S + 1);     // per-token mode: [2 wg][2 parity][kGT][129] tile sums
  int* tchosen = reinterpret_cast<int*>(tbuf + 4 * kGT * 129);   // [8 warps][64]
  int* sbeg = tchosen + 8 * 64;   // per-token mode: first compressed key of each selection block (item-relative)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = blockIdx.y;
  int Q, t0, t1;
  float* tok_scr = nullptr;   // per-token mode: [2 kGT tokens][max_slc_b] scores of this CTA (per-SM slot)
  if constexpr (kTok > 0) {
    const int qa = c.tok_cg[2 * blockIdx.x], qe = c.tok_cg[2 * blockIdx.x + 1];
    if (qe <= qa) return;                             // past the last group (uniform per CTA)
    Q = qa;
    t0 = c.off[SSA_LEVEL_Q][qa];
    t1 = c.off[SSA_LEVEL_Q][qe];
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (smid >= unsigned(kTokSlots)) __trap();
    tok_scr = c.tok_sc + size_t(smid) * (2 * kGT) * c.max_slc_b;   // one resident CTA per SM (smem)
  } else {
    Q = c.q_order[blockIdx.x];
    if (Q < c.q_begin || Q >= c.q_end) return;        // not owned by this shard (uniform per CTA)
    t0 = c.off[SSA_LEVEL_Q][Q];
    t1 = c.off[SSA_LEVEL_Q][Q + 1];
  }
  const int b = c.q_batch[Q];
  const int c0 = c.bb[SSA_LEVEL_CMP][b], nk = c.bb[SSA_LEVEL_CMP][b + 1] - c0;
  const int s0 = c.bb[SSA_LEVEL_SLC][b], ns = c.bb[SSA_LEVEL_SLC][b + 1] - s0;
  const int rows = (t1 - t0) * c.h_s;
  const int n_rt = (rows + kTile - 1) / kTile, n_kt = (nk + kTile - 1) / kTile;
  const int n_pair = (n_rt + 1) / 2;
  const int qrow0 = (g * c.N + t0) * c.h_s;
  const int krow0 = g * c.n_blk[SSA_LEVEL_CMP] + c0;

  if (tid == 0) {
    mbar_init(&S->q_full, 1);
    mbar_init(&S->q_empty, 2);                       // one arrival per MMA issuer
    for (int i = 0; i < kCmpStages; ++i) {
      mbar_init(&S->k_full[i], 1);
      mbar_init(&S->k_empty[i], 2);
      mbar_init(&S->v_full[i], 1);
      mbar_init(&S->v_empty[i], 2);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&S->s_full[i], 1);
      mbar_init(&S->s_empty[i], 128);
      mbar_init(&S->p_full[i], 128);
      mbar_init(&S->p_free[i], 1);
      mbar_init(&S->o_full[i], 1);
      mbar_init(&S->o_empty[i], 128);
    }
    fence_barrier_init();
  }
  if (warp == 8 && lane == 0) { tma_prefetch(&tmQ); tma_prefetch(&tmKh); tma_prefetch(&tmKl); tma_prefetch(&tmV); }
  if (warp == 9) tmem_alloc<512>(&S->tmem);
  if constexpr (kTok == 0)
    for (int i = tid; i < nk; i += kCmpThreads) { sc_cmp0[i] = 0.f; sc_cmp1[i] = 0.f; }
  if constexpr (kTok > 0)
    for (int i = tid; i <= ns; i += kCmpThreads) sbeg[i] = c.slc_cmp_begin[s0 + i] - c0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S->tmem;
#ifdef SSA_TRACE
  int tr_n = 0;
#endif

  if (warp == 8) {
    // ---------------------------------------------------------------- TMA producer
    // K (hi, lo) every pass, V in pass 1 only; separate rings so K(kt+1) never waits behind V(kt)
    Ring kr(kCmpStages), vr(kCmpStages);
    uint32_t qph = 0;
    for (int pr = 0; pr < n_pair; ++pr) {
      const bool bval = 2 * pr + 1 < n_rt;
      mbar_wait(&S->q_empty, qph ^ 1u);
      qph ^= 1u;
      if (lane == 0) {
        mbar_expect_tx(&S->q_full, bval ? 32768u : 16384u);
        tma_load_2d(sQ, &tmQ, &S->q_full, 0, qrow0 + 2 * pr * kTile);
        if (bval) tma_load_2d(sQ + 16384, &tmQ, &S->q_full, 0, qrow0 + (2 * pr + 1) * kTile);
      }
      for (int pass = 1; pass <= 2; ++pass) {
        for (int kt = 0; kt < n_kt; ++kt) {
          mbar_wait(&S->k_empty[kr.idx], kr.ph ^ 1u);
          TRACE_R(0, pass, kt);
          if (lane == 0) {
            uint8_t* st = sK + kr.idx * 32768;
            mbar_expect_tx(&S->k_full[kr.idx], 32768u);
            tma_load_2d(st, &tmKh, &S->k_full[kr.idx], 0, krow0 + kt * kTile);
            tma_load_2d(st + 16384, &tmKl, &S->k_full[kr.idx], 0, krow0 + kt * kTile);
          }
          __syncwarp();
          kr.next();
          if (pass == 1) {
            mbar_wait(&S->v_empty[vr.idx], vr.ph ^ 1u);
            if (lane == 0) {
              mbar_expect_tx(&S->v_full[vr.idx], 16384u);
              tma_load_2d(sV + vr.idx * 16384, &tmV, &S->v_full[vr.idx], 0, krow0 + kt * kTile);
            }
            __syncwarp();
            vr.next();
          }
        }
      }
    }
  } else if (warp >= 9) {
    // ---------------------------------------------------------------- MMA issuers
    // warp 9 issues for warpgroup 0, warp 10 for warpgroup 1 (tcgen05.mma issue is nearly synchronous
    // with execution, so one issuer would make each warpgroup's S wait behind the other's P.V).
    // Per warpgroup, in order: S(kt+1) as soon as S(kt) has been read, then P.V(kt).
    const int w = warp - 9;
    const uint32_t idS = idesc_bf16(128, 128, false, false);
    const uint32_t idO = idesc_f16(128, 64, false, true);   // P from TMEM, V MN-major
    Ring kr(kCmpStages), vr(kCmpStages), sb(1);
    uint32_t qph = 0, pph = 0, oph = 0;
    auto mma_s = [&](int ki, bool transposed) {
      const uint32_t aq = smem_u32(sQ + w * 16384), ak = smem_u32(sK + ki * 32768);
      const uint32_t d = tmem + w * 128;
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t dq = desc_sw128(aq + k * 32, 0, 1024), dk = desc_sw128(ak + h * 16384 + k * 32, 0, 1024);
          umma_bf16(d, transposed ? dk : dq, transposed ? dq : dk, idS, (h | k) ? 1u : 0u);
        }
      umma_commit(&S->s_full[w]);
    };
    for (int pr = 0; pr < n_pair; ++pr) {
      const bool mine = w == 0 || 2 * pr + 1 < n_rt;  // warpgroup 1 sits out the last, odd pair
      mbar_wait(&S->q_full, qph);
      qph ^= 1u;
      tc_fence_after();
      if (lane == 0) {
        if (!mine) {
          // keep the shared K / V rings moving: release each stage after it has been filled
          for (int pass = 1; pass <= 2; ++pass)
            for (int kt = 0; kt < n_kt; ++kt) {
              mbar_wait(&S->k_full[kr.idx], kr.ph);
              mbar_arrive(&S->k_empty[kr.idx]);
              kr.next();
              if (pass == 1) {
                mbar_wait(&S->v_full[vr.idx], vr.ph);
                mbar_arrive(&S->v_empty[vr.idx]);
                vr.next();
              }
            }
          mbar_arrive(&S->q_empty);
        } else {
          // pass 1: S(0); then per tile S(kt+1), P.V(kt)
          auto issue_s_next = [&](bool transposed) {
            mbar_wait(&S->k_full[kr.idx], kr.ph);
            mbar_wait(&S->s_empty[w], sb.ph ^ 1u);
            tc_fence_after();
            mma_s(kr.idx, transposed);
            umma_commit(&S->k_empty[kr.idx]);
            sb.next();
            kr.next();
          };
          issue_s_next(false);
          if (w == 0) TRACE_R(1, 3, 0);
          mbar_wait(&S->o_empty[w], oph ^ 1u);
          oph ^= 1u;
          for (int kt = 0; kt < n_kt; ++kt) {
            if (kt + 1 < n_kt) {
              issue_s_next(false);
              if (w == 0) TRACE_R(1, 3, kt + 1);
            }
            mbar_wait(&S->v_full[vr.idx], vr.ph);
            mbar_wait(&S->p_full[w], pph);
            pph ^= 1u;
            tc_fence_after();
            const uint32_t sv = smem_u32(sV + vr.idx * 16384);
#pragma unroll
            for (int k = 0; k < 8; ++k)
              umma_ts(tmem + 256 + w * 64, tmem + 384 + w * 64 + k * 8, desc_sw128(sv + k * 2048, 0, 1024), idO,
                      (kt > 0 || k > 0) ? 1u : 0u);
            umma_commit(&S->p_free[w]);          // P_w may be rewritten, O_w is up to date
            umma_commit(&S->v_empty[vr.idx]);
            vr.next();
            if (w == 0) TRACE_R(1, 5 + w, kt);
          }
          umma_commit(&S->o_full[w]);
          // pass 2: S^T per tile
          for (int kt = 0; kt < n_kt; ++kt) {
            issue_s_next(true);
            if (w == 0) TRACE_R(1, 4, kt);
          }
          umma_commit(&S->q_empty);
        }
      }
      __syncwarp();   // lanes 1-31 only track q_full; the ring cursors live in lane 0
    }
  } else {
    // ---------------------------------------------------------------- softmax warpgroup wg (128 threads)
    const int wg = warp >> 2, t = tid & 127;
    const uint32_t lrow = uint32_t((warp & 3) * 32) << 16;
    const uint32_t s_base = tmem + lrow + wg * 128, o_base = tmem + lrow + 256 + wg * 64;
    const uint32_t p_base = tmem + lrow + 384 + wg * 64;
    const float cl2 = c.scale * kLog2e;
    float* sc_cmp = wg ? sc_cmp1 : sc_cmp0;
    float* lse_s = S->lse[wg];
    Ring sb(1);
    uint32_t fph = 1u, oph = 0;
    // MUFU ping-pong: the two warpgroups take turns in their exponential loops (named barriers 4 / 5),
    // so each loop runs at the full MUFU rate while the other warpgroup loads S, waits or stores.
    // Warpgroup 1 hands warpgroup 0 the first turn.
    if (kCmpP1PingPong && wg == 1 && n_rt >= 2) named_bar_arrive(4, 256);
    for (int pr = 0; pr < n_pair; ++pr) {
      const int rt = 2 * pr + wg;
      if (rt >= n_rt) break;                          // warpgroup 1 sits out the last, odd pair
      const int r = rt * kTile + t;
      const bool rvalid = r < rows;
      const bool duo = 2 * pr + 1 < n_rt;             // both warpgroups in this pair
      auto turn_begin = [&]() { if (duo) named_bar_sync(4 + wg, 256); };
      auto turn_end = [&]() { if (duo) named_bar_arrive(5 - wg, 256); };
      // ---- pass 1: online softmax, P -> TMEM, O += P V
      float m = -1e30f, l = 0.f;
      for (int kt = 0; kt < n_kt; ++kt) {
        mbar_wait(&S->s_full[wg], sb.ph);
        if (warp == 0) TRACE_R(2, 7, kt);
        tc_fence_after();
        const int nv = min(kTile, nk - kt * kTile);
        float v[128];
        tmem_ld32(s_base, v);
        tmem_ld32(s_base + 32, v + 32);
        tmem_ld32(s_base + 64, v + 64);
        tmem_ld32(s_base + 96, v + 96);
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(&S->s_empty[wg]);
        sb.next();
        if (nv < kTile) {
#pragma unroll
          for (int i = 0; i < 128; ++i) v[i] = i < nv ? v[i] : -INFINITY;   // padded keys: p = 0
        }
        const float mx = max128(v) * cl2;
        const bool bump = mx > m + kRescale;
        const float m_new = bump ? mx : m;
        const float alpha = ex2(m - m_new);           // 1 when the reference does not move
        // P_w(kt-1) consumed and O_w up to date
        mbar_wait(&S->p_free[wg], fph);
        fph ^= 1u;
        tc_fence_after();
        if (warp == 0) TRACE_R(2, 9, kt);
        l *= alpha;
        m = m_new;
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        if (kCmpP1PingPong) turn_begin();
#pragma unroll
        for (int cc = 0; cc < 128; cc += 32) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const float p0 = ex2(fmaf(v[cc + i], cl2, -m)), p1 = ex2(fmaf(v[cc + i + 1], cl2, -m));
            acc[(i >> 1) & 3] += p0 + p1;
            pk[i >> 1] = pack_f16(p0, p1);
          }
          tmem_st16(p_base + cc / 2, pk);
        }
        if (kCmpP1PingPong) turn_end();
        l += (acc[0] + acc[1]) + (acc[2] + acc[3]);
        // the reference max moved: rescale O_w (P.V(kt-1) has completed: p_free)
        if (kt > 0 && __any_sync(0xffffffffu, bump)) {
#pragma unroll
          for (int cc = 0; cc < kD; cc += 16) {
            float o[16];
            tmem_ld16(o_base + cc, o);
            tmem_wait_ld();
            uint32_t ou[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) ou[i] = __float_as_uint(o[i] * alpha);
            tmem_st16(o_base + cc, ou);
          }
        }
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&S->p_full[wg]);
        if (warp == 0) TRACE_R(2, 11, kt);
      }
      // ---- O = (sum_j p_j v_j) / l, LSE (log2 domain)
      const float lse2 = rvalid ? m + lg2(l) : INFINITY;   // padded rows: p = 0 in pass 2
      const float inv_l = 1.f / l;
      mbar_wait(&S->o_full[wg], oph);
      oph ^= 1u;
      tc_fence_after();
      float* oc = static_cast<float*>(c.o[0]) + int64_t(qrow0 + r) * kD;
#pragma unroll
      for (int cc = 0; cc < kD; cc += 32) {
        float o[32];
        tmem_ld32(o_base + cc, o);
        tmem_wait_ld();
        if (rvalid) {
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<float4*>(oc + cc + i) =
                make_float4(o[i] * inv_l, o[i + 1] * inv_l, o[i + 2] * inv_l, o[i + 3] * inv_l);
        }
      }
      tc_fence_before();
      mbar_arrive(&S->o_empty[wg]);
      if (rvalid) c.lse[0][qrow0 + r] = lse2;   // saved LSEs are log2-domain
      named_bar_sync(1 + wg, 128);     // this warpgroup's previous pass 2 finished reading lse_s
      lse_s[t] = lse2;
      named_bar_sync(1 + wg, 128);
      // ---- pass 2: thread = key; exact fp32 Eq. 8 column sums of exp2(S^T c - LSE)
      if constexpr (kTok > 0) {
        // per token (kTok consecutive rows): column sums -> tile buffer -> selection-block scores
        float* gsc = tok_scr + size_t(wg * kGT) * c.max_slc_b;
        int Bcur = 0;   // first selection block intersecting the current key tile (uniform)
        for (int kt = 0; kt < n_kt; ++kt) {
          const int k0 = kt * kTile, k1 = min(nk, k0 + kTile);
          const bool kvalid = k0 + t < nk;
          mbar_wait(&S->s_full[wg], sb.ph);
          tc_fence_after();
          float cs[kGT];
#pragma unroll
          for (int j = 0; j < kGT; ++j) cs[j] = 0.f;
#pragma unroll
          for (int c00 = 0; c00 < kTile; c00 += 32) {
            float v[32];
            tmem_ld32(s_base + c00, v);
            tmem_wait_ld();
            if (c00 == kTile - 32) {
              tc_fence_before();
              mbar_arrive(&S->s_empty[wg]);
            }
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              const float4 L = ld_shared_f4(&lse_s[c00 + i]);
              cs[(c00 + i) / kTok] += ex2(fmaf(v[i], cl2, -L.x));
              cs[(c00 + i + 1) / kTok] += ex2(fmaf(v[i + 1], cl2, -L.y));
              cs[(c00 + i + 2) / kTok] += ex2(fmaf(v[i + 2], cl2, -L.z));
              cs[(c00 + i + 3) / kTok] += ex2(fmaf(v[i + 3], cl2, -L.w));
            }
          }
          sb.next();
          float* bw = tbuf + (wg * 2 + (kt & 1)) * (kGT * 129);
#pragma unroll
          for (int j = 0; j < kGT; ++j) bw[j * 129 + t] = kvalid ? cs[j] : 0.f;
          named_bar_sync(1 + wg, 128);   // (also orders the previous tile's score updates)
          {   // the selection block holding key k0: binary search in the staged block starts (blocks non-empty)
            int hi = ns;
            while (hi - Bcur > 1) {
              const int mid = (Bcur + hi) >> 1;
              if (sbeg[mid] <= k0) Bcur = mid; else hi = mid;
            }
          }
          for (int pi = t;; pi += 128) {
            const int B = Bcur + pi / kGT, j = pi % kGT;
            if (B >= ns) break;
            const int a0 = sbeg[B];
            if (a0 >= k1) break;
            const int e0 = sbeg[B + 1];
            const int lo = max(a0, k0) - k0, hi = min(e0, k1) - k0;
            float sum = 0.f;
            for (int k = lo; k < hi; ++k) sum += bw[j * 129 + k];
            float* dst = gsc + size_t(j) * c.max_slc_b + B;
            if (a0 >= k0) *dst = sum;      // first tile of block B
            else *dst += sum;              // B continues from the previous tile
          }
        }
      } else
      for (int kt = 0; kt < n_kt; ++kt) {
        const bool kvalid = kt * kTile + t < nk;
        mbar_wait(&S->s_full[wg], sb.ph);
        if (warp == 0) TRACE_R(2, 8, kt);
        tc_fence_after();
        float cs[4] = {0.f, 0.f, 0.f, 0.f};
        if (kCmpP2PingPong) turn_begin();
#pragma unroll
        for (int c00 = 0; c00 < kTile; c00 += 32) {
          float v[32];
          tmem_ld32(s_base + c00, v);
          tmem_wait_ld();
          if (c00 == kTile - 32) {
            tc_fence_before();
            mbar_arrive(&S->s_empty[wg]);
          }
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 L = ld_shared_f4(&lse_s[c00 + i]);
            cs[0] += ex2(fmaf(v[i], cl2, -L.x));
            cs[1] += ex2(fmaf(v[i + 1], cl2, -L.y));
            cs[2] += ex2(fmaf(v[i + 2], cl2, -L.z));
            cs[3] += ex2(fmaf(v[i + 3], cl2, -L.w));
          }
        }
        if (kCmpP2PingPong) turn_end();
        sb.next();
        if (kvalid) sc_cmp[kt * kTile + t] += (cs[0] + cs[1]) + (cs[2] + cs[3]);
      }
    }
    if constexpr (kTok > 0) {
      // ---- per-token top-k: warp w takes tokens w, w + 8, ... (scores copied to shared memory when
      // they fit the freed tile buffers, else read in place from the scratch)
      __threadfence_block();
      named_bar_sync(3, 256);
      constexpr int kPerWarp = 4 * kGT * 129 / 8;
      float* wrow = tbuf + warp * kPerWarp;
      int* wch = tchosen + warp * 64;
      const int ntok = t1 - t0;
      const int Teff = min(c.T, ns);
      for (int j = warp; j < ntok; j += 8) {
        float* src = tok_scr + size_t(j) * c.max_slc_b;
        const int64_t qj = int64_t(Q + j) * c.h_kv + g;   // query block of token j (m_q = 1)
        if (c.save_scores)
          for (int B = lane; B < ns; B += 32) c.scores[qj * c.max_slc_b + B] = src[B];
        float* row = src;
        if (ns <= kPerWarp) {
          for (int B = lane; B < ns; B += 32) wrow[B] = src[B];
          row = wrow;
        }
        __syncwarp();
        if (Teff <= 8) {
          // one pass: every lane keeps its own top 8 (descending value, ascending index on ties: its
          // blocks are scanned in ascending order and only a strictly larger value moves ahead), then
          // Teff rounds of a warp argmax over the lanes' heads (same order), the winner pops its head
          float tv[8];
          int ti[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) { tv[k] = -2.f; ti[k] = 0x7fffffff; }
          for (int B = lane; B < ns; B += 32) {
            float v = row[B];
            int bi = B;
            if (v > tv[7]) {
#pragma unroll
              for (int k = 0; k < 8; ++k)
                if (v > tv[k]) {
                  const float fv = tv[k];
                  const int fi = ti[k];
                  tv[k] = v; ti[k] = bi;
                  v = fv; bi = fi;
                }
            }
          }
          for (int it = 0; it < Teff; ++it) {
            float best = tv[0];
            int bidx = ti[0];
#pragma unroll
            for (int o = 16; o; o >>= 1) {
              const float ov = __shfl_xor_sync(0xffffffffu, best, o);
              const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
              if (ov > best || (ov == best && oi < bidx)) { best = ov; bidx = oi; }
            }
            if ((bidx & 31) == lane && bidx == ti[0]) {   // the owner pops its head
#pragma unroll
              for (int k = 0; k < 7; ++k) { tv[k] = tv[k + 1]; ti[k] = ti[k + 1]; }
              tv[7] = -2.f; ti[7] = 0x7fffffff;
            }
            if (lane == 0) wch[it] = bidx;
          }
          __syncwarp();
        } else {
          for (int it = 0; it < Teff; ++it) {
            float best = -2.f;
            int bidx = 0x7fffffff;
            for (int B = lane; B < ns; B += 32) {
              const float v = row[B];
              if (v > best) { best = v; bidx = B; }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
              const float ov = __shfl_xor_sync(0xffffffffu, best, o);
              const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
              if (ov > best || (ov == best && oi < bidx)) { best = ov; bidx = oi; }
            }
            if (lane == 0) { wch[it] = bidx; row[bidx] = -1.f; }
            __syncwarp();
          }
        }
        if (lane == 0)
          for (int i = 1; i < Teff; ++i) {
            const int v = wch[i];
            int k = i - 1;
            while (k >= 0 && wch[k] > v) { wch[k + 1] = wch[k]; --k; }
            wch[k + 1] = v;
          }
        __syncwarp();
        for (int jj = lane; jj < c.T; jj += 32) c.I[qj * c.T + jj] = jj < Teff ? s0 + wch[jj] : -1;
        __syncwarp();
      }
    } else {
    // ---- Eq. 8 selection-block scores and top-k (both softmax warpgroups, 256 threads)
    named_bar_sync(3, 256);
    for (int B = tid; B < ns; B += 256) {
      float s = 0.f;
      for (int i = c.slc_cmp_begin[s0 + B]; i < c.slc_cmp_begin[s0 + B + 1]; ++i)
        s += sc_cmp0[i - c0] + sc_cmp1[i - c0];
      sc_slc[B] = s;
      if (c.save_scores) c.scores[(int64_t(Q) * c.h_kv + g) * c.max_slc_b + B] = s;
    }
    named_bar_sync(3, 256);
    const int Teff = min(c.T, ns);
    for (int it = 0; it < Teff; ++it) {
      float best = -2.f;
      int bidx = 0x7fffffff;
      for (int B = tid; B < ns; B += 256) {
        const float v = sc_slc[B];
        if (v > best) { best = v; bidx = B; }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
        if (ov > best || (ov == best && oi < bidx)) { best = ov; bidx = oi; }
      }
      if (lane == 0) { S->bv[warp] = best; S->bi[warp] = bidx; }
      named_bar_sync(3, 256);
      if (tid == 0) {
        float bb = S->bv[0];
        int ii = S->bi[0];
        for (int w = 1; w < 8; ++w)
          if (S->bv[w] > bb || (S->bv[w] == bb && S->bi[w] < ii)) { bb = S->bv[w]; ii = S->bi[w]; }
        S->chosen[it] = ii;
        sc_slc[ii] = -1.f;
      }
      named_bar_sync(3, 256);
    }
    if (tid == 0) {
      for (int i = 1; i < Teff; ++i) {
        const int v = S->chosen[i];
        int j = i - 1;
        while (j >= 0 && S->chosen[j] > v) { S->chosen[j + 1] = S->chosen[j]; --j; }
        S->chosen[j + 1] = v;
      }
    }
    named_bar_sync(3, 256);
    for (int j = tid; j < c.T; j += 256) c.I[(int64_t(Q) * c.h_kv + g) * c.T + j] = j < Teff ? s0 + S->chosen[j] : -1;
    }
  }
#ifdef SSA_TRACE
  if (TRACE_ON && (warp == 8 || warp == 9 || warp == 0)) {
    const int role = warp == 8 ? 0 : (warp == 9 ? 1 : 2);
    for (int i = 0; i < tr_n; ++i) g_trace[role][i] = S->trace[role][i];
    g_trace_cnt[role] = tr_n;
  }
#endif
  tc_fence_before();
  __syncthreads();
  if (warp == 9) tmem_dealloc<512>(tmem);
}

// ================================================================================================
// selection + window attention + gated sum
// ================================================================================================
// 352 threads, same roles as the compression kernel: warpgroups 0 / 1 own the two 128-row tiles of a
// row-tile pair (thread i <-> TMEM lane i), warp 8 = TMA producer, warps 9 / 10 = MMA issuers.
// Online softmax with lazy rescaling; P (fp16) goes to TMEM and O += P V runs with A from TMEM.
// TMEM per warpgroup w (256 columns at w * 256): S [0, 128) | P [128, 192) | O [192, 256).
// Key tiles: the T selected blocks (ascending), then the window (== the query block: m_win == m_q);
// at the branch boundary the selection O is normalised and stored, and O restarts from zero.
constexpr int kMaxTiles = 4 * 64 + 8;
constexpr int kMaxSegs = 2 * kMaxTiles + 8;
constexpr int kSwThreads = 352;
struct SwSmem {
  uint64_t q_full[2], q_empty[2], kv_full[kStages], kv_empty[kStages], s_full[2], s_empty[2], p_full[2], p_free[2],
      o_full[2], o_empty[2], p_half[2];
  uint32_t tmem;
  int n_tiles, n_slc_tiles;
  // packed key tiles: tile j = segments [tile_seg[j], tile_seg[j + 1]); segment = 8-row-aligned run of one
  // block's keys (seg_row: first key row; seg_dst_len: destination slot << 8 | rows), tile_mask = valid keys
  int tile_seg[kMaxTiles + 1];
  uint32_t tile_mask[kMaxTiles][4];
  int seg_row[kMaxSegs];
  int seg_dst_len[kMaxSegs];
  int blk_a0[kMaxTiles], blk_a1[kMaxTiles];   // key ranges of the selected blocks (T <= kMaxTiles)
  alignas(16) uint8_t gran_slot[kMaxTiles][16];   // selection slot of every 8-key granule (0xff: none / window)
};

// Per-warp staging of 32 rows x 64 fp32 (8 KB): the thread that owns a row (TMEM lane) writes it with
// 16-byte chunks XOR-swizzled by the row, then the warp reads it back two rows per instruction (lanes
// 0-15 row 2i, 16-31 row 2i+1) so every global access of the epilogue is a coalesced 512-byte row pair
// instead of 32 rows touched by one instruction (measured: the per-row form cost ~10 us per row-tile
// pair). Both directions are bank-conflict free.
__device__ __forceinline__ void stage_row(float* wbuf, int lane, const float* v, float scale, int c0, int n) {
#pragma unroll
  for (int j = 0; j < n; j += 4) {
    const int ch = (c0 + j) >> 2;
    *reinterpret_cast<float4*>(wbuf + lane * 64 + 4 * (ch ^ (lane & 15))) =
        make_float4(v[j] * scale, v[j + 1] * scale, v[j + 2] * scale, v[j + 3] * scale);
  }
}
__device__ __forceinline__ float4 staged_chunk(const float* wbuf, int rl, int ch) {
  return *reinterpret_cast<const float4*>(wbuf + rl * 64 + 4 * (ch ^ (rl & 15)));
}
// half-width staging (kEpiHalf): 32 rows x 32 fp32 (4 KB) per warp, chunks XOR-swizzled by row & 7; read back
// four rows per instruction (lanes 8i..8i+7 take row 4k+i), every global access a 128-B row segment
__device__ __forceinline__ void stage_row_h(float* wbuf, int lane, const float* v, float scale) {
#pragma unroll
  for (int j = 0; j < 32; j += 4)
    *reinterpret_cast<float4*>(wbuf + lane * 32 + 4 * ((j >> 2) ^ (lane & 7))) =
        make_float4(v[j] * scale, v[j + 1] * scale, v[j + 2] * scale, v[j + 3] * scale);
}
__device__ __forceinline__ float4 staged_h(const float* wbuf, int rl, int ch) {
  return *reinterpret_cast<const float4*>(wbuf + rl * 32 + 4 * (ch ^ (rl & 7)));
}

// kMask: the per-row union-slot masks of small query blocks (pertoken.cu); a separate instantiation so
// the query-block path carries none of its registers
template <bool kMask, bool kPartial = false>
__global__ void __launch_bounds__(kSwThreads, 1)
k_tc_slcwin_fwd(Ctx c, __grid_constant__ const CUtensorMap tmQ, __grid_constant__ const TmapSet4 tmK,
                __grid_constant__ const TmapSet4 tmV) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = sm;                          // 2 x 16 KB (row tiles of the pair)
  uint8_t* sKV = sm + 32768;                 // kStages x {K, V} 32 KB
  uint8_t* sEpi = sKV + kStages * 32768;     // epilogue staging: kEpiBytes / 8 per softmax warp
  SwSmem* S = reinterpret_cast<SwSmem*>(sEpi + kEpiBytes);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int Q = c.q_order[blockIdx.x], g = blockIdx.y;
  if (Q < c.q_begin || Q >= c.q_end) return;          // not owned by this shard (uniform per CTA)
#ifdef SSA_TRACE
  const unsigned long long stamp0 = gtimer();
#endif
  const int t0 = c.off[SSA_LEVEL_Q][Q], t1 = c.off[SSA_LEVEL_Q][Q + 1];
  if (t1 <= t0) return;                               // empty virtual query block (uniform per CTA)
  const int rows = (t1 - t0) * c.h_s;
  const int n_rt = (rows + kTile - 1) / kTile;
  const int n_pair = (n_rt + 1) / 2;
  const int qrow0 = (g * c.N + t0) * c.h_s;
  const int krow_g = g * c.N;

  if (warp == 0) {   // the selected blocks' key ranges, fetched by all lanes at once
    for (int j = lane; j < c.T; j += 32) {
      const int B = c.I[(int64_t(Q) * c.h_kv + g) * c.T + j];
      S->blk_a0[j] = B >= 0 ? c.off[SSA_LEVEL_SLC][B] : 0;
      S->blk_a1[j] = B >= 0 ? c.off[SSA_LEVEL_SLC][B + 1] : 0;
    }
    __syncwarp();
  }
  if (tid == 0) {
    // per-warpgroup Q slots: slot w is released by its MMA issuer once the pair's last S MMA has read it,
    // so the next pair's Q load overlaps the last tile's softmax, P.V and epilogue
    for (int w = 0; w < 2; ++w) { mbar_init(&S->q_full[w], 1); mbar_init(&S->q_empty[w], 1); }
    for (int i = 0; i < kStages; ++i) { mbar_init(&S->kv_full[i], 1); mbar_init(&S->kv_empty[i], 2); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&S->s_full[i], 1);
      mbar_init(&S->s_empty[i], 128);
      mbar_init(&S->p_full[i], 128);
      mbar_init(&S->p_half[i], 128);
      mbar_init(&S->p_free[i], 1);
      mbar_init(&S->o_full[i], 1);
      mbar_init(&S->o_empty[i], 128);
    }
    fence_barrier_init();
    // Key tiles: the selected blocks' keys packed back to back in 8-row granules (a block of n keys takes
    // ceil(n / 8) granules, so a 128-key tile mixes blocks instead of padding each block to 128), then
    // the window (= the query block) from a fresh tile. Granules are TMA boxes of 8..64 rows at 1024-B
    // aligned slots, so the 128-B swizzle pattern is the one a single 128-row box would produce.
    int n = 0, ns = 0, pos = kTile;
    uint32_t mk[4] = {0u, 0u, 0u, 0u};            // mask of the open tile, flushed when it closes
    auto flush = [&]() {
      if (n > 0) for (int w = 0; w < 4; ++w) S->tile_mask[n - 1][w] = mk[w];
    };
    auto add_block = [&](int a0, int a1, int slot) {
      const int len = a1 - a0, l8 = (len + 7) & ~7;
      for (int x = 0; x < l8 && n <= kMaxTiles;) {
        if (pos == kTile) {
          flush();
          if (n == kMaxTiles) { n = kMaxTiles + 1; break; }
          S->tile_seg[n] = ns;
          mk[0] = mk[1] = mk[2] = mk[3] = 0u;
          for (int gq = 0; gq < 16; ++gq) S->gran_slot[n][gq] = 0xffu;
          ++n;
          pos = 0;
        }
        const int take = min(l8 - x, kTile - pos), valid = max(0, min(take, len - x));
        for (int gq = pos / 8; gq < (pos + take) / 8; ++gq) S->gran_slot[n - 1][gq] = uint8_t(slot);
        if (ns < kMaxSegs) { S->seg_row[ns] = a0 + x; S->seg_dst_len[ns] = (pos << 8) | take; ++ns; }
#pragma unroll
        for (int w = 0; w < 4; ++w) {              // bits [pos, pos + valid) of the 128-bit mask
          const int lo = max(pos, 32 * w), hi = min(pos + valid, 32 * w + 32);
          if (hi > lo) mk[w] |= (hi - lo == 32 ? 0xffffffffu : ((1u << (hi - lo)) - 1u)) << (lo - 32 * w);
        }
        pos += take;
        x += take;
      }
    };
    for (int j = 0; j < c.T; ++j) add_block(S->blk_a0[j], S->blk_a1[j], j);   // (unselected: empty range)
    S->n_slc_tiles = min(n, kMaxTiles);
    pos = kTile;                                  // the window starts a fresh tile
    if (!c.no_win) {                              // the window holding the query block (SSA_NO_WINDOW: none)
      const int wb = c.tok_block[SSA_LEVEL_WIN][t0];
      add_block(c.off[SSA_LEVEL_WIN][wb], c.off[SSA_LEVEL_WIN][wb + 1], 0xff);
    }
    if (n <= kMaxTiles) flush();
    n = min(n, kMaxTiles);
    S->tile_seg[n] = ns;
    S->n_tiles = n;
  }
  // zero the K/V stages once: slots a packed tile leaves unfilled must hold finite values (P = 0 there)
  for (int i = tid; i < kStages * 32768 / 16; i += kSwThreads)
    *reinterpret_cast<uint4*>(sKV + 16 * i) = make_uint4(0u, 0u, 0u, 0u);
  fence_proxy_async_smem();
  if (warp == 8 && lane == 0) {
    tma_prefetch(&tmQ);
    for (int b = 0; b < 4; ++b) { tma_prefetch(&tmK.m[b]); tma_prefetch(&tmV.m[b]); }
  }
  if (warp == 9) tmem_alloc<512>(&S->tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S->tmem;
  const int n_tiles = S->n_tiles, n_slc_tiles = S->n_slc_tiles;
#ifdef SSA_TRACE
  int sw_n = 0;
#endif

  if (warp == 8) {
    // ---------------------------------------------------------------- TMA producer
    Ring kv(kStages);
    uint32_t qph[2] = {0u, 0u};
    for (int pr = 0; pr < n_pair; ++pr) {
      const bool duo = 2 * pr + 1 < n_rt;
      for (int w = 0; w < (duo ? 2 : 1); ++w) {
        mbar_wait(&S->q_empty[w], qph[w] ^ 1u);
        qph[w] ^= 1u;
        TRACE_SW(0, 1, pr * 2 + w);
        if (lane == 0) {
          mbar_expect_tx(&S->q_full[w], 16384u);
          tma_load_2d(sQ + w * 16384, &tmQ, &S->q_full[w], 0, qrow0 + (2 * pr + w) * kTile);
        }
        __syncwarp();
      }
      for (int j = 0; j < n_tiles; ++j) {
        mbar_wait(&S->kv_empty[kv.idx], kv.ph ^ 1u);
        if (lane == 0) {
          uint8_t* st = sKV + kv.idx * 32768;
          const int s0 = S->tile_seg[j], s1 = S->tile_seg[j + 1];
          uint32_t rows_in = 0;
          for (int q = s0; q < s1; ++q) rows_in += uint32_t(S->seg_dst_len[q] & 0xff);
          mbar_expect_tx(&S->kv_full[kv.idx], rows_in * 256u);
          for (int q = s0; q < s1; ++q) {
            const int dst = S->seg_dst_len[q] >> 8, len = S->seg_dst_len[q] & 0xff, src = krow_g + S->seg_row[q];
            for (int off = 0; off < len;) {   // boxes of 64 / 32 / 16 / 8 rows
              const int b = len - off >= 64 ? 0 : (len - off >= 32 ? 1 : (len - off >= 16 ? 2 : 3));
              tma_load_2d(st + (dst + off) * 128, &tmK.m[b], &S->kv_full[kv.idx], 0, src + off);
              tma_load_2d(st + 16384 + (dst + off) * 128, &tmV.m[b], &S->kv_full[kv.idx], 0, src + off);
              off += 64 >> b;
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
    const uint32_t idS = idesc_bf16(128, 128, false, false);
    const uint32_t idO = idesc_f16(128, 64, false, true);    // P from TMEM, V MN-major
    const uint32_t aQ = smem_u32(sQ + w * 16384);
    const uint32_t tS = tmem + w * 256, tP = tS + 128, tO = tS + 192;
    Ring kv(kStages), sb(1);
    uint32_t qph = 0, pph = 0, oph = 0;
    for (int pr = 0; pr < n_pair; ++pr) {
      const bool mine = w == 0 || 2 * pr + 1 < n_rt;
      if (mine) {
        mbar_wait(&S->q_full[w], qph);
        qph ^= 1u;
        tc_fence_after();
      }
      if (lane == 0) {
        if (!mine) {
          for (int j = 0; j < n_tiles; ++j) {   // keep the shared K/V ring moving
            mbar_wait(&S->kv_full[kv.idx], kv.ph);
            mbar_arrive(&S->kv_empty[kv.idx]);
            kv.next();
          }
        } else {
          Ring kv_pv = kv;
          int n_s = 0;
          auto issue_s = [&]() {
            mbar_wait(&S->kv_full[kv.idx], kv.ph);
            mbar_wait(&S->s_empty[w], sb.ph ^ 1u);
            tc_fence_after();
            const uint32_t sk = smem_u32(sKV + kv.idx * 32768);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_bf16(tS, desc_sw128(aQ + k * 32, 0, 1024), desc_sw128(sk + k * 32, 0, 1024), idS, k > 0);
            umma_commit(&S->s_full[w]);
            if (w == 0) TRACE_SW(1, 3, n_s);
            if (++n_s == n_tiles) umma_commit(&S->q_empty[w]);   // last S of the pair: Q slot w is free
            kv.next();
            sb.next();
          };
          issue_s();
          mbar_wait(&S->o_empty[w], oph ^ 1u);
          oph ^= 1u;
          for (int j = 0; j < n_tiles; ++j) {
            if (j + 1 < n_tiles) issue_s();
            const uint32_t sv = smem_u32(sKV + kv_pv.idx * 32768 + 16384);
            const bool fresh = j == 0 || j == n_slc_tiles;   // first tile of a branch: O restarts
            // P.V in two halves: keys 0-63 as soon as the softmax has stored them (mid-turn), keys 64-127
            // after the turn, so only the second half's MMAs sit between the turn and p_free
            mbar_wait(&S->p_half[w], pph);
            if (w == 0) TRACE_SW(1, 14, j);
            tc_fence_after();
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_ts(tO, tP + k * 8, desc_sw128(sv + k * 2048, 0, 1024), idO, (!fresh || k > 0) ? 1u : 0u);
            mbar_wait(&S->p_full[w], pph);
            if (w == 0) TRACE_SW(1, 13, j);
            pph ^= 1u;
            tc_fence_after();
#pragma unroll
            for (int k = 4; k < 8; ++k)
              umma_ts(tO, tP + k * 8, desc_sw128(sv + k * 2048, 0, 1024), idO, 1u);
            umma_commit(&S->p_free[w]);
            if (w == 0) TRACE_SW(1, 5, j);
            umma_commit(&S->kv_empty[kv_pv.idx]);
            kv_pv.next();
          }
          umma_commit(&S->o_full[w]);
        }
      }
      __syncwarp();   // the ring cursors live in lane 0
    }
  } else {
    // ---------------------------------------------------------------- softmax warpgroup wg
    const int wg = warp >> 2, t = tid & 127;
    const uint32_t lrow = uint32_t((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + lrow + wg * 256, tP = tS + 128, tO = tS + 192;
    const float cl2 = c.scale * kLog2e;
    Ring sb(1);
    uint32_t fph = 1u, oph = 0;
    if (kSwPingPong && wg == 1 && n_rt >= 2) named_bar_arrive(4, 256);   // warpgroup 0 takes the first turn
    for (int pr = 0; pr < n_pair; ++pr) {
      const int rt = 2 * pr + wg;
      if (rt >= n_rt) break;                          // warpgroup 1 sits out the last, odd pair
      const bool duo = 2 * pr + 1 < n_rt;
      const int r = rt * kTile + t;
      const bool rvalid = r < rows;
      const int64_t row = qrow0 + (rvalid ? r : 0);
      const int wrow0 = rt * kTile + (warp & 3) * 32;   // first row of this warp
      float* wbuf = reinterpret_cast<float*>(sEpi + wg * (kEpiBytes / 2) + (warp & 3) * (kEpiBytes / 8));
      if (wrow0 + lane < rows && !kPartial) {
        // pull this warp's O_cmp rows (HBM) and gates toward L2 now; the epilogue reads them a pair later
        const char* pc = reinterpret_cast<const char*>(static_cast<const float*>(c.o[0]) + (qrow0 + wrow0 + lane) * int64_t(kD));
        asm volatile("prefetch.global.L2 [%0];\n\tprefetch.global.L2 [%1];" :: "l"(pc), "l"(pc + 128));
        if ((lane & 7) == 0) asm volatile("prefetch.global.L2 [%0];" :: "l"(c.gs + (qrow0 + wrow0 + lane) * 3));
      }
      float lse_slc = 0.f;
      float m = -1e30f, l = 0.f;
      // small query blocks (virtual level): the selection slots this row's query block selected
      const int64_t mi = (int64_t(t0 + (rvalid ? r : 0) / c.h_s) * c.h_kv + g) * 2;
      const unsigned long long rm0 = (kMask && rvalid) ? c.umask[mi] : ~0ull, rm1 = (kMask && rvalid) ? c.umask[mi + 1] : ~0ull;
      for (int j = 0; j < n_tiles; ++j) {
        const bool fresh = j == 0 || j == n_slc_tiles;
        const bool closed = j == n_slc_tiles && j > 0;
        if (closed) {             // close the selection branch -> saved O_slc (fp32), after P.V(j-1)
          mbar_wait(&S->p_free[wg], fph);
          fph ^= 1u;
          tc_fence_after();
          const float inv = 1.f / l;
          float* os = static_cast<float*>(c.o[1]);
          if (kEpiHalf) {
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              float o[32];
              tmem_ld32(tO + 32 * hf, o);
              tmem_wait_ld();
              stage_row_h(wbuf, lane, o, inv);
              __syncwarp();
#pragma unroll 4
              for (int i = 0; i < 8; ++i) {
                const int rl = 4 * i + (lane >> 3), ch = lane & 7, rr = wrow0 + rl;
                if (rr < rows)
                  *reinterpret_cast<float4*>(os + (qrow0 + rr) * int64_t(kD) + 32 * hf + 4 * ch) = staged_h(wbuf, rl, ch);
              }
              __syncwarp();
            }
          } else {
#pragma unroll
            for (int cc = 0; cc < kD; cc += 32) {
              float o[32];
              tmem_ld32(tO + cc, o);
              tmem_wait_ld();
              stage_row(wbuf, lane, o, inv, cc, 32);
            }
            __syncwarp();
#pragma unroll 4
            for (int i = 0; i < 16; ++i) {
              const int rl = 2 * i + (lane >> 4), ch = lane & 15, rr = wrow0 + rl;
              if (rr < rows) *reinterpret_cast<float4*>(os + (qrow0 + rr) * int64_t(kD) + 4 * ch) = staged_chunk(wbuf, rl, ch);
            }
            __syncwarp();
          }
          lse_slc = m + lg2(l);
          m = -1e30f;
          l = 0.f;
        }
        if (warp == 0) TRACE_SW(2, 6, j);
        mbar_wait(&S->s_full[wg], sb.ph);
        if (warp == 0) TRACE_SW(2, 7, j);
        tc_fence_after();
        const uint32_t mk0 = S->tile_mask[j][0], mk1 = S->tile_mask[j][1], mk2 = S->tile_mask[j][2], mk3 = S->tile_mask[j][3];
        float v[128];
        tmem_ld32(tS, v);
        tmem_ld32(tS + 32, v + 32);
        tmem_ld32(tS + 64, v + 64);
        tmem_ld32(tS + 96, v + 96);
        tmem_wait_ld();
        if (warp == 0) TRACE_SW(2, 11, j);
        tc_fence_before();
        mbar_arrive(&S->s_empty[wg]);
        sb.next();
        if ((mk0 & mk1 & mk2 & mk3) != 0xffffffffu) {   // granule padding / unfilled slots: p = 0
          const uint32_t mk[4] = {mk0, mk1, mk2, mk3};
#pragma unroll
          for (int gr = 0; gr < kTile / 8; ++gr) {      // only granules with padding pay the selects
            const uint32_t bits = (mk[gr >> 2] >> (8 * (gr & 3))) & 0xffu;
            if (bits != 0xffu) {
#pragma unroll
              for (int i = 0; i < 8; ++i) v[8 * gr + i] = (bits >> i) & 1u ? v[8 * gr + i] : -INFINITY;
            }
          }
        }
        if (kMask && j < n_slc_tiles) {   // granules of blocks this row's query block did not select
          const uint4 gs4 = *reinterpret_cast<const uint4*>(&S->gran_slot[j][0]);
          const uint32_t gw[4] = {gs4.x, gs4.y, gs4.z, gs4.w};
#pragma unroll
          for (int gr = 0; gr < kTile / 8; ++gr) {
            const uint32_t slot = (gw[gr >> 2] >> (8 * (gr & 3))) & 0xffu;
            if (slot < 128u && !(((slot < 64u ? rm0 : rm1) >> (slot & 63u)) & 1ull)) {
#pragma unroll
              for (int i = 0; i < 8; ++i) v[8 * gr + i] = -INFINITY;
            }
          }
        }
        // the max first: it overlaps the wait for P.V(j-1) below
        // (a tile may hold no key of this row at all under a per-row mask: keep the max finite)
        const float mx0 = max128(v) * cl2;
        const float mx = kMask ? fmaxf(mx0, -1e30f) : mx0;
        const bool bump = fresh || mx > m + kRescale;
        const float m_new = bump ? mx : m;
        const float alpha = ex2(m - m_new);           // 1 when the reference does not move
        if (!closed) {   // P.V(j-1) complete: O is up to date and P may be rewritten
          mbar_wait(&S->p_free[wg], fph);
          fph ^= 1u;
          tc_fence_after();
        }
        if (warp == 0) TRACE_SW(2, 12, j);
        l *= alpha;
        m = m_new;
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        // the reference max moved inside a branch (rare): this warp rescales its rows of O after the turn and
        // only then releases the first P.V half, which reads O (P.V(j-1) has completed: p_free)
        const bool rescale = __any_sync(0xffffffffu, bump && !fresh);
        if (warp == 0) TRACE_SW(2, 8, j);
        if (kSwPingPong && duo) named_bar_sync(4 + wg, 256);
        if (warp == 0) TRACE_SW(2, 9, j);
#pragma unroll
        for (int cc = 0; cc < kTile; cc += 32) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const float p0 = ex2(fmaf(v[cc + i], cl2, -m)), p1 = ex2(fmaf(v[cc + i + 1], cl2, -m));
            acc[(i >> 1) & 3] += p0 + p1;
            pk[i >> 1] = pack_f16(p0, p1);
          }
          if (cc == 64 && !rescale) {   // keys 0-63 stored (their stores completed while these exps ran)
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&S->p_half[wg]);
          }
          tmem_st16(tP + cc / 2, pk);
        }
        if (kSwPingPong && duo) named_bar_arrive(5 - wg, 256);
        if (warp == 0) TRACE_SW(2, 10, j);
        l += (acc[0] + acc[1]) + (acc[2] + acc[3]);
        if (rescale) {
#pragma unroll
          for (int cc = 0; cc < kD; cc += 16) {
            float o[16];
            tmem_ld16(tO + cc, o);
            tmem_wait_ld();
            uint32_t ou[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) ou[i] = __float_as_uint(fresh ? o[i] : o[i] * alpha);
            tmem_st16(tO + cc, ou);
          }
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(&S->p_half[wg]);
        }
        tmem_wait_st();
        if (warp == 0) TRACE_SW(2, 15, j);
        tc_fence_before();
        mbar_arrive(&S->p_full[wg]);
      }
      const float* os_g = static_cast<const float*>(c.o[1]);
      const float* ocm_g = static_cast<const float*>(c.o[0]);
      float* ow = static_cast<float*>(c.o[c.no_win ? 1 : 2]);
      // gated sum of one staged 4-column chunk of row rr (Eq. 6), O_win (or O_slc under SSA_NO_WINDOW) stored
      auto combine = [&](int rr, int col, const float4& wn, const float4& sl_in, const float4& cm, const float* w3,
                         int dst) {
        const int64_t grow = qrow0 + rr;
        const float4 sl = c.no_win ? wn : sl_in;
        const float w0 = w3[0], w1 = w3[1], w2 = c.no_win ? 0.f : w3[2];
        *reinterpret_cast<float4*>(ow + grow * kD + col) = wn;
        if (kPartial) return;           // per-block selection pass: O and LSE only
        if (col >= c.Dc) return;             // zero-padded head dims (d = 32) are not output
        __nv_bfloat16* out = static_cast<__nv_bfloat16*>(c.out) + (int64_t(dst) * c.H + g * c.h_s + rr % c.h_s) * c.Dc + col;
        float4 y = make_float4(w0 * cm.x + w1 * sl.x + w2 * wn.x, w0 * cm.y + w1 * sl.y + w2 * wn.y,
                               w0 * cm.z + w1 * sl.z + w2 * wn.z, w0 * cm.w + w1 * sl.w + w2 * wn.w);
        if (c.accumulate) {   // SSA_ACCUMULATE: add to the caller's out (e.g. the shifted-window pass)
          const uint2 old = *reinterpret_cast<const uint2*>(out);
          const float2 a = unpack_bf16(old.x), b = unpack_bf16(old.y);
          y.x += a.x; y.y += a.y; y.z += b.x; y.w += b.y;
        }
        *reinterpret_cast<uint2*>(out) = make_uint2(pack_bf16(y.x, y.y), pack_bf16(y.z, y.w));
      };
      if (kEpiHalf) {
        // Epilogue (gated sum, Eq. 6), 32 columns at a time: the window output is staged through the warp's
        // 4 KB slot and read back four rows per instruction (lanes 8i..8i+7: row 4k+i, four columns each);
        // the gated sum's global operands (O_slc written at the branch close, O_cmp, gates, destination
        // rows) come in batches of four row quads, the first issued before O is ready.
        const int ch = lane & 7;
        float4 h_sl[4], h_cm[4];
        float h_w[4][3];
        int h_dst[4];
        auto epi_load_h = [&](int hf, int bt) {
          if (kPartial) return;
#pragma unroll
          for (int ii = 0; ii < 4; ++ii) {
            const int rl = 4 * (bt * 4 + ii) + (lane >> 3), rr = min(wrow0 + rl, rows - 1);   // clamp: valid memory
            const int64_t grow = qrow0 + rr;
            if (!c.no_win) h_sl[ii] = *reinterpret_cast<const float4*>(os_g + grow * kD + 32 * hf + 4 * ch);
            h_cm[ii] = *reinterpret_cast<const float4*>(ocm_g + grow * kD + 32 * hf + 4 * ch);
            h_w[ii][0] = c.gs[grow * 3];
            h_w[ii][1] = c.gs[grow * 3 + 1];
            h_w[ii][2] = c.gs[grow * 3 + 2];
            const int tok = t0 + rr / c.h_s;
            h_dst[ii] = c.sorted_input ? tok : c.perm[tok];
          }
        };
        epi_load_h(0, 0);
        if (warp == 0) TRACE_SW(2, 13, pr);
        mbar_wait(&S->o_full[wg], oph);
        oph ^= 1u;
        if (warp == 0) TRACE_SW(2, 14, pr);
        tc_fence_after();
        const float inv = 1.f / l;
        if (rvalid) {
          // window-only: keep the "no keys" sentinel of the selection LSE (api.cu); no-window: the O in
          // TMEM is the selection branch's (its tiles were the last ones)
          if (n_slc_tiles > 0 && !c.no_win) c.lse[1][row] = lse_slc;
          c.lse[c.no_win ? 1 : 2][row] = m + lg2(l);
        }
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          {
            float o[32];
            tmem_ld32(tO + 32 * hf, o);
            tmem_wait_ld();
            stage_row_h(wbuf, lane, o, inv);
          }
          if (hf == 1) {                 // O fully read: the next pair's P.V may overwrite it
            tc_fence_before();
            mbar_arrive(&S->o_empty[wg]);
          }
          __syncwarp();
          if (warp == 0) TRACE_SW(2, 0, pr);
#pragma unroll
          for (int bt = 0; bt < 2; ++bt) {
            if (hf + bt > 0) epi_load_h(hf, bt);
#pragma unroll
            for (int ii = 0; ii < 4; ++ii) {
              const int rl = 4 * (bt * 4 + ii) + (lane >> 3), rr = wrow0 + rl;
              if (rr < rows) combine(rr, 32 * hf + 4 * ch, staged_h(wbuf, rl, ch), h_sl[ii], h_cm[ii], h_w[ii], h_dst[ii]);
            }
          }
          __syncwarp();
        }
      } else {
        // Epilogue (gated sum, Eq. 6). The window output is staged through the warp's shared slot so every
        // global access is a coalesced row pair (lanes 0-15 / 16-31 take rows 2i / 2i+1, four columns
        // each); the gated sum's global operands (O_slc written at the branch close, O_cmp, gates,
        // destination rows) come in two batches of 8 row pairs, the first issued before O is ready.
        const int ch = lane & 15;
        float4 e_sl[8], e_cm[8];
        float e_w[8][3];
        int e_dst[8];
        auto epi_load = [&](int bt) {
          if (kPartial) return;
#pragma unroll
          for (int ii = 0; ii < 8; ++ii) {
            const int rl = 2 * (bt * 8 + ii) + (lane >> 4), rr = min(wrow0 + rl, rows - 1);   // clamp: valid memory
            const int64_t grow = qrow0 + rr;
            if (!c.no_win) e_sl[ii] = *reinterpret_cast<const float4*>(os_g + grow * kD + 4 * ch);
            e_cm[ii] = *reinterpret_cast<const float4*>(ocm_g + grow * kD + 4 * ch);
            e_w[ii][0] = c.gs[grow * 3];
            e_w[ii][1] = c.gs[grow * 3 + 1];
            e_w[ii][2] = c.gs[grow * 3 + 2];
            const int tok = t0 + rr / c.h_s;
            e_dst[ii] = c.sorted_input ? tok : c.perm[tok];
          }
        };
        epi_load(0);
        if (warp == 0) TRACE_SW(2, 13, pr);
        mbar_wait(&S->o_full[wg], oph);
        oph ^= 1u;
        if (warp == 0) TRACE_SW(2, 14, pr);
        tc_fence_after();
        const float inv = 1.f / l;
#pragma unroll
        for (int cc = 0; cc < kD; cc += 32) {
          float o[32];
          tmem_ld32(tO + cc, o);
          tmem_wait_ld();
          stage_row(wbuf, lane, o, inv, cc, 32);
        }
        tc_fence_before();
        mbar_arrive(&S->o_empty[wg]);
        if (rvalid) {
          if (n_slc_tiles > 0 && !c.no_win) c.lse[1][row] = lse_slc;
          c.lse[c.no_win ? 1 : 2][row] = m + lg2(l);
        }
        __syncwarp();
        if (warp == 0) TRACE_SW(2, 0, pr);
#pragma unroll
        for (int bt = 0; bt < 2; ++bt) {
          if (bt == 1) epi_load(1);
          if (warp == 0) TRACE_SW(2, 2 + 2 * bt, pr);
#pragma unroll
          for (int ii = 0; ii < 8; ++ii) {
            const int rl = 2 * (bt * 8 + ii) + (lane >> 4), rr = wrow0 + rl;
            if (rr < rows) combine(rr, 4 * ch, staged_chunk(wbuf, rl, ch), e_sl[ii], e_cm[ii], e_w[ii], e_dst[ii]);
          }
        }
      }
      __syncwarp();
      if (warp == 0) TRACE_SW(2, 15, pr);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) tmem_dealloc<512>(tmem);
#ifdef SSA_TRACE
  if (tid == 0 && blockIdx.x * gridDim.y + blockIdx.y < 2 * 4096) {
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    auto* st = g_cta_stamp[blockIdx.y * gridDim.x + blockIdx.x];
    st[0] = stamp0; st[1] = gtimer(); st[2] = smid;
  }
#endif
}

}  // namespace

bool tc_available() { return true; }

size_t tc_fwd_ws_bytes(int64_t N, int H, int h_kv, int D) {
  (void)H;
  // bf16 hi/lo K^cmp + fp16 V^cmp (n_cmp <= N) + fp16 copy of V
  return size_t(4) * size_t(h_kv) * size_t(N) * size_t(D) * 2 + 4 * 256;
}

// groups of GS consecutive query blocks (one token each, m_q = 1) of one batch item, inside the owned
// range [q_begin, q_end): cg[v] = [qa, qe), empty past the last group. One CTA.
__global__ void k_tok_groups(Ctx c, int GS, int32_t* __restrict__ pref, int32_t* __restrict__ cg, int bound) {
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int b = 0; b < c.batch; ++b) {
      pref[b] = acc;
      const int qa = max(c.bb[SSA_LEVEL_Q][b], c.q_begin), qe = min(c.bb[SSA_LEVEL_Q][b + 1], c.q_end);
      acc += qe > qa ? (qe - qa + GS - 1) / GS : 0;
    }
    pref[c.batch] = acc;
  }
  __syncthreads();
  const int total = pref[c.batch];
  for (int v = threadIdx.x; v < bound; v += blockDim.x) {
    if (v >= total) { cg[2 * v] = cg[2 * v + 1] = 0; continue; }
    int lo = 0, hi = c.batch;   // last item b with pref[b] <= v (non-empty: pref[b + 1] > v)
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (pref[mid] <= v) lo = mid; else hi = mid;
    }
    const int qb0 = max(c.bb[SSA_LEVEL_Q][lo], c.q_begin), qb1 = min(c.bb[SSA_LEVEL_Q][lo + 1], c.q_end);
    const int qa = qb0 + (v - pref[lo]) * GS;
    cg[2 * v] = qa;
    cg[2 * v + 1] = min(qa + GS, qb1);
  }
}

int tok_cmp_hs(int m_q, int h_s) {
  const char* e = getenv("SSA_TOK_CMP");       // A/B knob: 0 = CTA per query block also at m_q = 1
  if (e && atoi(e) == 0) return 0;
  return m_q == 1 && (h_s == 4 || h_s == 8 || h_s == 16) ? h_s : 0;
}
static int tok_bound(int n_q, int batch, int h_s) { return n_q / (2 * kTile / h_s) + batch + 1; }
size_t tok_cmp_ws_bytes(int n_q, int batch, int h_s, int max_slc_b) {
  if (h_s <= 0) return 0;
  return size_t(batch + 1) * 4 + 256 + size_t(tok_bound(n_q, batch, h_s)) * 8 + 256 +
         size_t(kTokSlots) * (2 * kTile / h_s) * max_slc_b * 4 + 256;
}
template <int kTok>
static size_t cmp_smem_bytes(const Ctx& c) {
  const size_t base = 1024 + 32768 + kCmpStages * 49152 + sizeof(CmpSmem) + 16;
  if (kTok == 0) return base + (2 * size_t(c.max_cmp_b) + c.max_slc_b) * sizeof(float);
  // tile buffers + chosen lists; at least 120 KB so that one CTA is resident per SM (per-SM scratch slot)
  return std::max<size_t>(base + (4 * (kTile / std::max(kTok, 1)) * 129 + 8 * 64 + size_t(c.max_slc_b) + 2) * 4,
                          120 * 1024);
}
template <int kTok>
static ssa_status launch_cmp(const Ctx& c, const TcArgs& a, const CUtensorMap& tmQ, const CUtensorMap& tmKh,
                             const CUtensorMap& tmKl, const CUtensorMap& tmVc, int grid, cudaStream_t st) {
  const size_t smem = cmp_smem_bytes<kTok>(c);
  if (smem > 232448) { set_error("compression tile state exceeds shared memory"); return SSA_ERR_UNSUPPORTED; }
  SSA_CUDA_TRY(cudaFuncSetAttribute(k_tc_cmp_fwd<kTok>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  ProfScope ps("tc_cmp_fwd", st);
  k_tc_cmp_fwd<kTok><<<dim3(grid, c.h_kv), kCmpThreads, smem, st>>>(a, tmQ, tmKh, tmKl, tmVc);
  SSA_LAUNCH_CHECK("k_tc_cmp_fwd");
  return SSA_OK;
}

bool tc_plan_ok(const ssa_plan_info& info, int top_k) {
  const size_t smem = 1024 + 32768 + kCmpStages * 49152 + sizeof(CmpSmem) + 16 +
                      (2 * size_t(info.max_blocks_per_batch[SSA_LEVEL_CMP]) + info.max_blocks_per_batch[SSA_LEVEL_SLC]) * 4;
  const int slc_tiles = (info.max_fill[SSA_LEVEL_SLC] + 95) / 96;      // dQ key tiles of 96 (tc_bwd.cu)
  const int dq_tiles = (info.max_blocks_per_batch[SSA_LEVEL_CMP] + 95) / 96 + top_k * slc_tiles + slc_tiles;
  return smem <= 232448 && dq_tiles <= 64 + 4 * 64 * 2 + 16 && top_k * ((info.max_fill[SSA_LEVEL_SLC] + 127) / 128) +
         (info.max_fill[SSA_LEVEL_SLC] + 127) / 128 <= 4 * 64 + 8;
}

ssa_status tc_forward(const Ctx& c, void* ws, cudaStream_t st, cudaEvent_t kv_ev, bool gather_keys_late) {
  const int n_cmp = c.n_blk[SSA_LEVEL_CMP];
  Carve cw(ws, tc_fwd_ws_bytes(c.N, c.H, c.h_kv, c.D));
  __nv_bfloat16* kc_hi = cw.take<__nv_bfloat16>(size_t(c.h_kv) * n_cmp * kD);
  __nv_bfloat16* kc_lo = cw.take<__nv_bfloat16>(size_t(c.h_kv) * n_cmp * kD);
  __half* vc = cw.take<__half>(size_t(c.h_kv) * n_cmp * kD);
  __half* vs16 = cw.take<__half>(size_t(c.h_kv) * c.N * kD);
  const int64_t n = int64_t(c.h_kv) * c.N * kD;   // >= h_kv * n_cmp * kD
  // raw k / v pending (cfg.kv_event, sharded mode 2): only the pooled keys are prepared before the
  // compression kernel; the wait, the key gather and the V conversion follow it
  const bool split = kv_ev != nullptr || gather_keys_late;
  if (split) {
    const int64_t nc = int64_t(c.h_kv) * n_cmp * kD;
    k_tc_prep<<<unsigned(std::max<int64_t>(1, (nc / 4 + 255) / 256)), 256, 0, st>>>(c, kc_hi, kc_lo, vc, vs16, 1);
  } else {
    k_tc_prep<<<unsigned((n / 4 + 255) / 256), 256, 0, st>>>(c, kc_hi, kc_lo, vc, vs16, 3);
  }
  SSA_LAUNCH_CHECK("k_tc_prep");
  CUtensorMap tmQ, tmKh, tmKl, tmVc;
  const uint64_t qrows = uint64_t(c.h_kv) * c.N * c.h_s, crows = uint64_t(c.h_kv) * n_cmp, krows = uint64_t(c.h_kv) * c.N;
  if (!make_tmap_bf16_2d(&tmQ, c.qs, qrows, kTile) || !make_tmap_bf16_2d(&tmKh, kc_hi, crows, kTile) ||
      !make_tmap_bf16_2d(&tmKl, kc_lo, crows, kTile) || !make_tmap_bf16_2d(&tmVc, vc, crows, kTile))
    return SSA_ERR_CUDA;
  TcArgs a{c, kc_hi, kc_lo, vc};
  const int nq = c.n_blk[SSA_LEVEL_Q];
  if (!c.win_only) {
    ssa_status s = SSA_OK;
    if (c.tok_cmp) {   // per-token compression: token groups, per-SM score scratch
      Carve tw(c.tok_ws, tok_cmp_ws_bytes(nq, c.batch, c.tok_cmp, c.max_slc_b));
      int32_t* pref = tw.take<int32_t>(c.batch + 1);
      const int bound = tok_bound(nq, c.batch, c.tok_cmp);
      int32_t* cg = tw.take<int32_t>(size_t(bound) * 2);
      a.c.tok_cg = cg;
      a.c.tok_sc = tw.take<float>(size_t(kTokSlots) * (2 * kTile / c.tok_cmp) * c.max_slc_b);
      k_tok_groups<<<1, 256, 0, st>>>(c, 2 * kTile / c.tok_cmp, pref, cg, bound);
      SSA_LAUNCH_CHECK("k_tok_groups");
      if (c.tok_cmp == 4) s = launch_cmp<4>(c, a, tmQ, tmKh, tmKl, tmVc, bound, st);
      else if (c.tok_cmp == 8) s = launch_cmp<8>(c, a, tmQ, tmKh, tmKl, tmVc, bound, st);
      else s = launch_cmp<16>(c, a, tmQ, tmKh, tmKl, tmVc, bound, st);
    } else {
      s = launch_cmp<0>(c, a, tmQ, tmKh, tmKl, tmVc, nq, st);
    }
    if (s != SSA_OK) return s;
  }
  if (split) {
    if (kv_ev) SSA_CUDA_TRY(cudaStreamWaitEvent(st, kv_ev, 0));
    if (c.n_peer > 0) {   // one-sided fetch of the selected blocks (needs this CTA grid's indices: done)
      ssa_status s = fetch_selected(c, true, st);
      if (s != SSA_OK) return s;
    }
    if (gather_keys_late) {
      ssa_status s = gather_inputs(c, true, st, false, /*rows=*/false, /*keys=*/true, /*gates=*/false);
      if (s != SSA_OK) return s;
    }
    k_tc_prep<<<unsigned((n / 4 + 255) / 256), 256, 0, st>>>(c, kc_hi, kc_lo, vc, vs16, 2);
    SSA_LAUNCH_CHECK("k_tc_prep(v)");
  }
  Ctx cv = c;   // query blocks smaller than the selection blocks: the virtual level (pertoken.cu)
  if (c.vq_ws) {
    ssa_status s = build_virtual_level(c, c.vq_S, c.vq_ws, st, &cv, /*plain=*/c.blk_ws != nullptr);
    if (s != SSA_OK) return s;
  }
  {
    const int nq = cv.n_blk[SSA_LEVEL_Q];
    const size_t smem = 1024 + 32768 + kStages * 32768 + kEpiBytes + sizeof(SwSmem);
    static_assert(1024 + 32768 + kStages * 32768 + kEpiBytes + sizeof(SwSmem) <= 232448, "selection/window shared memory");
    SSA_CUDA_TRY(cudaFuncSetAttribute(k_tc_slcwin_fwd<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    SSA_CUDA_TRY(cudaFuncSetAttribute(k_tc_slcwin_fwd<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    TmapSet4 tk, tv;
    for (int b = 0; b < 4; ++b)
      if (!make_tmap_bf16_2d(&tk.m[b], c.ks, krows, 64u >> b) || !make_tmap_bf16_2d(&tv.m[b], vs16, krows, 64u >> b))
        return SSA_ERR_CUDA;
    if (c.blk_ws) {
      // per-token selection: every (token, selected block) pair once (pertoken.cu), partial O / LSE merged
      // into O_slc / LSE_slc; the virtual level then runs the window branch + gated sum alone
      ProfScope pb("tc_slc_blk_fwd", st);
      BlkPass bp;
      ssa_status s = blk_build(c, c.blk_ws, st, &bp);
      if (s != SSA_OK) return s;
      const Ctx ce = blk_context(c, bp);
      CUtensorMap tmQe;
      if (!make_tmap_bf16_2d(&tmQe, bp.q_exp, uint64_t(bp.n_exp) * c.h_s, kTile)) return SSA_ERR_CUDA;
      SSA_CUDA_TRY(cudaFuncSetAttribute(k_tc_slcwin_fwd<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      k_tc_slcwin_fwd<false, true><<<dim3(unsigned(bp.bound), 1), kSwThreads, smem, st>>>(ce, tmQe, tk, tv);
      SSA_LAUNCH_CHECK("k_tc_slcwin_fwd(blocks)");
      if ((s = blk_merge(c, bp, st)) != SSA_OK) return s;
      // (the plain virtual level has empty selection lists and no slot masks: window + gated sum only)
    }
    ProfScope ps("tc_slc_win_fwd", st);
    if (cv.umask) k_tc_slcwin_fwd<true><<<dim3(nq, c.h_kv), kSwThreads, smem, st>>>(cv, tmQ, tk, tv);
    else k_tc_slcwin_fwd<false><<<dim3(nq, c.h_kv), kSwThreads, smem, st>>>(cv, tmQ, tk, tv);
    SSA_LAUNCH_CHECK("k_tc_slcwin_fwd");
  }
  return SSA_OK;
}

}  // namespace ssa

#ifdef SSA_TRACE
extern "C" int ssa_debug_trace_sw(unsigned long long* host, int cap) {
  int cnt[3];
  unsigned long long buf[3][512];
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(cnt, ssa::g_trace_sw_cnt, sizeof(cnt));
  cudaMemcpyFromSymbol(buf, ssa::g_trace_sw, sizeof(buf));
  int n = 0;
  for (int r = 0; r < 3; ++r)
    for (int i = 0; i < cnt[r] && n < cap; ++i) host[n++] = buf[r][i];
  return n;
}
extern "C" int ssa_debug_cta_stamps(unsigned long long* host, int n) {   // [n][3] start, end, smid
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(host, ssa::g_cta_stamp, size_t(n) * 3 * 8) == cudaSuccess ? n : -1;
}
extern "C" int ssa_debug_trace(unsigned long long* host, int cap) {
  int cnt[3];
  unsigned long long buf[3][128];
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(cnt, ssa::g_trace_cnt, sizeof(cnt));
  cudaMemcpyFromSymbol(buf, ssa::g_trace, sizeof(buf));
  int n = 0;
  for (int r = 0; r < 3; ++r)
    for (int i = 0; i < cnt[r] && n < cap; ++i) host[n++] = buf[r][i];
  return n;
}
#endif
