// learned.cu — SURVEY §8f row 2: the learned compression delta of Eq. 7 and the gate projection of
// Eq. 6, forward and backward (readings R17, R18).
//
//   Eq. 7, reading R17: k^cmp_B = (1/n_B) sum_{t in B} W[loc(t), g] (k_t + PE[loc(t), g]) + b[g]
//     — a sparse 3D convolution with kernel = stride = m_cmp (one weight matrix per intra-block offset,
//     grouped per kv head) over the active tokens, followed by the sparse mean pooling (division by the
//     active count). W [m^3][h_kv][d_out = d][d_in = d] fp32 applied as W x; b [h_kv][d] fp32.
//   Eq. 6 gates, reading R18: omega = sigmoid(x W_g + b_g), x [N][C] (caller order, dtype),
//     W_g [C][3 h_q] fp32 (column h*3 + c: head h, branch c), b_g [3 h_q] fp32.
//
// All reductions are in a fixed order (deterministic, no atomics).
#include <cfloat>

#include "internal.h"

namespace ssa {
namespace {

__device__ __forceinline__ float ldx(const float* p) { return *p; }
__device__ __forceinline__ float ldx(const __nv_bfloat16* p) { return __bfloat162float(*p); }
__device__ __forceinline__ void stx(float* p, float v) { *p = v; }
__device__ __forceinline__ void stx(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }
inline unsigned nb(int64_t n, int t) { return unsigned((n + t - 1) / t); }

__device__ __forceinline__ int local_offset(const Ctx& c, int p) {
  const int4 cc = reinterpret_cast<const int4*>(c.sorted_coords)[p];
  const int m = c.m_cmp;
  return ((cc.y % m) * m + (cc.z % m)) * m + (cc.w % m);
}

// ---------------------------------------------------------------------------------------------
// Tokens grouped by intra-block offset loc (R17 applies one weight matrix per offset): a stable
// counting sort of the plan positions by loc. Each compression block holds at most one token per
// offset, so the list of offset loc is "the token at loc of every block that has one", in plan order.
// One warp per chunk of kLocChunk tokens; ranks among equal offsets from __match_any_sync.
// ---------------------------------------------------------------------------------------------
constexpr int kLocChunk = 2048;
__global__ void k_loc_count(Ctx c, int n_chunk, int32_t* __restrict__ cnt_lm) {   // cnt_lm[loc][chunk]
  __shared__ int cnt[512];
  const int m3 = c.m_cmp * c.m_cmp * c.m_cmp, lane = threadIdx.x, ch = blockIdx.x;
  for (int l = lane; l < m3; l += 32) cnt[l] = 0;
  __syncwarp();
  const int t0 = ch * kLocChunk, t1 = min(c.N, t0 + kLocChunk);
  for (int b = t0; b < t1; b += 32) {
    const int t = b + lane;
    const int loc = t < t1 ? local_offset(c, t) : -1;
    const unsigned same = __match_any_sync(0xffffffffu, loc);
    if (loc >= 0 && lane == __ffs(same) - 1) cnt[loc] += __popc(same);
    __syncwarp();
  }
  for (int l = lane; l < m3; l += 32) cnt_lm[l * n_chunk + ch] = cnt[l];
}
__global__ void k_loc_scatter(Ctx c, int n_chunk, const int32_t* __restrict__ off_lm, int32_t* __restrict__ list) {
  __shared__ int cnt[512];
  const int m3 = c.m_cmp * c.m_cmp * c.m_cmp, lane = threadIdx.x, ch = blockIdx.x;
  for (int l = lane; l < m3; l += 32) cnt[l] = off_lm[l * n_chunk + ch];
  __syncwarp();
  const int t0 = ch * kLocChunk, t1 = min(c.N, t0 + kLocChunk);
  for (int b = t0; b < t1; b += 32) {
    const int t = b + lane;
    const int loc = t < t1 ? local_offset(c, t) : -1;
    const unsigned same = __match_any_sync(0xffffffffu, loc);
    if (loc >= 0) list[cnt[loc] + __popc(same & ((1u << lane) - 1u))] = t;
    __syncwarp();
    if (loc >= 0 && lane == __ffs(same) - 1) cnt[loc] += __popc(same);
    __syncwarp();
  }
}

// Forward learned conv (R17), grouped by offset: CTA per (loc, kv head, sub-range of the loc's token
// list), 128 threads. W[loc, g] of k and v staged transposed in shared memory (conflict-free: lane =
// output e); warp per token: y_t = W[loc] (x_t + PE[loc]) for k and v -> Y (fp32 [2][h_kv][N][D]).
constexpr int kConvSubs = 8;
template <class T>
__global__ void __launch_bounds__(128) k_conv_apply(Ctx c, const int32_t* __restrict__ loc_off,
                                                     const int32_t* __restrict__ list, float* __restrict__ Y) {
  constexpr int D = 64;
  __shared__ float wk[D][D + 1], wv[D][D + 1];     // [f][e]
  const int loc = blockIdx.x, g = blockIdx.y, sub = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t wo = (int64_t(loc) * c.h_kv + g) * D * D;
  for (int i = threadIdx.x; i < D * D; i += 128) {
    const int e = i / D, f = i % D;                // W[e][f] coalesced reads
    wk[f][e] = c.conv_kw[wo + i];
    wv[f][e] = c.conv_vw[wo + i];
  }
  __syncthreads();
  const int a0 = loc_off[loc], a1 = loc_off[loc + 1], len = a1 - a0;
  const int s0 = a0 + int(int64_t(len) * sub / kConvSubs), s1 = a0 + int(int64_t(len) * (sub + 1) / kConvSubs);
  const T* ks = static_cast<const T*>(c.ks);
  const T* vs = static_cast<const T*>(c.vs);
  const T* pek = static_cast<const T*>(c.pe_k);
  const T* pev = static_cast<const T*>(c.pe_v);
  const int64_t pi = (int64_t(loc) * c.h_kv + g) * D;
  const float pk0 = pek ? ldx(pek + pi + lane) : 0.f, pk1 = pek ? ldx(pek + pi + lane + 32) : 0.f;
  const float pv0 = pev ? ldx(pev + pi + lane) : 0.f, pv1 = pev ? ldx(pev + pi + lane + 32) : 0.f;
  const int64_t plane = int64_t(c.h_kv) * c.N * D;
  for (int i = s0 + warp; i < s1; i += 4) {
    const int t = list[i];
    const int64_t xi = (int64_t(g) * c.N + t) * D;
    const float xk0 = ldx(ks + xi + lane) + pk0, xk1 = ldx(ks + xi + lane + 32) + pk1;
    const float xv0 = ldx(vs + xi + lane) + pv0, xv1 = ldx(vs + xi + lane + 32) + pv1;
    float ak0 = 0.f, ak1 = 0.f, av0 = 0.f, av1 = 0.f;
#pragma unroll 16
    for (int f = 0; f < D; ++f) {
      const float fk = __shfl_sync(0xffffffffu, f < 32 ? xk0 : xk1, f & 31);
      const float fv = __shfl_sync(0xffffffffu, f < 32 ? xv0 : xv1, f & 31);
      ak0 += wk[f][lane] * fk;
      ak1 += wk[f][lane + 32] * fk;
      av0 += wv[f][lane] * fv;
      av1 += wv[f][lane + 32] * fv;
    }
    Y[xi + lane] = ak0;
    Y[xi + lane + 32] = ak1;
    Y[plane + xi + lane] = av0;
    Y[plane + xi + lane + 32] = av1;
  }
}
// ... then the sparse mean pooling of Y per compression block (+ bias): CTA per (block, kv head), D threads
__global__ void k_pool_y(Ctx c, const float* __restrict__ Y) {
  const int j = blockIdx.x, g = blockIdx.y, e = threadIdx.x;
  const int t0 = c.off[SSA_LEVEL_CMP][j], t1 = c.off[SSA_LEVEL_CMP][j + 1];
  const int64_t plane = int64_t(c.h_kv) * c.N * c.D;
  float sk = 0.f, sv = 0.f;
  for (int t = t0; t < t1; ++t) {
    const int64_t xi = (int64_t(g) * c.N + t) * c.D + e;
    sk += Y[xi];
    sv += Y[plane + xi];
  }
  const float inv = 1.f / float(t1 - t0);
  const int64_t o = (int64_t(g) * c.n_blk[SSA_LEVEL_CMP] + j) * c.D + e;
  static_cast<float*>(c.kc)[o] = sk * inv + (c.conv_kb ? c.conv_kb[g * c.D + e] : 0.f);
  static_cast<float*>(c.vc)[o] = sv * inv + (c.conv_vb ? c.conv_vb[g * c.D + e] : 0.f);
}

// dW of the learned conv (R17): CTA per (loc, kv head, sub-range of the loc's list), 256 threads;
// thread owns row e = tid / 4 and inputs f = (tid % 4) * 16 .. +16 of dW_k and dW_v; tokens in list
// order, 32 per shared-memory batch: part[sub][loc][g][e][f] += dy_B[e] (x_t + PE[loc])[f] / n_B.
template <class T>
__global__ void __launch_bounds__(256) k_conv_dw(Ctx c, const int32_t* __restrict__ loc_off,
                                                  const int32_t* __restrict__ list, float* __restrict__ part) {
  constexpr int D = 64;
  __shared__ float yk[32][D], yv[32][D], xk[32][D], xv[32][D];
  const int loc = blockIdx.x, g = blockIdx.y, sub = blockIdx.z, tid = threadIdx.x;
  const int e = tid >> 2, fb = (tid & 3) * 16;
  const T* ks = static_cast<const T*>(c.ks);
  const T* vs = static_cast<const T*>(c.vs);
  const T* pek = static_cast<const T*>(c.pe_k);
  const T* pev = static_cast<const T*>(c.pe_v);
  const int a0 = loc_off[loc], a1 = loc_off[loc + 1], len = a1 - a0;
  const int s0 = a0 + int(int64_t(len) * sub / kConvSubs), s1 = a0 + int(int64_t(len) * (sub + 1) / kConvSubs);
  float ak[16], av[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) ak[u] = av[u] = 0.f;
  for (int b0 = s0; b0 < s1; b0 += 32) {
    const int nb_ = min(32, s1 - b0);
    __syncthreads();
    for (int i = tid; i < nb_ * D; i += 256) {
      const int r = i / D, f = i % D, tt = list[b0 + r];
      const int j = c.tok_block[SSA_LEVEL_CMP][tt];
      const float inv = 1.f / float(c.off[SSA_LEVEL_CMP][j + 1] - c.off[SSA_LEVEL_CMP][j]);
      const int64_t yi = (int64_t(g) * c.n_blk[SSA_LEVEL_CMP] + j) * D + f;
      yk[r][f] = c.dkc[yi] * inv;
      yv[r][f] = c.dvc[yi] * inv;
      const int64_t xi = (int64_t(g) * c.N + tt) * D + f, pi = (int64_t(loc) * c.h_kv + g) * D + f;
      xk[r][f] = ldx(ks + xi) + (pek ? ldx(pek + pi) : 0.f);
      xv[r][f] = ldx(vs + xi) + (pev ? ldx(pev + pi) : 0.f);
    }
    __syncthreads();
    for (int r = 0; r < nb_; ++r) {
      const float a = yk[r][e], b = yv[r][e];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        ak[u] += a * xk[r][fb + u];
        av[u] += b * xv[r][fb + u];
      }
    }
  }
  const int64_t per = int64_t(c.m_cmp) * c.m_cmp * c.m_cmp * c.h_kv * D * D;   // one sub's slab (k part)
  const int64_t o = int64_t(sub) * 2 * per + ((int64_t(loc) * c.h_kv + g) * D + e) * D + fb;
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    part[o + u] = ak[u];
    part[o + per + u] = av[u];
  }
}
__global__ void k_conv_dw_reduce(Ctx c, const float* __restrict__ part) {
  const int64_t per = int64_t(c.m_cmp) * c.m_cmp * c.m_cmp * c.h_kv * c.D * c.D;
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= per) return;
  float sk = 0.f, sv = 0.f;
  for (int s = 0; s < kConvSubs; ++s) {
    sk += part[int64_t(s) * 2 * per + i];
    sv += part[int64_t(s) * 2 * per + per + i];
  }
  c.conv_dkw[i] = sk;
  c.conv_dvw[i] = sv;
}
// db of the learned conv: chunk partials over 64 compression blocks, then a fixed-order sum
__global__ void k_conv_db_part(Ctx c, float* __restrict__ part) {
  const int ch = blockIdx.x, g = blockIdx.y, e = threadIdx.x;
  const int j0 = ch * 64, j1 = min(c.n_blk[SSA_LEVEL_CMP], j0 + 64);
  float sk = 0.f, sv = 0.f;
  for (int j = j0; j < j1; ++j) {
    const int64_t yi = (int64_t(g) * c.n_blk[SSA_LEVEL_CMP] + j) * c.D + e;
    sk += c.dkc[yi];
    sv += c.dvc[yi];
  }
  const int64_t o = (int64_t(ch) * c.h_kv + g) * c.D * 2 + e;
  part[o] = sk;
  part[o + c.D] = sv;
}
__global__ void k_conv_db_reduce(Ctx c, const float* __restrict__ part, int n_ch) {
  const int g = blockIdx.x, e = threadIdx.x;
  float sk = 0.f, sv = 0.f;
  for (int ch = 0; ch < n_ch; ++ch) {
    const int64_t o = (int64_t(ch) * c.h_kv + g) * c.D * 2 + e;
    sk += part[o];
    sv += part[o + c.D];
  }
  if (c.conv_dkb) c.conv_dkb[g * c.D + e] = sk;
  if (c.conv_dvb) c.conv_dvb[g * c.D + e] = sv;
}

// ---------------------------------------------------------------------------------------------
// Gate projection GEMMs (R18), register-tiled SIMT (fp32 accumulate). J = 3 h_q <= 96.
//   proj: Z[p][col] = sum_f x[p][f] W_g[f][col]        (64 rows x J per CTA, 4 rows x 3 cols per thread)
//   dx:   dx[p][f]  = sum_col dz[p][col] W_g[f][col]   (64 rows x 64 f per CTA, 4 x 4 per thread)
//   dW:   dW[f][col] = sum_p x[p][f] dz[p][col]        (row-chunk partials, 64 f x J per CTA)
// dz / gates live in the internal [h_kv][N][h_s][3] layout: column col = h*3 + c of row p.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ int64_t gate_index(const Ctx& c, int p, int col) {
  const int h = col / 3, br = col - 3 * h, g = h / c.h_s, s = h - g * c.h_s;
  return ((int64_t(g) * c.N + p) * c.h_s + s) * 3 + br;
}
constexpr int kGK = 32;   // K step (features) of the proj GEMM
template <class T>
__global__ void __launch_bounds__(256) k_gate_proj(Ctx c) {
  __shared__ float xs[kGK][64 + 4];   // [f][row]
  __shared__ float ws[kGK][96];       // [f][col]
  const int J = 3 * c.H, tid = threadIdx.x;
  const int tr = tid / 32, tc = tid % 32;      // rows tr*4..+4? -> 8 x 4 = 32 rows... see below
  // thread tile: rows r0 = (tid / 32) * 8 .. +8, cols col = tc, tc + 32, tc + 64 (J <= 96)
  const int p0 = c.row_lo + blockIdx.x * 64;
  const T* x = static_cast<const T*>(c.gx);
  float acc[8][3];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) acc[a][b] = 0.f;
  for (int f0 = 0; f0 < c.gC; f0 += kGK) {
    __syncthreads();
    for (int i = tid; i < 64 * kGK; i += 256) {
      const int r = i / kGK, f = i % kGK, p = p0 + r;
      float v = 0.f;
      if (p < c.row_hi && f0 + f < c.gC) {
        const int src = c.sorted_input ? p : c.perm[p];
        v = ldx(x + (int64_t(src) - c.row_base) * c.gC + f0 + f);
      }
      xs[f][r] = v;
    }
    for (int i = tid; i < kGK * J; i += 256) {
      const int f = i / J, col = i % J;
      ws[f][col] = f0 + f < c.gC ? c.gw[int64_t(f0 + f) * J + col] : 0.f;
    }
    __syncthreads();
#pragma unroll 4
    for (int f = 0; f < kGK; ++f) {
      float xv[8], wv[3];
#pragma unroll
      for (int a = 0; a < 8; ++a) xv[a] = xs[f][tr * 8 + a];
#pragma unroll
      for (int b = 0; b < 3; ++b) wv[b] = tc + 32 * b < J ? ws[f][tc + 32 * b] : 0.f;
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) acc[a][b] += xv[a] * wv[b];
    }
  }
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    const int p = p0 + tr * 8 + a;
    if (p >= c.row_hi) continue;
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const int col = tc + 32 * b;
      if (col < J) c.gs[gate_index(c, p, col)] = 1.f / (1.f + __expf(-(acc[a][b] + c.gb[col])));
    }
  }
}

template <class T>
__global__ void __launch_bounds__(256) k_gate_dx(Ctx c) {
  __shared__ float dzs[96][64 + 4];   // [col][row]
  __shared__ float ws[96][32 + 4];    // [col][f] (32-feature chunks)
  const int J = 3 * c.H, tid = threadIdx.x;
  const int tr = tid / 16, tf = tid % 16;        // 16 x 16 threads, 4 rows x 2 features each
  const int p0 = c.row_lo + blockIdx.x * 64;
  for (int i = tid; i < 64 * J; i += 256) {
    const int r = i / J, col = i % J, p = p0 + r;
    dzs[col][r] = p < c.row_hi ? c.dz[gate_index(c, p, col)] : 0.f;
  }
  T* dx = static_cast<T*>(c.gdx);
  for (int f0 = 0; f0 < c.gC; f0 += 32) {
    __syncthreads();
    for (int i = tid; i < 32 * J; i += 256) {
      const int f = i / J, col = i % J;
      ws[col][f] = f0 + f < c.gC ? c.gw[int64_t(f0 + f) * J + col] : 0.f;
    }
    __syncthreads();
    float acc[4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a) acc[a][0] = acc[a][1] = 0.f;
    for (int col = 0; col < J; ++col) {
      float dv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) dv[a] = dzs[col][tr * 4 + a];
      const float w0 = ws[col][tf], w1 = ws[col][tf + 16];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        acc[a][0] += dv[a] * w0;
        acc[a][1] += dv[a] * w1;
      }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int p = p0 + tr * 4 + a;
      if (p >= c.row_hi) continue;
      const int dst = c.sorted_input ? p : c.perm[p];
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int f = f0 + tf + 16 * b;
        if (f < c.gC) stx(dx + (int64_t(dst) - c.row_base) * c.gC + f, acc[a][b]);
      }
    }
  }
}

// dW_g partials: grid (row chunks of kGateRowsPerChunk, C / 64); 64 features x J per CTA, thread =
// 4 features x 3 columns (col = tc, tc+32, tc+64); rows in order, 32 per shared-memory batch.
constexpr int kGateRowsPerChunk = 1024;
template <class T>
__global__ void __launch_bounds__(256) k_gate_dw(Ctx c, float* __restrict__ part, float* __restrict__ part_b) {
  __shared__ float xs[32][64 + 4];
  __shared__ float dzs[32][96];
  const int J = 3 * c.H, tid = threadIdx.x;
  const int tfr = tid / 32, tc = tid % 32;      // features tfr*8 .. +8 (8 x 8 = 64), cols tc + 32 b
  const int f0 = blockIdx.y * 64;
  const int r0 = c.row_lo + blockIdx.x * kGateRowsPerChunk;
  const int r1 = min(c.row_hi, r0 + kGateRowsPerChunk);
  const T* x = static_cast<const T*>(c.gx);
  float acc[8][3], accb[3] = {0.f, 0.f, 0.f};
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) acc[a][b] = 0.f;
  for (int pb = r0; pb < r1; pb += 32) {
    __syncthreads();
    for (int i = tid; i < 32 * 64; i += 256) {
      const int r = i / 64, f = i % 64, p = pb + r;
      float v = 0.f;
      if (p < r1 && f0 + f < c.gC) {
        const int src = c.sorted_input ? p : c.perm[p];
        v = ldx(x + (int64_t(src) - c.row_base) * c.gC + f0 + f);
      }
      xs[r][f] = v;
    }
    for (int i = tid; i < 32 * J; i += 256) {
      const int r = i / J, col = i % J, p = pb + r;
      dzs[r][col] = p < r1 ? c.dz[gate_index(c, p, col)] : 0.f;
    }
    __syncthreads();
#pragma unroll 4
    for (int r = 0; r < 32; ++r) {
      float xv[8], dv[3];
#pragma unroll
      for (int a = 0; a < 8; ++a) xv[a] = xs[r][tfr * 8 + a];
#pragma unroll
      for (int b = 0; b < 3; ++b) dv[b] = tc + 32 * b < J ? dzs[r][tc + 32 * b] : 0.f;
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) acc[a][b] += xv[a] * dv[b];
#pragma unroll
      for (int b = 0; b < 3; ++b) accb[b] += dv[b];
    }
  }
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    const int f = f0 + tfr * 8 + a;
    if (f >= c.gC) continue;
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const int col = tc + 32 * b;
      if (col < J) part[(int64_t(blockIdx.x) * c.gC + f) * J + col] = acc[a][b];
    }
  }
  if (blockIdx.y == 0 && tfr == 0)
#pragma unroll
    for (int b = 0; b < 3; ++b)
      if (tc + 32 * b < J) part_b[int64_t(blockIdx.x) * J + tc + 32 * b] = accb[b];
}
// dW_g = sum of the chunk partials in chunk order; db_g likewise
__global__ void k_gate_dw_reduce(Ctx c, const float* __restrict__ part, const float* __restrict__ part_b, int n_chunk) {
  const int J = 3 * c.H;
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < int64_t(c.gC) * J) {
    float s = 0.f;
    for (int k = 0; k < n_chunk; ++k) s += part[int64_t(k) * c.gC * J + i];
    c.gdw[i] = s;
  }
  if (i < J && c.gdb) {
    float s = 0.f;
    for (int k = 0; k < n_chunk; ++k) s += part_b[int64_t(k) * J + i];
    c.gdb[i] = s;
  }
}

}  // namespace

static int loc_chunks(int64_t N) { return int((N + kLocChunk - 1) / kLocChunk); }
static size_t loc_ws_bytes(int64_t N, int m3) {
  const int nch = std::max(1, loc_chunks(N));
  return size_t(m3) * nch * 4 * 2 + 1024 + size_t(N) * 4 + size_t(m3 + 1) * 4 + scan_ws_bytes(int64_t(m3) * nch) + 1024;
}
// per-offset token lists (stable counting sort by intra-block offset); returns list / loc_off
static ssa_status build_loc_lists(const Ctx& c, Carve& cw, int32_t** list_out, int32_t** off_out, cudaStream_t st) {
  const int m3 = c.m_cmp * c.m_cmp * c.m_cmp;
  const int nch = std::max(1, loc_chunks(c.N));
  int32_t* cnt = cw.take<int32_t>(size_t(m3) * nch + 1);
  int32_t* off = cw.take<int32_t>(size_t(m3) * nch + 1);
  int32_t* list = cw.take<int32_t>(size_t(c.N) + 1);
  int32_t* loc_off = cw.take<int32_t>(size_t(m3) + 1);
  void* sws = cw.take<char>(scan_ws_bytes(int64_t(m3) * nch));
  if (m3 > 512) { set_error("learned delta: m_cmp^3 must be <= 512"); return SSA_ERR_UNSUPPORTED; }
  k_loc_count<<<nch, 32, 0, st>>>(c, nch, cnt);
  SSA_LAUNCH_CHECK("k_loc_count");
  ssa_status s = exclusive_scan(cnt, off, int64_t(m3) * nch, off + int64_t(m3) * nch, sws, st);
  if (s != SSA_OK) return s;
  k_loc_scatter<<<nch, 32, 0, st>>>(c, nch, off, list);
  SSA_LAUNCH_CHECK("k_loc_scatter");
  // loc_off[l] = off[l * nch] (l < m3), loc_off[m3] = N
  SSA_CUDA_TRY(cudaMemcpy2DAsync(loc_off, 4, off, size_t(nch) * 4, 4, m3 + 1 > 0 ? m3 : 0, cudaMemcpyDeviceToDevice, st));
  SSA_CUDA_TRY(cudaMemcpyAsync(loc_off + m3, off + int64_t(m3) * nch, 4, cudaMemcpyDeviceToDevice, st));
  *list_out = list;
  *off_out = loc_off;
  return SSA_OK;
}

size_t learned_fwd_ws_bytes(const Ctx& c) {
  if (!c.conv_kw) return 0;
  const int m3 = c.m_cmp * c.m_cmp * c.m_cmp;
  return size_t(2) * c.h_kv * size_t(c.N) * c.D * 4 + loc_ws_bytes(c.N, m3) + 1024;
}

size_t gate_bwd_ws_bytes(int64_t N, int H, int C) {     // dz + dW_g / db_g chunk partials
  const int64_t chunks = (N + kGateRowsPerChunk - 1) / kGateRowsPerChunk + 1;
  return size_t(N) * H * 3 * 4 + size_t(chunks) * (size_t(C) + 1) * 3 * H * 4 + 2048;
}
size_t conv_bwd_ws_bytes(int64_t N, int h_kv, int m_cmp, int n_cmp, int D) {   // conv dW / db partials + lists
  const int m3 = m_cmp * m_cmp * m_cmp;
  return size_t(kConvSubs) * 2 * m3 * h_kv * D * D * 4 + loc_ws_bytes(N, m3) +
         size_t((n_cmp + 63) / 64 + 1) * h_kv * D * 2 * 4 + 2048;
}

ssa_status learned_checks(const Ctx& c) {
  if ((c.conv_kw || c.gx) && (c.D != 64 || c.Dc != 64)) { set_error("the learned delta / gate projection kernels need d == 64"); return SSA_ERR_UNSUPPORTED; }
  if (c.gx && (c.gC < 1 || c.H > 32)) {
    set_error("gate projection: h_q must be <= 32 and C >= 1");
    return SSA_ERR_UNSUPPORTED;
  }
  if (c.conv_kw && c.m_cmp * c.m_cmp * c.m_cmp > 512) { set_error("learned delta: m_cmp^3 must be <= 512"); return SSA_ERR_UNSUPPORTED; }
  return SSA_OK;
}

// forward: learned pool into c.kc / c.vc (replaces pool_forward); ws of learned_fwd_ws_bytes
ssa_status learned_pool_forward(const Ctx& c, bool bf16, void* ws, cudaStream_t st) {
  Carve cw(ws, learned_fwd_ws_bytes(c));
  float* Y = cw.take<float>(size_t(2) * c.h_kv * c.N * c.D);
  int32_t *list, *loc_off;
  ssa_status s = build_loc_lists(c, cw, &list, &loc_off, st);
  if (s != SSA_OK) return s;
  if (c.n_blk[SSA_LEVEL_CMP] == 0) return SSA_OK;
  const int m3 = c.m_cmp * c.m_cmp * c.m_cmp;
  ProfScope ps("k_pool_learned", st);
  if (bf16) k_conv_apply<__nv_bfloat16><<<dim3(m3, c.h_kv, kConvSubs), 128, 0, st>>>(c, loc_off, list, Y);
  else k_conv_apply<float><<<dim3(m3, c.h_kv, kConvSubs), 128, 0, st>>>(c, loc_off, list, Y);
  SSA_LAUNCH_CHECK("k_conv_apply");
  k_pool_y<<<dim3(c.n_blk[SSA_LEVEL_CMP], c.h_kv), c.D, 0, st>>>(c, Y);
  SSA_LAUNCH_CHECK("k_pool_y");
  return SSA_OK;
}

// forward: gates from the projection into c.gs (owned rows)
ssa_status gate_proj_forward(const Ctx& c, bool bf16, cudaStream_t st) {
  const int rows = c.row_hi - c.row_lo;
  if (rows <= 0) return SSA_OK;
  ProfScope ps("k_gate_proj", st);
  if (bf16) k_gate_proj<__nv_bfloat16><<<nb(rows, 64), 256, 0, st>>>(c);
  else k_gate_proj<float><<<nb(rows, 64), 256, 0, st>>>(c);
  SSA_LAUNCH_CHECK("k_gate_proj");
  return SSA_OK;
}

// backward of the gate projection (needs c.dz from the row prologue): dx, dW_g, db_g
ssa_status gate_proj_backward(const Ctx& c, bool bf16, void* part_ws, cudaStream_t st) {
  const int rows = c.row_hi - c.row_lo;
  const int J = 3 * c.H;
  if (c.gdx && rows > 0) {
    if (bf16) k_gate_dx<__nv_bfloat16><<<nb(rows, 64), 256, 0, st>>>(c);
    else k_gate_dx<float><<<nb(rows, 64), 256, 0, st>>>(c);
    SSA_LAUNCH_CHECK("k_gate_dx");
  }
  if (c.gdw) {
    const int n_chunk = std::max(1, (rows + kGateRowsPerChunk - 1) / kGateRowsPerChunk);
    float* part = static_cast<float*>(part_ws);
    float* part_b = part + size_t(n_chunk) * c.gC * J;
    if (rows > 0) {
      dim3 grid(n_chunk, (c.gC + 63) / 64);
      if (bf16) k_gate_dw<__nv_bfloat16><<<grid, 256, 0, st>>>(c, part, part_b);
      else k_gate_dw<float><<<grid, 256, 0, st>>>(c, part, part_b);
      SSA_LAUNCH_CHECK("k_gate_dw");
    } else {
      SSA_CUDA_TRY(cudaMemsetAsync(part, 0, size_t(c.gC + 1) * J * 4, st));
    }
    k_gate_dw_reduce<<<nb(int64_t(c.gC) * J, 256), 256, 0, st>>>(c, part, part_b, rows > 0 ? n_chunk : 1);
    SSA_LAUNCH_CHECK("k_gate_dw_reduce");
  }
  return SSA_OK;
}

// backward of the learned pool's parameters (needs c.dkc / c.dvc and the gathered keys c.ks / c.vs)
ssa_status learned_pool_backward_params(const Ctx& c, bool bf16, void* ws, cudaStream_t st) {
  const int m3 = c.m_cmp * c.m_cmp * c.m_cmp;
  Carve cw(ws, conv_bwd_ws_bytes(c.N, c.h_kv, c.m_cmp, c.n_blk[SSA_LEVEL_CMP], c.D));
  float* part = cw.take<float>(size_t(kConvSubs) * 2 * m3 * c.h_kv * c.D * c.D);
  int32_t *list, *loc_off;
  ssa_status s = build_loc_lists(c, cw, &list, &loc_off, st);
  if (s != SSA_OK) return s;
  if (c.conv_dkw && c.conv_dvw) {
    if (bf16) k_conv_dw<__nv_bfloat16><<<dim3(m3, c.h_kv, kConvSubs), 256, 0, st>>>(c, loc_off, list, part);
    else k_conv_dw<float><<<dim3(m3, c.h_kv, kConvSubs), 256, 0, st>>>(c, loc_off, list, part);
    SSA_LAUNCH_CHECK("k_conv_dw");
    k_conv_dw_reduce<<<nb(int64_t(m3) * c.h_kv * c.D * c.D, 256), 256, 0, st>>>(c, part);
    SSA_LAUNCH_CHECK("k_conv_dw_reduce");
  }
  if (c.conv_dkb || c.conv_dvb) {
    const int n_ch = std::max(1, (c.n_blk[SSA_LEVEL_CMP] + 63) / 64);
    float* pb = cw.take<float>(size_t(n_ch) * c.h_kv * c.D * 2);
    k_conv_db_part<<<dim3(n_ch, c.h_kv), c.D, 0, st>>>(c, pb);
    SSA_LAUNCH_CHECK("k_conv_db_part");
    k_conv_db_reduce<<<c.h_kv, c.D, 0, st>>>(c, pb, n_ch);
    SSA_LAUNCH_CHECK("k_conv_db_reduce");
  }
  return SSA_OK;
}

}  // namespace ssa
