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

// W [loc][g][e][f] -> Wt [loc][g][f][e] (so a warp's 32 lanes = 32 consecutive outputs e read one
// 128-B line per input f)
__global__ void k_transpose_w(const float* __restrict__ w, float* __restrict__ wt, int64_t mats, int D) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= mats * D * D) return;
  const int64_t mat = i / (D * D);
  const int r = int(i % (D * D)) / D, col = int(i % D);
  wt[mat * D * D + int64_t(col) * D + r] = w[i];
}

// Forward learned pool (R17): CTA per (compression block j, kv head g), 4 warps; warp w takes the
// block's tokens w, w+4, ...; lane owns outputs e = lane, lane + 32. Partial sums reduced over the 4
// warps in a fixed order. Inputs k / v from the internal [h_kv][N][D] layout (+ optional PE).
template <class T>
__global__ void __launch_bounds__(128) k_pool_learned(Ctx c, const float* __restrict__ wtk, const float* __restrict__ wtv) {
  constexpr int D = 64;
  __shared__ float red[4][2][D];
  const int j = blockIdx.x, g = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t0 = c.off[SSA_LEVEL_CMP][j], t1 = c.off[SSA_LEVEL_CMP][j + 1];
  const T* ks = static_cast<const T*>(c.ks);
  const T* vs = static_cast<const T*>(c.vs);
  const T* pek = static_cast<const T*>(c.pe_k);
  const T* pev = static_cast<const T*>(c.pe_v);
  float ak0 = 0.f, ak1 = 0.f, av0 = 0.f, av1 = 0.f;
  for (int t = t0 + warp; t < t1; t += 4) {
    const int loc = local_offset(c, t);
    const int64_t xi = (int64_t(g) * c.N + t) * D;
    float xk0 = ldx(ks + xi + lane), xk1 = ldx(ks + xi + lane + 32);
    float xv0 = ldx(vs + xi + lane), xv1 = ldx(vs + xi + lane + 32);
    const int64_t pi = (int64_t(loc) * c.h_kv + g) * D;
    if (pek) { xk0 += ldx(pek + pi + lane); xk1 += ldx(pek + pi + lane + 32); }
    if (pev) { xv0 += ldx(pev + pi + lane); xv1 += ldx(pev + pi + lane + 32); }
    const float* wk = wtk + (int64_t(loc) * c.h_kv + g) * D * D;
    const float* wv = wtv + (int64_t(loc) * c.h_kv + g) * D * D;
#pragma unroll 8
    for (int f = 0; f < D; ++f) {
      const float fk = __shfl_sync(0xffffffffu, f < 32 ? xk0 : xk1, f & 31);
      const float fv = __shfl_sync(0xffffffffu, f < 32 ? xv0 : xv1, f & 31);
      ak0 += wk[f * D + lane] * fk;
      ak1 += wk[f * D + lane + 32] * fk;
      av0 += wv[f * D + lane] * fv;
      av1 += wv[f * D + lane + 32] * fv;
    }
  }
  red[warp][0][lane] = ak0;
  red[warp][0][lane + 32] = ak1;
  red[warp][1][lane] = av0;
  red[warp][1][lane + 32] = av1;
  __syncthreads();
  if (threadIdx.x < 2 * D) {
    const int kv = threadIdx.x / D, e = threadIdx.x % D;
    const float s = ((red[0][kv][e] + red[1][kv][e]) + red[2][kv][e]) + red[3][kv][e];
    const float* bias = kv == 0 ? c.conv_kb : c.conv_vb;
    const float val = s / float(t1 - t0) + (bias ? bias[g * D + e] : 0.f);
    const int64_t o = (int64_t(g) * c.n_blk[SSA_LEVEL_CMP] + j) * D + e;
    static_cast<float*>(kv == 0 ? c.kc : c.vc)[o] = val;
  }
}

// Gate projection forward (R18): CTA per 32 rows p (plan order, owned range), 256 threads;
// x chunk [32][64] and W_g chunk [64][3H] staged in shared memory; omega written to the internal
// [h_kv][N][h_s][3] layout. Dynamic smem: (32 * 64 + 64 * 3H) floats.
template <class T>
__global__ void __launch_bounds__(256) k_gate_proj(Ctx c) {
  extern __shared__ float sm[];
  const int J = 3 * c.H;
  float* xs = sm;              // [32][64]
  float* ws = sm + 32 * 64;    // [64][J]
  const int p0 = c.row_lo + blockIdx.x * 32;
  const T* x = static_cast<const T*>(c.gx);
  float acc[12];
  const int per = (32 * J + 255) / 256;   // outputs per thread (<= 12 for h_q <= 32; checked on the host)
#pragma unroll
  for (int u = 0; u < 12; ++u) acc[u] = 0.f;
  for (int f0 = 0; f0 < c.gC; f0 += 64) {
    __syncthreads();
    for (int i = threadIdx.x; i < 32 * 64; i += 256) {
      const int r = i / 64, f = i % 64, p = p0 + r;
      float v = 0.f;
      if (p < c.row_hi && f0 + f < c.gC) {
        const int src = c.sorted_input ? p : c.perm[p];
        v = ldx(x + (int64_t(src) - c.row_base) * c.gC + f0 + f);
      }
      xs[i] = v;
    }
    for (int i = threadIdx.x; i < 64 * J; i += 256) {
      const int f = i / J;
      ws[i] = f0 + f < c.gC ? c.gw[int64_t(f0 + f) * J + i % J] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 12; ++u) {
      const int o = threadIdx.x + u * 256;
      if (u < per && o < 32 * J) {
        const int r = o / J, col = o % J;
        float a = acc[u];
#pragma unroll 16
        for (int f = 0; f < 64; ++f) a += xs[r * 64 + f] * ws[f * J + col];
        acc[u] = a;
      }
    }
  }
#pragma unroll
  for (int u = 0; u < 12; ++u) {
    const int o = threadIdx.x + u * 256;
    if (u < per && o < 32 * J) {
      const int r = o / J, col = o % J, p = p0 + r;
      if (p < c.row_hi) {
        const int h = col / 3, br = col % 3, g = h / c.h_s, s = h % c.h_s;
        const float z = acc[u] + c.gb[col];
        c.gs[((int64_t(g) * c.N + p) * c.h_s + s) * 3 + br] = 1.f / (1.f + __expf(-z));
      }
    }
  }
}

// dx = dz W_g^T: CTA per 32 rows, 256 threads; dz tile [32][J] and a W_g chunk [64][J] in shared
// memory; thread = (row, input feature) pairs of the chunk.
template <class T>
__global__ void __launch_bounds__(256) k_gate_dx(Ctx c) {
  extern __shared__ float sm[];
  const int J = 3 * c.H;
  float* dzs = sm;             // [32][J]
  float* ws = sm + 32 * J;     // [64][J]
  const int p0 = c.row_lo + blockIdx.x * 32;
  for (int i = threadIdx.x; i < 32 * J; i += 256) {
    const int r = i / J, col = i % J, p = p0 + r;
    const int h = col / 3, br = col % 3, g = h / c.h_s, s = h % c.h_s;
    dzs[i] = p < c.row_hi ? c.dz[((int64_t(g) * c.N + p) * c.h_s + s) * 3 + br] : 0.f;
  }
  T* dx = static_cast<T*>(c.gdx);
  for (int f0 = 0; f0 < c.gC; f0 += 64) {
    __syncthreads();
    for (int i = threadIdx.x; i < 64 * J; i += 256) {
      const int f = i / J;
      ws[i] = f0 + f < c.gC ? c.gw[int64_t(f0 + f) * J + i % J] : 0.f;
    }
    __syncthreads();
    for (int o = threadIdx.x; o < 32 * 64; o += 256) {
      const int r = o / 64, f = o % 64, p = p0 + r;
      if (p >= c.row_hi || f0 + f >= c.gC) continue;
      float a = 0.f;
      for (int col = 0; col < J; ++col) a += dzs[r * J + col] * ws[f * J + col];
      const int dst = c.sorted_input ? p : c.perm[p];
      stx(dx + (int64_t(dst) - c.row_base) * c.gC + f0 + f, a);
    }
  }
}

// dW_g partials: grid (row chunks, C / 64); CTA sums x[p][f0 + f] dz[p][col] over its chunk's rows
// (in row order) into part[chunk][f][col]; 256 threads x 12 outputs (J <= 48 per pass, looped).
constexpr int kGateRowsPerChunk = 1024;
template <class T>
__global__ void __launch_bounds__(256) k_gate_dw(Ctx c, float* __restrict__ part) {
  __shared__ float xs[32][64];
  __shared__ float dzs[32][48];
  const int J = 3 * c.H;
  const int f0 = blockIdx.y * 64;
  const int r0 = c.row_lo + blockIdx.x * kGateRowsPerChunk;
  const int r1 = min(c.row_hi, r0 + kGateRowsPerChunk);
  const T* x = static_cast<const T*>(c.gx);
  for (int c0 = 0; c0 < J; c0 += 48) {
    const int nc = min(48, J - c0);
    float acc[12];
#pragma unroll
    for (int u = 0; u < 12; ++u) acc[u] = 0.f;
    for (int pb = r0; pb < r1; pb += 32) {
      __syncthreads();
      for (int i = threadIdx.x; i < 32 * 64; i += 256) {
        const int r = i / 64, f = i % 64, p = pb + r;
        float v = 0.f;
        if (p < r1 && f0 + f < c.gC) {
          const int src = c.sorted_input ? p : c.perm[p];
          v = ldx(x + (int64_t(src) - c.row_base) * c.gC + f0 + f);
        }
        xs[r][f] = v;
      }
      for (int i = threadIdx.x; i < 32 * 48; i += 256) {
        const int r = i / 48, col = c0 + i % 48, p = pb + r;
        float v = 0.f;
        if (p < r1 && col < J) {
          const int h = col / 3, br = col % 3, g = h / c.h_s, s = h % c.h_s;
          v = c.dz[((int64_t(g) * c.N + p) * c.h_s + s) * 3 + br];
        }
        dzs[r][i % 48] = v;
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < 12; ++u) {
        const int o = threadIdx.x + u * 256;   // o in [0, 64 * 48)
        const int f = o / 48, col = o % 48;
        float a = acc[u];
#pragma unroll 8
        for (int r = 0; r < 32; ++r) a += xs[r][f] * dzs[r][col];
        acc[u] = a;
      }
    }
#pragma unroll
    for (int u = 0; u < 12; ++u) {
      const int o = threadIdx.x + u * 256;
      const int f = o / 48, col = o % 48;
      if (col < nc && f0 + f < c.gC)
        part[(int64_t(blockIdx.x) * c.gC + f0 + f) * J + c0 + col] = acc[u];
    }
  }
}
// dW_g = sum of the chunk partials in chunk order; db_g[col] = sum over the owned rows of dz (row order)
__global__ void k_gate_dw_reduce(Ctx c, const float* __restrict__ part, int n_chunk) {
  const int J = 3 * c.H;
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < int64_t(c.gC) * J) {
    float s = 0.f;
    for (int k = 0; k < n_chunk; ++k) s += part[int64_t(k) * c.gC * J + i];
    c.gdw[i] = s;
  }
  if (i < J && c.gdb) {
    const int h = int(i) / 3, br = int(i) % 3, g = h / c.h_s, s = h % c.h_s;
    float a = 0.f;
    for (int p = c.row_lo; p < c.row_hi; ++p) a += c.dz[((int64_t(g) * c.N + p) * c.h_s + s) * 3 + br];
    c.gdb[i] = a;
  }
}

// dW of the learned pool (R17): CTA per (intra-block offset loc, kv head g), 256 threads; thread owns
// row e = tid / 4 and inputs f = (tid % 4) * 16 .. +16 of both dW_k and dW_v. Tokens are scanned in
// plan order in windows of 256; those at offset loc are compacted in order (ballots) and accumulated
// in that order: dW[loc][g][e][f] += dy_B[e] (x_t + PE[loc])[f] / n_B.
template <class T>
__global__ void __launch_bounds__(256) k_conv_dw(Ctx c) {
  constexpr int D = 64;
  __shared__ int list[256];
  __shared__ int wcount[8];
  __shared__ float yk[32][D], yv[32][D], xk[32][D], xv[32][D];
  const int loc = blockIdx.x, g = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int e = tid >> 2, fb = (tid & 3) * 16;
  const T* ks = static_cast<const T*>(c.ks);
  const T* vs = static_cast<const T*>(c.vs);
  const T* pek = static_cast<const T*>(c.pe_k);
  const T* pev = static_cast<const T*>(c.pe_v);
  float ak[16], av[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) ak[u] = av[u] = 0.f;
  for (int w0 = 0; w0 < c.N; w0 += 256) {
    const int t = w0 + tid;
    const bool hit = t < c.N && local_offset(c, t) == loc;
    const unsigned bal = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) wcount[warp] = __popc(bal);
    __syncthreads();
    int base = 0, total = 0;
    for (int w = 0; w < 8; ++w) {
      if (w < warp) base += wcount[w];
      total += wcount[w];
    }
    if (hit) list[base + __popc(bal & ((1u << lane) - 1u))] = t;
    __syncthreads();
    for (int b0 = 0; b0 < total; b0 += 32) {
      const int nb_ = min(32, total - b0);
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
      __syncthreads();
    }
  }
  const int64_t o = ((int64_t(loc) * c.h_kv + g) * D + e) * D + fb;
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    c.conv_dkw[o + u] = ak[u];
    c.conv_dvw[o + u] = av[u];
  }
}
// db of the learned pool: db[g][e] = sum over compression blocks of dy (block order)
__global__ void k_conv_db(Ctx c) {
  const int g = blockIdx.x, e = threadIdx.x;
  float sk = 0.f, sv = 0.f;
  for (int j = 0; j < c.n_blk[SSA_LEVEL_CMP]; ++j) {
    const int64_t yi = (int64_t(g) * c.n_blk[SSA_LEVEL_CMP] + j) * c.D + e;
    sk += c.dkc[yi];
    sv += c.dvc[yi];
  }
  if (c.conv_dkb) c.conv_dkb[g * c.D + e] = sk;
  if (c.conv_dvb) c.conv_dvb[g * c.D + e] = sv;
}

}  // namespace

size_t learned_fwd_ws_bytes(const Ctx& c) {
  if (!c.conv_kw) return 0;
  return size_t(2) * c.m_cmp * c.m_cmp * c.m_cmp * c.h_kv * c.D * c.D * 4 + 512;
}

size_t learned_bwd_ws_bytes(int64_t N, int H, int h_kv, int C) {
  const int64_t rows = N * H;
  const int64_t chunks = (N + kGateRowsPerChunk - 1) / kGateRowsPerChunk + 1;   // as carved in api.cu
  return size_t(rows) * 3 * 4 + size_t(chunks) * size_t(C) * 3 * H * 4 + 1024;
}

ssa_status learned_checks(const Ctx& c) {
  if ((c.conv_kw || c.gx) && c.D != 64) { set_error("the learned delta / gate projection kernels need d == 64"); return SSA_ERR_UNSUPPORTED; }
  if (c.gx && (c.gC < 1 || c.H > 32)) {
    set_error("gate projection: h_q must be <= 32 and C >= 1");
    return SSA_ERR_UNSUPPORTED;
  }
  return SSA_OK;
}

// forward: learned pool into c.kc / c.vc (replaces pool_forward); ws of learned_fwd_ws_bytes
ssa_status learned_pool_forward(const Ctx& c, bool bf16, void* ws, cudaStream_t st) {
  const int64_t mats = int64_t(c.m_cmp) * c.m_cmp * c.m_cmp * c.h_kv;
  Carve cw(ws, learned_fwd_ws_bytes(c));
  float* wtk = cw.take<float>(size_t(mats) * c.D * c.D);
  float* wtv = cw.take<float>(size_t(mats) * c.D * c.D);
  k_transpose_w<<<nb(mats * c.D * c.D, 256), 256, 0, st>>>(c.conv_kw, wtk, mats, c.D);
  SSA_LAUNCH_CHECK("k_transpose_w");
  k_transpose_w<<<nb(mats * c.D * c.D, 256), 256, 0, st>>>(c.conv_vw, wtv, mats, c.D);
  SSA_LAUNCH_CHECK("k_transpose_w");
  if (c.n_blk[SSA_LEVEL_CMP] == 0) return SSA_OK;
  dim3 grid(c.n_blk[SSA_LEVEL_CMP], c.h_kv);
  ProfScope ps("k_pool_learned", st);
  if (bf16) k_pool_learned<__nv_bfloat16><<<grid, 128, 0, st>>>(c, wtk, wtv);
  else k_pool_learned<float><<<grid, 128, 0, st>>>(c, wtk, wtv);
  SSA_LAUNCH_CHECK("k_pool_learned");
  return SSA_OK;
}

// forward: gates from the projection into c.gs (owned rows)
ssa_status gate_proj_forward(const Ctx& c, bool bf16, cudaStream_t st) {
  const int rows = c.row_hi - c.row_lo;
  if (rows <= 0) return SSA_OK;
  const size_t smem = size_t(32 * 64 + 64 * 3 * c.H) * 4;
  ProfScope ps("k_gate_proj", st);
  if (bf16) {
    SSA_CUDA_TRY(cudaFuncSetAttribute(k_gate_proj<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    k_gate_proj<__nv_bfloat16><<<nb(rows, 32), 256, smem, st>>>(c);
  } else {
    SSA_CUDA_TRY(cudaFuncSetAttribute(k_gate_proj<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    k_gate_proj<float><<<nb(rows, 32), 256, smem, st>>>(c);
  }
  SSA_LAUNCH_CHECK("k_gate_proj");
  return SSA_OK;
}

// backward of the gate projection (needs c.dz from the row prologue): dx, dW_g, db_g
ssa_status gate_proj_backward(const Ctx& c, bool bf16, void* part_ws, cudaStream_t st) {
  const int rows = c.row_hi - c.row_lo;
  const int J = 3 * c.H;
  if (c.gdx && rows > 0) {
    const size_t smem = size_t(32 * J + 64 * J) * 4;
    if (bf16) {
      SSA_CUDA_TRY(cudaFuncSetAttribute(k_gate_dx<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      k_gate_dx<__nv_bfloat16><<<nb(rows, 32), 256, smem, st>>>(c);
    } else {
      SSA_CUDA_TRY(cudaFuncSetAttribute(k_gate_dx<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      k_gate_dx<float><<<nb(rows, 32), 256, smem, st>>>(c);
    }
    SSA_LAUNCH_CHECK("k_gate_dx");
  }
  if (c.gdw) {
    const int n_chunk = std::max(1, (rows + kGateRowsPerChunk - 1) / kGateRowsPerChunk);
    float* part = static_cast<float*>(part_ws);
    if (rows > 0) {
      dim3 grid(n_chunk, (c.gC + 63) / 64);
      if (bf16) k_gate_dw<__nv_bfloat16><<<grid, 256, 0, st>>>(c, part);
      else k_gate_dw<float><<<grid, 256, 0, st>>>(c, part);
      SSA_LAUNCH_CHECK("k_gate_dw");
    } else {
      SSA_CUDA_TRY(cudaMemsetAsync(part, 0, size_t(c.gC) * J * 4, st));
    }
    k_gate_dw_reduce<<<nb(int64_t(c.gC) * J, 256), 256, 0, st>>>(c, part, rows > 0 ? n_chunk : 1);
    SSA_LAUNCH_CHECK("k_gate_dw_reduce");
  }
  return SSA_OK;
}

// backward of the learned pool's parameters (needs c.dkc / c.dvc and the gathered keys c.ks / c.vs)
ssa_status learned_pool_backward_params(const Ctx& c, bool bf16, cudaStream_t st) {
  const int m3 = c.m_cmp * c.m_cmp * c.m_cmp;
  if (c.conv_dkw && c.conv_dvw) {
    if (bf16) k_conv_dw<__nv_bfloat16><<<dim3(m3, c.h_kv), 256, 0, st>>>(c);
    else k_conv_dw<float><<<dim3(m3, c.h_kv), 256, 0, st>>>(c);
    SSA_LAUNCH_CHECK("k_conv_dw");
  }
  if (c.conv_dkb || c.conv_dvb) {
    k_conv_db<<<c.h_kv, c.D, 0, st>>>(c);
    SSA_LAUNCH_CHECK("k_conv_db");
  }
  return SSA_OK;
}

}  // namespace ssa
