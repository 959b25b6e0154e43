// simt.cu — CUDA-core kernels of the SSA path: input permutation (a2), compression pool (a3, Eq. 7),
// gated combine (a8, Eq. 6), backward prologue/epilogue, inverse selection CSR, and the SIMT fp32
// attention kernels (a4-a7, a9). The SIMT attention kernels are the fp32 mode (SSA_F32; tolerance
// 1e-4 rules out TF32 tensor cores) and the SSA_FORCE_SIMT path; bf16 with d = 64 runs the tcgen05
// kernels in tc_fwd.cu / tc_bwd.cu.
//
// Internal layouts (plan-sorted token order p): rows  [h_kv][N][h_s][D]  (row = (p, s) of group g),
// keys [h_kv][N][D], compressed keys [h_kv][n_cmp][D], per-row fp32 stats [h_kv][N][h_s].
#include <cfloat>

#include "internal.h"

namespace ssa {
namespace {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

__device__ __forceinline__ float ld(const float* p) { return *p; }
__device__ __forceinline__ float ld(const __nv_bfloat16* p) { return __bfloat162float(*p); }
__device__ __forceinline__ void st(float* p, float v) { *p = v; }
__device__ __forceinline__ void st(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }

inline unsigned nblk(int64_t n, int t) { return unsigned((n + t - 1) / t); }

// ---------------------------------------------------------------------------------------------
// a2: gather caller tensors into the internal block-sorted layouts.
// ---------------------------------------------------------------------------------------------
// Both layouts keep the h_s heads of one (token, group) contiguous (h_s * D elements), so each thread
// moves 16 B with coalesced reads and writes.
template <class T>
__global__ void k_gather_rows(Ctx c, const T* __restrict__ src, T* __restrict__ dst) {
  const int per = c.h_s * c.D * int(sizeof(T)) / 16;     // 16-B chunks per (token, group)
  const int i = blockIdx.x * blockDim.x + threadIdx.x;   // 32-bit index math: N * H * D * esz / 16 < 2^31
  if (i >= c.N * c.h_kv * per) return;
  const int ch = i % per;
  const int g = (i / per) % c.h_kv;
  const int p = i / (per * c.h_kv);
  uint4* d4 = reinterpret_cast<uint4*>(dst + (int64_t(g) * c.N + p) * c.h_s * c.D);
  if (p < c.row_lo || p >= c.row_hi) {   // rows of other shards are never read; zeros keep the padded
    d4[ch] = make_uint4(0u, 0u, 0u, 0u); // tail of a row tile finite (TMA loads whole 128-row tiles)
    return;
  }
  const int src_p = c.sorted_input ? p : c.perm[p];
  if (c.Dc == c.D) {
    const uint4* s4 = reinterpret_cast<const uint4*>(src + (int64_t(src_p) * c.H + g * c.h_s) * c.D);
    d4[ch] = s4[ch];
  } else {   // caller head dim Dc < D: zero-padded heads (d = 32 on the tcgen05 path)
    const int hc = c.D * int(sizeof(T)) / 16, s = ch / hc, cc = ch % hc, e = cc * 16 / int(sizeof(T));
    d4[ch] = e < c.Dc ? *reinterpret_cast<const uint4*>(src + (int64_t(src_p) * c.H + g * c.h_s + s) * c.Dc + e)
                      : make_uint4(0u, 0u, 0u, 0u);
  }
}

template <class T>
__global__ void k_gather_keys(Ctx c, const T* __restrict__ k, const T* __restrict__ v, T* __restrict__ ks,
                              T* __restrict__ vs) {
  const int per = c.D * int(sizeof(T)) / 16;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= c.N * c.h_kv * per) return;
  const int ch = i % per;
  const int g = (i / per) % c.h_kv;
  const int p = i / (per * c.h_kv);
  const int src_p = c.sorted_input ? p : c.perm[p];
  const int64_t so = (int64_t(src_p) * c.h_kv + g) * c.Dc, dof = (int64_t(g) * c.N + p) * c.D;
  const int e = ch * 16 / int(sizeof(T));
  const bool in = e < c.Dc;                      // zero-padded heads when Dc < D (d = 32 on tcgen05)
  reinterpret_cast<uint4*>(ks + dof)[ch] = in ? *reinterpret_cast<const uint4*>(k + so + e) : make_uint4(0u, 0u, 0u, 0u);
  reinterpret_cast<uint4*>(vs + dof)[ch] = in ? *reinterpret_cast<const uint4*>(v + so + e) : make_uint4(0u, 0u, 0u, 0u);
}

template <class T>
__global__ void k_gather_gates(Ctx c, const T* __restrict__ gates, float* __restrict__ gs) {
  // one thread per (token, head): its 3 gates; 32-bit index math (N * H < 2^31)
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= c.N * c.H) return;
  const int h = i % c.H, p = i / c.H;
  const int g = h / c.h_s, s = h % c.h_s;
  if (p < c.row_lo || p >= c.row_hi) {                   // rows of other shards are never read
    float* z = gs + ((int64_t(g) * c.N + p) * c.h_s + s) * 3;
    z[0] = z[1] = z[2] = 0.f;
    return;
  }
  const int src_p = c.sorted_input ? p : c.perm[p];
  const T* src = gates + (int64_t(src_p) * c.H + h) * 3;
  float* dst = gs + ((int64_t(g) * c.N + p) * c.h_s + s) * 3;
  dst[0] = ld(src);
  dst[1] = ld(src + 1);
  dst[2] = ld(src + 2);
}

// ---------------------------------------------------------------------------------------------
// a3: compression pool, Eq. 7 with delta = masked mean (reading R4), optional intra-block PE.
// grid (n_cmp, h_kv), block D threads.
// ---------------------------------------------------------------------------------------------
template <class T>
__global__ void k_pool(Ctx c) {
  const int j = blockIdx.x, g = blockIdx.y, e = threadIdx.x;
  const int t0 = c.off[SSA_LEVEL_CMP][j], t1 = c.off[SSA_LEVEL_CMP][j + 1];
  const T* ks = static_cast<const T*>(c.ks);
  const T* vs = static_cast<const T*>(c.vs);
  const T* pek = static_cast<const T*>(c.pe_k);
  const T* pev = static_cast<const T*>(c.pe_v);
  const int m = c.m_cmp;
  float sk = 0.f, sv = 0.f;
  for (int p = t0; p < t1; ++p) {
    int64_t idx = (int64_t(g) * c.N + p) * c.D + e;
    float kk = ld(ks + idx), vv = ld(vs + idx);
    if (pek || pev) {
      const int4 cc = reinterpret_cast<const int4*>(c.sorted_coords)[p];
      int loc = ((cc.y % m) * m + (cc.z % m)) * m + (cc.w % m);
      int64_t pi = (int64_t(loc) * c.h_kv + g) * c.D + e;
      if (pek) kk += ld(pek + pi);
      if (pev) vv += ld(pev + pi);
    }
    sk += kk;
    sv += vv;
  }
  const float inv = 1.f / float(t1 - t0);
  int64_t o = (int64_t(g) * c.n_blk[SSA_LEVEL_CMP] + j) * c.D + e;
  static_cast<float*>(c.kc)[o] = sk * inv;
  static_cast<float*>(c.vc)[o] = sv * inv;
}

// ---------------------------------------------------------------------------------------------
// a4 + a5 (SIMT): compression attention (two passes) + Eq. 8 block scores + top-k, one CTA per
// (query block, kv group), query blocks in LPT order. Thread = row (t, s).
// ---------------------------------------------------------------------------------------------
constexpr int kRows = 128;
constexpr int kKT = 32;   // keys per smem tile

template <class T, int D>
__global__ void __launch_bounds__(kRows) k_cmp_fwd(Ctx c) {
  extern __shared__ float sm[];
  float* Kt = sm;                       // [kKT][D]
  float* Vt = Kt + kKT * D;             // [kKT][D]
  float* Pt = Vt + kKT * D;             // [kRows][kKT+1]
  float* red = Pt + kRows * (kKT + 1);  // [4][kKT]
  float* sc_cmp = red + 4 * kKT;        // [max_cmp_b]
  float* sc_slc = sc_cmp + c.max_cmp_b; // [max_slc_b]
  __shared__ float bv[kRows / 32];
  __shared__ int bi[kRows / 32];
  __shared__ int chosen[64];

  const int Q = c.q_order[blockIdx.x], g = blockIdx.y, tid = threadIdx.x;
  if (Q < c.q_begin || Q >= c.q_end) return;          // not owned by this shard
  const int t0 = c.off[SSA_LEVEL_Q][Q], t1 = c.off[SSA_LEVEL_Q][Q + 1];
  const int b = c.q_batch[Q];
  const int c0 = c.bb[SSA_LEVEL_CMP][b], c1 = c.bb[SSA_LEVEL_CMP][b + 1], nk = c1 - c0;
  const int s0 = c.bb[SSA_LEVEL_SLC][b], s1 = c.bb[SSA_LEVEL_SLC][b + 1], ns = s1 - s0;
  const int rows = (t1 - t0) * c.h_s;
  const T* qs = static_cast<const T*>(c.qs);
  const float* kc = static_cast<const float*>(c.kc);
  const float* vc = static_cast<const float*>(c.vc);
  const int n_cmp = c.n_blk[SSA_LEVEL_CMP];
  const float qscale = c.scale * kLog2e;
  for (int i = tid; i < nk; i += kRows) sc_cmp[i] = 0.f;
  const int64_t row_base = (int64_t(g) * c.N + t0) * c.h_s;

  for (int r0 = 0; r0 < rows; r0 += kRows) {
    const int r = r0 + tid;
    const bool valid = r < rows;
    float q[D];
#pragma unroll
    for (int e = 0; e < D; ++e) q[e] = valid ? ld(qs + (row_base + r) * D + e) * qscale : 0.f;
    // pass 1: log2-domain LSE over all compressed keys of the batch item
    float m = -FLT_MAX, l = 0.f;
    for (int k0 = 0; k0 < nk; k0 += kKT) {
      const int nt = min(kKT, nk - k0);
      __syncthreads();
      for (int i = tid; i < nt * D; i += kRows)
        Kt[i] = ld(kc + (int64_t(g) * n_cmp + c0 + k0) * D + i);
      __syncthreads();
      for (int j = 0; j < nt; ++j) {
        float x = 0.f;
#pragma unroll
        for (int e = 0; e < D; ++e) x += q[e] * Kt[j * D + e];
        float mn = fmaxf(m, x);
        l = l * exp2f(m - mn) + exp2f(x - mn);
        m = mn;
      }
    }
    const float lse2 = m + log2f(l);
    // pass 2: P = exp(S - LSE), O = P V, column sums of P into sc_cmp
    float o[D];
#pragma unroll
    for (int e = 0; e < D; ++e) o[e] = 0.f;
    for (int k0 = 0; k0 < nk; k0 += kKT) {
      const int nt = min(kKT, nk - k0);
      __syncthreads();
      for (int i = tid; i < nt * D; i += kRows) {
        Kt[i] = ld(kc + (int64_t(g) * n_cmp + c0 + k0) * D + i);
        Vt[i] = ld(vc + (int64_t(g) * n_cmp + c0 + k0) * D + i);
      }
      __syncthreads();
      for (int j = 0; j < kKT; ++j) {
        float p = 0.f;
        if (j < nt) {
          float x = 0.f;
#pragma unroll
          for (int e = 0; e < D; ++e) x += q[e] * Kt[j * D + e];
          p = valid ? exp2f(x - lse2) : 0.f;
#pragma unroll
          for (int e = 0; e < D; ++e) o[e] += p * Vt[j * D + e];
        }
        Pt[tid * (kKT + 1) + j] = p;
      }
      __syncthreads();
      {
        const int col = tid & (kKT - 1), part = tid / kKT;
        float s = 0.f;
        for (int i = part * 32; i < part * 32 + 32; ++i) s += Pt[i * (kKT + 1) + col];
        red[part * kKT + col] = s;
      }
      __syncthreads();
      if (tid < nt) sc_cmp[k0 + tid] += (red[tid] + red[kKT + tid]) + (red[2 * kKT + tid] + red[3 * kKT + tid]);
    }
    if (valid) {
      float* oc = static_cast<float*>(c.o[0]);
#pragma unroll
      for (int e = 0; e < D; ++e) oc[(row_base + r) * D + e] = o[e];
      c.lse[0][row_base + r] = lse2;   // saved LSEs are log2-domain
    }
  }
  __syncthreads();
  // Eq. 8: selection-block score = sum over its compression blocks (contiguous range)
  for (int B = tid; B < ns; B += kRows) {
    float s = 0.f;
    for (int i = c.slc_cmp_begin[s0 + B]; i < c.slc_cmp_begin[s0 + B + 1]; ++i) s += sc_cmp[i - c0];
    sc_slc[B] = s;
    if (c.save_scores) c.scores[(int64_t(Q) * c.h_kv + g) * c.max_slc_b + B] = s;
  }
  __syncthreads();
  // top-k: T rounds of block argmax (value desc, index asc); scores >= 0 so -1 marks "taken"
  const int Teff = min(c.T, ns);
  for (int it = 0; it < Teff; ++it) {
    float best = -2.f;
    int bidx = 0x7fffffff;
    for (int B = tid; B < ns; B += kRows) {
      float v = sc_slc[B];
      if (v > best) { best = v; bidx = B; }   // strided ascending scan keeps the lowest index on ties
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      float ov = __shfl_xor_sync(0xffffffffu, best, o);
      int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
      if (ov > best || (ov == best && oi < bidx)) { best = ov; bidx = oi; }
    }
    if ((tid & 31) == 0) { bv[tid >> 5] = best; bi[tid >> 5] = bidx; }
    __syncthreads();
    if (tid == 0) {
      float bb = bv[0];
      int ii = bi[0];
      for (int w = 1; w < kRows / 32; ++w)
        if (bv[w] > bb || (bv[w] == bb && bi[w] < ii)) { bb = bv[w]; ii = bi[w]; }
      chosen[it] = ii;
      sc_slc[ii] = -1.f;
    }
    __syncthreads();
  }
  if (tid == 0) {
    for (int i = 1; i < Teff; ++i) {   // ascending block index
      int v = chosen[i], j = i - 1;
      while (j >= 0 && chosen[j] > v) { chosen[j + 1] = chosen[j]; --j; }
      chosen[j + 1] = v;
    }
  }
  __syncthreads();
  for (int j = tid; j < c.T; j += kRows)
    c.I[(int64_t(Q) * c.h_kv + g) * c.T + j] = j < Teff ? s0 + chosen[j] : -1;
}

// ---------------------------------------------------------------------------------------------
// a6 / a7 (SIMT): single-pass online-softmax attention over a list of key segments.
// mode 1 = selection (CTA per (query block, g), segments = selected blocks I, Alg. 1),
// mode 2 = window    (CTA per (window, g), one segment = the window itself).
// ---------------------------------------------------------------------------------------------
template <class T, int D>
__global__ void __launch_bounds__(kRows) k_attn_fwd(Ctx c, int mode) {
  __shared__ float Kt[kKT * D];
  __shared__ float Vt[kKT * D];
  __shared__ int seg_s[64], seg_e[64];
  __shared__ int nseg;
  const int g = blockIdx.y, tid = threadIdx.x;
  int t0, t1;
  if (mode == 1) {
    const int Q = c.q_order[blockIdx.x];
    if (Q < c.q_begin || Q >= c.q_end) return;
    t0 = c.off[SSA_LEVEL_Q][Q];
    t1 = c.off[SSA_LEVEL_Q][Q + 1];
    if (tid == 0) {
      int n = 0;
      for (int j = 0; j < c.T; ++j) {
        int B = c.I[(int64_t(Q) * c.h_kv + g) * c.T + j];
        if (B >= 0) { seg_s[n] = c.off[SSA_LEVEL_SLC][B]; seg_e[n] = c.off[SSA_LEVEL_SLC][B + 1]; ++n; }
      }
      nseg = n;
    }
  } else {
    const int W = blockIdx.x;
    if (c.q_end - c.q_begin < c.n_blk[SSA_LEVEL_Q] && (W < c.q_begin || W >= c.q_end)) return;  // m_win == m_q
    t0 = c.off[SSA_LEVEL_WIN][W];
    t1 = c.off[SSA_LEVEL_WIN][W + 1];
    if (tid == 0) { seg_s[0] = t0; seg_e[0] = t1; nseg = 1; }
  }
  __syncthreads();
  const int rows = (t1 - t0) * c.h_s;
  const T* qs = static_cast<const T*>(c.qs);
  const T* ks = static_cast<const T*>(c.ks);
  const T* vs = static_cast<const T*>(c.vs);
  const float qscale = c.scale * kLog2e;
  const int64_t row_base = (int64_t(g) * c.N + t0) * c.h_s;
  const int br = mode;  // branch index: 1 = slc, 2 = win
  for (int r0 = 0; r0 < rows; r0 += kRows) {
    const int r = r0 + tid;
    const bool valid = r < rows;
    float q[D], o[D];
#pragma unroll
    for (int e = 0; e < D; ++e) {
      q[e] = valid ? ld(qs + (row_base + r) * D + e) * qscale : 0.f;
      o[e] = 0.f;
    }
    float m = -FLT_MAX, l = 0.f;
    for (int sgi = 0; sgi < nseg; ++sgi) {
      for (int k0 = seg_s[sgi]; k0 < seg_e[sgi]; k0 += kKT) {
        const int nt = min(kKT, seg_e[sgi] - k0);
        __syncthreads();
        for (int i = tid; i < nt * D; i += kRows) {
          Kt[i] = ld(ks + (int64_t(g) * c.N + k0) * D + i);
          Vt[i] = ld(vs + (int64_t(g) * c.N + k0) * D + i);
        }
        __syncthreads();
        for (int j = 0; j < nt; ++j) {
          float x = 0.f;
#pragma unroll
          for (int e = 0; e < D; ++e) x += q[e] * Kt[j * D + e];
          float mn = fmaxf(m, x);
          float a = exp2f(m - mn), p = exp2f(x - mn);
          l = l * a + p;
#pragma unroll
          for (int e = 0; e < D; ++e) o[e] = o[e] * a + p * Vt[j * D + e];
          m = mn;
        }
      }
    }
    if (valid) {
      const float inv = 1.f / l;
      float* ob = static_cast<float*>(c.o[br]);
#pragma unroll
      for (int e = 0; e < D; ++e) ob[(row_base + r) * D + e] = o[e] * inv;
      c.lse[br][row_base + r] = m + log2f(l);
    }
  }
}

// ---------------------------------------------------------------------------------------------
// a8: gated sum (Eq. 6) + scatter to caller order. Thread per (p, h, e).
// ---------------------------------------------------------------------------------------------
template <class T>
__global__ void k_combine(Ctx c) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  int64_t total = int64_t(c.N) * c.H * c.D;
  if (i >= total) return;
  int e = int(i % c.D);
  int h = int((i / c.D) % c.H);
  int p = int(i / (int64_t(c.D) * c.H));
  int g = h / c.h_s, s = h % c.h_s;
  if (p < c.off[SSA_LEVEL_Q][c.q_begin] || p >= c.off[SSA_LEVEL_Q][c.q_end]) return;
  int64_t row = (int64_t(g) * c.N + p) * c.h_s + s;
  const float* w = c.gs + row * 3;
  float v = w[0] * static_cast<const float*>(c.o[0])[row * c.D + e] +
            w[1] * static_cast<const float*>(c.o[1])[row * c.D + e] +
            w[2] * static_cast<const float*>(c.o[2])[row * c.D + e];
  int dst = c.sorted_input ? p : c.perm[p];
  st(static_cast<T*>(c.out) + (int64_t(dst) * c.H + h) * c.D + e, v);
}

// ---------------------------------------------------------------------------------------------
// Backward prologue: dgate_c = <dO, O_c> (caller order, dtype), D_c = omega_c * dgate_c (fp32).
// ---------------------------------------------------------------------------------------------
template <class T>
__global__ void k_bwd_pre(Ctx c) {
  // D/8 lanes per row (g, p, s), 8 elements each, reduced with shuffles
  const int lpr = c.D / 8;
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t row = t / lpr;
  const int sub = int(t % lpr);
  const bool valid = row < int64_t(c.N) * c.H;
  const int64_t rr = valid ? row : 0;
  const T* dos = static_cast<const T*>(c.dos) + rr * c.D + sub * 8;
  float acc[3] = {0.f, 0.f, 0.f};
  float d[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) d[e] = ld(dos + e);
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    const float4* o = reinterpret_cast<const float4*>(static_cast<const float*>(c.o[b]) + rr * c.D + sub * 8);
    const float4 x = o[0], y = o[1];
    acc[b] = d[0] * x.x + d[1] * x.y + d[2] * x.z + d[3] * x.w + d[4] * y.x + d[5] * y.y + d[6] * y.z + d[7] * y.w;
  }
  for (int o = lpr / 2; o; o >>= 1)
#pragma unroll
    for (int b = 0; b < 3; ++b) acc[b] += __shfl_xor_sync(0xffffffffu, acc[b], o);
  if (!valid || sub != 0) return;
  const int s = int(row % c.h_s);
  const int p = int((row / c.h_s) % c.N);
  if (p < c.off[SSA_LEVEL_Q][c.q_begin] || p >= c.off[SSA_LEVEL_Q][c.q_end]) return;
  const int g = int(row / (int64_t(c.h_s) * c.N));
  const int h = g * c.h_s + s;
  const int dst = c.sorted_input ? p : c.perm[p];
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    const float wb = c.gs[row * 3 + b];
    if (c.dz) c.dz[row * 3 + b] = acc[b] * wb * (1.f - wb);   // gate projection backward (R18)
    c.Dd[b][row] = wb * acc[b];
    st(static_cast<T*>(c.dgates) + (int64_t(dst) * c.H + h) * 3 + b, acc[b]);
  }
}

// ---------------------------------------------------------------------------------------------
// Inverse selection CSR: for every (selection block B, g), the ascending list of query blocks whose
// top-k contains B. Each (B, g, Q) is unique, so its dense index (B*h_kv + g)*n_q + Q marked in a
// bitmap and ranked by popcount prefix sums IS its position in the (key, Q)-sorted list: a counting
// sort with no comparisons and a deterministic result (same trick as the block build).
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ int32_t bit_rank(const uint32_t* bm, const int32_t* chunk_pre, int64_t bit) {
  const int64_t w = bit >> 5, ch = bit >> 10;
  int32_t r = chunk_pre[ch];
  for (int64_t i = ch * 32; i < w; ++i) r += __popc(bm[i]);
  return r + __popc(bm[w] & ((1u << (bit & 31)) - 1u));
}
__global__ void k_inv_mark(Ctx c, uint32_t* bm) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= int64_t(c.n_blk[SSA_LEVEL_Q]) * c.h_kv * c.T) return;
  const int B = c.I[i];
  if (B < 0) return;
  const int g = int((i / c.T) % c.h_kv);
  const int Q = int(i / (int64_t(c.T) * c.h_kv));
  if (Q < c.q_begin || Q >= c.q_end) return;          // selections of rows this shard does not own
  const int64_t bit = (int64_t(B) * c.h_kv + g) * c.n_blk[SSA_LEVEL_Q] + Q;
  atomicOr(bm + (bit >> 5), 1u << (bit & 31));
}
__global__ void k_inv_chunk_popc(const uint32_t* __restrict__ bm, int64_t n_chunks, int32_t* __restrict__ cnt) {
  const int64_t ch = int64_t(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (ch >= n_chunks) return;
  int v = __popc(bm[ch * 32 + (threadIdx.x & 31)]);
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) cnt[ch] = v;
}
__global__ void k_inv_place(Ctx c, const uint32_t* bm, const int32_t* chunk_pre) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= int64_t(c.n_blk[SSA_LEVEL_Q]) * c.h_kv * c.T) return;
  const int B = c.I[i];
  if (B < 0) return;
  const int g = int((i / c.T) % c.h_kv);
  const int Q = int(i / (int64_t(c.T) * c.h_kv));
  if (Q < c.q_begin || Q >= c.q_end) return;
  const int64_t bit = (int64_t(B) * c.h_kv + g) * c.n_blk[SSA_LEVEL_Q] + Q;
  c.inv_list[bit_rank(bm, chunk_pre, bit)] = Q;
}
__global__ void k_inv_offsets(Ctx c, const uint32_t* bm, const int32_t* chunk_pre, int64_t total_bits) {
  const int64_t key = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nkeys = int64_t(c.n_blk[SSA_LEVEL_SLC]) * c.h_kv;
  if (key > nkeys) return;
  const int64_t bit = key * c.n_blk[SSA_LEVEL_Q];
  c.inv_off[key] = bit < total_bits ? bit_rank(bm, chunk_pre, bit) : bit_rank(bm, chunk_pre, total_bits - 1) +
                                                                       int((bm[(total_bits - 1) >> 5] >> ((total_bits - 1) & 31)) & 1u);
}

// ---------------------------------------------------------------------------------------------
// a9 (SIMT) dQ, Q-outer over the compression keys and the selected blocks (CTA per (Q, g)).
// dS = P (dP - D_c), dP = omega_c <dO, v_j>, dq += scale * dS * k_j.
// ---------------------------------------------------------------------------------------------
template <class T, int D>
__global__ void __launch_bounds__(kRows) k_dq(Ctx c) {
  __shared__ float Kt[kKT * D];
  __shared__ float Vt[kKT * D];
  __shared__ int seg_s[65], seg_e[65];
  __shared__ int nseg;
  const int Q = c.q_order[blockIdx.x], g = blockIdx.y, tid = threadIdx.x;
  if (Q < c.q_begin || Q >= c.q_end) return;
  const int t0 = c.off[SSA_LEVEL_Q][Q], t1 = c.off[SSA_LEVEL_Q][Q + 1];
  const int b = c.q_batch[Q];
  const int rows = (t1 - t0) * c.h_s;
  if (tid == 0) {
    seg_s[0] = c.bb[SSA_LEVEL_CMP][b];
    seg_e[0] = c.bb[SSA_LEVEL_CMP][b + 1];
    int n = 1;
    for (int j = 0; j < c.T; ++j) {
      int B = c.I[(int64_t(Q) * c.h_kv + g) * c.T + j];
      if (B >= 0) { seg_s[n] = c.off[SSA_LEVEL_SLC][B]; seg_e[n] = c.off[SSA_LEVEL_SLC][B + 1]; ++n; }
    }
    nseg = n;
  }
  __syncthreads();
  const T* qs = static_cast<const T*>(c.qs);
  const T* dos = static_cast<const T*>(c.dos);
  const int64_t row_base = (int64_t(g) * c.N + t0) * c.h_s;
  const float l2s = c.scale * kLog2e;
  for (int r0 = 0; r0 < rows; r0 += kRows) {
    const int r = r0 + tid;
    const bool valid = r < rows;
    const int64_t row = row_base + (valid ? r : 0);
    float q[D], dO[D], dq[D];
#pragma unroll
    for (int e = 0; e < D; ++e) {
      q[e] = ld(qs + row * D + e);
      dO[e] = ld(dos + row * D + e);
      dq[e] = 0.f;
    }
    for (int sgi = 0; sgi < nseg; ++sgi) {
      const int br = sgi == 0 ? 0 : 1;
      const T* kb = static_cast<const T*>(c.ks);
      const T* vb = static_cast<const T*>(c.vs);
      const float* kcf = static_cast<const float*>(c.kc);
      const float* vcf = static_cast<const float*>(c.vc);
      const int64_t kbase = int64_t(g) * (br == 0 ? c.n_blk[SSA_LEVEL_CMP] : c.N);
      const float lse2 = c.lse[br][row];
      const float w = c.gs[row * 3 + br];
      const float Dv = c.Dd[br][row];
      for (int k0 = seg_s[sgi]; k0 < seg_e[sgi]; k0 += kKT) {
        const int nt = min(kKT, seg_e[sgi] - k0);
        __syncthreads();
        for (int i = tid; i < nt * D; i += kRows) {
          Kt[i] = br == 0 ? kcf[(kbase + k0) * D + i] : ld(kb + (kbase + k0) * D + i);
          Vt[i] = br == 0 ? vcf[(kbase + k0) * D + i] : ld(vb + (kbase + k0) * D + i);
        }
        __syncthreads();
        for (int j = 0; j < nt; ++j) {
          float x = 0.f, dp = 0.f;
#pragma unroll
          for (int e = 0; e < D; ++e) {
            x += q[e] * Kt[j * D + e];
            dp += dO[e] * Vt[j * D + e];
          }
          const float p = exp2f(x * l2s - lse2);
          const float ds = p * (w * dp - Dv) * c.scale;
#pragma unroll
          for (int e = 0; e < D; ++e) dq[e] += ds * Kt[j * D + e];
        }
      }
    }
    if (valid) {
#pragma unroll
      for (int e = 0; e < D; ++e) c.dq_acc[row * D + e] = dq[e];
    }
  }
}

// ---------------------------------------------------------------------------------------------
// KV-outer helper: a pair of threads owns one key (half the channels each). For every staged row:
// s = scale <q_r, k_j>, p = exp(s - lse_r), dv_j += p w_r dO_r, dp = w_r <dO_r, v_j>,
// ds = p (dp - D_r), dk_j += scale ds q_r.
// ---------------------------------------------------------------------------------------------
template <int D>
struct KvAcc {
  float k[D / 2], v[D / 2], dk[D / 2], dv[D / 2];
};

template <class T, int D>
__device__ __forceinline__ void kv_rows_tile(KvAcc<D>& a, bool kvalid, int half, const float* Qt, const float* Ot,
                                             const float* st_lse2, const float* st_w, const float* st_D, int nr,
                                             float scale) {
  const float l2s = scale * kLog2e;
  // two-level summation: the tile's rows are summed into fresh registers, then added to the running
  // totals once per tile (fp32 error growth ~ rows/tile + tiles instead of all rows of a popular key
  // block — the fp32 mode's 1e-4 bound at C2, where a key collects ~3e5 row terms)
  float tdk[D / 2], tdv[D / 2];
#pragma unroll
  for (int e = 0; e < D / 2; ++e) tdk[e] = tdv[e] = 0.f;
  for (int rr = 0; rr < nr; ++rr) {
    float x = 0.f, dp = 0.f;
#pragma unroll
    for (int e = 0; e < D / 2; ++e) {
      x += Qt[rr * D + half * (D / 2) + e] * a.k[e];
      dp += Ot[rr * D + half * (D / 2) + e] * a.v[e];
    }
    x += __shfl_xor_sync(0xffffffffu, x, 1);
    dp += __shfl_xor_sync(0xffffffffu, dp, 1);
    if (!kvalid) continue;
    const float p = exp2f(x * l2s - st_lse2[rr]);
    const float w = st_w[rr];
    const float ds = p * (w * dp - st_D[rr]) * scale;
    const float pw = p * w;
#pragma unroll
    for (int e = 0; e < D / 2; ++e) {
      tdv[e] += pw * Ot[rr * D + half * (D / 2) + e];
      tdk[e] += ds * Qt[rr * D + half * (D / 2) + e];
    }
  }
#pragma unroll
  for (int e = 0; e < D / 2; ++e) {
    a.dv[e] += tdv[e];
    a.dk[e] += tdk[e];
  }
}

template <class T, int D>
__device__ __forceinline__ void stage_rows(const Ctx& c, int br, int64_t row0, int nr, float* Qt, float* Ot,
                                           float* st_lse2, float* st_w, float* st_D) {
  const T* qs = static_cast<const T*>(c.qs);
  const T* dos = static_cast<const T*>(c.dos);
  __syncthreads();
  for (int i = threadIdx.x; i < nr * D; i += blockDim.x) {
    Qt[i] = ld(qs + row0 * D + i);
    Ot[i] = ld(dos + row0 * D + i);
  }
  for (int i = threadIdx.x; i < nr; i += blockDim.x) {
    st_lse2[i] = c.lse[br][row0 + i];
    st_w[i] = c.gs[(row0 + i) * 3 + br];
    st_D[i] = c.Dd[br][row0 + i];
  }
  __syncthreads();
}

constexpr int kRT = 32;  // rows per staged tile in KV-outer kernels

// selection branch dK/dV: CTA per (selection block B, g); assigns dk_acc / dv_acc of B's tokens.
template <class T, int D>
__global__ void __launch_bounds__(128) k_slc_dkdv(Ctx c) {
  __shared__ float Qt[kRT * D], Ot[kRT * D], s_l[kRT], s_w[kRT], s_D[kRT];
  const int B = blockIdx.x, g = blockIdx.y;
  const int kk0 = c.off[SSA_LEVEL_SLC][B], kk1 = c.off[SSA_LEVEL_SLC][B + 1];
  const int half = threadIdx.x & 1;
  const int64_t key = int64_t(B) * c.h_kv + g;
  const int la = c.inv_off[key], le = c.inv_off[key + 1];
  const T* ks = static_cast<const T*>(c.ks);
  const T* vs = static_cast<const T*>(c.vs);
  for (int j0 = kk0; j0 < kk1; j0 += 64) {
    const int j = j0 + (threadIdx.x >> 1);
    const bool kvalid = j < kk1;
    KvAcc<D> a;
#pragma unroll
    for (int e = 0; e < D / 2; ++e) {
      int64_t idx = (int64_t(g) * c.N + (kvalid ? j : kk0)) * D + half * (D / 2) + e;
      a.k[e] = ld(ks + idx);
      a.v[e] = ld(vs + idx);
      a.dk[e] = 0.f;
      a.dv[e] = 0.f;
    }
    for (int li = la; li < le; ++li) {
      const int Q = c.inv_list[li];
      const int q0 = c.off[SSA_LEVEL_Q][Q], q1 = c.off[SSA_LEVEL_Q][Q + 1];
      const int64_t rb = (int64_t(g) * c.N + q0) * c.h_s;
      const int rows = (q1 - q0) * c.h_s;
      for (int r0 = 0; r0 < rows; r0 += kRT) {
        const int nr = min(kRT, rows - r0);
        stage_rows<T, D>(c, 1, rb + r0, nr, Qt, Ot, s_l, s_w, s_D);
        kv_rows_tile<T, D>(a, kvalid, half, Qt, Ot, s_l, s_w, s_D, nr, c.scale);
      }
    }
    if (kvalid) {
#pragma unroll
      for (int e = 0; e < D / 2; ++e) {
        int64_t idx = (int64_t(g) * c.N + j) * D + half * (D / 2) + e;
        c.dk_acc[idx] = a.dk[e];
        c.dv_acc[idx] = a.dv[e];
      }
    }
  }
}

// window branch backward: CTA per (window W, g). dq_acc += (row-thread pass), dk/dv_acc += (key pass).
template <class T, int D>
__global__ void __launch_bounds__(128) k_win_bwd(Ctx c) {
  __shared__ float Qt[kRT * D], Ot[kRT * D], s_l[kRT], s_w[kRT], s_D[kRT];
  const int W = blockIdx.x, g = blockIdx.y, tid = threadIdx.x;
  if (c.q_end - c.q_begin < c.n_blk[SSA_LEVEL_Q] && (W < c.q_begin || W >= c.q_end)) return;  // m_win == m_q
  const int t0 = c.off[SSA_LEVEL_WIN][W], t1 = c.off[SSA_LEVEL_WIN][W + 1];
  const int rows = (t1 - t0) * c.h_s;
  const int64_t rb = (int64_t(g) * c.N + t0) * c.h_s;
  const T* ks = static_cast<const T*>(c.ks);
  const T* vs = static_cast<const T*>(c.vs);
  const T* qs = static_cast<const T*>(c.qs);
  const T* dos = static_cast<const T*>(c.dos);
  const float l2s = c.scale * kLog2e;
  // dq: thread = row, keys staged through Qt/Ot (reused as K/V tiles)
  for (int r0 = 0; r0 < rows; r0 += 128) {
    const int r = r0 + tid;
    const bool valid = r < rows;
    const int64_t row = rb + (valid ? r : 0);
    float q[D], dO[D], dq[D];
#pragma unroll
    for (int e = 0; e < D; ++e) {
      q[e] = ld(qs + row * D + e);
      dO[e] = ld(dos + row * D + e);
      dq[e] = 0.f;
    }
    const float lse2 = c.lse[2][row], w = c.gs[row * 3 + 2], Dv = c.Dd[2][row];
    for (int k0 = t0; k0 < t1; k0 += kRT) {
      const int nt = min(kRT, t1 - k0);
      __syncthreads();
      for (int i = tid; i < nt * D; i += 128) {
        Qt[i] = ld(ks + (int64_t(g) * c.N + k0) * D + i);
        Ot[i] = ld(vs + (int64_t(g) * c.N + k0) * D + i);
      }
      __syncthreads();
      for (int j = 0; j < nt; ++j) {
        float x = 0.f, dp = 0.f;
#pragma unroll
        for (int e = 0; e < D; ++e) {
          x += q[e] * Qt[j * D + e];
          dp += dO[e] * Ot[j * D + e];
        }
        const float p = exp2f(x * l2s - lse2);
        const float ds = p * (w * dp - Dv) * c.scale;
#pragma unroll
        for (int e = 0; e < D; ++e) dq[e] += ds * Qt[j * D + e];
      }
    }
    if (valid) {
#pragma unroll
      for (int e = 0; e < D; ++e) c.dq_acc[row * D + e] += dq[e];
    }
  }
  // dk/dv: key pairs
  const int half = tid & 1;
  for (int j0 = t0; j0 < t1; j0 += 64) {
    const int j = j0 + (tid >> 1);
    const bool kvalid = j < t1;
    KvAcc<D> a;
#pragma unroll
    for (int e = 0; e < D / 2; ++e) {
      int64_t idx = (int64_t(g) * c.N + (kvalid ? j : t0)) * D + half * (D / 2) + e;
      a.k[e] = ld(ks + idx);
      a.v[e] = ld(vs + idx);
      a.dk[e] = 0.f;
      a.dv[e] = 0.f;
    }
    for (int r0 = 0; r0 < rows; r0 += kRT) {
      const int nr = min(kRT, rows - r0);
      stage_rows<T, D>(c, 2, rb + r0, nr, Qt, Ot, s_l, s_w, s_D);
      kv_rows_tile<T, D>(a, kvalid, half, Qt, Ot, s_l, s_w, s_D, nr, c.scale);
    }
    if (kvalid) {
#pragma unroll
      for (int e = 0; e < D / 2; ++e) {
        int64_t idx = (int64_t(g) * c.N + j) * D + half * (D / 2) + e;
        c.dk_acc[idx] += a.dk[e];
        c.dv_acc[idx] += a.dv[e];
      }
    }
  }
}

// compression branch dK^cmp/dV^cmp partials: grid (cmp tile, g, chunk). Tile = 128 compressed keys
// of one batch item (processed as two 64-key halves); chunk = a contiguous 1/n_chunk share of the
// batch item's rows.
template <class T, int D>
__global__ void __launch_bounds__(128) k_cmp_dkdv(Ctx c) {
  __shared__ float Qt[kRT * D], Ot[kRT * D], s_l[kRT], s_w[kRT], s_D[kRT];
  const int tile = blockIdx.x, g = blockIdx.y, chunk = blockIdx.z;
  const int b = c.cmp_tiles[2 * tile], jt = c.cmp_tiles[2 * tile + 1];
  const int c1 = min(c.bb[SSA_LEVEL_CMP][b + 1], jt + 128);
  const int n_cmp = c.n_blk[SSA_LEVEL_CMP];
  const int half = threadIdx.x & 1;
  const float* kc = static_cast<const float*>(c.kc);
  const float* vc = static_cast<const float*>(c.vc);
  const int bt0 = max(c.batch_tokens[b], c.off[SSA_LEVEL_Q][c.q_begin]);
  const int bt1 = max(bt0, min(c.batch_tokens[b + 1], c.off[SSA_LEVEL_Q][c.q_end]));   // owned rows only
  const int64_t rows = int64_t(bt1 - bt0) * c.h_s;
  const int64_t per = (rows + c.n_chunk - 1) / c.n_chunk;
  const int64_t ra = min(rows, per * chunk), re = min(rows, per * (chunk + 1));
  const int64_t rb = (int64_t(g) * c.N + bt0) * c.h_s;
  for (int j0 = jt; j0 < c1; j0 += 64) {
    const int j = j0 + (threadIdx.x >> 1);
    const bool kvalid = j < c1;
    KvAcc<D> a;
#pragma unroll
    for (int e = 0; e < D / 2; ++e) {
      int64_t idx = (int64_t(g) * n_cmp + (kvalid ? j : j0)) * D + half * (D / 2) + e;
      a.k[e] = kc[idx];
      a.v[e] = vc[idx];
      a.dk[e] = 0.f;
      a.dv[e] = 0.f;
    }
    for (int64_t r0 = ra; r0 < re; r0 += kRT) {
      const int nr = int((re - r0) < kRT ? (re - r0) : kRT);
      stage_rows<T, D>(c, 0, rb + r0, nr, Qt, Ot, s_l, s_w, s_D);
      kv_rows_tile<T, D>(a, kvalid, half, Qt, Ot, s_l, s_w, s_D, nr, c.scale);
    }
    if (kvalid) {
#pragma unroll
      for (int e = 0; e < D / 2; ++e) {
        int64_t idx = ((int64_t(chunk) * c.h_kv + g) * n_cmp + j) * D + half * (D / 2) + e;
        c.dkc_part[idx] = a.dk[e];
        c.dvc_part[idx] = a.dv[e];
      }
    }
  }
}

__global__ void k_cmp_reduce(Ctx c) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  int64_t per = int64_t(c.h_kv) * c.n_blk[SSA_LEVEL_CMP] * c.D;
  if (i >= per) return;
  float sk = 0.f, sv = 0.f;
  for (int ch = 0; ch < c.n_chunk; ++ch) {
    sk += c.dkc_part[ch * per + i];
    sv += c.dvc_part[ch * per + i];
  }
  c.dkc[i] = sk;
  c.dvc[i] = sv;
}

// epilogue: dq -> caller order; dk/dv = raw-token part + mean-pool backward of dk^cmp/dv^cmp
template <class T>
__global__ void k_bwd_final_q(Ctx c) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  int64_t total = int64_t(c.N) * c.H * c.D;
  if (i >= total) return;
  int e = int(i % c.D);
  int h = int((i / c.D) % c.H);
  int p = int(i / (int64_t(c.D) * c.H));
  int g = h / c.h_s, s = h % c.h_s;
  if (p < c.off[SSA_LEVEL_Q][c.q_begin] || p >= c.off[SSA_LEVEL_Q][c.q_end]) return;
  int dst = c.sorted_input ? p : c.perm[p];
  st(static_cast<T*>(c.dq) + (int64_t(dst) * c.H + h) * c.D + e,
     c.dq_acc[((int64_t(g) * c.N + p) * c.h_s + s) * c.D + e]);
}
template <class T>
__global__ void k_bwd_final_kv(Ctx c) {
  // 4 consecutive elements per thread (D is a multiple of 4), 32-bit index math
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int dq4 = c.D >> 2;
  if (i >= c.N * c.h_kv * dq4) return;
  const int e = (i % dq4) * 4;
  const int g = (i / dq4) % c.h_kv;
  const int p = i / (dq4 * c.h_kv);
  const int j = c.tok_block[SSA_LEVEL_CMP][p];
  const float inv = 1.f / float(c.off[SSA_LEVEL_CMP][j + 1] - c.off[SSA_LEVEL_CMP][j]);
  const int64_t ki = (int64_t(g) * c.N + p) * c.D + e;
  const int64_t ci = (int64_t(g) * c.n_blk[SSA_LEVEL_CMP] + j) * c.D + e;
  const int dst = c.sorted_input ? p : c.perm[p];
  if (e >= c.Dc) return;                         // zero-padded head dims (d = 32 on tcgen05) are not output
  const int64_t o = (int64_t(dst) * c.h_kv + g) * c.Dc + e;
  const float4 ak = *reinterpret_cast<const float4*>(c.dk_acc + ki), av = *reinterpret_cast<const float4*>(c.dv_acc + ki);
  float4 ck = *reinterpret_cast<const float4*>(c.dkc + ci), cv = *reinterpret_cast<const float4*>(c.dvc + ci);
  if (c.conv_kw) {
    // learned delta (R17): d(k_t) = W[loc(t), g]^T dk^cmp_B / n_B (the 1/n_B is applied below)
    const int m = c.m_cmp;
    const int4 cc = reinterpret_cast<const int4*>(c.sorted_coords)[p];
    const int loc = ((cc.y % m) * m + (cc.z % m)) * m + (cc.w % m);
    const float* wk = c.conv_kw + (int64_t(loc) * c.h_kv + g) * c.D * c.D + e;
    const float* wv = c.conv_vw + (int64_t(loc) * c.h_kv + g) * c.D * c.D + e;
    const float* yk = c.dkc + (int64_t(g) * c.n_blk[SSA_LEVEL_CMP] + j) * c.D;
    const float* yv = c.dvc + (int64_t(g) * c.n_blk[SSA_LEVEL_CMP] + j) * c.D;
    float4 sk = make_float4(0.f, 0.f, 0.f, 0.f), sv = sk;
    for (int r = 0; r < c.D; ++r) {
      const float4 a = *reinterpret_cast<const float4*>(wk + int64_t(r) * c.D);
      const float4 b = *reinterpret_cast<const float4*>(wv + int64_t(r) * c.D);
      const float y1 = yk[r], y2 = yv[r];
      sk.x += a.x * y1; sk.y += a.y * y1; sk.z += a.z * y1; sk.w += a.w * y1;
      sv.x += b.x * y2; sv.y += b.y * y2; sv.z += b.z * y2; sv.w += b.w * y2;
    }
    ck = sk;
    cv = sv;
  }
  const float gk[4] = {ak.x + ck.x * inv, ak.y + ck.y * inv, ak.z + ck.z * inv, ak.w + ck.w * inv};
  const float gv[4] = {av.x + cv.x * inv, av.y + cv.y * inv, av.z + cv.z * inv, av.w + cv.w * inv};
  if (c.kv_grad_f32) {
    float4* pk = reinterpret_cast<float4*>(static_cast<float*>(c.dk) + o);
    float4* pv = reinterpret_cast<float4*>(static_cast<float*>(c.dv) + o);
    float4 ak4 = make_float4(gk[0], gk[1], gk[2], gk[3]), av4 = make_float4(gv[0], gv[1], gv[2], gv[3]);
    if (c.accumulate) {
      const float4 a = *pk, b = *pv;
      ak4.x += a.x; ak4.y += a.y; ak4.z += a.z; ak4.w += a.w;
      av4.x += b.x; av4.y += b.y; av4.z += b.z; av4.w += b.w;
    }
    *pk = ak4;
    *pv = av4;
  } else {
#pragma unroll
    for (int u = 0; u < 4; ++u) {   // SSA_ACCUMULATE: add to the caller's dk / dv
      st(static_cast<T*>(c.dk) + o + u, c.accumulate ? gk[u] + ld(static_cast<const T*>(c.dk) + o + u) : gk[u]);
      st(static_cast<T*>(c.dv) + o + u, c.accumulate ? gv[u] + ld(static_cast<const T*>(c.dv) + o + u) : gv[u]);
    }
  }
}

template <class T, int D>
ssa_status simt_fwd_t(const Ctx& c, cudaStream_t st, bool attention_only) {
  const int nq = c.n_blk[SSA_LEVEL_Q];
  if (!attention_only) {
    size_t smem = (2 * kKT * D + kRows * (kKT + 1) + 4 * kKT + c.max_cmp_b + c.max_slc_b) * sizeof(float);
    if (smem > 227 * 1024) { set_error("too many blocks per batch item for the SIMT kernel"); return SSA_ERR_UNSUPPORTED; }
    SSA_CUDA_TRY(cudaFuncSetAttribute(k_cmp_fwd<T, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    {
      ProfScope ps_("k_cmp_fwd", st);
      k_cmp_fwd<T, D><<<dim3(nq, c.h_kv), kRows, smem, st>>>(c);
      SSA_LAUNCH_CHECK("k_cmp_fwd");
    }
  }
  {
    ProfScope ps_("k_attn_fwd(slc)", st);
    k_attn_fwd<T, D><<<dim3(nq, c.h_kv), kRows, 0, st>>>(c, 1);
    SSA_LAUNCH_CHECK("k_attn_fwd(slc)");
  }
  {
    ProfScope ps_("k_attn_fwd(win)", st);
    k_attn_fwd<T, D><<<dim3(c.n_blk[SSA_LEVEL_WIN], c.h_kv), kRows, 0, st>>>(c, 2);
    SSA_LAUNCH_CHECK("k_attn_fwd(win)");
  }
  return SSA_OK;
}

template <class T, int D>
ssa_status simt_bwd_t(const Ctx& c, cudaStream_t st) {
  const int nq = c.n_blk[SSA_LEVEL_Q];
  {
    ProfScope ps_("k_dq", st);
    k_dq<T, D><<<dim3(nq, c.h_kv), kRows, 0, st>>>(c);
    SSA_LAUNCH_CHECK("k_dq");
  }
  {
    ProfScope ps_("k_slc_dkdv", st);
    k_slc_dkdv<T, D><<<dim3(c.n_blk[SSA_LEVEL_SLC], c.h_kv), 128, 0, st>>>(c);
    SSA_LAUNCH_CHECK("k_slc_dkdv");
  }
  {
    ProfScope ps_("k_win_bwd", st);
    k_win_bwd<T, D><<<dim3(c.n_blk[SSA_LEVEL_WIN], c.h_kv), 128, 0, st>>>(c);
    SSA_LAUNCH_CHECK("k_win_bwd");
  }
  {
    ProfScope ps_("k_cmp_dkdv", st);
    k_cmp_dkdv<T, D><<<dim3(c.n_cmp_tiles, c.h_kv, c.n_chunk), 128, 0, st>>>(c);
    SSA_LAUNCH_CHECK("k_cmp_dkdv");
  }
  return cmp_reduce(c, st);
}

template <class T>
ssa_status dispatch_d_fwd(const Ctx& c, cudaStream_t st, bool ao) {
  switch (c.D) {
    case 16: return simt_fwd_t<T, 16>(c, st, ao);
    case 32: return simt_fwd_t<T, 32>(c, st, ao);
    case 64: return simt_fwd_t<T, 64>(c, st, ao);
  }
  set_error("SIMT kernels support head dim 16, 32 or 64");
  return SSA_ERR_UNSUPPORTED;
}
template <class T>
ssa_status dispatch_d_bwd(const Ctx& c, cudaStream_t st) {
  switch (c.D) {
    case 16: return simt_bwd_t<T, 16>(c, st);
    case 32: return simt_bwd_t<T, 32>(c, st);
    case 64: return simt_bwd_t<T, 64>(c, st);
  }
  set_error("SIMT kernels support head dim 16, 32 or 64");
  return SSA_ERR_UNSUPPORTED;
}
}  // namespace

ssa_status gather_inputs(const Ctx& c, bool bf16, cudaStream_t st, bool with_dout, bool rows, bool keys, bool gates) {
  const int esz = bf16 ? 2 : 4;
  const int64_t nr = int64_t(c.N) * c.h_kv * (c.h_s * c.D * esz / 16), nk = int64_t(c.N) * c.h_kv * (c.D * esz / 16);
  const int64_t ng = int64_t(c.N) * c.H * 3;
  if (bf16) {
    using T = __nv_bfloat16;
    if (with_dout && rows) {
      k_gather_rows<T><<<nblk(nr, 256), 256, 0, st>>>(c, static_cast<const T*>(c.dout), static_cast<T*>(c.dos));
      SSA_LAUNCH_CHECK("k_gather_rows(dout)");
    }
    if (rows) {
      k_gather_rows<T><<<nblk(nr, 256), 256, 0, st>>>(c, static_cast<const T*>(c.q), static_cast<T*>(c.qs));
      SSA_LAUNCH_CHECK("k_gather_rows");
    }
    if (keys) {
      k_gather_keys<T><<<nblk(nk, 256), 256, 0, st>>>(c, static_cast<const T*>(c.k), static_cast<const T*>(c.v),
                                                      static_cast<T*>(c.ks), static_cast<T*>(c.vs));
      SSA_LAUNCH_CHECK("k_gather_keys");
    }
    if (gates) {
      k_gather_gates<T><<<nblk(ng / 3, 256), 256, 0, st>>>(c, static_cast<const T*>(c.gates), c.gs);
      SSA_LAUNCH_CHECK("k_gather_gates");
    }
  } else {
    using T = float;
    if (with_dout) {
      k_gather_rows<T><<<nblk(nr, 256), 256, 0, st>>>(c, static_cast<const T*>(c.dout), static_cast<T*>(c.dos));
      SSA_LAUNCH_CHECK("k_gather_rows(dout)");
    }
    k_gather_rows<T><<<nblk(nr, 256), 256, 0, st>>>(c, static_cast<const T*>(c.q), static_cast<T*>(c.qs));
    SSA_LAUNCH_CHECK("k_gather_rows");
    if (keys) {
      k_gather_keys<T><<<nblk(nk, 256), 256, 0, st>>>(c, static_cast<const T*>(c.k), static_cast<const T*>(c.v),
                                                      static_cast<T*>(c.ks), static_cast<T*>(c.vs));
      SSA_LAUNCH_CHECK("k_gather_keys");
    }
    if (gates) {
      k_gather_gates<T><<<nblk(ng / 3, 256), 256, 0, st>>>(c, static_cast<const T*>(c.gates), c.gs);
      SSA_LAUNCH_CHECK("k_gather_gates");
    }
  }
  return SSA_OK;
}

// ssa_pool (sharded mode 2): Eq. 7 (delta = mean, reading R4, optional PE) straight from the caller's
// plan-order k, v, for the compression blocks inside the owned rows [row_lo, row_hi); every other
// block is written as 0 so that a sum over ranks assembles the complete pooled keys. k, v point at
// row row_lo (SSA_LOCAL_ROWS) or row 0. grid (n_cmp, h_kv), block D threads.
template <class T>
__global__ void k_pool_rows(Ctx c, const T* __restrict__ k, const T* __restrict__ v, int64_t row_base,
                            float* __restrict__ kc, float* __restrict__ vc) {
  const int j = blockIdx.x, g = blockIdx.y, e = threadIdx.x;
  const int t0 = c.off[SSA_LEVEL_CMP][j], t1 = c.off[SSA_LEVEL_CMP][j + 1];
  const int64_t o = (int64_t(g) * c.n_blk[SSA_LEVEL_CMP] + j) * c.D + e;
  if (t0 < c.row_lo || t1 > c.row_hi) {           // not owned (compression blocks nest in query blocks)
    kc[o] = 0.f;
    vc[o] = 0.f;
    return;
  }
  const T* pek = static_cast<const T*>(c.pe_k);
  const T* pev = static_cast<const T*>(c.pe_v);
  const int m = c.m_cmp;
  float sk = 0.f, sv = 0.f;
  for (int p = t0; p < t1; ++p) {
    const int64_t idx = ((int64_t(p) - row_base) * c.h_kv + g) * c.D + e;
    float kk = ld(k + idx), vv = ld(v + idx);
    if (pek || pev) {
      const int4 cc = reinterpret_cast<const int4*>(c.sorted_coords)[p];
      const int loc = ((cc.y % m) * m + (cc.z % m)) * m + (cc.w % m);
      const int64_t pi = (int64_t(loc) * c.h_kv + g) * c.D + e;
      if (pek) kk += ld(pek + pi);
      if (pev) vv += ld(pev + pi);
    }
    sk += kk;
    sv += vv;
  }
  const float inv = 1.f / float(t1 - t0);
  kc[o] = sk * inv;
  vc[o] = sv * inv;
}

ssa_status pool_rows(const Ctx& c, bool bf16, const void* k, const void* v, float* kc, float* vc, cudaStream_t st) {
  if (c.n_blk[SSA_LEVEL_CMP] == 0) return SSA_OK;
  dim3 grid(c.n_blk[SSA_LEVEL_CMP], c.h_kv);
  if (bf16)
    k_pool_rows<__nv_bfloat16><<<grid, c.D, 0, st>>>(c, static_cast<const __nv_bfloat16*>(k),
                                                      static_cast<const __nv_bfloat16*>(v), c.row_base, kc, vc);
  else
    k_pool_rows<float><<<grid, c.D, 0, st>>>(c, static_cast<const float*>(k), static_cast<const float*>(v), c.row_base, kc, vc);
  SSA_LAUNCH_CHECK("k_pool_rows");
  return SSA_OK;
}

ssa_status pool_forward(const Ctx& c, bool bf16, cudaStream_t st) {
  dim3 grid(c.n_blk[SSA_LEVEL_CMP], c.h_kv);
  if (bf16) k_pool<__nv_bfloat16><<<grid, c.D, 0, st>>>(c);
  else k_pool<float><<<grid, c.D, 0, st>>>(c);
  SSA_LAUNCH_CHECK("k_pool");
  return SSA_OK;
}

ssa_status combine_forward(const Ctx& c, bool bf16, cudaStream_t st) {
  int64_t n = int64_t(c.N) * c.H * c.D;
  if (bf16) k_combine<__nv_bfloat16><<<nblk(n, 256), 256, 0, st>>>(c);
  else k_combine<float><<<nblk(n, 256), 256, 0, st>>>(c);
  SSA_LAUNCH_CHECK("k_combine");
  return SSA_OK;
}

ssa_status simt_forward(const Ctx& c, bool bf16, cudaStream_t st, bool attention_only) {
  return bf16 ? dispatch_d_fwd<__nv_bfloat16>(c, st, attention_only) : dispatch_d_fwd<float>(c, st, attention_only);
}

size_t inverse_csr_ws_bytes(int n_slc, int h_kv, int n_q) {
  const int64_t bits = int64_t(n_slc) * h_kv * n_q + 1;
  const int64_t n_chunks = (bits + 1023) / 1024;
  return size_t(n_chunks) * 128 + size_t(n_chunks) * 8 + scan_ws_bytes(n_chunks) + 3 * 256;
}

ssa_status build_inverse_csr(const Ctx& c, void* ws, cudaStream_t st) {
  const int64_t bits = int64_t(c.n_blk[SSA_LEVEL_SLC]) * c.h_kv * c.n_blk[SSA_LEVEL_Q] + 1;
  const int64_t n_chunks = (bits + 1023) / 1024;
  const int64_t nI = int64_t(c.n_blk[SSA_LEVEL_Q]) * c.h_kv * c.T;
  Carve cw(ws, inverse_csr_ws_bytes(c.n_blk[SSA_LEVEL_SLC], c.h_kv, c.n_blk[SSA_LEVEL_Q]));
  uint32_t* bm = cw.take<uint32_t>(n_chunks * 32);
  int32_t* cnt = cw.take<int32_t>(n_chunks);
  int32_t* pre = cw.take<int32_t>(n_chunks);
  void* scan_ws = cw.take<char>(scan_ws_bytes(n_chunks));
  SSA_CUDA_TRY(cudaMemsetAsync(bm, 0, size_t(n_chunks) * 128, st));
  k_inv_mark<<<nblk(nI, 256), 256, 0, st>>>(c, bm);
  SSA_LAUNCH_CHECK("k_inv_mark");
  k_inv_chunk_popc<<<nblk(n_chunks * 32, 256), 256, 0, st>>>(bm, n_chunks, cnt);
  SSA_LAUNCH_CHECK("k_inv_chunk_popc");
  ssa_status s = exclusive_scan(cnt, pre, n_chunks, nullptr, scan_ws, st);
  if (s != SSA_OK) return s;
  k_inv_place<<<nblk(nI, 256), 256, 0, st>>>(c, bm, pre);
  SSA_LAUNCH_CHECK("k_inv_place");
  const int64_t nkeys = int64_t(c.n_blk[SSA_LEVEL_SLC]) * c.h_kv;
  k_inv_offsets<<<nblk(nkeys + 1, 256), 256, 0, st>>>(c, bm, pre, bits - 1);
  SSA_LAUNCH_CHECK("k_inv_offsets");
  return SSA_OK;
}

ssa_status bwd_prologue(const Ctx& c, bool bf16, cudaStream_t st) {
  int64_t rows = int64_t(c.N) * c.H * (c.D / 8);
  if (bf16) k_bwd_pre<__nv_bfloat16><<<nblk(rows, 256), 256, 0, st>>>(c);
  else k_bwd_pre<float><<<nblk(rows, 256), 256, 0, st>>>(c);
  SSA_LAUNCH_CHECK("k_bwd_pre");
  return SSA_OK;
}

ssa_status cmp_reduce(const Ctx& c, cudaStream_t st) {
  int64_t per = int64_t(c.h_kv) * c.n_blk[SSA_LEVEL_CMP] * c.D;
  k_cmp_reduce<<<nblk(per, 256), 256, 0, st>>>(c);
  SSA_LAUNCH_CHECK("k_cmp_reduce");
  return SSA_OK;
}

ssa_status bwd_epilogue(const Ctx& c, bool bf16, cudaStream_t st, bool skip_q) {
  int64_t nq = int64_t(c.N) * c.H * c.D, nk = int64_t(c.N) * c.h_kv * c.D;
  if (bf16) {
    if (!skip_q) {
      k_bwd_final_q<__nv_bfloat16><<<nblk(nq, 256), 256, 0, st>>>(c);
      SSA_LAUNCH_CHECK("k_bwd_final_q");
    }
    k_bwd_final_kv<__nv_bfloat16><<<nblk(nk / 4, 256), 256, 0, st>>>(c);
    SSA_LAUNCH_CHECK("k_bwd_final_kv");
  } else {
    if (!skip_q) {
      k_bwd_final_q<float><<<nblk(nq, 256), 256, 0, st>>>(c);
      SSA_LAUNCH_CHECK("k_bwd_final_q");
    }
    k_bwd_final_kv<float><<<nblk(nk / 4, 256), 256, 0, st>>>(c);
    SSA_LAUNCH_CHECK("k_bwd_final_kv");
  }
  return SSA_OK;
}

ssa_status simt_backward(const Ctx& c, bool bf16, cudaStream_t st) {
  return bf16 ? dispatch_d_bwd<__nv_bfloat16>(c, st) : dispatch_d_bwd<float>(c, st);
}

// ---------------------------------------------------------------------------------------------
// One-sided fetch of the selected K/V blocks: k_fetch_mark flags every selection
// block an owned query block selected; k_fetch_copy copies the flagged blocks owned by another rank
// from that rank's rows (peer pointer) into the caller's full-size k / v. Blocks are contiguous in plan
// order, [rows][h_kv][d]; one CTA per block, 16-byte vectors.
// ---------------------------------------------------------------------------------------------
namespace {
__global__ void k_fetch_mark(Ctx c) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t n = int64_t(c.q_end - c.q_begin) * c.h_kv * c.T;
  if (i >= n) return;
  const int B = c.I[int64_t(c.q_begin) * c.h_kv * c.T + i];
  if (B >= 0) c.fetch_mark[B] = 1;
}
__global__ void k_fetch_copy(Ctx c, int esz) {
  const int B = blockIdx.x;
  if (!c.fetch_mark[B]) return;
  const int t0 = c.off[SSA_LEVEL_SLC][B], t1 = c.off[SSA_LEVEL_SLC][B + 1];
  int owner = 0;
  while (owner + 1 < c.n_peer && c.peer_tok[owner + 1] <= t0) ++owner;
  if (owner == c.my_rank) return;
  const int64_t row_bytes = int64_t(c.h_kv) * c.Dc * esz;
  const int64_t n16 = int64_t(t1 - t0) * row_bytes / 16;
  const uint4* sk = reinterpret_cast<const uint4*>(static_cast<const char*>(c.peer_k[owner]) + (t0 - c.peer_tok[owner]) * row_bytes);
  const uint4* sv = reinterpret_cast<const uint4*>(static_cast<const char*>(c.peer_v[owner]) + (t0 - c.peer_tok[owner]) * row_bytes);
  uint4* dk = reinterpret_cast<uint4*>(static_cast<char*>(const_cast<void*>(c.k)) + int64_t(t0) * row_bytes);
  uint4* dv = reinterpret_cast<uint4*>(static_cast<char*>(const_cast<void*>(c.v)) + int64_t(t0) * row_bytes);
  for (int64_t j = threadIdx.x; j < n16; j += blockDim.x) {
    dk[j] = sk[j];
    dv[j] = sv[j];
  }
}
}  // namespace

ssa_status fetch_selected(const Ctx& c, bool bf16, cudaStream_t st) {
  const int n_slc = c.n_blk[SSA_LEVEL_SLC];
  SSA_CUDA_TRY(cudaMemsetAsync(c.fetch_mark, 0, size_t(n_slc) * 4, st));
  const int64_t n = int64_t(c.q_end - c.q_begin) * c.h_kv * c.T;
  if (n > 0) {
    k_fetch_mark<<<nblk(n, 256), 256, 0, st>>>(c);
    SSA_LAUNCH_CHECK("k_fetch_mark");
  }
  if (n_slc > 0) {
    ProfScope ps("k_fetch_copy", st);
    k_fetch_copy<<<n_slc, 256, 0, st>>>(c, bf16 ? 2 : 4);
    SSA_LAUNCH_CHECK("k_fetch_copy");
  }
  return SSA_OK;
}

}  // namespace ssa
