// pertoken.cu — query blocks smaller than the selection blocks (m_q | m_slc, m_q < m_slc; m_q = 1 is the
// paper's per-token selection, I in R^{N x h_kv x T}, Alg. 1 P:182 / P:188) on the tcgen05 kernels.
//
// The compression kernel runs per query block (its Eq. 8 scores and top-k ARE per query block). The
// selection / window and dQ / KV-outer kernels would then see one query block's few rows per 128-row
// tile, so they run on a "virtual" query level instead: each selection block's query blocks are cut
// into sub-groups of consecutive query blocks (contiguous rows) — greedily, up to S query blocks (S chosen
// on the host so that a sub-group fills a row-tile pair) while the union of the sub-group's selections
// stays within kVqSlots = 128 blocks and kVqKeyCap keys for every kv group; a sub-group's key set is that
// union, and every row keeps only its own query block's blocks through a 128-bit slot mask
// (umask[token][g][2]): the softmax loops set the other granules' logits to -inf (forward, dQ), the
// KV-outer producer gives the rows of query blocks that did not select the key block an LSE of +inf
// (p = 0). Same arithmetic per row as the query-block path; only the row / key grouping changes. A
// sub-group closed by a cap holds at least kmin query blocks (vq_bound), which bounds their number.
#include <climits>
#include <cstdlib>

#include "internal.h"

namespace ssa {
namespace {

inline unsigned nb(int64_t n, int t) { return unsigned((n + t - 1) / t); }

// query-block range [qa, qe) of selection block B
__device__ __forceinline__ void slc_qblocks(const Ctx& c, int B, int* qa, int* qe) {
  const int t0 = c.off[SSA_LEVEL_SLC][B], t1 = c.off[SSA_LEVEL_SLC][B + 1];
  *qa = c.tok_block[SSA_LEVEL_Q][t0];
  *qe = c.tok_block[SSA_LEVEL_Q][t1 - 1] + 1;
}

// Greedy sub-groups of chunk ch (2 S consecutive query blocks) of selection block B (one warp per chunk):
// walk its query blocks in order, closing the open sub-group before a query block whose selections would
// push any kv group's union past kVqSlots blocks or kVqKeyCap keys (the tile capacity of the selection /
// dQ kernels), or when it holds S query blocks. With qa = the chunk's first query block, per sub-group k
// (k < count <= its query blocks): first[qa + k] = its first query block, un[((qa + k) * h_kv + g) *
// kVqSlots + j] = its union for kv group g (order of first appearance, -1 padded); cnt[B * cmax + ch] =
// count; umask[(t * h_kv + g) * 2 + w] = word w of the union slots of token t's own query block's
// selections (bits stay valid: the union only grows by appending). The open unions live in shared memory;
// membership of the T candidates (one per lane) is tested against the union held four entries per lane,
// by ballot.
constexpr int kVqWarps = 4;
constexpr int kVqMaxG = 8;                         // kv groups of the virtual level (vq_group)
__global__ void __launch_bounds__(32 * kVqWarps) k_vq_count(Ctx c, int S, int cmax, int32_t* __restrict__ cnt,
                                                            int32_t* __restrict__ first, int32_t* __restrict__ un,
                                                            unsigned long long* __restrict__ umask) {
  extern __shared__ int vq_u[];                    // [warp][g][kVqSlots]
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int w = blockIdx.x * kVqWarps + wid;       // (selection block, chunk of 2 S query blocks)
  const int B = w / cmax, ch = w % cmax;
  if (B >= c.n_blk[SSA_LEVEL_SLC]) return;         // warp-uniform
  int* u = vq_u + wid * c.h_kv * kVqSlots;
  int qa, qe;
  slc_qblocks(c, B, &qa, &qe);
  // chunks are walked independently (a sub-group never spans two): the serial walk is at most 2 S long
  qa += ch * 2 * S;
  if (qa >= qe) {
    if (lane == 0) cnt[w] = 0;
    return;
  }
  qe = min(qe, qa + 2 * S);
  int n_open = 0, size = 0, start = qa;
  int nu_lane = 0, nk_lane = 0;                    // lane g < h_kv: union size / keys of kv group g
  auto flush = [&](int k) {                        // write the open sub-group's unions as sub-group k
    for (int g = 0; g < c.h_kv; ++g) {
      const int nu = __shfl_sync(0xffffffffu, nu_lane, g);
      int32_t* o = un + (int64_t(qa + k) * c.h_kv + g) * kVqSlots;
#pragma unroll
      for (int q4 = 0; q4 < kVqSlots / 32; ++q4) o[lane + 32 * q4] = lane + 32 * q4 < nu ? u[g * kVqSlots + lane + 32 * q4] : -1;
    }
  };
  // candidates of the next query block, loaded one query block ahead (lane j < T: block I[q][g][j])
  int nxt[kVqMaxG];
#pragma unroll
  for (int g = 0; g < kVqMaxG; ++g) nxt[g] = g < c.h_kv && lane < c.T && qa < qe ? c.I[(int64_t(qa) * c.h_kv + g) * c.T + lane] : -1;
  int nxt_t = c.off[SSA_LEVEL_Q][qa];               // token range of the next query block, also one ahead
  for (int q = qa; q < qe; ++q) {
    int cand[kVqMaxG], ckeys[kVqMaxG];
#pragma unroll
    for (int g = 0; g < kVqMaxG; ++g) {
      cand[g] = nxt[g];
      ckeys[g] = cand[g] >= 0 ? c.off[SSA_LEVEL_SLC][cand[g] + 1] - c.off[SSA_LEVEL_SLC][cand[g]] : 0;
      nxt[g] = g < c.h_kv && lane < c.T && q + 1 < qe ? c.I[(int64_t(q + 1) * c.h_kv + g) * c.T + lane] : -1;
    }
    const int tq0 = nxt_t;
    nxt_t = c.off[SSA_LEVEL_Q][q + 1];
    const int tq1 = nxt_t;
    // membership of q's candidates in the open unions: slot or -1
    int slot[kVqMaxG];
    bool over = false;
#pragma unroll
    for (int g = 0; g < kVqMaxG; ++g) {
      slot[g] = -1;
      if (g >= c.h_kv) continue;
      const int Bj = cand[g];
      const int nu = __shfl_sync(0xffffffffu, nu_lane, g), nk = __shfl_sync(0xffffffffu, nk_lane, g);
      int uu[kVqSlots / 32];
#pragma unroll
      for (int q4 = 0; q4 < kVqSlots / 32; ++q4) uu[q4] = lane + 32 * q4 < nu ? u[g * kVqSlots + lane + 32 * q4] : -2;
      for (int j = 0; j < c.T; ++j) {
        const int b = __shfl_sync(0xffffffffu, Bj, j);
        int pos = -1;
#pragma unroll
        for (int q4 = kVqSlots / 32 - 1; q4 >= 0; --q4) {
          const unsigned h = __ballot_sync(0xffffffffu, uu[q4] == b);
          if (h) pos = 32 * q4 + __ffs(h) - 1;
        }
        if (lane == j && b >= 0) slot[g] = pos;
      }
      const bool is_new = Bj >= 0 && slot[g] < 0;
      const int nnew = __popc(__ballot_sync(0xffffffffu, is_new));
      const int knew = __reduce_add_sync(0xffffffffu, is_new ? ckeys[g] : 0);
      over |= nu + nnew > kVqSlots || nk + knew > kVqKeyCap;
    }
    if (size > 0 && (size == S || over)) {         // close the open sub-group before q
      flush(n_open);
      __syncwarp();                                 // flush's reads of the union before its reuse
      if (lane == 0) first[qa + n_open] = start;
      ++n_open;
      start = q;
      size = 0;
      nu_lane = 0;
      nk_lane = 0;
#pragma unroll
      for (int g = 0; g < kVqMaxG; ++g) slot[g] = -1;
    }
#pragma unroll
    for (int g = 0; g < kVqMaxG; ++g) {            // insert q's new blocks, q's slot mask
      if (g >= c.h_kv) continue;
      const int Bj = cand[g];
      const int nu = __shfl_sync(0xffffffffu, nu_lane, g);
      int sl = slot[g];
      const bool is_new = Bj >= 0 && sl < 0;
      const unsigned mk = __ballot_sync(0xffffffffu, is_new);
      const int knew = __reduce_add_sync(0xffffffffu, is_new ? ckeys[g] : 0);
      if (is_new) {
        sl = nu + __popc(mk & ((1u << lane) - 1u));
        u[g * kVqSlots + sl] = Bj;
      }
      __syncwarp();
      if (lane == g) {
        nu_lane = nu + __popc(mk);
        nk_lane += knew;
      }
      const bool hit = Bj >= 0 && sl >= 0;
      const uint32_t b0 = hit && sl < 32 ? 1u << sl : 0u, b1 = hit && sl >= 32 && sl < 64 ? 1u << (sl - 32) : 0u;
      const uint32_t b2 = hit && sl >= 64 && sl < 96 ? 1u << (sl - 64) : 0u, b3 = hit && sl >= 96 ? 1u << (sl - 96) : 0u;
      const unsigned long long m0 = (unsigned long long)__reduce_or_sync(0xffffffffu, b1) << 32 | __reduce_or_sync(0xffffffffu, b0);
      const unsigned long long m1 = (unsigned long long)__reduce_or_sync(0xffffffffu, b3) << 32 | __reduce_or_sync(0xffffffffu, b2);
      for (int t = tq0 + lane; t < tq1; t += 32) {
        umask[(int64_t(t) * c.h_kv + g) * 2] = m0;
        umask[(int64_t(t) * c.h_kv + g) * 2 + 1] = m1;
      }
    }
    ++size;
  }
  if (size > 0) flush(n_open);
  if (lane == 0) {
    if (size > 0) first[qa + n_open] = start;
    cnt[w] = n_open + (size > 0 ? 1 : 0);
  }
}

// plain sub-groups (no unions: the per-block selection pass empties the selection lists): chunk ch of
// selection block B as sub-groups of S consecutive query blocks
__global__ void k_vq_count_plain(Ctx c, int S, int cmax, int32_t* __restrict__ cnt, int32_t* __restrict__ first) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  const int B = w / cmax, ch = w % cmax;
  if (B >= c.n_blk[SSA_LEVEL_SLC]) return;
  int qa, qe;
  slc_qblocks(c, B, &qa, &qe);
  qa += ch * 2 * S;
  if (qa >= qe) { cnt[w] = 0; return; }
  qe = min(qe, qa + 2 * S);
  int k = 0;
  for (int q = qa; q < qe; q += S) first[qa + k++] = q;
  cnt[w] = k;
}

// sub-group v of selection block B covers query blocks [qa_v, qe_v): token offsets off_v, batch item,
// identity work order; slots past the real count are empty (off = N) so their CTAs do nothing
__global__ void k_vq_fill(Ctx c, int vT, int S, int cmax, const int32_t* __restrict__ start, const int32_t* __restrict__ first,
                          const int32_t* __restrict__ un, int32_t* __restrict__ I_u, int32_t* __restrict__ off_v,
                          int32_t* __restrict__ qrange, int32_t* __restrict__ batch_v, int32_t* __restrict__ order_v,
                          int bound) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v > bound) return;
  const int total = start[c.n_blk[SSA_LEVEL_SLC] * cmax];
  if (v < bound) order_v[v] = v;
  if (v >= total) {
    off_v[v] = c.N;
    if (v < bound) {
      qrange[2 * v] = qrange[2 * v + 1] = 0;
      batch_v[v] = 0;
      for (int j = 0; j < c.h_kv * vT; ++j) I_u[int64_t(v) * c.h_kv * vT + j] = -1;   // selects nothing
    }
    return;
  }
  int lo = 0, hi = c.n_blk[SSA_LEVEL_SLC] * cmax;   // chunk w with start[w] <= v < start[w + 1]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (start[mid] <= v) lo = mid; else hi = mid;
  }
  const int w = lo, B = w / cmax, ch = w % cmax;
  int qa, qe;
  slc_qblocks(c, B, &qa, &qe);
  qa += ch * 2 * S;
  qe = min(qe, qa + 2 * S);
  const int k = v - start[w];
  const int a = first[qa + k], e = k + 1 < start[w + 1] - start[w] ? first[qa + k + 1] : qe;
  off_v[v] = c.off[SSA_LEVEL_Q][a];
  qrange[2 * v] = a;
  qrange[2 * v + 1] = e;
  batch_v[v] = c.q_batch[a];
  for (int g = 0; g < c.h_kv; ++g)
    for (int j = 0; j < vT; ++j)
      I_u[(int64_t(v) * c.h_kv + g) * vT + j] = un ? un[(int64_t(qa + k) * c.h_kv + g) * kVqSlots + j] : -1;
}

}  // namespace

// KV-outer work-item size on the virtual level, in virtual query blocks (build knob SSA_VQ_QB_PER_ITEM;
// the partial-sum buffers scale with 1 / this)
// (knobs are read per call, so a test can switch them between calls)
int vq_qb_per_item() {
  const char* e = getenv("SSA_VQ_QB_PER_ITEM");
  const int x = e ? atoi(e) : 0;
  return x > 0 ? x : 128;
}
// the virtual level can be switched off (A/B knob SSA_VQ=0: the query-block tiles run as they are)
bool vq_enabled() {
  const char* e = getenv("SSA_VQ");
  return !(e && atoi(e) == 0);
}

int vq_slots(int S, int T) { return S * T < kVqSlots ? S * T : kVqSlots; }
// every sub-group but the last of a chunk holds S query blocks or was closed by a cap: by the slot cap it
// then holds > (128 - T) / T, i.e. >= floor(128 / T), query blocks; by the key cap (each query block adds
// at most T * max_fill keys) >= floor(kVqKeyCap / (T * max_fill)); one short sub-group per chunk of 2 S
int vq_kmin(int S, int T, int max_fill_slc) {
  int k = S < kVqSlots / T ? S : kVqSlots / T;
  const int kk = kVqKeyCap / (T * (max_fill_slc > 0 ? max_fill_slc : 1));
  k = k < kk ? k : kk;
  return k > 1 ? k : 1;
}
int64_t vq_bound(int n_slc, int n_q, int S, int T, int max_fill_slc) {
  const int kmin = vq_kmin(S, T, max_fill_slc);
  return int64_t(n_slc) * 2 + int64_t(n_q) / (2 * S) + (int64_t(n_q) + kmin - 1) / kmin + 1;
}
// chunks of 2 S query blocks per selection block (a selection block holds at most max_fill_slc of them,
// its most-populated one exactly that many tokens); the (selection block, chunk) grid is n_slc x cmax
static int vq_cmax(int max_fill_slc, int S) { return (max_fill_slc + 2 * S - 1) / (2 * S); }
size_t vq_ws_bytes(int64_t N, int h_kv, int n_slc, int n_q, int S, int T, int max_fill_slc) {
  const int64_t bound = vq_bound(n_slc, n_q, S, T, max_fill_slc);
  const int64_t chunks = int64_t(n_slc) * vq_cmax(max_fill_slc, S);
  return size_t(chunks + 2) * 4 * 2 + scan_ws_bytes(chunks + 1) + size_t(bound + 2) * 4 * 5 + size_t(n_q + 1) * 4 +
         size_t(n_q) * h_kv * kVqSlots * 4 +
         size_t(bound) * h_kv * vq_slots(S, T) * 4 + size_t(N) * h_kv * 16 + 18 * 256;
}

// Build the virtual query level (see the header) with sub-groups of at most S query blocks from the per-query-
// block selections c.I and return in *v the context the selection / window, dQ and KV-outer kernels run
// with.
ssa_status build_virtual_level(const Ctx& c, int S, void* ws, cudaStream_t st, Ctx* v, bool plain) {
  const int n_slc = c.n_blk[SSA_LEVEL_SLC], n_q = c.n_blk[SSA_LEVEL_Q];
  const int vT = vq_slots(S, c.T);
  if (S < 2 || c.T > 32) { set_error("virtual query level: bad sub-group size"); return SSA_ERR_UNSUPPORTED; }
  const int64_t bound = vq_bound(n_slc, n_q, S, c.T, c.max_fill[SSA_LEVEL_SLC]);
  Carve cw(ws, vq_ws_bytes(c.N, c.h_kv, n_slc, n_q, S, c.T, c.max_fill[SSA_LEVEL_SLC]));
  const int cmax = vq_cmax(c.max_fill[SSA_LEVEL_SLC], S);
  const int64_t nw = int64_t(n_slc) * cmax;
  int32_t* cnt = cw.take<int32_t>(nw + 1);
  int32_t* start = cw.take<int32_t>(nw + 1);
  int32_t* first = cw.take<int32_t>(n_q + 1);
  int32_t* un = cw.take<int32_t>(size_t(n_q) * c.h_kv * kVqSlots);
  void* sws = cw.take<char>(scan_ws_bytes(nw + 1));
  int32_t* off_v = cw.take<int32_t>(bound + 1);
  int32_t* qrange = cw.take<int32_t>(2 * bound + 2);
  int32_t* batch_v = cw.take<int32_t>(bound + 1);
  int32_t* order_v = cw.take<int32_t>(bound + 1);
  int32_t* I_u = cw.take<int32_t>(size_t(bound) * c.h_kv * vT);
  unsigned long long* umask = cw.take<unsigned long long>(size_t(c.N) * c.h_kv * 2);
  if (n_slc > 0) {
    if (plain) k_vq_count_plain<<<nb(nw, 128), 128, 0, st>>>(c, S, cmax, cnt, first);
    else k_vq_count<<<nb(nw, kVqWarps), 32 * kVqWarps, size_t(kVqWarps) * c.h_kv * kVqSlots * 4, st>>>(c, S, cmax, cnt, first, un, umask);
    SSA_LAUNCH_CHECK("k_vq_count");
  }
  ssa_status s = exclusive_scan(cnt, start, nw, start + nw, sws, st);
  if (s != SSA_OK) return s;
  k_vq_fill<<<nb(bound + 1, 256), 256, 0, st>>>(c, vT, S, cmax, start, first, plain ? nullptr : un, I_u, off_v, qrange, batch_v, order_v, int(bound));
  SSA_LAUNCH_CHECK("k_vq_fill");
  *v = c;
  v->tok_I = c.I;            // the per-query-block selections (KV-outer row masks)
  v->tok_T = c.T;
  v->tok_qb = c.tok_block[SSA_LEVEL_Q];
  v->off[SSA_LEVEL_Q] = off_v;
  v->n_blk[SSA_LEVEL_Q] = int32_t(bound);
  v->q_order = order_v;
  v->q_batch = batch_v;
  v->q_begin = 0;
  v->q_end = int32_t(bound);
  v->I = I_u;
  v->T = vT;
  v->umask = plain ? nullptr : umask;
  v->qb_per_item = vq_qb_per_item();     // KV-outer work items in virtual query blocks (bounds the partial buffers)
  return SSA_OK;
}


// ================================================================================================
// Per-block selection pass for per-token selection (m_q = 1). The union-based virtual level makes a row
// attend to its sub-group's union of selected blocks (masked), which with diverse per-token selections is
// many times the T blocks the row needs. This pass instead attends every (token, selected block) pair
// exactly once: for every (selection block B, kv group g), the tokens that selected B (the inverse
// selection CSR, ascending) are laid out contiguously in an "expanded" token space e, their q rows
// gathered into Q_exp [e][h_s][D]; the selection/window kernel runs on it with the single key block B per
// virtual query block of <= 32 expanded tokens (no window, epilogue = O and LSE only), and a merge
// combines each row's T partial results by their LSEs (log2 domain):
//   LSE = log2 sum_j 2^{LSE_j},  O_slc = sum_j 2^{LSE_j - LSE} O_j
// which is the softmax over the union of the T blocks' keys (Alg. 1's per-token selection attention).
// ================================================================================================
namespace {

constexpr int kBlkChunk = 32;   // expanded tokens per virtual query block (h_s = 8: a row-tile pair)

__device__ __forceinline__ int key_of(const int32_t* __restrict__ inv_off, int nkeys, int64_t e) {
  int lo = 0, hi = nkeys;         // largest key with inv_off[key] <= e
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (inv_off[mid] <= e) lo = mid; else hi = mid;
  }
  return lo;
}

// entries of the inverse CSR = (key, query block) pairs; etok = exclusive scan of their token counts (the
// expanded token space: an entry's tokens are contiguous, each token a row group of h_s rows)
__global__ void k_blk_entry_tokens(Ctx c, int32_t* __restrict__ cnt, int64_t n_entries_bound) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_entries_bound) return;
  const int nkeys = c.n_blk[SSA_LEVEL_SLC] * c.h_kv;
  if (i >= c.inv_off[nkeys]) { cnt[i] = 0; return; }
  const int Q = c.inv_list[i];
  cnt[i] = c.off[SSA_LEVEL_Q][Q + 1] - c.off[SSA_LEVEL_Q][Q];
}
__device__ __forceinline__ int64_t entry_of(const int32_t* __restrict__ etok, int64_t n_entries, int64_t e) {
  int64_t lo = 0, hi = n_entries;   // largest entry with etok[entry] <= e (token counts are >= 1)
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (etok[mid] <= e) lo = mid; else hi = mid;
  }
  return lo;
}

__global__ void k_blk_count(Ctx c, const int32_t* __restrict__ etok, int32_t* __restrict__ cnt) {
  const int key = blockIdx.x * blockDim.x + threadIdx.x;
  const int nkeys = c.n_blk[SSA_LEVEL_SLC] * c.h_kv;
  if (key >= nkeys) return;
  const int len = etok[c.inv_off[key + 1]] - etok[c.inv_off[key]];
  cnt[key] = (len + kBlkChunk - 1) / kBlkChunk;
}

// virtual query block v: expanded tokens [off_e[v], off_e[v + 1]) of key (B, g), its one block B' = g n_slc + B
__global__ void k_blk_fill(Ctx c, const int32_t* __restrict__ etok, const int32_t* __restrict__ start,
                           int32_t* __restrict__ off_e, int32_t* __restrict__ I_e, int32_t* __restrict__ order_e, int bound) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v > bound) return;
  const int nkeys = c.n_blk[SSA_LEVEL_SLC] * c.h_kv;
  const int total = start[nkeys], n_e = etok[c.inv_off[nkeys]];
  if (v < bound) order_e[v] = v;
  if (v >= total) {
    off_e[v] = n_e;
    if (v < bound) I_e[v] = -1;
    return;
  }
  int lo = 0, hi = nkeys;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (start[mid] <= v) lo = mid; else hi = mid;
  }
  const int key = lo, B = key / c.h_kv, g = key % c.h_kv;
  off_e[v] = etok[c.inv_off[key]] + (v - start[key]) * kBlkChunk;
  I_e[v] = g * c.n_blk[SSA_LEVEL_SLC] + B;
}

// selection-level offsets of the expanded context: block B' = g n_slc + B covers key rows g N + [C_B, C_B+1)
__global__ void k_blk_slc_off(Ctx c, int32_t* __restrict__ off) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int n_slc = c.n_blk[SSA_LEVEL_SLC];
  if (j > n_slc * c.h_kv) return;
  off[j] = j == n_slc * c.h_kv ? c.h_kv * c.N : (j / n_slc) * c.N + c.off[SSA_LEVEL_SLC][j % n_slc];
}

// expanded token e -> (kv group, token): entry i holding e, its key and query block
// (one-token query blocks, m_q = 1: entries and expanded tokens coincide, no search)
__device__ __forceinline__ void exp_token(const Ctx& c, const int32_t* __restrict__ etok, int64_t e, int* g, int* t) {
  const int nkeys = c.n_blk[SSA_LEVEL_SLC] * c.h_kv;
  const int64_t i = c.n_blk[SSA_LEVEL_Q] == c.N ? e : entry_of(etok, c.inv_off[nkeys], e);
  *g = key_of(c.inv_off, nkeys, i) % c.h_kv;
  const int Q = c.inv_list[i];
  *t = c.off[SSA_LEVEL_Q][Q] + int(e - etok[i]);
}
// position of token t (query block Q) of key (B, g) in the expanded token space (Q is in the key's list)
__device__ __forceinline__ int64_t exp_index(const Ctx& c, const int32_t* __restrict__ etok, int B, int g, int Q, int t) {
  const int key = B * c.h_kv + g;
  int lo = c.inv_off[key], hi = c.inv_off[key + 1];   // ascending query blocks: binary search for Q
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (c.inv_list[mid] < Q) lo = mid + 1; else hi = mid;
  }
  return int64_t(etok[lo]) + (t - c.off[SSA_LEVEL_Q][Q]);
}

// Q_exp[e] = the h_s q rows (internal layout) of expanded token e; one warp per e
__global__ void k_blk_gather(Ctx c, const int32_t* __restrict__ etok, __nv_bfloat16* __restrict__ q_exp) {
  const int64_t e = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nkeys = c.n_blk[SSA_LEVEL_SLC] * c.h_kv;
  if (e >= etok[c.inv_off[nkeys]]) return;
  int g, t;
  exp_token(c, etok, e, &g, &t);
  const uint4* src = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(c.qs) + (int64_t(g) * c.N + t) * c.h_s * c.D);
  uint4* dst = reinterpret_cast<uint4*>(q_exp + e * c.h_s * c.D);
  for (int i = lane; i < c.h_s * c.D / 8; i += 32) dst[i] = src[i];
}

// per row (token t, group g, head s): combine the T partial results of its selected blocks (one warp per (t, g))
__global__ void k_blk_merge(Ctx c, const int32_t* __restrict__ etok, const float* __restrict__ o_exp,
                            const float* __restrict__ lse_exp) {
  const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= int64_t(c.N) * c.h_kv) return;
  const int t = int(w / c.h_kv), g = int(w % c.h_kv);
  const int Q = c.tok_block[SSA_LEVEL_Q][t];
  // lane j < T: the expanded index of (t, j-th selected block), or -1
  int64_t ej = -1;
  if (lane < c.T) {
    const int B = c.I[(int64_t(Q) * c.h_kv + g) * c.T + lane];
    if (B >= 0) ej = exp_index(c, etok, B, g, Q, t);
  }
  const int64_t row0 = (int64_t(g) * c.N + t) * c.h_s;
  float* O = static_cast<float*>(c.o[1]);
  for (int idx = lane * 4; idx < c.h_s * c.D; idx += 128) {
    const int s = idx / c.D, col = idx % c.D;
    float M = -INFINITY;
    for (int j = 0; j < c.T; ++j) {
      const int64_t e = __shfl_sync(0xffffffffu, ej, j);
      if (e >= 0) M = fmaxf(M, lse_exp[e * c.h_s + s]);
    }
    float L = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j = 0; j < c.T; ++j) {
      const int64_t e = __shfl_sync(0xffffffffu, ej, j);
      if (e < 0) continue;
      const float wgt = exp2f(lse_exp[e * c.h_s + s] - M);
      const float4 o = *reinterpret_cast<const float4*>(o_exp + (e * c.h_s + s) * c.D + col);
      L += wgt;
      acc.x += wgt * o.x; acc.y += wgt * o.y; acc.z += wgt * o.z; acc.w += wgt * o.w;
    }
    const float inv = L > 0.f ? 1.f / L : 0.f;
    *reinterpret_cast<float4*>(O + (row0 + s) * c.D + col) = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
    if (col == 0) c.lse[1][row0 + s] = L > 0.f ? M + log2f(L) : __int_as_float(0x7f7f7f7f);
  }
}

}  // namespace

bool blk_enabled() {
  const char* e = getenv("SSA_VQ_BLOCKSEL");
  return !(e && atoi(e) == 0);
}
bool blk_forced() {
  const char* e = getenv("SSA_VQ_BLOCKSEL");
  return e && atoi(e) == 2;
}
static int64_t blk_bound(int n_slc, int h_kv, int64_t n_exp) { return int64_t(n_slc) * h_kv + n_exp / kBlkChunk + 1; }
// entries (key, query block) <= n_q h_kv T; expanded tokens <= N h_kv T (a token is in <= T lists per group)
static size_t blk_entries_bytes(int64_t n_ent) { return size_t(n_ent + 2) * 4 * 2 + scan_ws_bytes(n_ent + 1) + 3 * 256; }
size_t blk_ws_bytes(int64_t N, int h_kv, int h_s, int D, int n_slc, int n_q, int T) {
  const int64_t n_ent = int64_t(n_q) * h_kv * T, n_exp = N * h_kv * T, nkeys = int64_t(n_slc) * h_kv;
  const int64_t bound = blk_bound(n_slc, h_kv, n_exp);
  return inverse_csr_ws_bytes(n_slc, h_kv, n_q) + size_t(nkeys + 2) * 4 * 3 + size_t(n_ent + 1) * 4 +
         blk_entries_bytes(n_ent) + scan_ws_bytes(nkeys + 1) + size_t(bound + 2) * 4 * 3 + size_t(nkeys + 2) * 4 +
         size_t(n_exp) * h_s * D * 2 + size_t(n_exp) * h_s * D * 4 + size_t(n_exp) * h_s * 4 + 16 * 256;
}
// etok over the inverse CSR's entries (exclusive scan of their token counts)
static ssa_status blk_entries(const Ctx& c, int64_t n_ent, Carve& cw, cudaStream_t st, int32_t** etok) {
  int32_t* tc = cw.take<int32_t>(n_ent + 2);
  *etok = cw.take<int32_t>(n_ent + 2);
  void* ws = cw.take<char>(scan_ws_bytes(n_ent + 1));
  k_blk_entry_tokens<<<nb(n_ent + 1, 256), 256, 0, st>>>(c, tc, n_ent + 1);
  SSA_LAUNCH_CHECK("k_blk_entry_tokens");
  return exclusive_scan(tc, *etok, n_ent + 1, nullptr, ws, st);
}

ssa_status blk_build(const Ctx& c, void* ws, cudaStream_t st, BlkPass* b) {
  const int n_slc = c.n_blk[SSA_LEVEL_SLC], n_q = c.n_blk[SSA_LEVEL_Q];
  const int64_t n_ent = int64_t(n_q) * c.h_kv * c.T, n_exp = int64_t(c.N) * c.h_kv * c.T;
  const int64_t nkeys = int64_t(n_slc) * c.h_kv, bound = blk_bound(n_slc, c.h_kv, n_exp);
  Carve cw(ws, blk_ws_bytes(c.N, c.h_kv, c.h_s, c.D, n_slc, n_q, c.T));
  void* inv_ws = cw.take<char>(inverse_csr_ws_bytes(n_slc, c.h_kv, n_q));
  Ctx ci = c;
  ci.inv_off = cw.take<int32_t>(nkeys + 2);
  ci.inv_list = cw.take<int32_t>(n_ent + 1);
  int32_t* cnt = cw.take<int32_t>(nkeys + 2);
  int32_t* start = cw.take<int32_t>(nkeys + 2);
  void* sws = cw.take<char>(scan_ws_bytes(nkeys + 1));
  b->off_e = cw.take<int32_t>(bound + 2);
  b->I_e = cw.take<int32_t>(bound + 2);
  b->order_e = cw.take<int32_t>(bound + 2);
  b->off_slc = cw.take<int32_t>(nkeys + 2);
  b->q_exp = cw.take<__nv_bfloat16>(size_t(n_exp) * c.h_s * c.D);
  b->o_exp = cw.take<float>(size_t(n_exp) * c.h_s * c.D);
  b->lse_exp = cw.take<float>(size_t(n_exp) * c.h_s);
  b->bound = bound;
  b->n_exp = n_exp;
  b->inv_off = ci.inv_off;
  b->inv_list = ci.inv_list;
  ssa_status s = build_inverse_csr(ci, inv_ws, st);
  if (s != SSA_OK) return s;
  if ((s = blk_entries(ci, n_ent, cw, st, &b->etok)) != SSA_OK) return s;
  if (!cw.ok()) { set_error("per-block selection: workspace carve"); return SSA_ERR_WORKSPACE; }
  k_blk_count<<<nb(nkeys, 256), 256, 0, st>>>(ci, b->etok, cnt);
  SSA_LAUNCH_CHECK("k_blk_count");
  if ((s = exclusive_scan(cnt, start, nkeys, start + nkeys, sws, st)) != SSA_OK) return s;
  k_blk_fill<<<nb(bound + 1, 256), 256, 0, st>>>(ci, b->etok, start, b->off_e, b->I_e, b->order_e, int(bound));
  SSA_LAUNCH_CHECK("k_blk_fill");
  k_blk_slc_off<<<nb(nkeys + 1, 256), 256, 0, st>>>(ci, b->off_slc);
  SSA_LAUNCH_CHECK("k_blk_slc_off");
  k_blk_gather<<<nb(n_exp * 32, 256), 256, 0, st>>>(ci, b->etok, b->q_exp);
  SSA_LAUNCH_CHECK("k_blk_gather");
  return SSA_OK;
}

// the expanded context the selection kernel runs on (h_kv = 1 view: blocks B' = g n_slc + B over all
// groups' key rows; no window; epilogue O / LSE only)
Ctx blk_context(const Ctx& c, const BlkPass& b) {
  Ctx e = c;
  e.h_kv = 1;
  e.N = int32_t(b.n_exp);
  e.T = 1;
  e.n_blk[SSA_LEVEL_Q] = int32_t(b.bound);
  e.n_blk[SSA_LEVEL_SLC] = c.n_blk[SSA_LEVEL_SLC] * c.h_kv;
  e.off[SSA_LEVEL_Q] = b.off_e;
  e.off[SSA_LEVEL_SLC] = b.off_slc;
  e.I = b.I_e;
  e.q_order = b.order_e;
  e.q_begin = 0;
  e.q_end = int32_t(b.bound);
  e.no_win = 1;
  e.accumulate = 0;
  e.sel_partial = 1;
  e.umask = nullptr;
  e.o[1] = b.o_exp;
  e.lse[1] = b.lse_exp;
  e.qs = b.q_exp;
  return e;
}

ssa_status blk_merge(const Ctx& c, const BlkPass& b, cudaStream_t st) {
  Ctx ci = c;
  ci.inv_off = b.inv_off;
  ci.inv_list = b.inv_list;
  const int64_t warps = int64_t(c.N) * c.h_kv;
  k_blk_merge<<<nb(warps * 32, 256), 256, 0, st>>>(ci, b.etok, b.o_exp, b.lse_exp);
  SSA_LAUNCH_CHECK("k_blk_merge");
  return SSA_OK;
}


// ---- backward: the selection branch's dQ per block ----------------------------------------------
namespace {
// expanded row operands: fp16 q / dO rows of token inv_list[e] in e's kv group, its selection-branch row
// stats (LSE, D) and gates; one warp per e
__global__ void k_blk_gather_bwd(Ctx c, const int32_t* __restrict__ etok, const __half* __restrict__ q16,
                                 const __half* __restrict__ do16, __half* __restrict__ q_e, __half* __restrict__ do_e,
                                 float* __restrict__ lse_e, float* __restrict__ D_e, float* __restrict__ gs_e) {
  const int64_t e = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nkeys = c.n_blk[SSA_LEVEL_SLC] * c.h_kv;
  if (e >= etok[c.inv_off[nkeys]]) return;
  int g, t;
  exp_token(c, etok, e, &g, &t);
  const int64_t r0 = (int64_t(g) * c.N + t) * c.h_s;
  const uint4* sq = reinterpret_cast<const uint4*>(q16 + r0 * c.D);
  const uint4* sd = reinterpret_cast<const uint4*>(do16 + r0 * c.D);
  uint4* dq_ = reinterpret_cast<uint4*>(q_e + e * c.h_s * c.D);
  uint4* dd_ = reinterpret_cast<uint4*>(do_e + e * c.h_s * c.D);
  for (int i = lane; i < c.h_s * c.D / 8; i += 32) {
    dq_[i] = sq[i];
    dd_[i] = sd[i];
  }
  for (int s = lane; s < c.h_s; s += 32) {
    lse_e[e * c.h_s + s] = c.lse[1][r0 + s];
    D_e[e * c.h_s + s] = c.Dd[1][r0 + s];
#pragma unroll
    for (int k = 0; k < 3; ++k) gs_e[(e * c.h_s + s) * 3 + k] = c.gs[(r0 + s) * 3 + k];
  }
}
// dq_extra of row (t, g, s) = sum over its selected blocks j (slot order) of the per-block partials
__global__ void k_blk_merge_bwd(Ctx c, const int32_t* __restrict__ etok, const float* __restrict__ dq_part,
                                float* __restrict__ dq_extra) {
  const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= int64_t(c.N) * c.h_kv) return;
  const int t = int(w / c.h_kv), g = int(w % c.h_kv);
  const int Q = c.tok_block[SSA_LEVEL_Q][t];
  int64_t ej = -1;
  if (lane < c.T) {
    const int B = c.I[(int64_t(Q) * c.h_kv + g) * c.T + lane];
    if (B >= 0) ej = exp_index(c, etok, B, g, Q, t);
  }
  const int64_t row0 = (int64_t(g) * c.N + t) * c.h_s;
  for (int idx = lane * 4; idx < c.h_s * c.D; idx += 128) {
    const int s = idx / c.D, col = idx % c.D;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j = 0; j < c.T; ++j) {
      const int64_t e = __shfl_sync(0xffffffffu, ej, j);
      if (e < 0) continue;
      const float4 x = *reinterpret_cast<const float4*>(dq_part + (e * c.h_s + s) * c.D + col);
      acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
    }
    *reinterpret_cast<float4*>(dq_extra + (row0 + s) * c.D + col) = acc;
  }
}
}  // namespace

size_t blk_bwd_ws_bytes(int64_t N, int h_kv, int h_s, int D, int n_slc, int n_q, int T) {
  const int64_t n_ent = int64_t(n_q) * h_kv * T, n_exp = N * h_kv * T, nkeys = int64_t(n_slc) * h_kv;
  const int64_t bound = blk_bound(n_slc, h_kv, n_exp), re = n_exp * h_s;
  return blk_entries_bytes(n_ent) + size_t(nkeys + 2) * 4 * 3 + scan_ws_bytes(nkeys + 1) + size_t(bound + 2) * 4 * 4 +
         size_t(re) * D * 2 * 2 + size_t(re) * 4 * 5 + size_t(re) * D * 4 + size_t(N) * h_kv * h_s * D * 4 + 20 * 256;
}

ssa_status blk_bwd_build(const Ctx& c, const __half* q16, const __half* do16, void* ws, cudaStream_t st, BlkPass* b,
                         Ctx* e, float** dq_extra) {
  const int n_slc = c.n_blk[SSA_LEVEL_SLC], n_q = c.n_blk[SSA_LEVEL_Q];
  const int64_t n_ent = int64_t(n_q) * c.h_kv * c.T, n_exp = int64_t(c.N) * c.h_kv * c.T;
  const int64_t nkeys = int64_t(n_slc) * c.h_kv, bound = blk_bound(n_slc, c.h_kv, n_exp), re = n_exp * c.h_s;
  Carve cw(ws, blk_bwd_ws_bytes(c.N, c.h_kv, c.h_s, c.D, n_slc, n_q, c.T));
  int32_t* cnt = cw.take<int32_t>(nkeys + 2);
  int32_t* start = cw.take<int32_t>(nkeys + 2);
  void* sws = cw.take<char>(scan_ws_bytes(nkeys + 1));
  b->off_e = cw.take<int32_t>(bound + 2);
  b->I_e = cw.take<int32_t>(bound + 2);
  b->order_e = cw.take<int32_t>(bound + 2);
  b->batch_e = cw.take<int32_t>(bound + 2);
  b->off_slc = cw.take<int32_t>(nkeys + 2);
  __half* q_e = cw.take<__half>(size_t(re) * c.D);
  __half* do_e = cw.take<__half>(size_t(re) * c.D);
  float* lse_e = cw.take<float>(re);
  float* D_e = cw.take<float>(re);
  float* gs_e = cw.take<float>(size_t(re) * 3);
  float* dq_part = cw.take<float>(size_t(re) * c.D);
  *dq_extra = cw.take<float>(size_t(c.N) * c.h_kv * c.h_s * c.D);
  if (!cw.ok()) { set_error("per-block selection dQ: workspace carve"); return SSA_ERR_WORKSPACE; }
  b->bound = bound;
  b->n_exp = n_exp;
  b->inv_off = c.inv_off;
  b->inv_list = c.inv_list;
  b->q_exp = nullptr;
  b->o_exp = nullptr;
  b->lse_exp = lse_e;
  b->dq_part = dq_part;
  ssa_status s = blk_entries(c, n_ent, cw, st, &b->etok);
  if (s != SSA_OK) return s;
  if (!cw.ok()) { set_error("per-block selection dQ: workspace carve"); return SSA_ERR_WORKSPACE; }
  k_blk_count<<<nb(nkeys, 256), 256, 0, st>>>(c, b->etok, cnt);
  SSA_LAUNCH_CHECK("k_blk_count");
  if ((s = exclusive_scan(cnt, start, nkeys, start + nkeys, sws, st)) != SSA_OK) return s;
  k_blk_fill<<<nb(bound + 1, 256), 256, 0, st>>>(c, b->etok, start, b->off_e, b->I_e, b->order_e, int(bound));
  SSA_LAUNCH_CHECK("k_blk_fill");
  k_blk_slc_off<<<nb(nkeys + 1, 256), 256, 0, st>>>(c, b->off_slc);
  SSA_LAUNCH_CHECK("k_blk_slc_off");
  SSA_CUDA_TRY(cudaMemsetAsync(b->batch_e, 0, size_t(bound + 2) * 4, st));
  k_blk_gather_bwd<<<nb(n_exp * 32, 256), 256, 0, st>>>(c, b->etok, q16, do16, q_e, do_e, lse_e, D_e, gs_e);
  SSA_LAUNCH_CHECK("k_blk_gather_bwd");
  Ctx x = c;
  x.h_kv = 1;
  x.N = int32_t(n_exp);
  x.T = 1;
  x.n_blk[SSA_LEVEL_Q] = int32_t(bound);
  x.n_blk[SSA_LEVEL_SLC] = n_slc * c.h_kv;
  x.off[SSA_LEVEL_Q] = b->off_e;
  x.off[SSA_LEVEL_SLC] = b->off_slc;
  x.I = b->I_e;
  x.q_order = b->order_e;
  x.q_batch = b->batch_e;
  x.q_begin = 0;
  x.q_end = int32_t(bound);
  x.no_win = 1;
  x.win_only = 0;
  x.accumulate = 0;
  x.sel_partial = 1;
  x.umask = nullptr;
  x.dq_extra = nullptr;
  x.dq_part = dq_part;
  for (int br = 0; br < 3; ++br) { x.lse[br] = lse_e; x.Dd[br] = D_e; }
  x.gs = gs_e;
  x.qs = q_e;        // (the tensor maps of the expanded rows are built from these two)
  x.dos = do_e;
  *e = x;
  return SSA_OK;
}

ssa_status blk_bwd_merge(const Ctx& c, const BlkPass& b, float* dq_extra, cudaStream_t st) {
  const int64_t warps = int64_t(c.N) * c.h_kv;
  k_blk_merge_bwd<<<nb(warps * 32, 256), 256, 0, st>>>(c, b.etok, b.dq_part, dq_extra);
  SSA_LAUNCH_CHECK("k_blk_merge_bwd");
  return SSA_OK;
}

}  // namespace ssa
