// build.cu — ssa_build_blocks: spatial block partition, token sort and block start offsets C.
// PAPER.md:143 (m^3 subgrids -> blocks), P:175 ("first sort the input tokens based on their block
// indices, then compute the starting index C"), Alg. 1 line 2.
//
// B200 design: instead of a comparison/radix sort, every token's hierarchical sort key is a dense
// mixed-radix cell index (b, coarse block, sub-block digits..., voxel-in-finest-block). Marking the
// occupied cells in a bitmap and taking popcount prefix sums gives every token its sorted rank
// directly (a counting sort over the dense key space): O(N + cells/32) work, fully coalesced, with
// duplicate detection for free (the bit was already set). Block starts of each level are then a
// flag + scan compaction over the sorted coordinates.
#include <algorithm>
#include <numeric>

#include "internal.h"

namespace ssa {
namespace {

struct KeySpec {
  int32_t batch;
  int32_t n_lv;          // number of distinct sizes
  int32_t ms[4];         // distinct sizes, descending
  int32_t coarse[3];     // number of coarsest blocks per axis
  int64_t cells;         // total key space
  int32_t grid[3];
};

enum : int32_t { kErrDup = 1, kErrRange = 2 };

__device__ __forceinline__ int64_t cell_key(const KeySpec& ks, int32_t b, int32_t x, int32_t y, int32_t z) {
  const int32_t m0 = ks.ms[0];
  int64_t key = b;
  key = key * ks.coarse[0] + x / m0;
  key = key * ks.coarse[1] + y / m0;
  key = key * ks.coarse[2] + z / m0;
  for (int l = 1; l < ks.n_lv; ++l) {
    const int32_t lo = ks.ms[l], r = ks.ms[l - 1] / lo;
    key = key * r + (x / lo) % r;
    key = key * r + (y / lo) % r;
    key = key * r + (z / lo) % r;
  }
  const int32_t ml = ks.ms[ks.n_lv - 1];
  key = key * ml + x % ml;
  key = key * ml + y % ml;
  key = key * ml + z % ml;
  return key;
}

__global__ void k_mark(const int4* __restrict__ coords, int64_t n, KeySpec ks, uint32_t* __restrict__ bitmap,
                       int64_t* __restrict__ keys, int32_t* __restrict__ err) {
  int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  int4 c = coords[t];
  if (c.x < 0 || c.x >= ks.batch || c.y < 0 || c.y >= ks.grid[0] || c.z < 0 || c.z >= ks.grid[1] || c.w < 0 ||
      c.w >= ks.grid[2]) {
    atomicOr(err, kErrRange);
    keys[t] = -1;
    return;
  }
  int64_t key = cell_key(ks, c.x, c.y, c.z, c.w);
  keys[t] = key;
  uint32_t bit = 1u << (key & 31);
  uint32_t old = atomicOr(bitmap + (key >> 5), bit);
  if (old & bit) atomicOr(err, kErrDup);
}

// popcount of 32-word (1024-bit) chunks
__global__ void k_chunk_popc(const uint32_t* __restrict__ bitmap, int64_t n_chunks, int32_t* __restrict__ cnt) {
  int64_t c = int64_t(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (c >= n_chunks) return;
  const int lane = threadIdx.x & 31;
  int v = __popc(bitmap[c * 32 + lane]);
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) cnt[c] = v;
}

__global__ void k_scatter(const int4* __restrict__ coords, const int64_t* __restrict__ keys, int64_t n,
                          const uint32_t* __restrict__ bitmap, const int32_t* __restrict__ chunk_pre,
                          int32_t* __restrict__ perm, int32_t* __restrict__ inv_perm, int4* __restrict__ sorted) {
  int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  int64_t key = keys[t];
  int64_t w = key >> 5, c = key >> 10;
  int32_t r = chunk_pre[c];
  for (int64_t i = c * 32; i < w; ++i) r += __popc(bitmap[i]);
  r += __popc(bitmap[w] & ((1u << (key & 31)) - 1u));
  perm[r] = int32_t(t);
  inv_perm[t] = r;
  sorted[r] = coords[t];
}

__device__ __forceinline__ bool same_block(int4 a, int4 b, int32_t m) {
  return a.x == b.x && a.y / m == b.y / m && a.z / m == b.z / m && a.w / m == b.w / m;
}

__global__ void k_flags(const int4* __restrict__ sorted, int64_t n, int32_t m, int32_t* __restrict__ flags) {
  int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  flags[p] = (p == 0 || !same_block(sorted[p], sorted[p - 1], m)) ? 1 : 0;
}

__global__ void k_blocks(const int4* __restrict__ sorted, int64_t n, int32_t m, const int32_t* __restrict__ flags,
                         const int32_t* __restrict__ excl, const int32_t* __restrict__ total,
                         int32_t* __restrict__ offsets, int4* __restrict__ bcoords, int32_t* __restrict__ tok_block) {
  int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  int32_t id = excl[p] + flags[p] - 1;
  tok_block[p] = id;
  if (flags[p]) {
    offsets[id] = int32_t(p);
    int4 c = sorted[p];
    bcoords[id] = make_int4(c.x, c.y / m, c.z / m, c.w / m);
  }
  if (p == n - 1) offsets[*total] = int32_t(n);
}

__global__ void k_max_fill(const int32_t* __restrict__ offsets, const int32_t* __restrict__ total,
                           int32_t* __restrict__ out) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  int32_t nb = *total;
  int32_t v = (i < nb) ? offsets[i + 1] - offsets[i] : 0;
#pragma unroll
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0 && v) atomicMax(out, v);
}

// batch_tokens[b] = first sorted token with batch >= b; batch_blocks[l][b] likewise for blocks
__global__ void k_batch(const int4* __restrict__ sorted, int64_t n, int32_t batch, int32_t* __restrict__ batch_tokens,
                        int32_t* const* tok_block, int32_t* const* batch_blocks, const int32_t* __restrict__ totals) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b > batch) return;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (sorted[mid].x < b) lo = mid + 1; else hi = mid;
  }
  batch_tokens[b] = int32_t(lo);
  for (int l = 0; l < kLevels; ++l) batch_blocks[l][b] = (lo < n) ? tok_block[l][lo] : totals[l];
}

__global__ void k_links(const int32_t* __restrict__ off_cmp, const int32_t* __restrict__ off_slc,
                        const int32_t* __restrict__ tb_cmp, const int32_t* __restrict__ tb_slc,
                        const int32_t* __restrict__ totals, int32_t* __restrict__ cmp_to_slc,
                        int32_t* __restrict__ slc_cmp_begin) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int32_t n_cmp = totals[SSA_LEVEL_CMP], n_slc = totals[SSA_LEVEL_SLC];
  if (i < n_cmp) cmp_to_slc[i] = tb_slc[off_cmp[i]];
  if (i < n_slc) slc_cmp_begin[i] = tb_cmp[off_slc[i]];
  if (i == n_slc) slc_cmp_begin[i] = n_cmp;
}

__global__ void k_q_batch(const int4* __restrict__ bcoords_q, const int32_t* __restrict__ totals,
                          int32_t* __restrict__ q_batch) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < totals[SSA_LEVEL_Q]) q_batch[i] = bcoords_q[i].x;
}

inline unsigned nblk(int64_t n, int t) { return unsigned((n + t - 1) / t); }

bool make_keyspec(int32_t batch, const int32_t grid[3], const int32_t m[4], KeySpec* ks, std::string* why) {
  std::vector<int32_t> ms(m, m + 4);
  for (int32_t v : ms)
    if (v < 1) { *why = "block sizes must be >= 1"; return false; }
  std::sort(ms.begin(), ms.end(), std::greater<int32_t>());
  ms.erase(std::unique(ms.begin(), ms.end()), ms.end());
  for (size_t i = 1; i < ms.size(); ++i)
    if (ms[i - 1] % ms[i]) { *why = "distinct block sizes must form a divisibility chain"; return false; }
  if (m[SSA_LEVEL_SLC] % m[SSA_LEVEL_CMP]) { *why = "m_slc must be a multiple of m_cmp (PAPER.md:166)"; return false; }
  ks->batch = batch;
  ks->n_lv = int32_t(ms.size());
  for (int i = 0; i < 4; ++i) ks->ms[i] = i < ks->n_lv ? ms[i] : 1;
  ks->cells = batch;
  for (int a = 0; a < 3; ++a) {
    ks->grid[a] = grid[a];
    ks->coarse[a] = (grid[a] + ms[0] - 1) / ms[0];
    ks->cells *= int64_t(ks->coarse[a]) * ms[0];
  }
  return true;
}

struct BuildWs {
  uint32_t* bitmap;
  int32_t* chunk_cnt;
  int64_t* keys;
  int32_t* flags;
  int32_t* excl;
  int32_t* dev_small;   // [0]=err, [1..4]=totals, [5..8]=max_fill
  int32_t** ptr_tab;    // device table of 8 pointers (tok_block[4], batch_blocks[4])
  void* scan_ws;
};

size_t carve_plan(Carve& c, Plan* p, int64_t n, int32_t batch) {
  p->perm = c.take<int32_t>(n);
  p->inv_perm = c.take<int32_t>(n);
  p->sorted_coords = c.take<int32_t>(4 * n);
  for (int l = 0; l < kLevels; ++l) {
    p->offsets[l] = c.take<int32_t>(n + 1);
    p->block_coords[l] = c.take<int32_t>(4 * n);
    p->tok_block[l] = c.take<int32_t>(n);
    p->batch_blocks[l] = c.take<int32_t>(batch + 1);
  }
  p->batch_tokens = c.take<int32_t>(batch + 1);
  p->cmp_to_slc = c.take<int32_t>(n);
  p->slc_cmp_begin = c.take<int32_t>(n + 1);
  p->q_order = c.take<int32_t>(n);
  p->q_batch = c.take<int32_t>(n);
  p->cmp_tiles = c.take<int32_t>(2 * (n + batch));
  return c.used;
}

size_t carve_ws(Carve& c, BuildWs* w, int64_t n, int64_t cells) {
  int64_t n_chunks = (cells + 1023) / 1024;
  w->bitmap = c.take<uint32_t>(n_chunks * 32);
  w->chunk_cnt = c.take<int32_t>(n_chunks);
  w->keys = c.take<int64_t>(n);
  w->flags = c.take<int32_t>(n);
  w->excl = c.take<int32_t>(std::max<int64_t>(n, n_chunks));
  w->dev_small = c.take<int32_t>(16);
  w->ptr_tab = c.take<int32_t*>(8);
  w->scan_ws = c.take<char>(scan_ws_bytes(std::max<int64_t>(n, n_chunks)));
  return c.used;
}
}  // namespace
}  // namespace ssa

using namespace ssa;

extern "C" ssa_status ssa_build_blocks_size(int64_t n, int32_t batch, const int32_t grid[3], int32_t m_cmp,
                                            int32_t m_slc, int32_t m_win, int32_t m_q, size_t* plan_bytes,
                                            size_t* ws_bytes) {
  if (n < 0 || batch < 1 || !grid || !plan_bytes || !ws_bytes) { set_error("bad argument"); return SSA_ERR_ARG; }
  const int32_t m[4] = {m_cmp, m_slc, m_win, m_q};
  KeySpec ks;
  std::string why;
  if (!make_keyspec(batch, grid, m, &ks, &why)) { set_error(why); return SSA_ERR_HIERARCHY; }
  if (ks.cells > (int64_t(1) << 34)) { set_error("key space exceeds 2^34 cells"); return SSA_ERR_UNSUPPORTED; }
  Plan p;
  Carve cp(nullptr, 0);
  *plan_bytes = carve_plan(cp, &p, std::max<int64_t>(n, 1), batch) + 256;
  BuildWs w;
  Carve cw(nullptr, 0);
  *ws_bytes = carve_ws(cw, &w, std::max<int64_t>(n, 1), ks.cells) + 256;
  return SSA_OK;
}

extern "C" ssa_status ssa_build_blocks(const int32_t* coords, int64_t n, int32_t batch, const int32_t grid[3],
                                       int32_t m_cmp, int32_t m_slc, int32_t m_win, int32_t m_q, void* plan_buf,
                                       size_t plan_bytes, void* ws, size_t ws_bytes, void* stream, ssa_plan* out) {
  if (!out || n < 1 || (n > 0 && !coords) || batch < 1 || !grid || !plan_buf || !ws) {
    set_error("bad argument (need n >= 1, non-null coords/plan_buf/ws/out)");
    return SSA_ERR_ARG;
  }
  if (n >= (int64_t(1) << 31)) { set_error("n must be < 2^31"); return SSA_ERR_UNSUPPORTED; }
  *out = nullptr;
  size_t need_plan, need_ws;
  ssa_status s = ssa_build_blocks_size(n, batch, grid, m_cmp, m_slc, m_win, m_q, &need_plan, &need_ws);
  if (s != SSA_OK) return s;
  if (plan_bytes < need_plan || ws_bytes < need_ws) { set_error("plan/ws buffer too small"); return SSA_ERR_WORKSPACE; }
  const int32_t m[4] = {m_cmp, m_slc, m_win, m_q};
  KeySpec ks;
  std::string why;
  make_keyspec(batch, grid, m, &ks, &why);
  cudaStream_t st = static_cast<cudaStream_t>(stream);

  Plan* p = new Plan();
  Carve cp(plan_buf, plan_bytes);
  carve_plan(cp, p, n, batch);
  BuildWs w;
  Carve cw(ws, ws_bytes);
  carve_ws(cw, &w, n, ks.cells);
  const int64_t n_chunks = (ks.cells + 1023) / 1024;
  auto fail = [&](ssa_status e) { delete p; return e; };

#define TRY(x) do { ssa_status _s = (x); if (_s != SSA_OK) return fail(_s); } while (0)
#define CTRY(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) return fail(cuda_status(_e, #x)); } while (0)
  CTRY(cudaMemsetAsync(w.bitmap, 0, size_t(n_chunks) * 128, st));
  CTRY(cudaMemsetAsync(w.dev_small, 0, 16 * sizeof(int32_t), st));
  const int4* c4 = reinterpret_cast<const int4*>(coords);
  k_mark<<<nblk(n, 256), 256, 0, st>>>(c4, n, ks, w.bitmap, w.keys, w.dev_small);
  count_launch();
  CTRY(cudaGetLastError());
  // validation needs the flags before the rank pass (a duplicate / out-of-range key breaks ranks)
  int32_t err = 0;
  CTRY(cudaMemcpyAsync(&err, w.dev_small, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CTRY(cudaStreamSynchronize(st));
  if (err & kErrRange) { set_error("coordinate or batch index out of range"); return fail(SSA_ERR_COORD_RANGE); }
  if (err & kErrDup) { set_error("duplicate coordinates"); return fail(SSA_ERR_DUP_COORD); }

  k_chunk_popc<<<nblk(n_chunks * 32, 256), 256, 0, st>>>(w.bitmap, n_chunks, w.chunk_cnt);
  count_launch();
  CTRY(cudaGetLastError());
  TRY(exclusive_scan(w.chunk_cnt, w.excl, n_chunks, nullptr, w.scan_ws, st));
  int4* sorted = reinterpret_cast<int4*>(p->sorted_coords);
  k_scatter<<<nblk(n, 256), 256, 0, st>>>(c4, w.keys, n, w.bitmap, w.excl, p->perm, p->inv_perm, sorted);
  count_launch();
  CTRY(cudaGetLastError());
  int32_t* totals = w.dev_small + 1;
  int32_t* maxfill = w.dev_small + 5;
  for (int l = 0; l < kLevels; ++l) {
    k_flags<<<nblk(n, 256), 256, 0, st>>>(sorted, n, m[l], w.flags);
    count_launch();
    CTRY(cudaGetLastError());
    TRY(exclusive_scan(w.flags, w.excl, n, totals + l, w.scan_ws, st));
    k_blocks<<<nblk(n, 256), 256, 0, st>>>(sorted, n, m[l], w.flags, w.excl, totals + l, p->offsets[l],
                                           reinterpret_cast<int4*>(p->block_coords[l]), p->tok_block[l]);
    count_launch();
    CTRY(cudaGetLastError());
    k_max_fill<<<nblk(n, 256), 256, 0, st>>>(p->offsets[l], totals + l, maxfill + l);
    count_launch();
    CTRY(cudaGetLastError());
  }
  int32_t* tab_h[8];
  for (int l = 0; l < kLevels; ++l) { tab_h[l] = p->tok_block[l]; tab_h[4 + l] = p->batch_blocks[l]; }
  CTRY(cudaMemcpyAsync(w.ptr_tab, tab_h, sizeof(tab_h), cudaMemcpyHostToDevice, st));
  k_batch<<<nblk(batch + 1, 128), 128, 0, st>>>(sorted, n, batch, p->batch_tokens, w.ptr_tab, w.ptr_tab + 4, totals);
  count_launch();
  CTRY(cudaGetLastError());
  k_links<<<nblk(n + 1, 256), 256, 0, st>>>(p->offsets[SSA_LEVEL_CMP], p->offsets[SSA_LEVEL_SLC],
                                            p->tok_block[SSA_LEVEL_CMP], p->tok_block[SSA_LEVEL_SLC], totals,
                                            p->cmp_to_slc, p->slc_cmp_begin);
  count_launch();
  CTRY(cudaGetLastError());
  k_q_batch<<<nblk(n, 256), 256, 0, st>>>(reinterpret_cast<const int4*>(p->block_coords[SSA_LEVEL_Q]), totals,
                                          p->q_batch);
  count_launch();
  CTRY(cudaGetLastError());

  int32_t small[16];
  CTRY(cudaMemcpyAsync(small, w.dev_small, sizeof(small), cudaMemcpyDeviceToHost, st));
  CTRY(cudaStreamSynchronize(st));
  ssa_plan_info& I = p->info;
  memset(&I, 0, sizeof(I));
  I.n = n;
  I.batch = batch;
  for (int a = 0; a < 3; ++a) I.grid[a] = grid[a];
  for (int l = 0; l < kLevels; ++l) {
    I.m[l] = m[l];
    I.n_blocks[l] = small[1 + l];
    I.max_fill[l] = small[5 + l];
    p->h_batch_blocks[l].resize(batch + 1);
    CTRY(cudaMemcpyAsync(p->h_batch_blocks[l].data(), p->batch_blocks[l], (batch + 1) * 4, cudaMemcpyDeviceToHost, st));
    CTRY(cudaStreamSynchronize(st));
    int32_t mb = 0;
    for (int b = 0; b < batch; ++b) mb = std::max(mb, p->h_batch_blocks[l][b + 1] - p->h_batch_blocks[l][b]);
    I.max_blocks_per_batch[l] = mb;
    I.offsets[l] = p->offsets[l];
    I.block_coords[l] = p->block_coords[l];
    I.batch_blocks[l] = p->batch_blocks[l];
  }
  p->h_batch_tokens.resize(batch + 1);
  CTRY(cudaMemcpyAsync(p->h_batch_tokens.data(), p->batch_tokens, (batch + 1) * 4, cudaMemcpyDeviceToHost, st));
  // LPT work order over query blocks (largest first; ties by index) — host side, n_q ints
  {
    const int32_t nq = I.n_blocks[SSA_LEVEL_Q];
    std::vector<int32_t> off(nq + 1), order(nq);
    CTRY(cudaMemcpyAsync(off.data(), p->offsets[SSA_LEVEL_Q], (nq + 1) * 4, cudaMemcpyDeviceToHost, st));
    CTRY(cudaStreamSynchronize(st));
    p->h_q_offsets = off;
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(),
                     [&](int32_t a, int32_t b) { return off[a + 1] - off[a] > off[b + 1] - off[b]; });
    CTRY(cudaMemcpyAsync(p->q_order, order.data(), nq * 4, cudaMemcpyHostToDevice, st));
    CTRY(cudaStreamSynchronize(st));
  }
  {  // 128-key compression tiles per batch item (KV-outer backward work list)
    std::vector<int32_t> tiles;
    const auto& bb = p->h_batch_blocks[SSA_LEVEL_CMP];
    for (int b = 0; b < batch; ++b)
      for (int32_t j = bb[b]; j < bb[b + 1]; j += 128) { tiles.push_back(b); tiles.push_back(j); }
    p->n_cmp_tiles = int32_t(tiles.size() / 2);
    if (!tiles.empty()) {
      CTRY(cudaMemcpyAsync(p->cmp_tiles, tiles.data(), tiles.size() * 4, cudaMemcpyHostToDevice, st));
      CTRY(cudaStreamSynchronize(st));
    }
  }
  I.perm = p->perm;
  I.inv_perm = p->inv_perm;
  I.sorted_coords = p->sorted_coords;
  I.batch_tokens = p->batch_tokens;
  I.cmp_to_slc = p->cmp_to_slc;
  *out = reinterpret_cast<ssa_plan>(p);
  return SSA_OK;
#undef TRY
#undef CTRY
}

extern "C" void ssa_plan_destroy(ssa_plan plan) { delete reinterpret_cast<Plan*>(plan); }

extern "C" ssa_status ssa_get_plan_info(ssa_plan plan, ssa_plan_info* out) {
  if (!plan || !out) { set_error("null plan/out"); return SSA_ERR_ARG; }
  *out = reinterpret_cast<Plan*>(plan)->info;
  return SSA_OK;
}
