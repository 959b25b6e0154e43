// internal.h — shared host-side declarations of libssa_b200 (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/ssa.h"

namespace ssa {

constexpr int kLevels = 4;  // cmp, slc, win, q

// Host handle behind ssa_plan. Device arrays live in the caller's plan_buf.
struct Plan {
  ssa_plan_info info;
  int32_t* perm = nullptr;
  int32_t* inv_perm = nullptr;
  int32_t* sorted_coords = nullptr;
  int32_t* offsets[kLevels] = {};
  int32_t* block_coords[kLevels] = {};
  int32_t* tok_block[kLevels] = {};
  int32_t* batch_blocks[kLevels] = {};
  int32_t* batch_tokens = nullptr;
  int32_t* cmp_to_slc = nullptr;
  int32_t* slc_cmp_begin = nullptr;   // [n_slc+1] first compression block of each selection block
  int32_t* q_order = nullptr;         // [n_q] query blocks, largest first (LPT work order)
  int32_t* q_batch = nullptr;         // [n_q] batch item of each query block
  int32_t* cmp_tiles = nullptr;       // [n_cmp_tiles][2] (batch item, first cmp block), 128-key tiles
  int32_t n_cmp_tiles = 0;
  std::vector<int32_t> h_batch_blocks[kLevels];
  std::vector<int32_t> h_batch_tokens;
  std::vector<int32_t> h_q_offsets;   // [n_q+1] token offsets of the query blocks (host copy)
};

// Everything a forward/backward kernel needs, by value (kernel parameter space).
struct Ctx {
  // problem
  int32_t N, H, h_kv, h_s, D, T, batch, m_cmp;
  int32_t Dc;                     // head dim of the caller's tensors (D = internal; 32 padded to 64 on tcgen05)
  int32_t n_blk[kLevels];
  int32_t max_cmp_b, max_slc_b;   // max compression / selection blocks of one batch item
  int32_t max_fill[kLevels];
  float scale;                    // softmax scale (natural)
  int32_t sorted_input;
  int32_t win_only;                   // SSA_WINDOW_ONLY: compression / selection branches skipped
  int32_t no_win;                     // SSA_NO_WINDOW: the window branch skipped (O_win = 0)
  int32_t accumulate;                 // SSA_ACCUMULATE: out / dq / dk / dv / dgates += instead of =
  int32_t q_begin, q_end;         // owned query blocks [q_begin, q_end) (plan order)
  int32_t tok_begin, tok_end;     // their token range
  int32_t row_lo, row_hi;         // rows (plan order) whose caller row tensors may be touched: the owned
                                  // range with a query-block range, [0, N) otherwise
  int64_t row_base;               // SSA_LOCAL_ROWS: first row held by the caller's row tensors (else 0)
  int32_t save_scores;
  int32_t kv_grad_f32;            // dk / dv written as fp32 (SSA_KV_GRAD_FP32)
  int32_t sel_partial;            // per-block selection pass (pertoken.cu): epilogue writes only O (o[1]) and LSE
                                  // (forward), fp32 dQ partials to dq_part (k_tc_dq), no compressed keys
  float* dq_part;                 // [expanded rows][D] fp32 dQ partials of the per-block pass (sel_partial)
  const float* dq_extra;          // [rows][D] fp32 added to dq before its bf16 store (per-block selection dQ)
  // plan (device)
  const int32_t *perm, *inv_perm, *sorted_coords;
  const int32_t *off[kLevels], *tok_block[kLevels], *bb[kLevels];
  const int32_t *batch_tokens, *slc_cmp_begin, *cmp_to_slc, *q_order, *q_batch;
  // caller tensors
  const void *q, *k, *v, *gates, *pe_k, *pe_v, *dout;
  void *out, *dq, *dk, *dv, *dgates;
  // internal tensors: layouts [h_kv][N][h_s][D] (rows), [h_kv][N][D] (keys)
  void *qs, *ks, *vs, *dos;
  float* gs;                      // [h_kv][N][h_s][3]
  void *kc, *vc;                  // [h_kv][n_cmp][D]
  void* o[3];                     // branch outputs (rows layout, dtype)
  float* lse[3];                  // [h_kv][N][h_s], log2 domain: log2 sum_j 2^(scale log2e q.k_j)
  int32_t* I;                     // [n_q][h_kv][T]
  float* scores;                  // [n_q][h_kv][max_slc_b] or null
  // backward scratch
  float* Dd[3];                   // [h_kv][N][h_s]  D_c = omega_c <dO, O_c>
  float *dq_acc, *dk_acc, *dv_acc;  // fp32 [rows] / [keys]
  float *dkc, *dvc;               // fp32 [h_kv][n_cmp][D]
  float *dkc_part, *dvc_part;     // fp32 [n_chunk][h_kv][n_cmp][D]
  int32_t n_chunk;
  int32_t qb_per_item;            // raw-key KV-outer work item size in query blocks (tc_qb_per_item)
  // query blocks smaller than the selection blocks on tcgen05 (pertoken.cu): the virtual-level context
  // carries the per-token slot masks and, for the KV-outer row masks, the per-query-block selections
  const unsigned long long* umask;  // [N][h_kv][2] 128-bit union-slot mask of every token, null on the plain path
  const int32_t* tok_I;             // [n_q][h_kv][tok_T] per-query-block selections
  int32_t tok_T;
  const int32_t* tok_qb;            // token -> query block
  void* vq_ws;                      // scratch of the virtual level (forward), null when it is not used
  void* blk_ws;                     // scratch of the per-block selection pass (forward, m_q = 1), or null
  int32_t vq_S;                     // its sub-group size in query blocks
  // per-token compression (m_q = 1, tc_fwd.cu k_tc_cmp_fwd<h_s>): tok_cmp = h_s when used, else 0
  int32_t tok_cmp;
  void* tok_ws;                     // its scratch (tok_cmp_ws_bytes), carved by tc_forward into:
  const int32_t* tok_cg;            // [bound][2] query-block range of each token group
  float* tok_sc;                    // [kTokSlots][2 * 128 / h_s][max_slc_b] per-SM selection-score scratch
  const uint32_t* do_amax;
  // §8f row 2 (learned.cu): learned compression delta (R17) and gate projection (R18)
  const float *conv_kw, *conv_kb, *conv_vw, *conv_vb;   // [m^3][h_kv][D][D], [h_kv][D]; null = mean pool
  float *conv_dkw, *conv_dkb, *conv_dvw, *conv_dvb;     // their gradients (backward outputs)
  const void* gx;                 // [N][gC] input features (caller order, dtype); null = gates are inputs
  int32_t gC;
  const float *gw, *gb;           // W_g [gC][3H], b_g [3H]
  void* gdx;                      // dx (dtype), dW_g, db_g (fp32) — backward outputs
  float *gdw, *gdb;
  float* dz;                      // [h_kv][N][h_s][3] gradients of the gate logits (row prologue)
  // one-sided fetch of the selected K/V blocks (cfg n_peer > 0)
  int32_t n_peer, my_rank;
  const void* peer_k[16];
  const void* peer_v[16];
  int32_t peer_tok[17];
  int32_t* fetch_mark;            // [n_slc] needed selection blocks        // tcgen05 backward: max |dO| (float bits) -> power-of-two operand scale
  int32_t *inv_off, *inv_list, *inv_cnt;   // inverse selection CSR over (slc block, g)
  int32_t *cmp_tiles;             // [n_cmp_tiles][2] (batch item, first cmp block) for the KV-outer cmp kernels
  int32_t n_cmp_tiles;
  // tcgen05 raw-key KV-outer work items (tc_bwd.cu)
  int32_t* kv_item_off;           // [n_slc * h_kv + 1] first work item of every (selection block, g)
  float *kv_part_k, *kv_part_v;   // [items_bound][max_fill_slc][D] partials of items 1..
  int32_t* kv_tile_off;           // [items + 1] first packed row tile of every raw-key work item
  int2* kv_desc;                  // [tiles][8] per 8-row granule of a packed row tile: {first row, meta} (tc_bwd.cu)
};

// SIMT kernels (simt.cu). Return SSA_OK or a launch error.
ssa_status simt_forward(const Ctx& c, bool bf16, cudaStream_t st, bool attention_only);
ssa_status simt_backward(const Ctx& c, bool bf16, cudaStream_t st);
// rows = false: only keys and gates are gathered (the tcgen05 backward reads q / dO rows itself)
ssa_status gather_inputs(const Ctx& c, bool bf16, cudaStream_t st, bool with_dout, bool rows = true, bool keys = true,
                         bool gates = true);
// one-sided fetch (simt.cu): mark the selection blocks owned query blocks selected, copy the peer-owned
// ones into the caller's full-size k / v (before the selection branch)
ssa_status fetch_selected(const Ctx& c, bool bf16, cudaStream_t st);
// pertoken.cu: the virtual query level of small query blocks (m_q < m_slc)
int vq_slots(int S, int T);
constexpr int kTokSlots = 256;      // per-SM scratch slots of the per-token compression kernel (>= %nsmid)
int tok_cmp_hs(int m_q, int h_s);   // h_s when the per-token compression kernel applies, else 0
size_t tok_cmp_ws_bytes(int n_q, int batch, int h_s, int max_slc_b);
int vq_qb_per_item();
bool vq_enabled();
// union capacity of a virtual query block: slots (mask bits) and keys (within the selection / dQ kernels'
// packed-tile capacity: 28 672 keys + 8-key granule padding of 128 blocks + a window block <= 264 x 128)
constexpr int kVqSlots = 128;
constexpr int kVqKeyCap = 28672;
int64_t vq_bound(int n_slc, int n_q, int S, int T, int max_fill_slc);
size_t vq_ws_bytes(int64_t N, int h_kv, int n_slc, int n_q, int S, int T, int max_fill_slc);
// plain: sub-groups of S query blocks with empty selection lists and no slot masks (the per-block pass)
ssa_status build_virtual_level(const Ctx& c, int S, void* ws, cudaStream_t st, Ctx* v, bool plain = false);
// pertoken.cu: per-block selection pass of per-token selection (m_q = 1)
struct BlkPass {
  int32_t *off_e, *I_e, *order_e, *off_slc, *inv_off, *inv_list;
  __nv_bfloat16* q_exp;
  float *o_exp, *lse_exp;
  int64_t bound, n_exp;
  int32_t* batch_e;               // zeros (the expanded context has no compressed keys)
  float* dq_part;                 // backward: fp32 dQ partials per expanded row
  int32_t* etok;                  // [entries + 1] first expanded token of every inverse-CSR entry
};
bool blk_enabled();
bool blk_forced();   // SSA_VQ_BLOCKSEL=2: the per-block pass also for m_q > 1
size_t blk_ws_bytes(int64_t N, int h_kv, int h_s, int D, int n_slc, int n_q, int T);
ssa_status blk_build(const Ctx& c, void* ws, cudaStream_t st, BlkPass* b);
Ctx blk_context(const Ctx& c, const BlkPass& b);
ssa_status blk_merge(const Ctx& c, const BlkPass& b, cudaStream_t st);
// backward (tc_bwd.cu): the selection branch's dQ per block; c = the real-level context with the inverse CSR
size_t blk_bwd_ws_bytes(int64_t N, int h_kv, int h_s, int D, int n_slc, int n_q, int T);
ssa_status blk_bwd_build(const Ctx& c, const __half* q16, const __half* do16, void* ws, cudaStream_t st, BlkPass* b,
                         Ctx* e, float** dq_extra);
ssa_status blk_bwd_merge(const Ctx& c, const BlkPass& b, float* dq_extra, cudaStream_t st);
// learned.cu
size_t learned_fwd_ws_bytes(const Ctx& c);
size_t gate_bwd_ws_bytes(int64_t N, int H, int C);
size_t conv_bwd_ws_bytes(int64_t N, int h_kv, int m_cmp, int n_cmp, int D);
ssa_status learned_checks(const Ctx& c);
ssa_status learned_pool_forward(const Ctx& c, bool bf16, void* ws, cudaStream_t st);
ssa_status gate_proj_forward(const Ctx& c, bool bf16, cudaStream_t st);
ssa_status gate_proj_backward(const Ctx& c, bool bf16, void* part_ws, cudaStream_t st);
ssa_status learned_pool_backward_params(const Ctx& c, bool bf16, void* ws, cudaStream_t st);
// ssa_pool's kernel: pooled keys of the owned compression blocks from caller-layout (sorted) k, v
ssa_status pool_rows(const Ctx& c, bool bf16, const void* k, const void* v, float* kc, float* vc, cudaStream_t st);
ssa_status pool_forward(const Ctx& c, bool bf16, cudaStream_t st);
ssa_status combine_forward(const Ctx& c, bool bf16, cudaStream_t st);
size_t inverse_csr_ws_bytes(int n_slc, int h_kv, int n_q);
ssa_status build_inverse_csr(const Ctx& c, void* ws, cudaStream_t st);
ssa_status bwd_prologue(const Ctx& c, bool bf16, cudaStream_t st);
ssa_status bwd_epilogue(const Ctx& c, bool bf16, cudaStream_t st, bool skip_q);
ssa_status cmp_reduce(const Ctx& c, cudaStream_t st);

// Optional per-kernel event timing (api.cu). Usage: { ProfScope ps("name", st); kernel<<<..., st>>>(); }
struct ProfScope {
  const char* name;
  cudaStream_t st;
  void* ev0 = nullptr;
  ProfScope(const char* n, cudaStream_t s);
  ~ProfScope();
};

// thread-local error text + launch counter (api.cu)
void set_error(const std::string& s);
void count_launch(int n = 1);
ssa_status cuda_status(cudaError_t e, const char* where);

#define SSA_CUDA_TRY(expr)                                              \
  do {                                                                  \
    cudaError_t _e = (expr);                                            \
    if (_e != cudaSuccess) return ::ssa::cuda_status(_e, #expr);        \
  } while (0)

#define SSA_LAUNCH_CHECK(name)                                          \
  do {                                                                  \
    ::ssa::count_launch();                                              \
    cudaError_t _e = cudaGetLastError();                                \
    if (_e != cudaSuccess) return ::ssa::cuda_status(_e, name);         \
  } while (0)

// Simple bump allocator over a caller buffer (device). Alignment 256 B.
struct Carve {
  char* base;
  size_t cap;
  size_t used = 0;
  Carve(void* b, size_t c) : base(static_cast<char*>(b)), cap(c) {}
  template <class T>
  T* take(size_t count) {
    size_t off = (used + 255) & ~size_t(255);
    used = off + count * sizeof(T);
    return base ? reinterpret_cast<T*>(base + off) : nullptr;
  }
  bool ok() const { return used <= cap; }
};

// ---- scan (scan.cu) ---------------------------------------------------------------------------
size_t scan_ws_bytes(int64_t n);
// exclusive prefix sum of int32 in[n] -> out[n]; *total (device) = sum. In-place allowed.
ssa_status exclusive_scan(const int32_t* in, int32_t* out, int64_t n, int32_t* total, void* ws,
                          cudaStream_t st);

}  // namespace ssa
