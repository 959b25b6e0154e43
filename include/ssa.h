/*
 * ssa.h — C ABI of the B200-native Spatial Sparse Attention library (libssa_b200.so).
 *
 * Spatial Sparse Attention (SSA) is the attention of Direct3D-S2 (arXiv 2505.17412, §4.1,
 * /root/reference/PAPER.md lines 129-226): sparse voxel tokens are grouped into m^3 spatial blocks
 * (P:143), each compression block's K/V are pooled into one block token (Eq. 7), the
 * compression attention scores pick the top-k selection blocks per query block (Eq. 8),
 * flash-style attention runs over the selected blocks (Algorithm 1) and over a local
 * m_win^3 window, and the three branch outputs are summed with gates (Eq. 6).
 *
 * Conventions shared by every entry point
 *   - Every tensor pointer is a DEVICE pointer (CUDA global memory) owned by the caller. The library
 *     never allocates device memory: sizes are queried first (ssa_*_size) and the caller passes the
 *     buffers. The host-side ssa_plan handle is the only host allocation (malloc, freed by
 *     ssa_plan_destroy).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream). All device work is
 *     enqueued on it. ssa_build_blocks synchronises the stream once (to read block counts and the
 *     validation flags); ssa_forward / ssa_backward are fully asynchronous: a device-side fault
 *     surfaces at the caller's next synchronisation.
 *   - Errors: no exceptions, no abort across the ABI. Host argument errors return immediately
 *     without enqueuing work. ssa_last_error() returns a thread-local text for the last failure.
 *   - Layouts are row-major, innermost index last. Token order is the CALLER's order unless
 *     SSA_INPUT_SORTED is set (then tensors are in the plan's block-sorted order).
 *   - Head layout (GQA, Alg. 1 signature P:182): q, out, dout, dq: [N, H, d] with
 *     H = h_kv * h_s; query head h = g*h_s + s uses kv head g; k, v, dk, dv: [N, h_kv, d];
 *     gates, dgates: [N, H, 3] with branch order (cmp, slc, win) of Eq. 6, values post-sigmoid.
 *   - Element type of q/k/v/gates/out/dout/dq/dk/dv/dgates: cfg->dtype (SSA_F32 or SSA_BF16). All
 *     accumulation, softmax statistics and scores are fp32.
 */
#ifndef SSA_B200_H
#define SSA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SSA_OK = 0,
  SSA_ERR_ARG = 1,          /* invalid host argument (null pointer, bad size, bad config)         */
  SSA_ERR_DUP_COORD = 2,    /* two tokens share a voxel                             */
  SSA_ERR_COORD_RANGE = 3,  /* coordinate outside [0,grid) or batch index outside [0,batch)        */
  SSA_ERR_HIERARCHY = 4,    /* block sizes do not form a divisibility chain / m_cmp !| m_slc*/
  SSA_ERR_BAD_STATE = 5,    /* plan / saved state mismatch                                        */
  SSA_ERR_WORKSPACE = 6,    /* caller buffer smaller than the queried size                        */
  SSA_ERR_UNSUPPORTED = 7,  /* configuration outside this build's kernels (reported in last_error) */
  SSA_ERR_CUDA = 8          /* CUDA runtime error (text in ssa_last_error)                        */
} ssa_status;

typedef enum { SSA_F32 = 0, SSA_BF16 = 1 } ssa_dtype;

/* Block levels of a plan. */
typedef enum { SSA_LEVEL_CMP = 0, SSA_LEVEL_SLC = 1, SSA_LEVEL_WIN = 2, SSA_LEVEL_Q = 3 } ssa_level;

typedef struct ssa_plan_s* ssa_plan;

/* ------------------------------------------------------------------------------------------------
 * ssa_build_blocks — spatial block partition + sort + start offsets C.
 * PAPER.md:143 ("divide the 3D space into subgrids of size m^3 ... grouped into one block")
 * ("first sort the input tokens based on their block indices, then compute the starting index C of
 * each block"), Alg. 1 line 2. Four levels are built at once: compression (m_cmp),
 * selection (m_slc), window (m_win) and query block (m_q; m_q = 1 is the paper's per-token query).
 * Sort order: hierarchical-lexicographic over the distinct sizes (coarse to fine), then voxel
 * order inside the finest block, within batch item b (reading R1). Every level is
 * contiguous in that order; empty blocks are not materialised.
 *
 *   coords      device int32 [n,4] rows (b,x,y,z), 0 <= b < batch, 0 <= x < grid[0] ...
 *   n           number of tokens, 1 <= n < 2^31 (an empty input, n = 0, is SSA_ERR_ARG: with no
 *               token there is no block, no query and nothing to attend; callers skip the call)
 *   grid        HOST int32[3] grid extent per axis (latent resolution, e.g. 128 at 1024^3)
 *   m_*         block edge lengths; the distinct values must form a divisibility chain and
 *               m_cmp | m_slc (relaxed to >=, reading R2)
 *   plan_buf    device buffer of ssa_build_blocks_size(...).plan_bytes, owned by the caller; it
 *               must stay alive and unmodified while the plan is used
 *   ws          device scratch of ws_bytes (may be reused after the call returns)
 *   out         receives a host handle (free with ssa_plan_destroy; does not free plan_buf)
 * Synchronises `stream` once. Errors: SSA_ERR_DUP_COORD, SSA_ERR_COORD_RANGE, SSA_ERR_HIERARCHY,
 * SSA_ERR_ARG, SSA_ERR_WORKSPACE, SSA_ERR_UNSUPPORTED (key space > 2^34 cells), SSA_ERR_CUDA.
 * ----------------------------------------------------------------------------------------------*/
ssa_status ssa_build_blocks_size(int64_t n, int32_t batch, const int32_t grid[3], int32_t m_cmp,
                                 int32_t m_slc, int32_t m_win, int32_t m_q, size_t* plan_bytes,
                                 size_t* ws_bytes);
ssa_status ssa_build_blocks(const int32_t* coords, int64_t n, int32_t batch, const int32_t grid[3],
                            int32_t m_cmp, int32_t m_slc, int32_t m_win, int32_t m_q, void* plan_buf,
                            size_t plan_bytes, void* ws, size_t ws_bytes, void* stream, ssa_plan* out);
void ssa_plan_destroy(ssa_plan plan);

/* Host-readable plan summary + device pointers into plan_buf (all int32, valid while plan_buf is).
 *   perm[n]        sorted position -> caller token index;  inv_perm[n] the inverse
 *   offsets[l]     [n_blocks[l]+1] token start of every block of level l (the paper's C)
 *   block_coords[l][n_blocks[l]*4] (b, x/m, y/m, z/m) of every block
 *   batch_blocks[l][batch+1] first block of every batch item;  batch_tokens[batch+1]
 *   cmp_to_slc[n_blocks[CMP]] enclosing selection block of every compression block          */
typedef struct {
  int64_t n;
  int32_t batch;
  int32_t grid[3];
  int32_t m[4];
  int32_t n_blocks[4];
  int32_t max_fill[4];            /* largest block (tokens) per level                          */
  int32_t max_blocks_per_batch[4];
  const int32_t* perm;
  const int32_t* inv_perm;
  const int32_t* sorted_coords;  /* [n,4] */
  const int32_t* offsets[4];
  const int32_t* block_coords[4];
  const int32_t* batch_blocks[4];
  const int32_t* batch_tokens;
  const int32_t* cmp_to_slc;
} ssa_plan_info;
ssa_status ssa_get_plan_info(ssa_plan plan, ssa_plan_info* out);

/* ------------------------------------------------------------------------------------------------
 * Attention configuration.
 *   h_q, h_kv, d : heads (h_q multiple of h_kv), head dim. top_k : T, the number of selected
 *   blocks (clamped per batch item to N_slc(b), padded slots hold -1, reading R9).
 *   scale        : softmax scale; <= 0 means 1/sqrt(d) (Eq. 5).
 *   dtype        : SSA_F32 (SIMT fp32 kernels, the fp32 mode) or SSA_BF16 (tcgen05 tensor-core
 *                  kernels: d == 64 — or d == 32, the paper's DiT head dim, run zero-padded to
 *                  64 inside the library: the logits and the outputs are unchanged — m_win == m_slc,
 *                  m_q dividing m_slc (m_q = 1: per-token selection, Alg. 1), block counts within the
 *                  kernels' on-chip limits). A bf16 request outside those returns SSA_ERR_UNSUPPORTED (reason in
 *                  ssa_last_error) unless SSA_FORCE_SIMT opts into the SIMT kernels — there is no
 *                  silent fallback. Every check happens before any work is enqueued.
 *   pe_k, pe_v   : optional device [m_cmp^3, h_kv, d] (dtype) intra-block PE tables added before
 *                  pooling (Eq. 7, reading R4); NULL = off. Not differentiated.
 *   flags        : SSA_INPUT_SORTED — tensors are already in plan order (no internal permute);
 *                  SSA_FORCE_SIMT   — use the SIMT kernels even where tcgen05 kernels exist;
 *                  SSA_SAVE_SCORES  — keep the fp32 selection scores in the saved state;
 *                  SSA_KV_GRAD_FP32 — dk, dv buffers are fp32 (exact partial sums across shards);
 *                  SSA_WINDOW_ONLY  — only the sparse 3D window branch is computed: the
 *                                     compression and selection branches are skipped (their saved
 *                                     outputs are 0, their LSEs the 0x7f7f7f7f sentinel, indices -1),
 *                                     out = omega_win * O_win, and the
 *                                     backward gives the window branch's gradients (dgates of the
 *                                     skipped branches are 0). With gates (0, 0, 1) this is sparse 3D
 *                                     window attention (the SS-VAE layer). tcgen05 path only
 *                                     (bf16, d = 64, m_win == m_slc == m_q); SSA_ERR_UNSUPPORTED otherwise.
 *                  SSA_NO_WINDOW    — the window branch is skipped (saved O_win = 0, LSE sentinel):
 *                                     out = omega_cmp O_cmp + omega_slc O_slc; dgates_win = 0.
 *                  SSA_ACCUMULATE   — out (forward) and dq, dk, dv, dgates (backward) are added to
 *                                     what the caller's buffers hold instead of overwriting them.
 *                                     Together: SSA with SHIFTED windows = one
 *                                     SSA_NO_WINDOW call on the plan of the coordinates, then one
 *                                     SSA_WINDOW_ONLY | SSA_ACCUMULATE call on the plan of the shifted
 *                                     coordinates (whose aligned windows are the shifted windows) with
 *                                     the same tensors (ssa.py: shifted_window_ssa). tcgen05 path only.
 * ----------------------------------------------------------------------------------------------*/
#define SSA_INPUT_SORTED 1u
#define SSA_FORCE_SIMT 2u
#define SSA_SAVE_SCORES 4u
#define SSA_KV_GRAD_FP32 8u   /* dk / dv are written as fp32 (partials of a query-block shard)    */
#define SSA_WINDOW_ONLY 16u   /* window branch only (sparse 3D window attention)                   */
#define SSA_LOCAL_ROWS 32u    /* q / gates / dout / out / dq / dgates hold only the owned rows       */
#define SSA_NO_WINDOW 64u     /* window branch skipped: O_win = 0 (its gate term vanishes)          */
#define SSA_ACCUMULATE 128u   /* out, dq, dk, dv, dgates are ADDED to the caller's buffers          */

/* ------------------------------------------------------------------------------------------------
 * Learned compression delta and gate projection (readings R17, R18).
 *   Eq. 7: k^cmp_B = (1/n_B) sum_{t in B} W_k[loc(t), g] (k_t + PE_k[loc(t), g]) + b_k[g] —
 *     a sparse 3D convolution with kernel = stride = m_cmp over the active tokens of each compression
 *     block (one d x d matrix per intra-block offset loc = ((x%m)*m + y%m)*m + z%m, grouped per kv head,
 *     applied as W x) followed by the sparse mean pooling. W [m_cmp^3][h_kv][d][d], b [h_kv][d], fp32,
 *     device. NULL conv_k_w: the masked mean pool (R4). V likewise with W_v, b_v.
 *   Eq. 6 gates: omega = sigmoid(x W_g + b_g) from the input features x [n][c] (dtype, caller
 *     order; SSA_LOCAL_ROWS: owned rows), W_g [c][3 h_q] (column h*3 + branch), b_g [3 h_q] fp32.
 *     NULL x: the gates are the `gates` input. The computed gates are kept in the saved state.
 *   Gradient outputs (written by ssa_backward where non-NULL): d_conv_* fp32 like their weights;
 *   dx [n][c] dtype; d_gate_w, d_gate_b fp32. tcgen05 / SIMT paths alike; d == 64 only.
 *   The pointers of this struct must be the same in the forward and the backward of one step.
 * ----------------------------------------------------------------------------------------------*/
typedef struct {
  const float* conv_k_w;
  const float* conv_k_b;
  const float* conv_v_w;
  const float* conv_v_b;
  const void* x;
  int32_t c;
  const float* gate_w;
  const float* gate_b;
  float* d_conv_k_w;
  float* d_conv_k_b;
  float* d_conv_v_w;
  float* d_conv_v_b;
  void* dx;
  float* d_gate_w;
  float* d_gate_b;
} ssa_learned;

typedef struct {
  int32_t h_q, h_kv, d, top_k;
  float scale;
  int32_t dtype;
  uint32_t flags;
  const void* pe_k;
  const void* pe_v;
  /* Query-block sharding (SURVEY §8e mode 2): compute only the rows of the query blocks
   * [q_begin, q_end) (plan order, SSA_LEVEL_Q; q_end <= 0 means all). Forward: only those rows of
   * out / saved state are written. Backward: dq and dgates are written for those rows only; dk and
   * dv receive the contributions of those rows to ALL keys (partials: the caller sums them across
   * shards, e.g. with a reduce-scatter). k, v must be complete (e.g. all-gathered). A strict range
   * requires m_win == m_q (a window is then exactly one query block). */
  int32_t q_begin, q_end;
  /* Query-block sharding, continued (SURVEY §8e mode 2, one shape over several GPUs):
   *   SSA_LOCAL_ROWS (needs SSA_INPUT_SORTED and a range): the row tensors q, gates, dout, out, dq,
   *     dgates hold ONLY the owned rows, i.e. plan-order tokens [C_q[q_begin], C_q[q_end]) — the rows a
   *     rank keeps; k, v stay complete. No kernel touches a row outside that range.
   *   kc_in, vc_in: optional device fp32 [h_kv][n_cmp][d] pooled keys / values (Eq. 7) supplied by
   *     the caller (e.g. every rank's ssa_pool output summed across ranks); the forward then does not
   *     pool and needs the raw k, v only for the selection and window branches.
   *   kv_event: optional cudaEvent_t. When set, the forward enqueues cudaStreamWaitEvent(stream,
   *     kv_event) right before its first read of the raw k, v — after the compression attention when
   *     kc_in / vc_in are given — so a K/V all-gather recorded on another stream overlaps the
   *     compression branch (a4/a5). NULL: k, v are ready when the call is made. */
  const void* kc_in;
  const void* vc_in;
  void* kv_event;
  const ssa_learned* learned;   /* NULL: delta = mean pool, gates are inputs (see ssa_learned) */
  /* One-sided fetch of the selected K/V blocks (mode 2 without the bulk all-gather):
   * n_peer > 0 ranks own contiguous plan-order token ranges [peer_tok[r], peer_tok[r+1]) of one
   * shape; peer_k[r] / peer_v[r] are device pointers (local, or peer mappings opened with
   * ssa_ipc_open — NVLink P2P on a multi-GPU node) to rank r's rows, layout [rows][h_kv][d].
   * Needs kc_in / vc_in. The forward then copies into the caller's full-size k, v buffers (which hold
   * this rank's own rows) exactly the rows of the selection blocks its owned query blocks selected —
   * after the compression attention and top-k, before the selection branch — instead of waiting for
   * a K/V all-gather; kv_event is not used. my_rank: this rank's index. */
  int32_t n_peer, my_rank;
  const void* peer_k[16];
  const void* peer_v[16];
  int32_t peer_tok[17];
} ssa_attn_cfg;

/* CUDA IPC helpers for the one-sided fetch: export a device allocation (base pointer) as a 64-byte
 * handle; open another process's handle (peer mapping; on one GPU a second mapping of the same memory)
 * and close it. Errors: SSA_ERR_ARG, SSA_ERR_CUDA. */
ssa_status ssa_ipc_handle(const void* base, void* handle64);
ssa_status ssa_ipc_open(const void* handle64, void** ptr);
ssa_status ssa_ipc_close(void* ptr);

/* ------------------------------------------------------------------------------------------------
 * ssa_pool — the compression pool alone (Eq. 7; delta = masked mean, reading R4, plus the
 * optional intra-block PE of cfg): kc[g][j][:] = mean over the tokens of compression block j of
 * k[t][g][:] (+ pe_k), likewise vc, fp32 [h_kv][n_cmp][d] (device, caller-owned). For sharded use
 * (SSA_LOCAL_ROWS + a query-block range) k, v hold the owned rows only and only the compression blocks
 * inside the owned rows are pooled; every other block of kc / vc is written as 0, so a SUM over ranks
 * (all-reduce) assembles the complete pooled keys. Needs SSA_INPUT_SORTED. No workspace.
 * Errors: SSA_ERR_ARG, SSA_ERR_BAD_STATE, SSA_ERR_CUDA.
 * ----------------------------------------------------------------------------------------------*/
ssa_status ssa_pool(ssa_plan plan, const ssa_attn_cfg* cfg, const void* k, const void* v, void* kc, void* vc,
                    void* stream);

/* ------------------------------------------------------------------------------------------------
 * ssa_forward — one SSA forward (Eq. 6): pool (Eq. 7) -> compression attention + Eq. 8 block
 * scores + top-k -> selection attention (Alg. 1, query-block granular) + window
 * attention -> gated sum (Eq. 6).
 *   q [n,h_q,d], k/v [n,h_kv,d], gates [n,h_q,3] (dtype, device) -> out [n,h_q,d] (dtype, device)
 *   saved      device buffer of saved_bytes; filled here, consumed by ssa_backward and the parity
 *              hooks below. Must not be modified between forward and backward.
 *   ws         device scratch of ws_bytes (forward-only lifetime).
 * Errors: SSA_ERR_ARG (bad cfg / null), SSA_ERR_BAD_STATE (plan null), SSA_ERR_WORKSPACE,
 * SSA_ERR_UNSUPPORTED, SSA_ERR_CUDA (launch failure).
 * ----------------------------------------------------------------------------------------------*/
ssa_status ssa_forward_size(ssa_plan plan, const ssa_attn_cfg* cfg, size_t* ws_bytes, size_t* saved_bytes);
ssa_status ssa_forward(ssa_plan plan, const ssa_attn_cfg* cfg, const void* q, const void* k,
                       const void* v, const void* gates, void* out, void* saved, size_t saved_bytes,
                       void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------------------------------
 * ssa_backward — gradients of ssa_forward with the block structure and the selected indices held
 * constant (hard routing, reading R15; the paper reports only the backward's speed,
 * P:391). Recomputes probabilities from the saved LSEs (flash-style).
 *   dout [n,h_q,d] -> dq [n,h_q,d], dk/dv [n,h_kv,d], dgates [n,h_q,3] (all dtype, device).
 *   q,k,v,gates must be the tensors given to the forward that filled `saved`.
 * ----------------------------------------------------------------------------------------------*/
ssa_status ssa_backward_size(ssa_plan plan, const ssa_attn_cfg* cfg, size_t* ws_bytes);
ssa_status ssa_backward(ssa_plan plan, const ssa_attn_cfg* cfg, const void* q, const void* k,
                        const void* v, const void* gates, const void* saved, size_t saved_bytes,
                        const void* dout, void* dq, void* dk, void* dv, void* dgates, void* ws,
                        size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------------------------------
 * Parity hooks into a filled saved state (device pointers, valid while `saved` is):
 *   idx      int32 [n_blocks[Q], h_kv, top_k]  selected selection-block ids (global), -1 padded
 *   scores   fp32 [n_blocks[Q], h_kv, max_blocks_per_batch[SLC]] (NULL unless SSA_SAVE_SCORES);
 *            row (Q,g) holds the Eq. 8 score of the selection blocks of Q's batch item (local index)
 *   o_branch, lse_branch: fp32 branch outputs / log2-domain LSEs (log2 sum 2^(scale q.k log2 e)), layout [h_kv][n][h_s][d] / [h_kv][n][h_s]
 *            in plan (sorted) order, branch 0=cmp 1=slc 2=win.
 * ----------------------------------------------------------------------------------------------*/
typedef struct {
  const int32_t* idx;
  const float* scores;
  const void* o_branch[3];
  const float* lse_branch[3];
  const void* k_cmp;   /* [h_kv][n_blocks[CMP]][d] fp32 */
  const void* v_cmp;
  int32_t used_tcgen05;  /* 1 if the forward ran the tcgen05 kernels */
  int32_t d_internal;    /* head dim of o_branch / k_cmp rows: d, or 64 when a d = 32 problem runs the
                            tcgen05 kernels zero-padded to 64 (padded entries are 0) */
} ssa_saved_view;
ssa_status ssa_saved_state(ssa_plan plan, const ssa_attn_cfg* cfg, const void* saved, size_t saved_bytes,
                           ssa_saved_view* out);

/* ------------------------------------------------------------------------------------------------
 * Kernel-timing hook (used by bench.py for the roofline of the dominant kernel). When enabled, the
 * library brackets each attention kernel launch with CUDA events recorded on the launch stream.
 * ssa_profile_read synchronises those events and returns the summed device time (ms) and launch
 * count of every launch whose kernel name equals `kernel` since the last reset.
 * ----------------------------------------------------------------------------------------------*/
void ssa_profile_enable(int on);
void ssa_profile_reset(void);
ssa_status ssa_profile_read(const char* kernel, double* total_ms, int64_t* launches);

const char* ssa_status_str(ssa_status s);
const char* ssa_last_error(void);
/* Kernels launched by this thread since the last reset (host counter; used by bench.py). */
int64_t ssa_launch_count(void);
void ssa_reset_launch_count(void);
const char* ssa_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* SSA_B200_H */
