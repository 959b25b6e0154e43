// api.cu — the C ABI of libssa_b200 (include/ssa.h): size queries, caller-buffer carving and the
// forward / backward orchestration. Every step of the path runs in this library's kernels.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "internal.h"
#include "tc.h"

namespace ssa {
namespace {
thread_local std::string g_err;
thread_local int64_t g_launches = 0;
}  // namespace

namespace {
struct ProfRec { std::string name; cudaEvent_t a, b; };
bool g_prof_on = false;
std::vector<ProfRec> g_prof;
}  // namespace

ProfScope::ProfScope(const char* n, cudaStream_t s) : name(n), st(s) {
  if (!g_prof_on) return;
  cudaEvent_t e;
  if (cudaEventCreate(&e) == cudaSuccess) { cudaEventRecord(e, st); ev0 = e; }
}
ProfScope::~ProfScope() {
  if (!ev0) return;
  cudaEvent_t e;
  if (cudaEventCreate(&e) == cudaSuccess) {
    cudaEventRecord(e, st);
    g_prof.push_back({name, static_cast<cudaEvent_t>(ev0), e});
  }
}

void set_error(const std::string& s) { g_err = s; }
void count_launch(int n) { g_launches += n; }
ssa_status cuda_status(cudaError_t e, const char* where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return SSA_ERR_CUDA;
}

namespace {

struct Dims {
  int64_t N;
  int H, h_kv, h_s, D, T;
  int Dc;   // caller head dim (D: internal, 64 when a d = 32 problem runs the tcgen05 kernels padded)
  size_t esz;
  int n_cmp, n_slc, n_win, n_q, max_slc_b;
};

bool use_tc(const Dims& d, const ssa_attn_cfg* cfg, const Plan* p);
// d = 32 (the paper's DiT head dim) on the tcgen05 path: heads are zero-padded to 64 in the
// internal layouts (zero features change neither q.k nor the first 32 output dims); every caller-
// facing read / write uses Dc = 32. Only where the whole tcgen05 path applies (no caller-supplied
// pooled keys, no learned delta: those interfaces are d = 64).
void pad_for_tc(Dims* d, const ssa_attn_cfg* cfg, const Plan* p) {
  if (d->Dc != 32 || cfg->dtype != SSA_BF16 || (cfg->flags & SSA_FORCE_SIMT) || cfg->kc_in || cfg->learned ||
      cfg->pe_k || cfg->pe_v)
    return;
  Dims t = *d;
  t.D = 64;
  if (use_tc(t, cfg, p)) d->D = 64;
}

ssa_status check_cfg(const Plan* p, const ssa_attn_cfg* cfg, Dims* d) {
  if (!p) { set_error("null plan"); return SSA_ERR_BAD_STATE; }
  if (!cfg) { set_error("null cfg"); return SSA_ERR_ARG; }
  if (cfg->h_kv < 1 || cfg->h_q < 1 || cfg->h_q % cfg->h_kv) { set_error("h_q must be a positive multiple of h_kv"); return SSA_ERR_ARG; }
  if (cfg->d < 1) { set_error("d must be >= 1"); return SSA_ERR_ARG; }
  if (cfg->top_k < 1 || cfg->top_k > 64) { set_error("top_k must be in [1, 64]"); return SSA_ERR_ARG; }
  if (cfg->dtype != SSA_F32 && cfg->dtype != SSA_BF16) { set_error("dtype must be SSA_F32 or SSA_BF16"); return SSA_ERR_ARG; }
  if (cfg->d != 16 && cfg->d != 32 && cfg->d != 64) { set_error("head dim must be 16, 32 or 64"); return SSA_ERR_UNSUPPORTED; }
  if (cfg->q_end > 0) {
    if (cfg->q_begin < 0 || cfg->q_begin > cfg->q_end || cfg->q_end > p->info.n_blocks[SSA_LEVEL_Q]) {
      set_error("query-block range outside [0, n_blocks[Q]]");
      return SSA_ERR_ARG;
    }
    if (p->info.m[SSA_LEVEL_WIN] != p->info.m[SSA_LEVEL_Q]) {
      set_error("a query-block range requires m_win == m_q");
      return SSA_ERR_UNSUPPORTED;
    }
  }
  if ((cfg->flags & SSA_LOCAL_ROWS) && (!(cfg->flags & SSA_INPUT_SORTED) || cfg->q_end <= 0)) {
    set_error("SSA_LOCAL_ROWS needs SSA_INPUT_SORTED and a query-block range");
    return SSA_ERR_ARG;
  }
  if ((cfg->kc_in == nullptr) != (cfg->vc_in == nullptr)) { set_error("kc_in and vc_in go together"); return SSA_ERR_ARG; }
  if (cfg->n_peer != 0) {
    if (cfg->n_peer < 1 || cfg->n_peer > 16 || cfg->my_rank < 0 || cfg->my_rank >= cfg->n_peer) {
      set_error("n_peer must be in [1, 16] and my_rank in [0, n_peer)");
      return SSA_ERR_ARG;
    }
    if (!cfg->kc_in || cfg->peer_tok[0] != 0 || cfg->peer_tok[cfg->n_peer] != p->info.n) {
      set_error("the one-sided fetch needs kc_in / vc_in and peer_tok covering [0, n)");
      return SSA_ERR_ARG;
    }
    for (int r = 0; r < cfg->n_peer; ++r)
      if (!cfg->peer_k[r] || !cfg->peer_v[r] || cfg->peer_tok[r] > cfg->peer_tok[r + 1]) {
        set_error("peer_k / peer_v / peer_tok invalid");
        return SSA_ERR_ARG;
      }
  }
  d->N = p->info.n;
  d->H = cfg->h_q;
  d->h_kv = cfg->h_kv;
  d->h_s = cfg->h_q / cfg->h_kv;
  d->D = cfg->d;
  d->T = cfg->top_k;
  d->esz = cfg->dtype == SSA_BF16 ? 2 : 4;
  d->n_cmp = p->info.n_blocks[SSA_LEVEL_CMP];
  d->n_slc = p->info.n_blocks[SSA_LEVEL_SLC];
  d->n_win = p->info.n_blocks[SSA_LEVEL_WIN];
  d->n_q = p->info.n_blocks[SSA_LEVEL_Q];
  d->max_slc_b = p->info.max_blocks_per_batch[SSA_LEVEL_SLC];
  d->Dc = cfg->d;
  pad_for_tc(d, cfg, p);
  return SSA_OK;
}

// The tcgen05 kernels assume bf16, d = 64 and that the window and the query block are the selection
// block (m_win = m_q = m_slc, true for every tensor-core config C2-C5); anything else runs SIMT.
bool use_tc(const Dims& d, const ssa_attn_cfg* cfg, const Plan* p) {
  const int32_t* m = p->info.m;
  return tc_available() && cfg->dtype == SSA_BF16 && d.D == 64 && !(cfg->flags & SSA_FORCE_SIMT) &&
         m[SSA_LEVEL_WIN] == m[SSA_LEVEL_SLC] && m[SSA_LEVEL_Q] <= m[SSA_LEVEL_SLC] &&
         m[SSA_LEVEL_SLC] % m[SSA_LEVEL_Q] == 0 && cfg->top_k <= 64 &&
         tc_plan_ok(p->info, cfg->top_k);
}
bool use_tc_bwd(const Dims& d, const ssa_attn_cfg* cfg, const Plan* p) {
  return tc_bwd_available() && use_tc(d, cfg, p);
}
// Why a bf16 request cannot take the tcgen05 path (nullptr if it can).
const char* tc_reason(const Dims& d, const ssa_attn_cfg* cfg, const Plan* p) {
  const int32_t* m = p->info.m;
  if (!tc_available()) return "library built without the tcgen05 kernels";
  if (d.D != 64) return "head dim not 32 or 64";
  if (m[SSA_LEVEL_WIN] != m[SSA_LEVEL_SLC] || m[SSA_LEVEL_Q] > m[SSA_LEVEL_SLC]) return "m_win != m_slc or m_q > m_slc";
  if (!tc_plan_ok(p->info, cfg->top_k)) return "a batch item's block counts exceed the kernels' on-chip limits";
  return nullptr;
}
// Path selection, before any work is enqueued: fp32 runs the SIMT kernels (the fp32 mode); bf16 runs
// the tcgen05 kernels, and a bf16 request they cannot take is an error unless the caller opts into the
// (100-500x slower) SIMT kernels with SSA_FORCE_SIMT — no silent fallback.
ssa_status choose_path(const Dims& d, const ssa_attn_cfg* cfg, const Plan* p, bool* tc) {
  *tc = use_tc(d, cfg, p);
  if ((cfg->flags & SSA_WINDOW_ONLY) && (cfg->flags & SSA_NO_WINDOW)) { set_error("SSA_WINDOW_ONLY and SSA_NO_WINDOW exclude each other"); return SSA_ERR_ARG; }
  if (cfg->flags & (SSA_WINDOW_ONLY | SSA_NO_WINDOW | SSA_ACCUMULATE)) {
    if (!*tc) {
      set_error("SSA_WINDOW_ONLY / SSA_NO_WINDOW / SSA_ACCUMULATE need the tcgen05 path (bf16, d = 64, m_win == m_slc == m_q)");
      return SSA_ERR_UNSUPPORTED;
    }
    return SSA_OK;
  }
  if (cfg->n_peer > 0 && !*tc) { set_error("the one-sided K/V fetch needs the tcgen05 path"); return SSA_ERR_UNSUPPORTED; }
  if (cfg->dtype == SSA_BF16 && !*tc && !(cfg->flags & SSA_FORCE_SIMT)) {
    set_error(std::string("bf16 request outside the tcgen05 kernels (") + tc_reason(d, cfg, p) +
              "); set SSA_FORCE_SIMT to run the SIMT kernels");
    return SSA_ERR_UNSUPPORTED;
  }
  return SSA_OK;
}

// saved state: kc, vc, o[3], lse[3], I, scores
void carve_saved(Carve& c, const Dims& d, const ssa_attn_cfg* cfg, Ctx* x) {
  const int64_t rows = d.N * d.H;
  // pooled K/V and branch outputs are kept in fp32 (precision of the saved state);
  // LSEs are stored in the log2 domain (what the kernels consume)
  x->kc = c.take<float>(size_t(d.h_kv) * d.n_cmp * d.D);
  x->vc = c.take<float>(size_t(d.h_kv) * d.n_cmp * d.D);
  for (int b = 0; b < 3; ++b) x->o[b] = c.take<float>(size_t(rows) * d.D);
  for (int b = 0; b < 3; ++b) x->lse[b] = c.take<float>(rows);
  x->I = c.take<int32_t>(size_t(d.n_q) * d.h_kv * d.T);
  x->scores = (cfg->flags & SSA_SAVE_SCORES) ? c.take<float>(size_t(d.n_q) * d.h_kv * std::max(d.max_slc_b, 1)) : nullptr;
}
// gates computed by the projection (ssa_learned.x) are part of the saved state, [h_kv][N][h_s][3] fp32
float* carve_saved_gates(Carve& c, const Dims& d, const ssa_attn_cfg* cfg) {
  return (cfg->learned && cfg->learned->x) ? c.take<float>(size_t(d.N) * d.H * 3) : nullptr;
}

void carve_inputs(Carve& c, const Dims& d, Ctx* x, bool with_dout) {
  const int64_t rows = d.N * d.H, keys = d.N * d.h_kv;
  x->qs = c.take<char>(size_t(rows) * d.D * d.esz);
  x->ks = c.take<char>(size_t(keys) * d.D * d.esz);
  x->vs = c.take<char>(size_t(keys) * d.D * d.esz);
  x->gs = c.take<float>(size_t(rows) * 3);
  x->dos = with_dout ? c.take<char>(size_t(rows) * d.D * d.esz) : nullptr;
}

// Row chunks of the compressed-key KV-outer backward: ~16 waves of 296 CTAs (148 SMs x 2 CTAs), so
// the last partial wave costs a few percent instead of up to a third (long CTAs, few waves).
// Row chunks per compressed-key tile for the KV-outer compression backward (one CTA per SM): the
// count in [8, 64] whose CTA total fills the last wave best (ties -> more chunks, better balance).
int pick_chunks(const Plan* p, int h_kv) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      sms = 148;
  }
  const int64_t tiles = std::max(1, p->n_cmp_tiles * h_kv);
  int best = 1;
  double best_eff = -1.0;
  for (int n = 1; n <= 64; ++n) {
    if (tiles * n < sms && n < 64) continue;               // at least one full wave when possible
    const int64_t ctas = tiles * n, waves = (ctas + sms - 1) / sms;
    const double eff = double(ctas) / double(waves * sms) - (n < 8 ? 0.05 : 0.0);
    if (eff >= best_eff - 1e-9) { best_eff = eff; best = n; }
  }
  return best;
}

// query blocks smaller than the selection blocks on the tcgen05 path run the selection / window, dQ and
// KV-outer kernels on a virtual query level (pertoken.cu): its block count bound and 64 union slots
// S = query blocks per sub-group (at most): enough for about SSA_VQ_ROWS (default 256: a row-tile pair, so both
// softmax warpgroups of the selection / dQ kernels work; measured C2 m_q = 1: 3.0 -> 2.0 ms, 3.0 -> 2.15 ms; 128, 192,
// 384, 512 rows all slower at C2 and C3) query rows at
// the plan's mean tokens per query block, at most 32 (k_vq_count also closes a sub-group before its union of
// selected blocks would exceed 64); 0 = no virtual level (m_q == m_slc, query blocks
// that fill a tile on their own, or a query-block range / SSA_LOCAL_ROWS, which the virtual level does
// not cut)
double env_or(const char* name, double dflt) {
  const char* e = getenv(name);
  const double x = e ? atof(e) : 0.0;
  return x > 0.0 ? x : dflt;
}
// per-token selection (m_q = 1) on the virtual level: the selection branch as a per-block pass + merge
// (pertoken.cu; it handles any m_q < m_slc, but for m_q = 2 / 4 the union-masked sub-groups measured faster:
// C2 m_q = 2 7.3 vs 7.7 ms — SSA_VQ_BLOCKSEL=2 forces it, for tests)
// (pertoken.cu) instead of the union-masked tiles; not with the window-only / no-window flags
bool use_blk(const Plan* p, const Dims& d, const ssa_attn_cfg* cfg, int vq_S) {
  return vq_S > 0 && (p->info.m[SSA_LEVEL_Q] == 1 || blk_forced()) && blk_enabled() &&
         !(cfg->flags & (SSA_WINDOW_ONLY | SSA_NO_WINDOW)) && d.h_kv >= 1;
}
double q_rows(const Dims& d) { return d.n_q > 0 ? double(d.N) / d.n_q * (d.H / d.h_kv) : 0.0; }
int vq_group(const Plan* p, const Dims& d, const ssa_attn_cfg* cfg) {
  if (p->info.m[SSA_LEVEL_Q] >= p->info.m[SSA_LEVEL_SLC] || !vq_enabled() || d.n_q <= 0 || d.T > 32 || d.h_kv > 8)
    return 0;
  // one query block's selections must fit a virtual block's key capacity
  if (int64_t(d.T) * p->info.max_fill[SSA_LEVEL_SLC] > kVqKeyCap) return 0;
  if (cfg->q_end > 0 && (cfg->q_begin > 0 || cfg->q_end < d.n_q)) return 0;
  const double target = env_or("SSA_VQ_ROWS", 256.0);
  const int S = std::min(32, std::max(1, int(target / q_rows(d) + 0.5)));
  return S >= 2 ? S : 0;
}
// The virtual level of the backward: dQ always runs on it (when S > 0); the KV-outer kernel only when
// query blocks are shorter than SSA_VQ_KV_ROWS rows (default 0: never), since its row walk packs the rows
// of the selecting query blocks into full 64-row tiles (8-row granules) and the union only adds masked rows.
struct VqBwd {
  int S = 0;
  bool kv = false;
  Dims dkv;        // sizes of the inverse CSR / KV-outer work items
  int qbpi = 0;    // KV-outer work-item size
};
VqBwd vq_backward(const Plan* p, const Dims& d, const ssa_attn_cfg* cfg, bool tc) {
  VqBwd v;
  v.S = tc ? vq_group(p, d, cfg) : 0;
  const double kv_rows = env_or("SSA_VQ_KV_ROWS", 0.0);
  v.kv = v.S > 0 && q_rows(d) < kv_rows;
  v.dkv = d;
  if (v.kv) {
    v.dkv.n_q = int(vq_bound(d.n_slc, d.n_q, v.S, d.T, p->info.max_fill[SSA_LEVEL_SLC]));
    v.dkv.T = vq_slots(v.S, d.T);
  }
  v.qbpi = v.kv ? vq_qb_per_item() : tc_qb_per_item(p->info.m[SSA_LEVEL_SLC], p->info.m[SSA_LEVEL_Q]);
  return v;
}

void carve_bwd(Carve& c, const Dims& d, const Plan* p, Ctx* x) {
  const int64_t rows = d.N * d.H, keys = d.N * d.h_kv;
  for (int b = 0; b < 3; ++b) x->Dd[b] = c.take<float>(rows);
  x->dq_acc = c.take<float>(size_t(rows) * d.D);
  x->dk_acc = c.take<float>(size_t(keys) * d.D);
  x->dv_acc = c.take<float>(size_t(keys) * d.D);
  x->dkc = c.take<float>(size_t(d.h_kv) * d.n_cmp * d.D);
  x->dvc = c.take<float>(size_t(d.h_kv) * d.n_cmp * d.D);
  x->n_chunk = pick_chunks(p, d.h_kv);
  x->dkc_part = c.take<float>(size_t(x->n_chunk) * d.h_kv * d.n_cmp * d.D);
  x->dvc_part = c.take<float>(size_t(x->n_chunk) * d.h_kv * d.n_cmp * d.D);
  const int64_t nkeys = int64_t(d.n_slc) * d.h_kv;
  x->inv_cnt = c.take<int32_t>(nkeys);
  x->inv_off = c.take<int32_t>(nkeys + 1);
  x->inv_list = c.take<int32_t>(size_t(d.n_q) * d.h_kv * d.T);
}

void fill_common(Ctx* x, const Plan* p, const Dims& d, const ssa_attn_cfg* cfg) {
  x->N = int32_t(d.N);
  x->H = d.H;
  x->h_kv = d.h_kv;
  x->h_s = d.h_s;
  x->D = d.D;
  x->Dc = d.Dc;
  x->T = d.T;
  x->batch = p->info.batch;
  x->m_cmp = p->info.m[SSA_LEVEL_CMP];
  for (int l = 0; l < kLevels; ++l) {
    x->n_blk[l] = p->info.n_blocks[l];
    x->max_fill[l] = p->info.max_fill[l];
    x->off[l] = p->offsets[l];
    x->tok_block[l] = p->tok_block[l];
    x->bb[l] = p->batch_blocks[l];
  }
  x->max_cmp_b = p->info.max_blocks_per_batch[SSA_LEVEL_CMP];
  x->qb_per_item = tc_qb_per_item(p->info.m[SSA_LEVEL_SLC], p->info.m[SSA_LEVEL_Q]);
  x->max_slc_b = p->info.max_blocks_per_batch[SSA_LEVEL_SLC];
  x->scale = cfg->scale > 0.f ? cfg->scale : 1.0f / std::sqrt(float(d.Dc));
  x->sorted_input = (cfg->flags & SSA_INPUT_SORTED) ? 1 : 0;
  x->win_only = (cfg->flags & SSA_WINDOW_ONLY) ? 1 : 0;
  x->no_win = (cfg->flags & SSA_NO_WINDOW) ? 1 : 0;
  x->accumulate = (cfg->flags & SSA_ACCUMULATE) ? 1 : 0;
  x->save_scores = (cfg->flags & SSA_SAVE_SCORES) ? 1 : 0;
  x->kv_grad_f32 = (cfg->flags & SSA_KV_GRAD_FP32) ? 1 : 0;
  x->perm = p->perm;
  x->inv_perm = p->inv_perm;
  x->sorted_coords = p->sorted_coords;
  x->batch_tokens = p->batch_tokens;
  x->slc_cmp_begin = p->slc_cmp_begin;
  x->cmp_to_slc = p->cmp_to_slc;
  x->q_order = p->q_order;
  x->q_batch = p->q_batch;
  x->cmp_tiles = p->cmp_tiles;
  x->n_cmp_tiles = p->n_cmp_tiles;
  x->pe_k = cfg->pe_k;
  x->pe_v = cfg->pe_v;
  const int nq = p->info.n_blocks[SSA_LEVEL_Q];
  x->q_begin = cfg->q_end > 0 ? std::max(0, cfg->q_begin) : 0;
  x->q_end = cfg->q_end > 0 ? std::min(nq, cfg->q_end) : nq;
  x->tok_begin = -1;   // resolved on device from the Q offsets (kernels read off[Q][q_begin / q_end])
  x->tok_end = -1;
  const bool ranged = cfg->q_end > 0 && p->h_q_offsets.size() == size_t(nq) + 1;
  x->row_lo = ranged ? p->h_q_offsets[x->q_begin] : 0;
  x->row_hi = ranged ? p->h_q_offsets[x->q_end] : int32_t(d.N);
  x->row_base = (cfg->flags & SSA_LOCAL_ROWS) ? x->row_lo : 0;
  if (const ssa_learned* L = cfg->learned) {
    x->conv_kw = L->conv_k_w; x->conv_kb = L->conv_k_b; x->conv_vw = L->conv_v_w; x->conv_vb = L->conv_v_b;
    x->conv_dkw = L->d_conv_k_w; x->conv_dkb = L->d_conv_k_b; x->conv_dvw = L->d_conv_v_w; x->conv_dvb = L->d_conv_v_b;
    x->gx = L->x; x->gC = L->c; x->gw = L->gate_w; x->gb = L->gate_b;
    x->gdx = L->dx; x->gdw = L->d_gate_w; x->gdb = L->d_gate_b;
  }
  x->n_peer = cfg->n_peer;
  x->my_rank = cfg->my_rank;
  for (int r = 0; r < 16; ++r) { x->peer_k[r] = cfg->peer_k[r]; x->peer_v[r] = cfg->peer_v[r]; }
  for (int r = 0; r < 17; ++r) x->peer_tok[r] = cfg->peer_tok[r];
}

// SSA_LOCAL_ROWS: the caller's row tensors start at row row_base; kernels index rows by their plan
// position p (p in [row_lo, row_hi) only), so the base pointers are moved back by row_base rows.
template <class P>
P rows_at(P ptr, const Ctx& x, int64_t elems_per_row, size_t esz) {
  using B = typename std::conditional<std::is_const<typename std::remove_pointer<P>::type>::value, const char*, char*>::type;
  return ptr ? reinterpret_cast<P>(reinterpret_cast<B>(ptr) - x.row_base * elems_per_row * int64_t(esz)) : ptr;
}
}  // namespace
}  // namespace ssa

using namespace ssa;

extern "C" ssa_status ssa_forward_size(ssa_plan plan, const ssa_attn_cfg* cfg, size_t* ws_bytes, size_t* saved_bytes) {
  Plan* p = reinterpret_cast<Plan*>(plan);
  Dims d;
  ssa_status s = check_cfg(p, cfg, &d);
  if (s != SSA_OK) return s;
  if (!ws_bytes || !saved_bytes) { set_error("null size pointer"); return SSA_ERR_ARG; }
  Ctx x{};
  Carve cs(nullptr, 0);
  carve_saved(cs, d, cfg, &x);
  carve_saved_gates(cs, d, cfg);
  *saved_bytes = cs.used + 256;
  Carve cw(nullptr, 0);
  carve_inputs(cw, d, &x, false);
  fill_common(&x, p, d, cfg);
  *ws_bytes = cw.used + tc_fwd_ws_bytes(d.N, d.H, d.h_kv, d.D) + learned_fwd_ws_bytes(x) + size_t(d.n_slc + 64) * 4 +
              (vq_group(p, d, cfg) ? vq_ws_bytes(d.N, d.h_kv, d.n_slc, d.n_q, vq_group(p, d, cfg), d.T, p->info.max_fill[SSA_LEVEL_SLC]) : 0) +
              (use_blk(p, d, cfg, vq_group(p, d, cfg)) ? blk_ws_bytes(d.N, d.h_kv, d.h_s, d.D, d.n_slc, d.n_q, d.T) + 256 : 0) +
              tok_cmp_ws_bytes(d.n_q, p->info.batch, tok_cmp_hs(p->info.m[SSA_LEVEL_Q], d.h_s), d.max_slc_b) + 2048;
  return SSA_OK;
}

extern "C" ssa_status ssa_forward(ssa_plan plan, const ssa_attn_cfg* cfg, const void* q, const void* k, const void* v,
                                  const void* gates, void* out, void* saved, size_t saved_bytes, void* ws,
                                  size_t ws_bytes, void* stream) {
  Plan* p = reinterpret_cast<Plan*>(plan);
  Dims d;
  ssa_status s = check_cfg(p, cfg, &d);
  if (s != SSA_OK) return s;
  const bool lgates = cfg->learned && cfg->learned->x;
  if (!q || !k || !v || !(gates || lgates) || !out || !saved || !ws) { set_error("null tensor pointer"); return SSA_ERR_ARG; }
  size_t need_ws, need_saved;
  s = ssa_forward_size(plan, cfg, &need_ws, &need_saved);
  if (s != SSA_OK) return s;
  if (ws_bytes < need_ws || saved_bytes < need_saved) { set_error("ws/saved buffer too small"); return SSA_ERR_WORKSPACE; }
  if (d.max_slc_b > 0 && p->info.max_blocks_per_batch[SSA_LEVEL_SLC] < 1) { set_error("empty plan"); return SSA_ERR_BAD_STATE; }
  bool tc = false;
  if ((s = choose_path(d, cfg, p, &tc)) != SSA_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Ctx x{};
  fill_common(&x, p, d, cfg);
  x.q = rows_at(q, x, int64_t(d.H) * d.Dc, d.esz);
  x.gates = rows_at(gates, x, int64_t(d.H) * 3, d.esz);
  x.out = rows_at(out, x, int64_t(d.H) * d.Dc, d.esz);
  x.k = k; x.v = v;
  if ((s = learned_checks(x)) != SSA_OK) return s;
  Carve cs(saved, saved_bytes);
  carve_saved(cs, d, cfg, &x);
  float* saved_gates = carve_saved_gates(cs, d, cfg);
  Carve cw(ws, ws_bytes);
  carve_inputs(cw, d, &x, false);
  void* tc_ws = cw.take<char>(tc_fwd_ws_bytes(d.N, d.H, d.h_kv, d.D));
  void* l_ws = cw.take<char>(learned_fwd_ws_bytes(x));
  x.fetch_mark = cw.take<int32_t>(size_t(d.n_slc) + 1);
  x.vq_S = tc ? vq_group(p, d, cfg) : 0;
  x.vq_ws = x.vq_S ? cw.take<char>(vq_ws_bytes(d.N, d.h_kv, d.n_slc, d.n_q, x.vq_S, d.T, p->info.max_fill[SSA_LEVEL_SLC])) : nullptr;
  x.blk_ws = use_blk(p, d, cfg, x.vq_S) ? cw.take<char>(blk_ws_bytes(d.N, d.h_kv, d.h_s, d.D, d.n_slc, d.n_q, d.T)) : nullptr;
  x.tok_cmp = tc ? tok_cmp_hs(p->info.m[SSA_LEVEL_Q], d.h_s) : 0;
  x.tok_ws = x.tok_cmp ? cw.take<char>(tok_cmp_ws_bytes(d.n_q, p->info.batch, x.tok_cmp, d.max_slc_b)) : nullptr;
  if (lgates) x.gs = saved_gates;
  const bool bf16 = cfg->dtype == SSA_BF16;
  // caller-supplied pooled keys (mode 2): no pooling; raw k / v are first read by the selection /
  // window branch, after cfg.kv_event (tcgen05 path) — the compression branch overlaps the K/V exchange
  const bool ext_kc = cfg->kc_in != nullptr;
  cudaEvent_t kv_ev = static_cast<cudaEvent_t>(cfg->kv_event);
  const size_t kc_bytes = size_t(d.h_kv) * d.n_cmp * d.D * 4;
  if (ext_kc) {
    SSA_CUDA_TRY(cudaMemcpyAsync(x.kc, cfg->kc_in, kc_bytes, cudaMemcpyDeviceToDevice, st));
    SSA_CUDA_TRY(cudaMemcpyAsync(x.vc, cfg->vc_in, kc_bytes, cudaMemcpyDeviceToDevice, st));
    if (!tc && kv_ev) SSA_CUDA_TRY(cudaStreamWaitEvent(st, kv_ev, 0));
    if ((s = gather_inputs(x, bf16, st, false, true, /*keys=*/!tc, /*gates=*/!lgates)) != SSA_OK) return s;
  } else {
    if (kv_ev) SSA_CUDA_TRY(cudaStreamWaitEvent(st, kv_ev, 0));
    if ((s = gather_inputs(x, bf16, st, false, true, true, /*gates=*/!lgates)) != SSA_OK) return s;
    if (x.conv_kw) {
      if ((s = learned_pool_forward(x, bf16, l_ws, st)) != SSA_OK) return s;
    } else if ((s = pool_forward(x, bf16, st)) != SSA_OK) {
      return s;
    }
  }
  if (lgates && (s = gate_proj_forward(x, bf16, st)) != SSA_OK) return s;
  if (x.win_only) {
    // skipped branches: O = 0, indices -1 (no selected blocks), LSE huge (p = exp2(s - LSE) = 0 anywhere)
    const int64_t rows = int64_t(d.N) * d.H;
    for (int b = 0; b < 2; ++b) {
      SSA_CUDA_TRY(cudaMemsetAsync(x.o[b], 0, size_t(rows) * d.D * 4, st));
      SSA_CUDA_TRY(cudaMemsetAsync(x.lse[b], 0x7f, size_t(rows) * 4, st));
    }
    SSA_CUDA_TRY(cudaMemsetAsync(x.I, 0xff, size_t(d.n_q) * d.h_kv * d.T * 4, st));
  }
  if (x.no_win) {   // skipped window branch: O_win = 0, LSE sentinel
    const int64_t rows = int64_t(d.N) * d.H;
    SSA_CUDA_TRY(cudaMemsetAsync(x.o[2], 0, size_t(rows) * d.D * 4, st));
    SSA_CUDA_TRY(cudaMemsetAsync(x.lse[2], 0x7f, size_t(rows) * 4, st));
  }
  if (tc) {
    if ((s = tc_forward(x, tc_ws, st, ext_kc ? kv_ev : nullptr, ext_kc)) != SSA_OK) return s;
  } else {
    if ((s = simt_forward(x, bf16, st, false)) != SSA_OK) return s;
    if ((s = combine_forward(x, bf16, st)) != SSA_OK) return s;
  }
  return SSA_OK;
}

extern "C" ssa_status ssa_backward_size(ssa_plan plan, const ssa_attn_cfg* cfg, size_t* ws_bytes) {
  Plan* p = reinterpret_cast<Plan*>(plan);
  Dims d;
  ssa_status s = check_cfg(p, cfg, &d);
  if (s != SSA_OK) return s;
  if (!ws_bytes) { set_error("null size pointer"); return SSA_ERR_ARG; }
  Ctx x{};
  Carve cw(nullptr, 0);
  const VqBwd vq = vq_backward(p, d, cfg, use_tc_bwd(d, cfg, p));
  carve_inputs(cw, d, &x, true);
  carve_bwd(cw, vq.dkv, p, &x);
  size_t scan = inverse_csr_ws_bytes(d.n_slc, d.h_kv, vq.dkv.n_q) + (vq.S ? vq_ws_bytes(d.N, d.h_kv, d.n_slc, d.n_q, vq.S, d.T, p->info.max_fill[SSA_LEVEL_SLC]) : 0) +
                (vq.S && use_blk(p, d, cfg, vq.S) && use_tc_bwd(d, cfg, p) && !vq.kv
                     ? blk_bwd_ws_bytes(d.N, d.h_kv, d.h_s, d.D, d.n_slc, d.n_q, d.T) + 256 : 0);
  if (cfg->learned && cfg->learned->x) scan += gate_bwd_ws_bytes(d.N, d.H, cfg->learned->c);
  if (cfg->learned && cfg->learned->conv_k_w) scan += conv_bwd_ws_bytes(d.N, d.h_kv, p->info.m[SSA_LEVEL_CMP], d.n_cmp, d.D);
  *ws_bytes = cw.used + scan + tc_bwd_ws_bytes(d.N, d.H, d.h_kv, d.D, d.n_slc, vq.dkv.n_q, vq.dkv.T,
                                               p->info.max_fill[SSA_LEVEL_SLC], vq.qbpi) + 1024;
  return SSA_OK;
}

extern "C" ssa_status ssa_backward(ssa_plan plan, const ssa_attn_cfg* cfg, const void* q, const void* k, const void* v,
                                   const void* gates, const void* saved, size_t saved_bytes, const void* dout,
                                   void* dq, void* dk, void* dv, void* dgates, void* ws, size_t ws_bytes,
                                   void* stream) {
  Plan* p = reinterpret_cast<Plan*>(plan);
  Dims d;
  ssa_status s = check_cfg(p, cfg, &d);
  if (s != SSA_OK) return s;
  const bool lgates = cfg->learned && cfg->learned->x;
  if (!q || !k || !v || !(gates || lgates) || !saved || !dout || !dq || !dk || !dv || !dgates || !ws) {
    set_error("null tensor pointer");
    return SSA_ERR_ARG;
  }
  size_t need_ws, need_ws_f, need_saved;
  if ((s = ssa_backward_size(plan, cfg, &need_ws)) != SSA_OK) return s;
  if ((s = ssa_forward_size(plan, cfg, &need_ws_f, &need_saved)) != SSA_OK) return s;
  if (saved_bytes < need_saved) { set_error("saved buffer smaller than this cfg's saved state"); return SSA_ERR_BAD_STATE; }
  if (ws_bytes < need_ws) { set_error("ws buffer too small"); return SSA_ERR_WORKSPACE; }
  bool tc_path = false;
  if ((s = choose_path(d, cfg, p, &tc_path)) != SSA_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Ctx x{};
  fill_common(&x, p, d, cfg);
  x.q = rows_at(q, x, int64_t(d.H) * d.Dc, d.esz);
  x.gates = rows_at(gates, x, int64_t(d.H) * 3, d.esz);
  x.dout = rows_at(dout, x, int64_t(d.H) * d.Dc, d.esz);
  x.dq = rows_at(dq, x, int64_t(d.H) * d.Dc, d.esz);
  x.dgates = rows_at(dgates, x, int64_t(d.H) * 3, d.esz);
  x.k = k; x.v = v; x.dk = dk; x.dv = dv;
  if ((s = learned_checks(x)) != SSA_OK) return s;
  Carve cs(const_cast<void*>(saved), saved_bytes);
  carve_saved(cs, d, cfg, &x);
  float* saved_gates = carve_saved_gates(cs, d, cfg);
  Carve cw(ws, ws_bytes);
  const VqBwd vq = vq_backward(p, d, cfg, tc_path);
  carve_inputs(cw, d, &x, true);
  carve_bwd(cw, vq.dkv, p, &x);
  void* scan_ws = cw.take<char>(inverse_csr_ws_bytes(d.n_slc, d.h_kv, vq.dkv.n_q));
  void* vq_ws = vq.S ? cw.take<char>(vq_ws_bytes(d.N, d.h_kv, d.n_slc, d.n_q, vq.S, d.T, p->info.max_fill[SSA_LEVEL_SLC])) : nullptr;
  void* tc_ws = cw.take<char>(tc_bwd_ws_bytes(d.N, d.H, d.h_kv, d.D, d.n_slc, vq.dkv.n_q, vq.dkv.T,
                                              p->info.max_fill[SSA_LEVEL_SLC], vq.qbpi));
  void* part_ws = nullptr;
  void* conv_ws = nullptr;
  if (lgates) {
    char* gw = cw.take<char>(gate_bwd_ws_bytes(d.N, d.H, cfg->learned->c));
    x.gs = saved_gates;
    x.dz = reinterpret_cast<float*>(gw);
    part_ws = gw + ((size_t(d.N) * d.H * 3 * 4 + 255) & ~size_t(255));
  }
  if (x.conv_kw) conv_ws = cw.take<char>(conv_bwd_ws_bytes(d.N, d.h_kv, p->info.m[SSA_LEVEL_CMP], d.n_cmp, d.D));
  const bool bf16 = cfg->dtype == SSA_BF16;
  const bool tc = use_tc_bwd(d, cfg, p);
  // the tcgen05 backward gathers the q / dO rows and computes D_c, dgates in its own row prologue
  if ((s = gather_inputs(x, bf16, st, true, /*rows=*/!tc, true, /*gates=*/!lgates)) != SSA_OK) return s;
  if (!tc && (s = bwd_prologue(x, bf16, st)) != SSA_OK) return s;
  x.blk_ws = (vq.S && use_blk(p, d, cfg, vq.S) && tc && !vq.kv)
                 ? cw.take<char>(blk_bwd_ws_bytes(d.N, d.h_kv, d.h_s, d.D, d.n_slc, d.n_q, d.T)) : nullptr;
  Ctx xq = x;                                      // the dQ context (virtual level for small m_q)
  if (vq.S && (s = build_virtual_level(x, vq.S, vq_ws, st, &xq, /*plain=*/x.blk_ws != nullptr)) != SSA_OK) return s;
  Ctx& xk = vq.kv ? xq : x;                        // the KV-outer context
  if ((s = build_inverse_csr(xk, scan_ws, st)) != SSA_OK) return s;
  if (tc) {
    if ((s = tc_backward(xq, xk, tc_ws, st)) != SSA_OK) return s;
    if (x.win_only) {   // no compressed-key gradients: the pool backward adds zeros
      SSA_CUDA_TRY(cudaMemsetAsync(x.dkc, 0, size_t(d.h_kv) * d.n_cmp * d.D * 4, st));
      SSA_CUDA_TRY(cudaMemsetAsync(x.dvc, 0, size_t(d.h_kv) * d.n_cmp * d.D * 4, st));
    } else if ((s = cmp_reduce(x, st)) != SSA_OK) {
      return s;
    }
  } else {
    if ((s = simt_backward(x, bf16, st)) != SSA_OK) return s;
  }
  if (x.conv_kw && (s = learned_pool_backward_params(x, bf16, conv_ws, st)) != SSA_OK) return s;
  if ((s = bwd_epilogue(x, bf16, st, /*skip_q=*/tc)) != SSA_OK) return s;
  if (lgates && (s = gate_proj_backward(x, bf16, part_ws, st)) != SSA_OK) return s;
  return SSA_OK;
}

extern "C" ssa_status ssa_pool(ssa_plan plan, const ssa_attn_cfg* cfg, const void* k, const void* v, void* kc, void* vc,
                               void* stream) {
  Plan* p = reinterpret_cast<Plan*>(plan);
  Dims d;
  ssa_status s = check_cfg(p, cfg, &d);
  if (s != SSA_OK) return s;
  if (!k || !v || !kc || !vc) { set_error("null tensor pointer"); return SSA_ERR_ARG; }
  if (!(cfg->flags & SSA_INPUT_SORTED)) { set_error("ssa_pool needs SSA_INPUT_SORTED (plan-order k, v)"); return SSA_ERR_ARG; }
  if (cfg->d != 64 && cfg->dtype == SSA_BF16) { set_error("ssa_pool / caller-supplied pooled keys need d == 64"); return SSA_ERR_UNSUPPORTED; }
  Ctx x{};
  fill_common(&x, p, d, cfg);
  return pool_rows(x, cfg->dtype == SSA_BF16, k, v, static_cast<float*>(kc), static_cast<float*>(vc),
                   static_cast<cudaStream_t>(stream));
}

extern "C" ssa_status ssa_ipc_handle(const void* base, void* handle64) {
  if (!base || !handle64) { set_error("null argument"); return SSA_ERR_ARG; }
  SSA_CUDA_TRY(cudaIpcGetMemHandle(static_cast<cudaIpcMemHandle_t*>(handle64), const_cast<void*>(base)));
  return SSA_OK;
}
extern "C" ssa_status ssa_ipc_open(const void* handle64, void** ptr) {
  if (!handle64 || !ptr) { set_error("null argument"); return SSA_ERR_ARG; }
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  SSA_CUDA_TRY(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return SSA_OK;
}
extern "C" ssa_status ssa_ipc_close(void* ptr) {
  if (!ptr) { set_error("null argument"); return SSA_ERR_ARG; }
  SSA_CUDA_TRY(cudaIpcCloseMemHandle(ptr));
  return SSA_OK;
}

extern "C" ssa_status ssa_saved_state(ssa_plan plan, const ssa_attn_cfg* cfg, const void* saved, size_t saved_bytes,
                                      ssa_saved_view* out) {
  Plan* p = reinterpret_cast<Plan*>(plan);
  Dims d;
  ssa_status s = check_cfg(p, cfg, &d);
  if (s != SSA_OK) return s;
  if (!saved || !out) { set_error("null saved/out"); return SSA_ERR_ARG; }
  Ctx x{};
  Carve cs(const_cast<void*>(saved), saved_bytes);
  carve_saved(cs, d, cfg, &x);
  if (!cs.ok()) { set_error("saved buffer too small"); return SSA_ERR_BAD_STATE; }
  out->idx = x.I;
  out->scores = x.scores;
  for (int b = 0; b < 3; ++b) { out->o_branch[b] = x.o[b]; out->lse_branch[b] = x.lse[b]; }
  out->k_cmp = x.kc;
  out->v_cmp = x.vc;
  out->used_tcgen05 = use_tc(d, cfg, p) ? 1 : 0;
  out->d_internal = d.D;
  return SSA_OK;
}

extern "C" const char* ssa_status_str(ssa_status s) {
  switch (s) {
    case SSA_OK: return "SSA_OK";
    case SSA_ERR_ARG: return "SSA_ERR_ARG";
    case SSA_ERR_DUP_COORD: return "SSA_ERR_DUP_COORD";
    case SSA_ERR_COORD_RANGE: return "SSA_ERR_COORD_RANGE";
    case SSA_ERR_HIERARCHY: return "SSA_ERR_HIERARCHY";
    case SSA_ERR_BAD_STATE: return "SSA_ERR_BAD_STATE";
    case SSA_ERR_WORKSPACE: return "SSA_ERR_WORKSPACE";
    case SSA_ERR_UNSUPPORTED: return "SSA_ERR_UNSUPPORTED";
    case SSA_ERR_CUDA: return "SSA_ERR_CUDA";
  }
  return "SSA_ERR_UNKNOWN";
}
extern "C" const char* ssa_last_error(void) { return g_err.c_str(); }
extern "C" void ssa_profile_enable(int on) { g_prof_on = on != 0; }
extern "C" void ssa_profile_reset(void) {
  for (auto& r : g_prof) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  g_prof.clear();
}
extern "C" ssa_status ssa_profile_read(const char* kernel, double* total_ms, int64_t* launches) {
  if (!kernel || !total_ms || !launches) { set_error("null argument"); return SSA_ERR_ARG; }
  double t = 0;
  int64_t n = 0;
  for (auto& r : g_prof) {
    if (r.name != kernel) continue;
    cudaError_t e = cudaEventSynchronize(r.b);
    if (e != cudaSuccess) return cuda_status(e, "ssa_profile_read");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    t += ms;
    ++n;
  }
  *total_ms = t;
  *launches = n;
  return SSA_OK;
}
extern "C" int64_t ssa_launch_count(void) { return g_launches; }
extern "C" void ssa_reset_launch_count(void) { g_launches = 0; }
extern "C" const char* ssa_build_info(void) {
  return tc_available() ? "libssa_b200 sm_100a: SIMT fp32 kernels + tcgen05/TMEM bf16 kernels"
                        : "libssa_b200 sm_100a: SIMT kernels only";
}
