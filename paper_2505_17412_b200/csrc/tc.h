// tc.h — tcgen05/TMEM/TMA (sm_100a) kernels of the bf16, d = 64 hot path (tc_fwd.cu, tc_bwd.cu).
#pragma once
#include "internal.h"

namespace ssa {
bool tc_available();
bool tc_bwd_available();
// the plan's block statistics fit the tcgen05 kernels' shared-memory score arrays and tile lists
bool tc_plan_ok(const ssa_plan_info& info, int top_k);
size_t tc_fwd_ws_bytes(int64_t N, int H, int h_kv, int D);
size_t tc_bwd_ws_bytes(int64_t N, int H, int h_kv, int D, int n_slc, int n_q, int T, int max_fill_slc, int qb_per_item);
// query blocks per raw-key KV-outer work item: the tuned 8 selection-block-sized query blocks, scaled by
// (m_slc / m_q)^3 when query blocks are smaller (per-token selection, m_q = 1)
int tc_qb_per_item(int m_slc, int m_q);
// forward after gather + pool: compression attention + scores + top-k, selection + window attention,
// gated combine (writes c.out and the saved state).
// kv_ev: wait for it before the first read of raw k / v; gather_keys_late: the key gather (k, v ->
// internal layout) has not been done yet and runs after the wait (pooled keys supplied by the caller)
ssa_status tc_forward(const Ctx& c, void* ws, cudaStream_t st, cudaEvent_t kv_ev = nullptr, bool gather_keys_late = false);
// backward after gather + prologue + inverse CSR: fills dq_acc, dk_acc, dv_acc, dkc, dvc. c: row prologue,
// dQ and compressed-key KV-outer; c_kv: raw-key KV-outer (its query level carries the inverse CSR).
ssa_status tc_backward(const Ctx& c, const Ctx& c_kv, void* ws, cudaStream_t st);
}  // namespace ssa
