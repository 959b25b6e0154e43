// tc_bwd.cu — tcgen05 backward kernels (bf16, d = 64). Until they land the backward runs the SIMT
// kernels on the tcgen05 forward's saved state (same layout).
#include "tc.h"
namespace ssa {
bool tc_bwd_available() { return false; }
size_t tc_bwd_ws_bytes(int64_t, int, int, int) { return 0; }
ssa_status tc_backward(const Ctx&, void*, cudaStream_t) { set_error("tcgen05 backward not built"); return SSA_ERR_UNSUPPORTED; }
}  // namespace ssa
