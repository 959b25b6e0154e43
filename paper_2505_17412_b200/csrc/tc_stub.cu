// tc_stub.cu — placeholder until the tcgen05 kernels land: reports them unavailable.
#include "tc.h"
namespace ssa {
bool tc_available() { return false; }
size_t tc_fwd_ws_bytes(int64_t, int, int, int) { return 0; }
size_t tc_bwd_ws_bytes(int64_t, int, int, int) { return 0; }
ssa_status tc_forward(const Ctx&, void*, cudaStream_t) { set_error("tcgen05 kernels not built"); return SSA_ERR_UNSUPPORTED; }
ssa_status tc_backward(const Ctx&, void*, cudaStream_t) { set_error("tcgen05 kernels not built"); return SSA_ERR_UNSUPPORTED; }
}  // namespace ssa
