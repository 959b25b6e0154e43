/* ssa_selftest.h — diagnostics exported by libssa_b200.so for the GPU test-suite (not part of the
 * SSA computation). ssa_selftest_umma runs ONE tcgen05.mma tile with the operand layouts the SSA
 * kernels use and writes the fp32 result, so descriptor encodings are checked in isolation:
 *   mode 0: d[128][n] = a[128][64] . b[n][64]^T       (K-major A and B, both TMA-loaded; n in 16..256)
 *   mode 1: d[128][64] = a[k][128]^T . b[k][64]        (MN-major A written by threads, MN-major B by TMA; k=128)
 *   mode 2: d[128][64] = a[128][k] . b[k][64]          (K-major A written by threads, MN-major B by TMA; k=64,96,128)
 *   mode 4: d[128][64] = a[128][k] . b[k][64]          (A in TMEM via tcgen05.st, MN-major B by TMA)
 *   mode 5: d[128][n]  = a[128][64] . b[n][64]^T       (A in TMEM via tcgen05.st, K-major B by TMA)
 * a, b: device bf16 row-major; d: device fp32 row-major. Synchronises `stream`. */
#ifndef SSA_SELFTEST_H
#define SSA_SELFTEST_H
#include "ssa.h"
#ifdef __cplusplus
extern "C" {
#endif
ssa_status ssa_selftest_umma(int mode, int n, int k, const void* a, const void* b, float* d, void* stream);
#ifdef __cplusplus
}
#endif
#endif
