/* fdmoe_dev.h — development entry points of libfdmoe_dev.so (tests and tools only).
 *
 * The product library libfdmoe.so exports only include/fdmoe.h. libfdmoe_dev.so is the same sources
 * built with -DFDMOE_DEV (ablation bits read from FDMOE_DEBUG, the MMA-warp chunk log, per-role wait
 * accounting) plus these diagnostics. Not part of the reference surface.
 */
#ifndef FDMOE_DEV_H
#define FDMOE_DEV_H
#include "fdmoe.h"
#ifdef __cplusplus
extern "C" {
#endif

/* The kernel's glibc-expf restatement on n host floats (runs on device 0). */
fdmoe_status fdmoe_debug_expf(const float* x, float* y, int64_t n);
/* One 128x128 tile through the layer's FFN machinery (weight rows -> registers -> TMEM operand,
 * token rows via TMA -> smem operand, tcgen05.mma, TMEM epilogue):
 * D[f][t] = sum_k W[f][k] * X[t][k]; W, X: 128 x K host row-major FP32 (K % 64 == 0). */
fdmoe_status fdmoe_debug_gemm(int32_t precision, int32_t K, const float* W, const float* X, float* D);
/* Issue-rate microbenchmark: SM cycles per tcgen05.mma (M=128, A from TMEM, N in {64,128,256})
 * when `nissuers` warps (1-2) each issue `iters` back-to-back MMAs into their own accumulator;
 * kind 0 = tf32, 1 = bf16. kind >= 16: the FFN pipeline skeleton (fdmoe_kernel.cu debug_pipe_kernel,
 * mode = kind - 16) on 148 CTAs, iters = half-stages of 12 MMAs; returns cycles per MMA. */
/* Latency probe (cycles): [0] issue of n tf32 N=128 MMAs, [1] issue -> commit completion,
 * [2] 8 x tcgen05.st.x16 + wait::st, [3] mbarrier wait with a 2000-cycle delayed arrive. */
fdmoe_status fdmoe_debug_latency(int32_t n, uint64_t* out4);
/* Debug: CTA 0's MMA-warp chunk timeline of the last launch (512 x {clock, wait tokens,
 * wait weights, issue}); enabled when FDMOE_CHUNKLOG is set at fdmoe_create. */
fdmoe_status fdmoe_read_chunklog(fdmoe_handle* h, uint64_t* out);
fdmoe_status fdmoe_debug_mma_rate(int32_t kind, int32_t nissuers, int32_t N, int32_t iters, double* cycles_per_mma);

#ifdef __cplusplus
}
#endif
#endif /* FDMOE_DEV_H */
