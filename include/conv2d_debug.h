/*
 * conv2d_debug.h -- diagnostics of libconv2d.so, not part of the computation (no PAPER.md passage:
 * this is instrumentation for the measurement step).
 */
#ifndef CONV2D_B200_DEBUG_H
#define CONV2D_B200_DEBUG_H

#ifdef __cplusplus
extern "C" {
#endif

/* Per-CTA timeline of the persistent GEMM core (gemm2sm_kernel), in %globaltimer nanoseconds.
 *   enable = 1: every later GEMM-core launch writes 8 stamps per CTA (CTA-major, up to 148 CTAs):
 *               [0] entry  [1] setup done (barriers, TMEM, cluster sync)  [2] first TMA issued
 *               [3] first stage consumed by the MMA (leader CTAs)  [4] first accumulator ready
 *               [5] last epilogue store issued  [6] stores drained  [7] exit;
 *               the buffer is zeroed.  Each launch overwrites the stamps of the CTAs it runs.
 *   enable = 0: stop stamping;  enable = -1: leave the state unchanged.
 * If `host` is non-NULL, copies min(n, 148*8) stamps to it (synchronous, device-wide) and returns
 * that count; returns 0 if nothing was copied and -1 on a CUDA error.  Costs one predicated
 * branch per stamp site when disabled.  Not thread-safe; for tools/ and bench diagnostics. */
int conv2d_debug_trace(int enable, unsigned long long* host, int n);

#ifdef __cplusplus
}
#endif
#endif
