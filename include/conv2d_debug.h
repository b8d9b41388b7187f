/*
 * conv2d_debug.h -- diagnostics of libconv2d.so, not part of the computation (no PAPER.md passage:
 * this is instrumentation for the measurement step).
 */
#ifndef CONV2D_B200_DEBUG_H
#define CONV2D_B200_DEBUG_H

#include "conv2d.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Per-CTA timelines of the tcgen05 GEMM kernels (gemm2sm_kernel, halo_kernel), %globaltimer ns.
 *   enable = 1: zero the buffer and restart the ring; every later launch (host call or CUDA-graph
 *               capture: the record index is fixed when the launch is issued) gets the next of 256
 *               records of 148 CTAs x 8 stamps (launch-major, then CTA, then stamp):
 *               [0] entry  [1] setup done (barriers, TMEM, cluster sync, PDL wait)  [2] first TMA
 *               issued  [3] first stage consumed by the MMA (leader CTAs)  [4] first accumulator
 *               ready  [5] last epilogue store issued  [6] stores drained  [7] exit
 *               (halo_kernel: [0], [1], [7] only); unused stamps stay 0.
 *   enable = 0: stop stamping;  enable = -1: leave the state unchanged.
 * If `host` is non-NULL, copies min(n, 256*148*8) stamps to it (synchronous, device-wide) and returns
 * that count; returns 0 if nothing was copied and -1 on a CUDA error.  Costs one predicated
 * branch per stamp site when disabled.  Not thread-safe; for tools/ and bench diagnostics. */
int conv2d_debug_trace(int enable, unsigned long long* host, int n);

/* K-split of the launch plan conv2d_forward(p, algo) would run now (with the variant currently recorded
 * for p): *splits = 1 (no split: every output is one accumulation over the whole K = KH*KW*C in a fixed
 * order), s > 1 (every tile's K range is cut into s parts, summed in fixed order by a reduce kernel), or
 * -s (remainder split: only the partial last wave's tiles are cut s ways).  Two plans with equal
 * *splits = 1 give bitwise identical outputs for the same image (the P11 shard check);
 * a split count depends on the tile count and so on the batch.  Status as conv2d_supports, plus
 * CONV2D_ERR_UNSUPPORTED when algo cannot run p.  Host-only, no device work. */
conv2d_status_t conv2d_debug_splits(const conv2d_params_t* p, conv2d_algo_t algo, int* splits);

#ifdef __cplusplus
}
#endif
#endif
