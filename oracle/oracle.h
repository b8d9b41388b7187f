/*
 * oracle.h -- CPU oracle for the fp32 NHWC conv2d forward pass.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may link, load or call
 * this library.  It shares no code, header, table or constant with the
 * product library (include/conv2d.h, paper_1904_04174_b200/csrc/).
 *
 * What it computes (the definition the paper's algorithms all reach,
 * PAPER.md:206-210 "a variety of different algorithms which all provide the
 * same numeric results"; index formula as restated in SPEC.md:120 and
 * SURVEY.md §8(c)):
 *
 *   y[n,ho,wo,f] = sum_{kh<Kh} sum_{kw<Kw} sum_{c<C}
 *                  x[n, ho*Sr + kh - pad_top, wo*Sc + kw - pad_left, c] * w[kh,kw,c,f]
 *
 * with out-of-bounds x contributing 0 (cross-correlation, no filter flip:
 * DESIGN.md reading R2).  Every product of two fp32 values is exact in
 * double; the sum is accumulated in double and rounded ONCE to fp32
 * (north_star "naive 7-loop convolution accumulating in
 * double").
 *
 * Layouts: input NHWC, filter HWCF, output N,Ho,Wo,F -- all dense, row-major,
 * channels/features fastest (reading R1).
 *
 * Shapes (reading R3):
 *   SAME : Ho = ceil(H/S);  VALID: Ho = floor((H-K)/S)+1 (requires K <= H)
 *   pad_total = max((Ho-1)*S + K - H, 0), pad_before = floor(pad_total/2),
 *   pad_after = pad_total - pad_before.   (VALID: all pads 0.)
 */
#ifndef CONV_ORACLE_H
#define CONV_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORACLE_SAME = 0, ORACLE_VALID = 1 };

typedef struct {
  int32_t batch, in_rows, in_cols, channels, features;
  int32_t window_rows, window_cols, stride_rows, stride_cols;
  int32_t padding; /* ORACLE_SAME / ORACLE_VALID */
} oracle_params;

/* Returns 0 and fills out_nhwf = {N, Ho, Wo, F}, pads_tblr = {top, bottom,
 * left, right}; returns 1 for invalid parameters (any dim < 1, bad padding
 * enum, VALID with window > input extent). */
int oracle_output_shape(const oracle_params* p, int32_t out_nhwf[4], int32_t pads_tblr[4]);

/* 2*N*Ho*Wo*Kh*Kw*C*F; 0 on invalid params. */
uint64_t oracle_flop_count(const oracle_params* p);

/* Full convolution.  out: N*Ho*Wo*F floats (double sum rounded once).
 * denom (nullable): N*Ho*Wo*F doubles, sum over taps of |x|*|w| -- the
 * denominator of the north_star error metric.  threads <= 0 means 1.
 * Returns 0 on success, 1 on invalid params. */
int oracle_conv2d(const oracle_params* p, const float* in, const float* filt, float* out,
                  double* denom, int threads);

/* One output element in double (unrounded) plus its |x||w| denominator.
 * Used for sampled checks at full size.  Returns 1 on invalid params or
 * out-of-range index. */
int oracle_conv2d_point(const oracle_params* p, const float* in, const float* filt,
                        int64_t n, int64_t ho, int64_t wo, int64_t f, double* y, double* denom);

/* Many points at once: idx is count x 4 int64 (n,ho,wo,f). */
int oracle_conv2d_points(const oracle_params* p, const float* in, const float* filt,
                         const int64_t* idx, int64_t count, double* y, double* denom, int threads);

/* ---- pooling (pool.c) -------------------------------
 * NHWC max / average pooling.  The window of output (n, ho, wo, c) is the in-bounds subset of
 * {(ho*Sr + kh - pad_top, wo*Sc + kw - pad_left)}; max = its maximum, avg = its double sum / its
 * count, rounded once.  Shapes: the convolution's (features := channels). */
enum { ORACLE_POOL_MAX = 0, ORACLE_POOL_AVG = 1 };

typedef struct {
  int32_t batch, in_rows, in_cols, channels;
  int32_t window_rows, window_cols, stride_rows, stride_cols;
  int32_t padding; /* ORACLE_SAME / ORACLE_VALID */
  int32_t op;      /* ORACLE_POOL_MAX / ORACLE_POOL_AVG */
} oracle_pool_params;

/* 0 and {N, Ho, Wo, C}, {top, bottom, left, right}; 1 on invalid params. */
int oracle_pool2d_shape(const oracle_pool_params* p, int32_t out_nhwc[4], int32_t pads_tblr[4]);
/* 0 on success, 1 invalid params, 2 if some window had no in-bounds element. */
int oracle_pool2d(const oracle_pool_params* p, const float* in, float* out, int threads);

#ifdef __cplusplus
}
#endif
#endif
