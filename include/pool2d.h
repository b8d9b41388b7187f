/*
 * pool2d.h -- NHWC max / average pooling on B200 (libconv2d.so; the library's
 * other primitive, "pooling and normalization layers"; semantics SPEC.md:361-401).
 *
 *   y[n,ho,wo,c] = max / mean over the IN-BOUNDS taps
 *                  { x[n, ho*Sr + kh - pad_top, wo*Sc + kw - pad_left, c] : kh < Kh, kw < Kw }
 *
 * SAME-padding positions are ignored (never -inf / never counted: SPEC.md:372, 381).  Shapes and pad
 * split are conv2d's (conv2d.h) with F := C.  Average: the sum is accumulated in double
 * in (kh, kw) order and divided by the in-bounds count in double, rounded once to fp32 -- so both
 * operations are bit-identical to the definition evaluated in double.
 *
 * Layouts: in NHWC fp32 (N*H*W*C), out N,Ho,Wo,C fp32; DEVICE pointers owned by the caller, 4-byte
 * aligned (16-byte alignment and C % 4 == 0 select the float4 path), not aliased.  Stream-ordered and
 * asynchronous on `stream` (a cudaStream_t; NULL = legacy default stream).  No workspace.
 * Errors: CONV2D_ERR_INVALID_PARAMS (dim < 1, bad enum, VALID window > input, > 2^40 elements),
 * CONV2D_ERR_NULL, CONV2D_ERR_ALIGNMENT (not 4-byte aligned), CONV2D_ERR_NO_DEVICE, CONV2D_ERR_CUDA --
 * all but the last returned before anything is launched.
 */
#ifndef POOL2D_B200_H
#define POOL2D_B200_H

#include "conv2d.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { POOL2D_MAX = 0, POOL2D_AVG = 1 } pool2d_op_t;

typedef struct {
  int32_t batch, in_rows, in_cols, channels;
  int32_t window_rows, window_cols, stride_rows, stride_cols;
  conv2d_padding_t padding;
  pool2d_op_t op;
} pool2d_params_t;

/* {N, Ho, Wo, C} and {top, bottom, left, right}; CONV2D_ERR_INVALID_PARAMS if invalid. Host only. */
conv2d_status_t pool2d_output_shape(const pool2d_params_t* p, int32_t out_nhwc[4], int32_t pads_tblr[4]);

/* One pooling pass over the whole tensor (one kernel launch). */
conv2d_status_t pool2d_forward(const pool2d_params_t* p, const float* in, float* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif
