/*
 * conv2d.h -- C-ABI of libconv2d.so: fp32 NHWC 2D-convolution forward on B200 (sm_100a).
 *
 * The operation (every algorithm below computes it; "a variety
 * of different algorithms which all provide the same numeric results"):
 *
 *   y[n,ho,wo,f] = sum_{kh,kw,c} x[n, ho*Sr + kh - pad_top, wo*Sc + kw - pad_left, c] * w[kh,kw,c,f]
 *
 * out-of-bounds x reads as 0; cross-correlation (no filter flip).  Parameter
 * space = SYCL-DNN's (Fig. 1 tuple "window size, stride, image
 * rows, image columns, input features, output features", plus batch and
 * SAME/VALID padding -- SPEC.md:40-45).  Shapes follow SPEC.md:48-56:
 *   SAME : Ho = ceil(H/S);   VALID: Ho = floor((H-K)/S)+1, requires K <= H
 *   pad_total = max((Ho-1)*S + K - H, 0); pad_top = floor(pad_total/2); pad_bottom = rest.
 *
 * Layouts (all dense, row-major, 64-bit indexed):
 *   in   : NHWC  fp32, N*H*W*C elements
 *   filt : HWCF  fp32 (Kh, Kw, C, F) -- i.e. a (Kh*Kw*C) x F row-major matrix
 *   out  : N,Ho,Wo,F fp32
 *
 * Ownership: the caller owns every buffer; all pointers passed to
 * conv2d_forward are DEVICE pointers, 16-byte aligned, and must not alias
 * (in/filt are read-only, out and ws are written).  The library never
 * allocates or frees device memory, and keeps no pointer after a call returns.
 *
 * Execution: conv2d_forward is stream-ordered and asynchronous on `stream`
 * (a cudaStream_t; NULL = legacy default stream).  Parameter errors are
 * returned synchronously before anything is launched.  Kernel launch errors
 * are returned as CONV2D_ERR_CUDA (detail in conv2d_last_error()).  Results
 * are bitwise reproducible for a fixed (params, algo, tuned variant -- see
 * conv2d_get_variant -- , device): no atomics, split-K partial sums are reduced
 * in a fixed order.
 *
 * Thread safety: every function may be called concurrently from several host
 * threads; the auto-selector cache is mutex-protected.
 */
#ifndef CONV2D_B200_H
#define CONV2D_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { CONV2D_PAD_SAME = 0, CONV2D_PAD_VALID = 1 } conv2d_padding_t;

/* Math mode of the tensor-core paths.
 *  FP32: fp32-faithful.  Tensor paths run 3xTF32 (a = a_hi + a_lo split;
 *        a_hi*b_hi + a_hi*b_lo + a_lo*b_hi, fp32 accumulation); CUDA-core paths
 *        run plain fp32 FFMA.  Tolerance max|err|/sum|x||w| <= 1e-5 (north_star).
 *  TF32: one TF32 MMA per product (reported separately; tolerance 2e-3).
 *        CUDA-core algorithms (direct, tiled) ignore it and stay exact fp32. */
typedef enum { CONV2D_MATH_FP32 = 0, CONV2D_MATH_TF32 = 1 } conv2d_math_t;

/* Algorithms.  Enum order is the auto-selector's tie-break order. */
typedef enum {
  CONV2D_ALGO_AUTO = 0,              /* measured-time argmin over supported algorithms, cached */
  CONV2D_ALGO_DIRECT = 1,            /* one thread per output vector, FFMA */
  CONV2D_ALGO_TILED = 2,             /* CTA output tile, smem halo, register blocking */
  CONV2D_ALGO_IMPLICIT_GEMM = 3,     /* tcgen05/TMEM GEMM over the never-materialised im2col matrix */
  CONV2D_ALGO_WINOGRAD_F2X2_3X3 = 4, /* Winograd F(2x2,3x3), tensor-core batched GEMM */
  CONV2D_ALGO_MATMUL_1X1 = 5,        /* 1x1/stride-1 conv as one GEMM */
  CONV2D_ALGO_WINOGRAD_F4X4_3X3 = 6  /* Winograd F(4x4,3x3) ("Winograd large"): 6x6 tiles, 36
                                        batched tensor-core GEMMs, 4x fewer multiplies than direct */
} conv2d_algo_t;
#define CONV2D_NUM_ALGOS 7

typedef struct {
  int32_t batch, in_rows, in_cols, channels, features;
  int32_t window_rows, window_cols, stride_rows, stride_cols;
  conv2d_padding_t padding;
  conv2d_math_t math;
} conv2d_params_t;

typedef enum {
  CONV2D_OK = 0,
  CONV2D_ERR_INVALID_PARAMS = 1, /* dim < 1, bad enum, VALID with K > H, element count overflow */
  CONV2D_ERR_UNSUPPORTED = 2,    /* algorithm incompatible with params (never silently replaced) */
  CONV2D_ERR_WORKSPACE = 3,      /* ws NULL or ws_bytes < conv2d_query_workspace() */
  CONV2D_ERR_ALIGNMENT = 4,      /* a device pointer is not 16-byte aligned */
  CONV2D_ERR_NULL = 5,           /* a required pointer argument is NULL */
  CONV2D_ERR_CUDA = 6,           /* a CUDA call failed; see conv2d_last_error() */
  CONV2D_ERR_NO_DEVICE = 7,      /* no sm_100 device is current */
  CONV2D_ERR_IO = 8              /* selection-table file could not be opened / written */
} conv2d_status_t;

/* Shape inference (no device needed).  out_nhwf = {N, Ho, Wo, F};
 * pads_tblr = {top, bottom, left, right} (either may be NULL). */
conv2d_status_t conv2d_output_shape(const conv2d_params_t* p, int32_t out_nhwf[4], int32_t pads_tblr[4]);

/* 2*N*Ho*Wo*Kh*Kw*C*F: direct-convolution flops, used for
 * GFLOP/s of every algorithm including Winograd (reading R8). */
conv2d_status_t conv2d_flop_count(const conv2d_params_t* p, uint64_t* flops);

/* *supported = 1 iff `algo` can run `p` (no device needed).  AUTO is always supported.
 *   DIRECT, TILED, IMPLICIT_GEMM : every valid params
 *   MATMUL_1X1                   : Kh = Kw = 1 and Sr = Sc = 1
 *   WINOGRAD_F2X2_3X3            : Kh = Kw = 3, Sr = Sc = 1, C >= 32 (reading R13/R16)
 *   WINOGRAD_F4X4_3X3            : as F2X2 and math = FP32 only -- in TF32 mode its larger transform
 *                                  constants put the error at the 2e-3 bound (reading R21) */
conv2d_status_t conv2d_supports(const conv2d_params_t* p, conv2d_algo_t algo, int* supported);

/* Device workspace bytes `algo` needs for `p` (AUTO: max over supported
 * algorithms).  0 means ws may be NULL. */
conv2d_status_t conv2d_query_workspace(const conv2d_params_t* p, conv2d_algo_t algo, size_t* bytes);

/* The forward pass.  in/filt/out/ws: device pointers (see Ownership).
 * ws_bytes must be >= conv2d_query_workspace(p, algo).  With AUTO on a cache
 * miss this tunes first (see conv2d_autotune: it SYNCHRONISES the stream and
 * uses out/ws as scratch), then runs the chosen algorithm.  Under stream capture
 * an AUTO cache miss returns CONV2D_ERR_UNSUPPORTED without touching the stream
 * (tune before capturing); a cached AUTO choice and concrete algorithms capture. */
conv2d_status_t conv2d_forward(const conv2d_params_t* p, conv2d_algo_t algo, const float* in,
                               const float* filt, float* out, void* ws, size_t ws_bytes, void* stream);

/* Auto-selector (PAPER.md:209-215 per-device algorithm choice):
 * time every supported algorithm on the caller's buffers (CUDA events, W warm-ups
 * then R reps, best-of-R), pick the argmin with ties broken by enum order, cache it
 * under (params incl. batch/padding/math, device), and write it to *chosen.
 * Synchronises `stream`.  ws must be sized for AUTO.  CONV2D_ERR_UNSUPPORTED if
 * `stream` is being captured (tuning cannot be captured). */
conv2d_status_t conv2d_autotune(const conv2d_params_t* p, const float* in, const float* filt, float* out,
                                void* ws, size_t ws_bytes, void* stream, conv2d_algo_t* chosen);

/* Cache query without tuning: CONV2D_OK and *chosen if cached, else
 * CONV2D_ERR_UNSUPPORTED and *chosen = AUTO. */
conv2d_status_t conv2d_selected(const conv2d_params_t* p, conv2d_algo_t* chosen);

/* Seed the cache explicitly (e.g. to replay a choice broadcast from rank 0).
 * Fails with CONV2D_ERR_UNSUPPORTED if `algo` cannot run `p`. */
conv2d_status_t conv2d_set_selected(const conv2d_params_t* p, conv2d_algo_t algo);

/* Tuned parameter variant of the implicit_gemm / matmul_1x1 / winograd_f2x2_3x3 kernels for `p` ("different
 * parameters for each algorithm"; the "/variant" of the selection table below).
 * implicit_gemm / matmul_1x1: a bit mask -- A-operand path, N tile, B path (bit 3; bit 5 on the 3x3 halo
 * path in 3xTF32), K split (igemm.cu).  Bit 0
 * (A path) on implicit_gemm: halo <-> im2col for 3x3/s1 with C % 32 == 0; 4-channel halo (0) <-> row-segment
 * boxes (1) for 3x3/s1 with C <= 4 and W*C % 4 == 0; space-to-depth halo <-> row segments for 7x7/s2 stems.
 * winograd_f2x2_3x3: 0 = transform kernels + batched tcgen05 GEMM (winograd.cu), 1 = the fused kernel
 * (input transform, 16 coordinate GEMMs and output transform in one cluster-of-2 launch; wino_fused.cu),
 * enumerated where C % 4 == 0, F % 4 == 0 and Ho >= 2.
 * get: *variant = the variant conv2d_autotune / load_selection / set_variant recorded, or 0 (the
 * default parameters) if none was.  set: seeds it (e.g. replaying rank 0's tuned choice on every rank);
 * CONV2D_ERR_INVALID_PARAMS unless `variant` is one the auto-selector enumerates for `p` and `algo`.
 * `algo` must be one of those three (CONV2D_ERR_INVALID_PARAMS otherwise; CONV2D_ERR_UNSUPPORTED if it cannot
 * run `p`).  Host-only. */
conv2d_status_t conv2d_get_variant(const conv2d_params_t* p, conv2d_algo_t algo, int* variant);
conv2d_status_t conv2d_set_variant(const conv2d_params_t* p, conv2d_algo_t algo, int variant);

/* Learned selector (tuning decisions "are a good candidate for a learned
 * solution rather than a hand tuned one"): the (algorithm, tuned variant) a decision tree trained on measured
 * B200 timings predicts to be fastest for `p` -- features are shape quantities (log M, N, C, K, window,
 * stride, padding, batch, math, tile count, arithmetic intensity); training data, cross-validated regret and
 * the generator: tools/selector_data.py, tools/train_selector.py, profiles/data/selector_model_r1.json.
 * Runs nothing on the device; the result always supports `p` (fallback implicit_gemm / 0). */
conv2d_status_t conv2d_predict(const conv2d_params_t* p, conv2d_algo_t* algo, int* variant);

/* What conv2d_forward(AUTO) does on a cache miss: MEASURE (default) tunes on the caller's buffers (see
 * conv2d_autotune; refused under stream capture); PREDICT caches conv2d_predict's choice instead -- no
 * timing, no synchronisation, so it also works inside a CUDA-graph capture; HYBRID tunes like MEASURE
 * (conv2d_autotune too) but times only the learned selector's top 3 candidates (CONV2D_HYBRID_TOPK).
 * Process-wide. */
typedef enum { CONV2D_AUTO_MEASURE = 0, CONV2D_AUTO_PREDICT = 1, CONV2D_AUTO_HYBRID = 2 } conv2d_auto_policy_t;
conv2d_status_t conv2d_set_auto_policy(conv2d_auto_policy_t policy);

/* Drop every cached choice. */
void conv2d_clear_selection_cache(void);

/* Cache-cold auto-selection: register a caller-owned DEVICE scratch buffer (e.g. 256 MiB, larger than the
 * 126 MB L2) that conv2d_autotune / conv2d_forward(AUTO) overwrite with cudaMemsetAsync before every timed
 * repetition, outside the timed events -- so candidates are compared with the cold caches a layer sees
 * inside a network rather than with their own inputs still in L2.  buf = NULL disables it (default).
 * The library keeps the pointer (the caller keeps the buffer alive while tuning may run) but never
 * allocates it.  CONV2D_ERR_INVALID_PARAMS if buf != NULL and bytes == 0. */
conv2d_status_t conv2d_set_autotune_flush(void* buf, size_t bytes);

/* Persisted selector table ("table serialization round-trips", SPEC.md:354's line format with
 * this library's full cache key).  One line per cached choice of the current device:
 *     N H W C F KH KW SH SW same|valid fp32|tf32 : algorithm[/variant]
 * (variant = the tuned algorithm parameters of implicit_gemm / matmul_1x1 / winograd_f2x2_3x3, see
 * conv2d_get_variant), then
 * `default : a,b,...` (algorithms by number of entries won; informative) and `#` comments.
 * save: CONV2D_ERR_IO if the file cannot be written.  load: parses and validates every line first
 * (CONV2D_ERR_INVALID_PARAMS for malformed lines / unknown names / invalid params / a variant the
 * auto-selector does not enumerate for that line's params,
 * CONV2D_ERR_UNSUPPORTED if an algorithm cannot run its params -- detail with file:line in
 * conv2d_last_error()); only a fully valid file is applied, seeding the cache (and variants) so
 * conv2d_forward(AUTO) uses the stored choices without tuning.  *loaded = entries applied (may be NULL).
 * Host-only: neither touches device memory. */
conv2d_status_t conv2d_save_selection(const char* path);
conv2d_status_t conv2d_load_selection(const char* path, int* loaded);

/* Last per-algorithm best times (microseconds) from the most recent autotune on
 * this thread; times[a] < 0 for algorithms not timed.  times must hold CONV2D_NUM_ALGOS.
 * A candidate whose launch is refused during tuning (e.g. a grid-limit error) is dropped
 * with a warning on stderr and reports < 0; a fault that leaves the stream
 * unusable is returned as CONV2D_ERR_CUDA instead. */
void conv2d_last_tune_times(double times_us[CONV2D_NUM_ALGOS]);

/* Number of kernel launches conv2d_forward(p, algo) issues (AUTO: of the cached choice,
 * or -1 if not cached).  Used by bench.py to report gpu_launches. */
int conv2d_launch_count(const conv2d_params_t* p, conv2d_algo_t algo);

/* Counter-based seeded generator on the device (NOT part of the convolution;
 * the device twin of paper_1904_04174_b200/synth.py, used to fill multi-GB bench
 * inputs quickly).  Writes count floats, element i = gen(key, offset + i);
 * dist 0 = uniform [-1,1), 1 = integers {-2..2}. */
conv2d_status_t conv2d_synth_fill(float* dst, uint64_t count, uint64_t key, uint64_t offset, int dist,
                                  void* stream);

const char* conv2d_status_string(conv2d_status_t s);
const char* conv2d_algo_name(conv2d_algo_t a);
/* Thread-local detail of the last error on this thread ("" if none). */
const char* conv2d_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* CONV2D_B200_H */
