// api.cpp -- the C-ABI of libconv2d.so (include/conv2d.h): validation, shape inference,
// workspace sizing, dispatch to the sm_100a kernels, and the measured-time auto-selector.
//
// Auto-selection follows the paper's adaptation model -- "the library can adapt to
// different hardware characteristics by either choosing different algorithms or
// different parameters for each algorithm", automated as planned in
// with SPEC.md:333-350's empirical argmin: every supported algorithm
// is timed with CUDA events (best of R after W warm-ups), ties go to enum order, and the
// choice is cached per (params, device).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <atomic>
#include <cmath>
#include <string>
#include <tuple>
#include <vector>
#include <cctype>
#include <cstdlib>

#include "internal.h"
#include "launch.cuh"
#include "selector_tree.h"
#include "../../include/conv2d_debug.h"
#include "../../include/pool2d.h"

using namespace conv2d;

namespace {

thread_local std::string g_last_error;
thread_local double g_tune_times[CONV2D_NUM_ALGOS] = {-1, -1, -1, -1, -1, -1, -1};

conv2d_status_t fail(conv2d_status_t s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

conv2d_status_t cuda_fail(cudaError_t e, const char* where) {
  g_last_error = std::string(where) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return CONV2D_ERR_CUDA;
}

bool shape_of(const conv2d_params_t* p, Problem* out, std::string* why) {
  if (!p) {
    *why = "params is NULL";
    return false;
  }
  if (p->batch < 1 || p->in_rows < 1 || p->in_cols < 1 || p->channels < 1 || p->features < 1 ||
      p->window_rows < 1 || p->window_cols < 1 || p->stride_rows < 1 || p->stride_cols < 1) {
    *why = "every dimension, window and stride must be >= 1";
    return false;
  }
  if (p->math != CONV2D_MATH_FP32 && p->math != CONV2D_MATH_TF32) {
    *why = "unknown math mode";
    return false;
  }
  Problem q{};
  q.N = p->batch; q.H = p->in_rows; q.W = p->in_cols; q.C = p->channels; q.F = p->features;
  q.KH = p->window_rows; q.KW = p->window_cols; q.SH = p->stride_rows; q.SW = p->stride_cols;
  q.math = p->math;
  // SPEC.md:48-56 shape algebra (reading R3: SAME pads floor-before / rest-after)
  if (p->padding == CONV2D_PAD_SAME) {
    q.HO = (q.H + q.SH - 1) / q.SH;
    q.WO = (q.W + q.SW - 1) / q.SW;
    const int64_t tr = std::max<int64_t>((int64_t)(q.HO - 1) * q.SH + q.KH - q.H, 0);
    const int64_t tc = std::max<int64_t>((int64_t)(q.WO - 1) * q.SW + q.KW - q.W, 0);
    q.pad_top = (int)(tr / 2);
    q.pad_left = (int)(tc / 2);
  } else if (p->padding == CONV2D_PAD_VALID) {
    if (q.KH > q.H || q.KW > q.W) {
      *why = "VALID padding requires window <= input extent";
      return false;
    }
    q.HO = (q.H - q.KH) / q.SH + 1;
    q.WO = (q.W - q.KW) / q.SW + 1;
    q.pad_top = q.pad_left = 0;
  } else {
    *why = "unknown padding mode";
    return false;
  }
  // overflow / index-width guard (reading R20): GEMM rows fit int32 tiles, sizes fit 2^40 elements
  const int64_t lim = int64_t(1) << 40;
  if (q.M() > INT_MAX - 256 || q.in_elems() > lim || q.out_elems() > lim || q.filt_elems() > lim ||
      q.K() > INT_MAX / 2) {
    *why = "tensor too large (element count overflow guard)";
    return false;
  }
  *out = q;
  return true;
}

bool algo_supports(const Problem& q, conv2d_algo_t a) {
  switch (a) {
    case CONV2D_ALGO_AUTO:
    case CONV2D_ALGO_DIRECT:
    case CONV2D_ALGO_IMPLICIT_GEMM:
      return true;
    case CONV2D_ALGO_TILED:
      return tiled_supported(q);
    case CONV2D_ALGO_MATMUL_1X1:
      return q.KH == 1 && q.KW == 1 && q.SH == 1 && q.SW == 1;
    case CONV2D_ALGO_WINOGRAD_F2X2_3X3:
      return q.KH == 3 && q.KW == 3 && q.SH == 1 && q.SW == 1 && q.C >= 32;
    case CONV2D_ALGO_WINOGRAD_F4X4_3X3:  // FP32 math only (reading R21)
      return q.KH == 3 && q.KW == 3 && q.SH == 1 && q.SW == 1 && q.C >= 32 && q.math == CONV2D_MATH_FP32;
  }
  return false;
}

size_t algo_workspace(const Problem& q, conv2d_algo_t a) {
  switch (a) {
    case CONV2D_ALGO_IMPLICIT_GEMM: return igemm_workspace(q, false);
    case CONV2D_ALGO_MATMUL_1X1: return igemm_workspace(q, true);
    case CONV2D_ALGO_WINOGRAD_F2X2_3X3: return winograd_workspace(q, 2);
    case CONV2D_ALGO_WINOGRAD_F4X4_3X3: return winograd_workspace(q, 4);
    default: return 0;
  }
}

int algo_launches(const Problem& q, conv2d_algo_t a) {
  switch (a) {
    case CONV2D_ALGO_DIRECT:
    case CONV2D_ALGO_TILED: return 1;
    case CONV2D_ALGO_IMPLICIT_GEMM: return igemm_launches(q, false);
    case CONV2D_ALGO_MATMUL_1X1: return igemm_launches(q, true);
    case CONV2D_ALGO_WINOGRAD_F2X2_3X3: return winograd_launches(q, 2);
    case CONV2D_ALGO_WINOGRAD_F4X4_3X3: return winograd_launches(q, 4);
    default: return -1;
  }
}

// ---- tuned parameter variants ("different parameters for each algorithm"):
// implicit_gemm / matmul_1x1 (igemm.cu: A path, N tile, B path, K split) and winograd_f2x2_3x3 (winograd.cu:
// 0 = transforms + batched GEMM, 1 = the fused kernel of wino_fused.cu)
bool has_variants(conv2d_algo_t a) {
  return a == CONV2D_ALGO_IMPLICIT_GEMM || a == CONV2D_ALGO_MATMUL_1X1 || a == CONV2D_ALGO_WINOGRAD_F2X2_3X3;
}
int algo_variants(const Problem& q, conv2d_algo_t a, int* masks) {
  if (a == CONV2D_ALGO_WINOGRAD_F2X2_3X3) return winograd_variants(q, masks);
  if (a == CONV2D_ALGO_IMPLICIT_GEMM || a == CONV2D_ALGO_MATMUL_1X1)
    return igemm_variants(q, a == CONV2D_ALGO_MATMUL_1X1, masks);
  masks[0] = 0;
  return 1;
}
void algo_set_variant(const Problem& q, conv2d_algo_t a, int v) {
  if (a == CONV2D_ALGO_WINOGRAD_F2X2_3X3) winograd_set_variant(q, v);
  else if (a == CONV2D_ALGO_IMPLICIT_GEMM || a == CONV2D_ALGO_MATMUL_1X1)
    igemm_set_variant(q, a == CONV2D_ALGO_MATMUL_1X1, v);
}
bool algo_get_variant(const Problem& q, conv2d_algo_t a, int* v) {
  if (a == CONV2D_ALGO_WINOGRAD_F2X2_3X3) return winograd_get_variant(q, v);
  if (a == CONV2D_ALGO_IMPLICIT_GEMM || a == CONV2D_ALGO_MATMUL_1X1)
    return igemm_get_variant(q, a == CONV2D_ALGO_MATMUL_1X1, v);
  return false;
}

// ---- device check (sm_100 only: the kernels are built for sm_100a exclusively)
std::mutex g_dev_mu;
std::map<int, bool> g_dev_ok;

conv2d_status_t check_device(int* dev_out) {
  int dev = -1;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  std::lock_guard<std::mutex> lk(g_dev_mu);
  auto it = g_dev_ok.find(dev);
  if (it == g_dev_ok.end()) {
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    it = g_dev_ok.emplace(dev, major == 10 && minor == 0).first;
  }
  if (!it->second) return fail(CONV2D_ERR_NO_DEVICE, "current device is not sm_100 (B200)");
  if (dev_out) *dev_out = dev;
  return CONV2D_OK;
}

// ---- selector cache: key = all params + device
using Key = std::tuple<int, int, int, int, int, int, int, int, int, int, int, int>;
Key key_of(const conv2d_params_t* p, int dev) {
  return Key(p->batch, p->in_rows, p->in_cols, p->channels, p->features, p->window_rows, p->window_cols,
             p->stride_rows, p->stride_cols, (int)p->padding, (int)p->math, dev);
}
std::mutex g_cache_mu;
std::map<Key, conv2d_algo_t> g_cache;

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

conv2d_status_t run_algo(const Problem& q, conv2d_algo_t a, const float* in, const float* filt, float* out, void* ws,
                         cudaStream_t s) {
  cudaError_t e = cudaSuccess;
  struct PdlHint {  // launch.cuh: programmatic dependent launch for small convs
    explicit PdlHint(bool on) { t_pdl_hint = on; }
    ~PdlHint() { t_pdl_hint = false; }
  } hint(2.0 * (double)q.M() * q.F * (double)q.K() <= 8e9 &&
         ((q.M() + 255) / 256) * ((q.F + (q.F <= 64 ? 63 : q.F <= 128 ? 127 : 255)) / (q.F <= 64 ? 64 : q.F <= 128 ? 128 : 256)) <= 2048);
  switch (a) {
    case CONV2D_ALGO_DIRECT: e = launch_direct(q, in, filt, out, s); break;
    case CONV2D_ALGO_TILED: e = launch_tiled(q, in, filt, out, s); break;
    case CONV2D_ALGO_IMPLICIT_GEMM: e = launch_igemm(q, false, in, filt, out, ws, s); break;
    case CONV2D_ALGO_MATMUL_1X1: e = launch_igemm(q, true, in, filt, out, ws, s); break;
    case CONV2D_ALGO_WINOGRAD_F2X2_3X3: e = launch_winograd(q, 2, in, filt, out, ws, s); break;
    case CONV2D_ALGO_WINOGRAD_F4X4_3X3: e = launch_winograd(q, 4, in, filt, out, ws, s); break;
    default: return fail(CONV2D_ERR_UNSUPPORTED, "no algorithm to run");
  }
  if (e != cudaSuccess) return cuda_fail(e, conv2d_algo_name(a));
  return CONV2D_OK;
}

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  if (!v || !*v) return dflt;
  return atoi(v);
}

// caller-owned scratch the auto-selector overwrites before every timed repetition (conv2d_set_autotune_flush)
std::mutex g_flush_mu;
void* g_flush_buf = nullptr;
size_t g_flush_bytes = 0;

// learned-selector ranking (defined with the selector below): the first `k` runnable (algorithm, variant)
// candidates for q in order of predicted log-regret; returns how many were written
int selector_topk(const conv2d_params_t* p, const Problem& q, int k, int* algos, int* variants);
int auto_policy();

conv2d_status_t autotune_impl(const conv2d_params_t* p, const Problem& q, int dev, const float* in, const float* filt,
                              float* out, void* ws, cudaStream_t s, conv2d_algo_t* chosen) {
  const int warm = std::max(1, env_int("CONV2D_AUTOTUNE_WARMUPS", 2));
  const int reps = std::max(1, env_int("CONV2D_AUTOTUNE_REPS", 5));
  void* flush = nullptr;
  size_t flush_bytes = 0;
  {
    std::lock_guard<std::mutex> lk(g_flush_mu);
    flush = g_flush_buf;
    flush_bytes = g_flush_bytes;
  }
  for (int i = 0; i < CONV2D_NUM_ALGOS; ++i) g_tune_times[i] = -1.0;
  bool failed_any = false;
  cudaEvent_t e0, e1;
  cudaError_t ce = cudaEventCreate(&e0);
  if (ce != cudaSuccess) return cuda_fail(ce, "cudaEventCreate");
  ce = cudaEventCreate(&e1);
  if (ce != cudaSuccess) {
    cudaEventDestroy(e0);
    return cuda_fail(ce, "cudaEventCreate");
  }
  conv2d_algo_t best = CONV2D_ALGO_AUTO;
  double best_t = 1e300;
  conv2d_status_t st = CONV2D_OK;
  // CONV2D_AUTO_HYBRID: time only the learned selector's top candidates (default 3)
  int top_a[32], top_v[32], ntop = 0;
  const bool hybrid = auto_policy() == CONV2D_AUTO_HYBRID;
  if (hybrid) ntop = selector_topk(p, q, std::min(32, std::max(1, env_int("CONV2D_HYBRID_TOPK", 3))), top_a, top_v);
  auto measured = [&](int a, int v) {
    if (!hybrid) return true;
    for (int i = 0; i < ntop; ++i)
      if (top_a[i] == a && top_v[i] == v) return true;
    return false;
  };
  for (int ai = 1; ai < CONV2D_NUM_ALGOS && st == CONV2D_OK; ++ai) {
    const conv2d_algo_t a = (conv2d_algo_t)ai;
    if (!algo_supports(q, a)) continue;
    // algorithm parameters: time every variant of the algorithm, keep its best
    const bool tuned = has_variants(a);
    int masks[32] = {0};
    const int nvar = algo_variants(q, a, masks);
    double t_best = 1e300;
    int v_best = 0;
    for (int vi = 0; vi < nvar && st == CONV2D_OK; ++vi) {
      const int v = masks[vi];
      if (!measured(ai, v)) continue;
      if (tuned) algo_set_variant(q, a, v);
      st = run_algo(q, a, in, filt, out, ws, s);
      if (st == CONV2D_ERR_CUDA) {
        // a measurement failure drops that candidate and logs a warning.  Only a launch that
        // was refused (non-sticky: the stream still synchronises cleanly) is skipped; a fault that
        // poisoned the context is returned to the caller.
        const std::string why = g_last_error;
        cudaGetLastError();
        if (cudaStreamSynchronize(s) != cudaSuccess) break;
        fprintf(stderr, "[conv2d] autotune: %s variant %d failed to launch (%s); candidate dropped\n",
                conv2d_algo_name(a), v, why.c_str());
        failed_any = true;
        st = CONV2D_OK;
        continue;
      }
      for (int w = 1; w < warm && st == CONV2D_OK; ++w) st = run_algo(q, a, in, filt, out, ws, s);
      for (int r = 0; r < reps && st == CONV2D_OK; ++r) {
        if (flush) {  // cache-cold repetition: evict L2 outside the timed events
          ce = cudaMemsetAsync(flush, r & 0xFF, flush_bytes, s);
          if (ce != cudaSuccess) {
            st = cuda_fail(ce, "autotune flush");
            break;
          }
        }
        cudaEventRecord(e0, s);
        st = run_algo(q, a, in, filt, out, ws, s);
        cudaEventRecord(e1, s);
        ce = cudaEventSynchronize(e1);
        if (ce != cudaSuccess) {
          st = cuda_fail(ce, "autotune sync");
          break;
        }
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < t_best) {
          t_best = ms;
          v_best = v;
        }
      }
    }
    if (st != CONV2D_OK) break;
    if (t_best >= 1e299) continue;  // hybrid: no variant of this algorithm was timed
    if (tuned) algo_set_variant(q, a, v_best);
    g_tune_times[ai] = t_best * 1000.0;
    if (t_best < best_t) {  // strict: ties keep the earlier enum
      best_t = t_best;
      best = a;
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (st != CONV2D_OK) return st;
  if (best == CONV2D_ALGO_AUTO)
    return fail(CONV2D_ERR_CUDA, failed_any ? "autotune: every candidate failed to launch" : "autotune: no candidate");
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    g_cache[key_of(p, dev)] = best;
  }
  if (chosen) *chosen = best;
  return CONV2D_OK;
}

size_t auto_workspace(const Problem& q) {
  size_t m = 0;
  for (int ai = 1; ai < CONV2D_NUM_ALGOS; ++ai)
    if (algo_supports(q, (conv2d_algo_t)ai)) m = std::max(m, algo_workspace(q, (conv2d_algo_t)ai));
  return m;
}

bool valid_algo(conv2d_algo_t a) { return (int)a >= 0 && (int)a < CONV2D_NUM_ALGOS; }

}  // namespace

// ---- learned selector: evaluation of the tree in selector_tree.h.
// Features in the order of tools/train_selector.py FEATURES (the two must stay in step; a CPU test walks the
// exported tree in Python with that script's features and compares with conv2d_predict).
static void selector_features(const conv2d_params_t* p, const Problem& q, double x[selector::kFeatures]) {
  const double m = (double)q.N * q.HO * q.WO;
  const double kk = (double)q.KH * q.KW * q.C;
  const int bn = q.F <= 64 ? 64 : q.F <= 128 ? 128 : 256;
  const double tiles = std::ceil(m / 256.0) * std::ceil((double)q.F / bn);
  const double flops = 2.0 * m * q.F * kk;
  const double bytes = 4.0 * ((double)q.N * q.H * q.W * q.C + kk * q.F + m * q.F);
  const double f[selector::kFeatures] = {std::log2(m), std::log2((double)q.F), std::log2((double)q.C), std::log2(kk),
                                         (double)q.KH, (double)q.SH, p->padding == CONV2D_PAD_VALID ? 1.0 : 0.0,
                                         std::log2((double)q.N), std::log2((double)q.HO * q.WO),
                                         q.math == CONV2D_MATH_TF32 ? 1.0 : 0.0, std::log2(tiles), std::log2(flops),
                                         flops / bytes};
  for (int i = 0; i < selector::kFeatures; ++i) x[i] = f[i];
}

static bool variant_enumerated(const Problem& q, conv2d_algo_t a, int v) {
  int masks[32];
  const int n = algo_variants(q, a, masks);
  for (int i = 0; i < n; ++i)
    if (masks[i] == v) return true;
  return false;
}

// the supported candidate of least predicted log-regret at the shape's leaf (fallback: implicit_gemm/0)
static std::atomic<int> g_auto_policy{CONV2D_AUTO_MEASURE};

namespace {
int auto_policy() { return g_auto_policy.load(); }

int selector_topk(const conv2d_params_t* p, const Problem& q, int k, int* algos, int* variants) {
  double x[selector::kFeatures];
  selector_features(p, q, x);
  int node = 0;
  while (selector::kFeature[node] >= 0)
    node = x[selector::kFeature[node]] <= selector::kThreshold[node] ? selector::kLeft[node] : selector::kRight[node];
  const float* lr = selector::kLogRegret[selector::kLeafRow[node]];
  int order[selector::kClasses];
  for (int i = 0; i < selector::kClasses; ++i) order[i] = i;
  std::stable_sort(order, order + selector::kClasses, [&](int a, int b) { return lr[a] < lr[b]; });
  int n = 0;
  for (int i = 0; i < selector::kClasses && n < k; ++i) {
    const conv2d_algo_t a = (conv2d_algo_t)selector::kClassAlgo[order[i]];
    const int v = selector::kClassVariant[order[i]];
    if (algo_supports(q, a) && variant_enumerated(q, a, v)) {
      algos[n] = a;
      variants[n] = v;
      ++n;
    }
  }
  if (n == 0) {  // nothing runnable ranked: implicit_gemm / 0 always is
    algos[0] = CONV2D_ALGO_IMPLICIT_GEMM;
    variants[0] = 0;
    n = 1;
  }
  return n;
}
}  // namespace

static void selector_predict(const conv2d_params_t* p, const Problem& q, conv2d_algo_t* algo, int* variant) {
  int a = 0, v = 0;
  selector_topk(p, q, 1, &a, &v);
  *algo = (conv2d_algo_t)a;
  *variant = v;
}

extern "C" {

conv2d_status_t conv2d_output_shape(const conv2d_params_t* p, int32_t out_nhwf[4], int32_t pads_tblr[4]) {
  Problem q;
  std::string why;
  if (!shape_of(p, &q, &why)) return fail(CONV2D_ERR_INVALID_PARAMS, why);
  if (out_nhwf) {
    out_nhwf[0] = q.N; out_nhwf[1] = q.HO; out_nhwf[2] = q.WO; out_nhwf[3] = q.F;
  }
  if (pads_tblr) {
    const int tr = std::max((q.HO - 1) * q.SH + q.KH - q.H, 0);
    const int tc = std::max((q.WO - 1) * q.SW + q.KW - q.W, 0);
    if (p->padding == CONV2D_PAD_VALID) {
      pads_tblr[0] = pads_tblr[1] = pads_tblr[2] = pads_tblr[3] = 0;
    } else {
      pads_tblr[0] = q.pad_top; pads_tblr[1] = tr - q.pad_top;
      pads_tblr[2] = q.pad_left; pads_tblr[3] = tc - q.pad_left;
    }
  }
  return CONV2D_OK;
}

conv2d_status_t conv2d_flop_count(const conv2d_params_t* p, uint64_t* flops) {
  Problem q;
  std::string why;
  if (!flops) return fail(CONV2D_ERR_NULL, "flops is NULL");
  if (!shape_of(p, &q, &why)) return fail(CONV2D_ERR_INVALID_PARAMS, why);
  *flops = 2ull * (uint64_t)q.M() * (uint64_t)q.K() * (uint64_t)q.F;
  return CONV2D_OK;
}

conv2d_status_t conv2d_supports(const conv2d_params_t* p, conv2d_algo_t algo, int* supported) {
  Problem q;
  std::string why;
  if (!supported) return fail(CONV2D_ERR_NULL, "supported is NULL");
  if (!shape_of(p, &q, &why)) return fail(CONV2D_ERR_INVALID_PARAMS, why);
  if (!valid_algo(algo)) return fail(CONV2D_ERR_INVALID_PARAMS, "unknown algorithm");
  *supported = algo_supports(q, algo) ? 1 : 0;
  return CONV2D_OK;
}

conv2d_status_t conv2d_query_workspace(const conv2d_params_t* p, conv2d_algo_t algo, size_t* bytes) {
  Problem q;
  std::string why;
  if (!bytes) return fail(CONV2D_ERR_NULL, "bytes is NULL");
  if (!shape_of(p, &q, &why)) return fail(CONV2D_ERR_INVALID_PARAMS, why);
  if (!valid_algo(algo)) return fail(CONV2D_ERR_INVALID_PARAMS, "unknown algorithm");
  if (!algo_supports(q, algo)) return fail(CONV2D_ERR_UNSUPPORTED, "algorithm does not support these params");
  *bytes = algo == CONV2D_ALGO_AUTO ? auto_workspace(q) : algo_workspace(q, algo);
  return CONV2D_OK;
}

static conv2d_status_t validate_call(const conv2d_params_t* p, conv2d_algo_t algo, const float* in, const float* filt,
                                     float* out, void* ws, size_t ws_bytes, Problem* q) {
  std::string why;
  if (!shape_of(p, q, &why)) return fail(CONV2D_ERR_INVALID_PARAMS, why);
  if (!valid_algo(algo)) return fail(CONV2D_ERR_INVALID_PARAMS, "unknown algorithm");
  if (!algo_supports(*q, algo))
    return fail(CONV2D_ERR_UNSUPPORTED, std::string(conv2d_algo_name(algo)) + " does not support these params");
  if (!in || !filt || !out) return fail(CONV2D_ERR_NULL, "in/filt/out must be non-NULL device pointers");
  if (!aligned16(in) || !aligned16(filt) || !aligned16(out) || (ws && !aligned16(ws)))
    return fail(CONV2D_ERR_ALIGNMENT, "device pointers must be 16-byte aligned");
  const size_t need = algo == CONV2D_ALGO_AUTO ? auto_workspace(*q) : algo_workspace(*q, algo);
  if (need > 0 && (!ws || ws_bytes < need))
    return fail(CONV2D_ERR_WORKSPACE, "workspace too small: need " + std::to_string(need) + " bytes");
  return CONV2D_OK;
}

static conv2d_status_t refuse_if_capturing(cudaStream_t s);

conv2d_status_t conv2d_forward(const conv2d_params_t* p, conv2d_algo_t algo, const float* in, const float* filt,
                               float* out, void* ws, size_t ws_bytes, void* stream) {
  Problem q;
  conv2d_status_t st = validate_call(p, algo, in, filt, out, ws, ws_bytes, &q);
  if (st != CONV2D_OK) return st;
  int dev = -1;
  st = check_device(&dev);
  if (st != CONV2D_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  conv2d_algo_t a = algo;
  if (a == CONV2D_ALGO_AUTO) {
    bool hit = false;
    {
      std::lock_guard<std::mutex> lk(g_cache_mu);
      auto it = g_cache.find(key_of(p, dev));
      if (it != g_cache.end()) {
        a = it->second;
        hit = true;
      }
    }
    if (!hit && g_auto_policy.load() == CONV2D_AUTO_PREDICT) {  // learned choice: no timing, capture-safe
      int v = 0;
      selector_predict(p, q, &a, &v);
      algo_set_variant(q, a, v);
      std::lock_guard<std::mutex> lk(g_cache_mu);
      g_cache[key_of(p, dev)] = a;
    } else if (!hit) {
      st = refuse_if_capturing(s);
      if (st != CONV2D_OK) return st;
      st = autotune_impl(p, q, dev, in, filt, out, ws, s, &a);
      if (st != CONV2D_OK) return st;
    }
  }
  return run_algo(q, a, in, filt, out, ws, s);
}

// Tuning times and synchronises the stream, which a stream capture forbids (and the failed call would
// invalidate the caller's capture): refuse up front instead.
static conv2d_status_t refuse_if_capturing(cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone)
    return fail(CONV2D_ERR_UNSUPPORTED,
                "auto-selection needs a cached choice while the stream is being captured: tune first "
                "(conv2d_autotune / conv2d_load_selection / conv2d_set_selected)");
  return CONV2D_OK;
}

conv2d_status_t conv2d_autotune(const conv2d_params_t* p, const float* in, const float* filt, float* out, void* ws,
                                size_t ws_bytes, void* stream, conv2d_algo_t* chosen) {
  Problem q;
  conv2d_status_t st = validate_call(p, CONV2D_ALGO_AUTO, in, filt, out, ws, ws_bytes, &q);
  if (st != CONV2D_OK) return st;
  int dev = -1;
  st = check_device(&dev);
  if (st != CONV2D_OK) return st;
  st = refuse_if_capturing(static_cast<cudaStream_t>(stream));
  if (st != CONV2D_OK) return st;
  return autotune_impl(p, q, dev, in, filt, out, ws, static_cast<cudaStream_t>(stream), chosen);
}

conv2d_status_t conv2d_selected(const conv2d_params_t* p, conv2d_algo_t* chosen) {
  Problem q;
  std::string why;
  if (!chosen) return fail(CONV2D_ERR_NULL, "chosen is NULL");
  *chosen = CONV2D_ALGO_AUTO;
  if (!shape_of(p, &q, &why)) return fail(CONV2D_ERR_INVALID_PARAMS, why);
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  std::lock_guard<std::mutex> lk(g_cache_mu);
  auto it = g_cache.find(key_of(p, dev));
  if (it == g_cache.end()) return fail(CONV2D_ERR_UNSUPPORTED, "not cached");
  *chosen = it->second;
  return CONV2D_OK;
}

conv2d_status_t conv2d_set_selected(const conv2d_params_t* p, conv2d_algo_t algo) {
  Problem q;
  std::string why;
  if (!shape_of(p, &q, &why)) return fail(CONV2D_ERR_INVALID_PARAMS, why);
  if (!valid_algo(algo) || algo == CONV2D_ALGO_AUTO) return fail(CONV2D_ERR_INVALID_PARAMS, "need a concrete algorithm");
  if (!algo_supports(q, algo)) return fail(CONV2D_ERR_UNSUPPORTED, "algorithm does not support these params");
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  std::lock_guard<std::mutex> lk(g_cache_mu);
  g_cache[key_of(p, dev)] = algo;
  return CONV2D_OK;
}

static conv2d_status_t variant_problem(const conv2d_params_t* p, conv2d_algo_t algo, Problem* q) {
  std::string why;
  if (!shape_of(p, q, &why)) return fail(CONV2D_ERR_INVALID_PARAMS, why);
  if (!has_variants(algo))
    return fail(CONV2D_ERR_INVALID_PARAMS, "variants exist for implicit_gemm / matmul_1x1 / winograd_f2x2_3x3 only");
  if (!algo_supports(*q, algo)) return fail(CONV2D_ERR_UNSUPPORTED, "algorithm does not support these params");
  return CONV2D_OK;
}

conv2d_status_t conv2d_get_variant(const conv2d_params_t* p, conv2d_algo_t algo, int* variant) {
  if (!variant) return fail(CONV2D_ERR_NULL, "variant is NULL");
  *variant = 0;
  Problem q;
  const conv2d_status_t st = variant_problem(p, algo, &q);
  if (st != CONV2D_OK) return st;
  int v = 0;
  if (algo_get_variant(q, algo, &v)) *variant = v;
  return CONV2D_OK;
}

conv2d_status_t conv2d_set_variant(const conv2d_params_t* p, conv2d_algo_t algo, int variant) {
  Problem q;
  const conv2d_status_t st = variant_problem(p, algo, &q);
  if (st != CONV2D_OK) return st;
  int masks[32];
  const int n = algo_variants(q, algo, masks);
  for (int i = 0; i < n; ++i)
    if (masks[i] == variant) {
      algo_set_variant(q, algo, variant);
      return CONV2D_OK;
    }
  return fail(CONV2D_ERR_INVALID_PARAMS, "variant " + std::to_string(variant) + " is not enumerated for these params");
}

conv2d_status_t conv2d_predict(const conv2d_params_t* p, conv2d_algo_t* algo, int* variant) {
  if (!algo || !variant) return fail(CONV2D_ERR_NULL, "algo / variant is NULL");
  Problem q;
  std::string why;
  if (!shape_of(p, &q, &why)) return fail(CONV2D_ERR_INVALID_PARAMS, why);
  selector_predict(p, q, algo, variant);
  return CONV2D_OK;
}

conv2d_status_t conv2d_set_auto_policy(conv2d_auto_policy_t policy) {
  if (policy != CONV2D_AUTO_MEASURE && policy != CONV2D_AUTO_PREDICT && policy != CONV2D_AUTO_HYBRID)
    return fail(CONV2D_ERR_INVALID_PARAMS, "unknown auto policy");
  g_auto_policy.store(policy);
  return CONV2D_OK;
}

// ---- persisted selector table (SPEC.md:354's line format, with the full key of this library's cache)
//   N H W C F KH KW SH SW same|valid fp32|tf32 : algo[/variant]
//   default : algo,algo,...        (ranking by win count over the entries; informative)
conv2d_status_t conv2d_save_selection(const char* path) {
  if (!path) return fail(CONV2D_ERR_NULL, "path is NULL");
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  std::vector<std::pair<Key, conv2d_algo_t>> rows;
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    for (const auto& kv : g_cache)
      if (std::get<11>(kv.first) == dev) rows.push_back(kv);
  }
  FILE* f = fopen(path, "w");
  if (!f) return fail(CONV2D_ERR_IO, std::string("cannot open for writing: ") + path);
  fprintf(f, "# conv2d selection table v1: N H W C F KH KW SH SW padding math : algorithm[/variant]\n");
  int wins[CONV2D_NUM_ALGOS] = {0};
  for (const auto& kv : rows) {
    const Key& k = kv.first;
    conv2d_params_t p{std::get<0>(k), std::get<1>(k), std::get<2>(k), std::get<3>(k), std::get<4>(k), std::get<5>(k),
                      std::get<6>(k), std::get<7>(k), std::get<8>(k), (conv2d_padding_t)std::get<9>(k),
                      (conv2d_math_t)std::get<10>(k)};
    fprintf(f, "%d %d %d %d %d %d %d %d %d %s %s : %s", p.batch, p.in_rows, p.in_cols, p.channels, p.features,
            p.window_rows, p.window_cols, p.stride_rows, p.stride_cols, p.padding == CONV2D_PAD_SAME ? "same" : "valid",
            p.math == CONV2D_MATH_FP32 ? "fp32" : "tf32", conv2d_algo_name(kv.second));
    Problem q;
    std::string why;
    int v = 0;
    if (has_variants(kv.second) && shape_of(&p, &q, &why) && algo_get_variant(q, kv.second, &v))
      fprintf(f, "/%d", v);
    fprintf(f, "\n");
    ++wins[kv.second];
  }
  fprintf(f, "default :");
  bool used[CONV2D_NUM_ALGOS] = {false};
  for (int n = 0, first = 1; n < CONV2D_NUM_ALGOS - 1; ++n) {
    int best = -1;
    for (int a = 1; a < CONV2D_NUM_ALGOS; ++a)  // most wins first, ties in enum order
      if (!used[a] && (best < 0 || wins[a] > wins[best])) best = a;
    used[best] = true;
    fprintf(f, "%s%s", first ? " " : ",", conv2d_algo_name((conv2d_algo_t)best));
    first = 0;
  }
  fprintf(f, "\n");
  const bool ok = fclose(f) == 0;
  return ok ? CONV2D_OK : fail(CONV2D_ERR_IO, std::string("write failed: ") + path);
}

conv2d_status_t conv2d_load_selection(const char* path, int* loaded) {
  if (!path) return fail(CONV2D_ERR_NULL, "path is NULL");
  if (loaded) *loaded = 0;
  FILE* f = fopen(path, "r");
  if (!f) return fail(CONV2D_ERR_IO, std::string("cannot open: ") + path);
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  struct Entry {
    conv2d_params_t p;
    conv2d_algo_t a;
    int variant;
  };
  std::vector<Entry> entries;
  char line[512];
  int lineno = 0;
  conv2d_status_t st = CONV2D_OK;
  std::string why;
  auto algo_by_name = [](const std::string& n) -> int {
    for (int a = 1; a < CONV2D_NUM_ALGOS; ++a)
      if (n == conv2d_algo_name((conv2d_algo_t)a)) return a;
    return -1;
  };
  while (st == CONV2D_OK && fgets(line, sizeof line, f)) {
    ++lineno;
    std::string l(line);
    const size_t hash = l.find('#');
    if (hash != std::string::npos) l.erase(hash);
    while (!l.empty() && isspace((unsigned char)l.back())) l.pop_back();
    size_t b = 0;
    while (b < l.size() && isspace((unsigned char)l[b])) ++b;
    l.erase(0, b);
    if (l.empty()) continue;
    const size_t colon = l.find(':');
    if (colon == std::string::npos) {
      st = CONV2D_ERR_INVALID_PARAMS;
      why = "missing ':'";
      break;
    }
    std::string lhs = l.substr(0, colon), rhs = l.substr(colon + 1);
    while (!rhs.empty() && isspace((unsigned char)rhs.front())) rhs.erase(0, 1);
    while (!lhs.empty() && isspace((unsigned char)lhs.back())) lhs.pop_back();
    if (lhs == "default") {  // validate the ranking; it is informative only
      size_t pos = 0;
      while (pos <= rhs.size()) {
        const size_t c = rhs.find(',', pos);
        std::string n = rhs.substr(pos, c == std::string::npos ? std::string::npos : c - pos);
        while (!n.empty() && isspace((unsigned char)n.back())) n.pop_back();
        while (!n.empty() && isspace((unsigned char)n.front())) n.erase(0, 1);
        if (algo_by_name(n) < 0) {
          st = CONV2D_ERR_INVALID_PARAMS;
          why = "unknown algorithm '" + n + "' in default ranking";
          break;
        }
        if (c == std::string::npos) break;
        pos = c + 1;
      }
      continue;
    }
    Entry e{};
    char pad[16] = {0}, math[16] = {0};
    int extra = 0;
    const int got = sscanf(lhs.c_str(), "%d %d %d %d %d %d %d %d %d %15s %15s %n", &e.p.batch, &e.p.in_rows,
                           &e.p.in_cols, &e.p.channels, &e.p.features, &e.p.window_rows, &e.p.window_cols,
                           &e.p.stride_rows, &e.p.stride_cols, pad, math, &extra);
    if (got != 11 || (size_t)extra != lhs.size()) {
      st = CONV2D_ERR_INVALID_PARAMS;
      why = "expected 'N H W C F KH KW SH SW padding math'";
      break;
    }
    const std::string ps(pad), ms(math);
    if ((ps != "same" && ps != "valid") || (ms != "fp32" && ms != "tf32")) {
      st = CONV2D_ERR_INVALID_PARAMS;
      why = "padding must be same|valid and math fp32|tf32";
      break;
    }
    e.p.padding = ps == "same" ? CONV2D_PAD_SAME : CONV2D_PAD_VALID;
    e.p.math = ms == "fp32" ? CONV2D_MATH_FP32 : CONV2D_MATH_TF32;
    e.variant = -1;
    std::string an = rhs;
    const size_t slash = rhs.find('/');
    if (slash != std::string::npos) {
      an = rhs.substr(0, slash);
      char* end = nullptr;
      const long v = strtol(rhs.c_str() + slash + 1, &end, 10);
      if (!end || *end != '\0' || v < 0 || v > 31) {
        st = CONV2D_ERR_INVALID_PARAMS;
        why = "bad variant";
        break;
      }
      e.variant = (int)v;
    }
    const int a = algo_by_name(an);
    if (a < 0) {
      st = CONV2D_ERR_INVALID_PARAMS;
      why = "unknown algorithm '" + an + "'";
      break;
    }
    e.a = (conv2d_algo_t)a;
    Problem q;
    std::string w;
    if (!shape_of(&e.p, &q, &w)) {
      st = CONV2D_ERR_INVALID_PARAMS;
      why = w;
      break;
    }
    if (!algo_supports(q, e.a)) {
      st = CONV2D_ERR_UNSUPPORTED;
      why = std::string(conv2d_algo_name(e.a)) + " does not support these params";
      break;
    }
    if (e.variant >= 0 && !has_variants(e.a)) {
      st = CONV2D_ERR_INVALID_PARAMS;
      why = "a variant is only defined for implicit_gemm / matmul_1x1 / winograd_f2x2_3x3";
      break;
    }
    if (e.variant >= 0) {  // only the variants the auto-selector enumerates for these params (as set_variant)
      int masks[32];
      const int n = algo_variants(q, e.a, masks);
      bool found = false;
      for (int i = 0; i < n; ++i) found = found || masks[i] == e.variant;
      if (!found) {
        st = CONV2D_ERR_INVALID_PARAMS;
        why = "variant " + std::to_string(e.variant) + " is not enumerated for these params";
        break;
      }
    }
    entries.push_back(e);
  }
  fclose(f);
  if (st != CONV2D_OK) return fail(st, std::string(path) + ":" + std::to_string(lineno) + ": " + why);
  {  // all lines valid: apply (an invalid file leaves the cache untouched)
    std::lock_guard<std::mutex> lk(g_cache_mu);
    for (const auto& e : entries) g_cache[key_of(&e.p, dev)] = e.a;
  }
  for (const auto& e : entries)
    if (e.variant >= 0) {
      Problem q;
      std::string w;
      shape_of(&e.p, &q, &w);
      algo_set_variant(q, e.a, e.variant);
    }
  if (loaded) *loaded = (int)entries.size();
  return CONV2D_OK;
}

conv2d_status_t conv2d_set_autotune_flush(void* buf, size_t bytes) {
  if (buf && bytes == 0) return fail(CONV2D_ERR_INVALID_PARAMS, "flush buffer of 0 bytes");
  std::lock_guard<std::mutex> lk(g_flush_mu);
  g_flush_buf = buf;
  g_flush_bytes = buf ? bytes : 0;
  return CONV2D_OK;
}

void conv2d_clear_selection_cache(void) {
  std::lock_guard<std::mutex> lk(g_cache_mu);
  g_cache.clear();
}

void conv2d_last_tune_times(double times_us[CONV2D_NUM_ALGOS]) {
  if (!times_us) return;
  for (int i = 0; i < CONV2D_NUM_ALGOS; ++i) times_us[i] = g_tune_times[i];
}

int conv2d_launch_count(const conv2d_params_t* p, conv2d_algo_t algo) {
  Problem q;
  std::string why;
  if (!shape_of(p, &q, &why) || !valid_algo(algo)) return -1;
  if (algo == CONV2D_ALGO_AUTO) {
    conv2d_algo_t a;
    if (conv2d_selected(p, &a) != CONV2D_OK) return -1;
    algo = a;
  }
  if (!algo_supports(q, algo)) return -1;
  return algo_launches(q, algo);
}

conv2d_status_t conv2d_synth_fill(float* dst, uint64_t count, uint64_t key, uint64_t offset, int dist, void* stream) {
  if (!dst && count) return fail(CONV2D_ERR_NULL, "dst is NULL");
  if (dist != 0 && dist != 1) return fail(CONV2D_ERR_INVALID_PARAMS, "dist must be 0 or 1");
  conv2d_status_t st = check_device(nullptr);
  if (st != CONV2D_OK) return st;
  cudaError_t e = launch_synth_fill(dst, count, key, offset, dist, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "synth_fill");
  return CONV2D_OK;
}

const char* conv2d_status_string(conv2d_status_t s) {
  switch (s) {
    case CONV2D_OK: return "CONV2D_OK";
    case CONV2D_ERR_INVALID_PARAMS: return "CONV2D_ERR_INVALID_PARAMS";
    case CONV2D_ERR_UNSUPPORTED: return "CONV2D_ERR_UNSUPPORTED";
    case CONV2D_ERR_WORKSPACE: return "CONV2D_ERR_WORKSPACE";
    case CONV2D_ERR_ALIGNMENT: return "CONV2D_ERR_ALIGNMENT";
    case CONV2D_ERR_NULL: return "CONV2D_ERR_NULL";
    case CONV2D_ERR_CUDA: return "CONV2D_ERR_CUDA";
    case CONV2D_ERR_NO_DEVICE: return "CONV2D_ERR_NO_DEVICE";
    case CONV2D_ERR_IO: return "CONV2D_ERR_IO";
  }
  return "CONV2D_ERR_UNKNOWN";
}

const char* conv2d_algo_name(conv2d_algo_t a) {
  switch (a) {
    case CONV2D_ALGO_AUTO: return "auto";
    case CONV2D_ALGO_DIRECT: return "direct";
    case CONV2D_ALGO_TILED: return "tiled";
    case CONV2D_ALGO_IMPLICIT_GEMM: return "implicit_gemm";
    case CONV2D_ALGO_WINOGRAD_F2X2_3X3: return "winograd_f2x2_3x3";
    case CONV2D_ALGO_WINOGRAD_F4X4_3X3: return "winograd_f4x4_3x3";
    case CONV2D_ALGO_MATMUL_1X1: return "matmul_1x1";
  }
  return "unknown";
}

const char* conv2d_last_error(void) { return g_last_error.c_str(); }

// ---- pooling (include/pool2d.h): shapes via the conv algebra with F := C
static bool pool_shape(const pool2d_params_t* p, Problem* q, std::string* why) {
  if (!p) {
    *why = "params is NULL";
    return false;
  }
  if (p->op != POOL2D_MAX && p->op != POOL2D_AVG) {
    *why = "bad pooling op";
    return false;
  }
  conv2d_params_t c{p->batch, p->in_rows, p->in_cols, p->channels, p->channels, p->window_rows, p->window_cols,
                    p->stride_rows, p->stride_cols, p->padding, CONV2D_MATH_FP32};
  return shape_of(&c, q, why);
}

conv2d_status_t pool2d_output_shape(const pool2d_params_t* p, int32_t out_nhwc[4], int32_t pads_tblr[4]) {
  Problem q;
  std::string why;
  if (!pool_shape(p, &q, &why)) return fail(CONV2D_ERR_INVALID_PARAMS, why);
  if (out_nhwc) {
    out_nhwc[0] = q.N; out_nhwc[1] = q.HO; out_nhwc[2] = q.WO; out_nhwc[3] = q.C;
  }
  if (pads_tblr) {
    pads_tblr[0] = q.pad_top;
    pads_tblr[1] = std::max(0, (q.HO - 1) * q.SH + q.KH - q.H - q.pad_top);
    pads_tblr[2] = q.pad_left;
    pads_tblr[3] = std::max(0, (q.WO - 1) * q.SW + q.KW - q.W - q.pad_left);
  }
  return CONV2D_OK;
}

conv2d_status_t pool2d_forward(const pool2d_params_t* p, const float* in, float* out, void* stream) {
  Problem q;
  std::string why;
  if (!pool_shape(p, &q, &why)) return fail(CONV2D_ERR_INVALID_PARAMS, why);
  if (!in || !out) return fail(CONV2D_ERR_NULL, "in/out is NULL");
  if ((reinterpret_cast<uintptr_t>(in) & 3) || (reinterpret_cast<uintptr_t>(out) & 3))
    return fail(CONV2D_ERR_ALIGNMENT, "pointers must be 4-byte aligned");
  conv2d_status_t st = check_device(nullptr);
  if (st != CONV2D_OK) return st;
  PoolProblem pp{q.N, q.H, q.W, q.C, q.KH, q.KW, q.SH, q.SW, q.HO, q.WO, q.pad_top, q.pad_left, p->op == POOL2D_AVG};
  cudaError_t e = launch_pool(pp, in, out, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? CONV2D_OK : cuda_fail(e, "pool2d");
}

int conv2d_debug_trace(int enable, unsigned long long* host, int n) {
  return conv2d::gemm2_trace(enable, host, n);
}

conv2d_status_t conv2d_debug_splits(const conv2d_params_t* p, conv2d_algo_t algo, int* splits) {
  if (!splits) return fail(CONV2D_ERR_NULL, "splits is NULL");
  Problem q;
  std::string why;
  if (!shape_of(p, &q, &why)) return fail(CONV2D_ERR_INVALID_PARAMS, why);
  if (!valid_algo(algo) || algo == CONV2D_ALGO_AUTO) return fail(CONV2D_ERR_INVALID_PARAMS, "need a concrete algorithm");
  if (!algo_supports(q, algo)) return fail(CONV2D_ERR_UNSUPPORTED, "algorithm does not support these params");
  switch (algo) {
    case CONV2D_ALGO_IMPLICIT_GEMM: *splits = igemm_split_desc(q, false); break;
    case CONV2D_ALGO_MATMUL_1X1: *splits = igemm_split_desc(q, true); break;
    case CONV2D_ALGO_WINOGRAD_F2X2_3X3: *splits = winograd_splits(q, 2); break;
    case CONV2D_ALGO_WINOGRAD_F4X4_3X3: *splits = winograd_splits(q, 4); break;
    default: *splits = 1;
  }
  return CONV2D_OK;
}

}  // extern "C"
