// internal.h -- host-side problem description shared by the dispatcher (api.cpp)
// and the kernel launchers (*.cu).  Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "../../include/conv2d.h"

namespace conv2d {

// Everything a launcher needs, derived once from conv2d_params_t.
struct Problem {
  int N, H, W, C, F;
  int KH, KW, SH, SW;
  int HO, WO;
  int pad_top, pad_left;  // bottom/right pads are implied by HO/WO
  conv2d_math_t math;
  int64_t M() const { return (int64_t)N * HO * WO; }      // GEMM rows (output pixels)
  int64_t K() const { return (int64_t)KH * KW * C; }      // GEMM depth (im2col columns)
  int64_t in_elems() const { return (int64_t)N * H * W * C; }
  int64_t out_elems() const { return M() * F; }
  int64_t filt_elems() const { return K() * F; }
};

// ---- pool.cu (include/pool2d.h)
struct PoolProblem {
  int N, H, W, C, KH, KW, SH, SW, HO, WO, PT, PL;
  bool avg;
};
cudaError_t launch_pool(const PoolProblem& p, const float* x, float* y, cudaStream_t s);

// ---- direct.cu
cudaError_t launch_direct(const Problem& p, const float* in, const float* filt, float* out, cudaStream_t s);
// ---- tiled.cu
cudaError_t launch_tiled(const Problem& p, const float* in, const float* filt, float* out, cudaStream_t s);
bool tiled_supported(const Problem& p);  // the tile's shared-memory chunk fits and the 1-D grid fits gridDim.x
// ---- igemm.cu (implicit GEMM and 1x1 matmul on tcgen05)
size_t igemm_workspace(const Problem& p, bool is_1x1);  // max over variants
int igemm_variants(const Problem& p, bool is_1x1, int* masks);  // tunable parameter masks (<= 8)
void igemm_set_variant(const Problem& p, bool is_1x1, int v);
bool igemm_get_variant(const Problem& p, bool is_1x1, int* v);  // false if never set
int igemm_launches(const Problem& p, bool is_1x1);
// K-split of the plan conv2d_forward would run now: 1 = none, s > 1 = every tile split s ways,
// -s = remainder split (the partial last wave's tiles split s ways)
int igemm_split_desc(const Problem& p, bool is_1x1);
cudaError_t launch_igemm(const Problem& p, bool is_1x1, const float* in, const float* filt, float* out, void* ws,
                         cudaStream_t s);
// ---- winograd.cu
size_t winograd_workspace(const Problem& p, int mt);  // mt = output tile: 2 (F2x2) or 4 (F4x4)
int winograd_launches(const Problem& p, int mt);
int winograd_splits(const Problem& p, int mt);  // K-split count of the batched GEMMs (1 = none)
// F(2x2) parameter variants (0 = transforms + batched GEMM, 1 = fused kernel where wino_fused_ok)
int winograd_variants(const Problem& p, int* masks);
bool winograd_get_variant(const Problem& p, int* v);  // false if never set
void winograd_set_variant(const Problem& p, int v);
cudaError_t launch_winograd(const Problem& p, int mt, const float* in, const float* filt, float* out, void* ws,
                            cudaStream_t s);
// filter transform U = G g G^T into Ut[xi][fpad][cpad] (hi, and lo when three_x; TF32: rna-rounded hi)
cudaError_t launch_wino_filter(int mt, const float* w, int C, int F, int64_t cpad, int64_t fpad, float* ut_hi,
                               float* ut_lo, bool three_x, cudaStream_t s);
// ---- wino_fused.cu: F(2x2,3x3) with the input transform, the 16 coordinate GEMMs and the output transform in
// one cluster kernel (V and M never leave the SM pair): F(2x2) parameter variant 1 where wino_fused_ok
bool wino_fused_ok(const Problem& p);
size_t wino_fused_workspace(const Problem& p);
cudaError_t launch_wino_fused(const Problem& p, const float* in, const float* filt, float* out, void* ws,
                              cudaStream_t s);
// ---- synth.cu
cudaError_t launch_synth_fill(float* dst, uint64_t count, uint64_t key, uint64_t offset, int dist, cudaStream_t s);

// gemm_common.cu
cudaError_t launch_split_reduce(const float* partial, float* d, int64_t rows, int64_t cols, int64_t ldd,
                                int splits, cudaStream_t s);

int gemm2_trace(int enable, unsigned long long* host, int n);  // gemm2sm.cu (conv2d_debug.h)

}  // namespace conv2d
