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

// ---- direct.cu
cudaError_t launch_direct(const Problem& p, const float* in, const float* filt, float* out, cudaStream_t s);
// ---- tiled.cu
cudaError_t launch_tiled(const Problem& p, const float* in, const float* filt, float* out, cudaStream_t s);
// ---- igemm.cu (implicit GEMM and 1x1 matmul on tcgen05)
size_t igemm_workspace(const Problem& p, bool is_1x1);
int igemm_launches(const Problem& p, bool is_1x1);
cudaError_t launch_igemm(const Problem& p, bool is_1x1, const float* in, const float* filt, float* out, void* ws,
                         cudaStream_t s);
// ---- winograd.cu
size_t winograd_workspace(const Problem& p);
int winograd_launches(const Problem& p);
cudaError_t launch_winograd(const Problem& p, const float* in, const float* filt, float* out, void* ws,
                            cudaStream_t s);
// ---- synth.cu
cudaError_t launch_synth_fill(float* dst, uint64_t count, uint64_t key, uint64_t offset, int dist, cudaStream_t s);

// Generic tcgen05 GEMM used by igemm and winograd (gemm_core.cuh instantiations live in igemm.cu).
//   D[b][m][n] = sum_k A[b](m,k) * Bt[b](n,k)      (Bt is K-major: row n holds k contiguous)
// A comes either from the im2col gather of an NHWC tensor (conv mode) or from a dense
// K-major matrix (dense mode, Winograd batched GEMMs).
struct GemmArgs {
  // A operand
  int a_mode;             // 0 = im2col of `in` (conv geometry from Problem), 1 = dense row-major [batch][M][lda]
  const float* a;         // in (mode 0) or dense A
  int64_t lda;            // dense mode row stride (floats), multiple of 4
  int64_t a_batch_stride; // dense mode
  // B operand, already split (hi, lo) and K-major, zero-padded to Kpad columns and Npad rows
  const float* bt_hi;
  const float* bt_lo;     // null in TF32 mode
  int64_t ldb;            // = Kpad
  int64_t b_batch_stride;
  // D
  float* d;
  int64_t ldd;            // row stride of D (floats)
  int64_t d_batch_stride;
  float* partial;         // split-K partials [splits][batch][M][ldd] (nullptr if splits == 1)
  int64_t M, N, K;        // logical sizes; K padded up to a multiple of 32 internally
  int batch;
  int splits;
  bool three_x;           // 3xTF32
  int block_n;            // 64, 128 or 256
};
cudaError_t launch_gemm(const Problem& conv, const GemmArgs& g, cudaStream_t s);
int gemm_choose_block_n(int64_t N, bool three_x);
int gemm_choose_splits(int64_t M, int64_t N, int64_t K, int batch, int block_n);
cudaError_t launch_split_reduce(const float* partial, float* d, int64_t rows, int64_t cols, int64_t ldd,
                                int splits, cudaStream_t s);
cudaError_t launch_filter_prep(const float* filt, int64_t K, int64_t F, int64_t kpad, int64_t npad, float* bt_hi,
                               float* bt_lo, cudaStream_t s);

}  // namespace conv2d
