// igemm.cu -- CONV2D_ALGO_IMPLICIT_GEMM and CONV2D_ALGO_MATMUL_1X1 launchers.
//
// Both lower the convolution to  Out[M x F] = A[M x K] * W[K x F]  with
// M = N*Ho*Wo, K = Kh*Kw*C (SPEC.md:231-248 im2col; SPEC.md:249-257 1x1 = matmul), but
// neither materialises A: the GEMM core (gemm_tcgen05.cu) gathers A tiles straight from
// the NHWC input (implicit GEMM) or reads the input as a dense (N*H*W) x C matrix (1x1).
//
// Launch sequence (stream-ordered):
//   1. filter_prep: W (K x F, HWCF) -> Bt (Fpad x Kpad, K-major), split into TF32 hi/lo
//      in FP32 (3xTF32) mode.  Workspace: Fpad*Kpad*4 B (x2 in FP32 mode).
//   2. gemm_tcgen05 (+ split_reduce when the tile count is below one wave).
#include "internal.h"

namespace conv2d {

namespace {
struct Plan {
  bool three_x;
  int block_n;
  int splits;
  int64_t kpad, npad;
  size_t bt_bytes, partial_bytes, total;
};

inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

Plan make_plan(const Problem& p) {
  Plan pl{};
  pl.three_x = p.math == CONV2D_MATH_FP32;
  pl.block_n = gemm_choose_block_n(p.F, pl.three_x);
  pl.kpad = round_up(p.K(), 32);
  pl.npad = round_up(p.F, pl.block_n);
  pl.splits = (p.F % 4 == 0) ? gemm_choose_splits(p.M(), p.F, p.K(), 1, pl.block_n) : 1;
  pl.bt_bytes = (size_t)pl.npad * pl.kpad * sizeof(float);
  const size_t bt_total = round_up((int64_t)pl.bt_bytes, 256) * (pl.three_x ? 2 : 1);
  pl.partial_bytes = pl.splits > 1 ? (size_t)pl.splits * p.M() * p.F * sizeof(float) : 0;
  pl.total = bt_total + pl.partial_bytes;
  return pl;
}
}  // namespace

size_t igemm_workspace(const Problem& p, bool) { return make_plan(p).total; }

int igemm_launches(const Problem& p, bool) { return 2 + (make_plan(p).splits > 1 ? 1 : 0); }

cudaError_t launch_igemm(const Problem& p, bool is_1x1, const float* in, const float* filt, float* out, void* ws,
                         cudaStream_t s) {
  const Plan pl = make_plan(p);
  uint8_t* w8 = static_cast<uint8_t*>(ws);
  float* bt_hi = reinterpret_cast<float*>(w8);
  float* bt_lo = pl.three_x ? reinterpret_cast<float*>(w8 + round_up((int64_t)pl.bt_bytes, 256)) : nullptr;
  float* partial = pl.splits > 1
                       ? reinterpret_cast<float*>(w8 + round_up((int64_t)pl.bt_bytes, 256) * (pl.three_x ? 2 : 1))
                       : nullptr;
  cudaError_t e = launch_filter_prep(filt, p.K(), p.F, pl.kpad, pl.npad, bt_hi, bt_lo, s);
  if (e != cudaSuccess) return e;
  GemmArgs g{};
  // 1x1/stride-1: the NHWC input is already the (N*H*W) x C A matrix (dense rows of C floats).
  const bool dense = is_1x1 && (p.C % 4 == 0);
  g.a_mode = dense ? 1 : 0;
  g.a = in;
  g.lda = p.C;
  g.a_batch_stride = 0;
  g.bt_hi = bt_hi;
  g.bt_lo = bt_lo;
  g.ldb = pl.kpad;
  g.b_batch_stride = 0;
  g.d = out;
  g.ldd = p.F;
  g.d_batch_stride = 0;
  g.partial = partial;
  g.M = p.M();
  g.N = p.F;
  g.K = p.K();
  g.batch = 1;
  g.splits = pl.splits;
  g.three_x = pl.three_x;
  g.block_n = pl.block_n;
  return launch_gemm(p, g, s);
}

}  // namespace conv2d
