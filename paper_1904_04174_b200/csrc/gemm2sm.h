// gemm2sm.h -- host interface of the persistent 2-CTA tcgen05 GEMM core (gemm2sm.cu).
#pragma once
#include <cuda.h>

#include "internal.h"

namespace conv2d {

enum { A_IM2COL = 0, A_DENSE = 1, A_GATHER = 2, A_NARROW = 3, A_ROWSEG = 4, A_HALO = 5, A_STEM = 6, A_S2D = 7, A_C4 = 8 };

struct Gemm2Args {
  int a_mode;              // A_IM2COL: a = NHWC input (C % 32 == 0), k = (r, s, c-block of 32)
                           // A_NARROW: gather_x = NHWC input with gather_c (% 4 == 0) channels, flat k =
                           //           (tap, channel quad): eight 128-px x 4-ch im2col boxes per k-block
                           // A_ROWSEG: gather_x = spatially padded NHWC input (Hp x Wp x gather_c); one
                           //           k-block per kernel row r holds the KW*gather_c contiguous floats of
                           //           each output pixel (5-D tiled TMA over overlapping strides); the CTA
                           //           tile is a 16 (wo) x 8 (ho) spatial block, the pair tile 16 x 16
                           // A_STEM  : same tiles and k order as A_ROWSEG, but TMA loads one compact input
                           //           halo per tile and the transform warps assemble each kernel row's
                           //           A tile from it (B resident); for the small-C stems
                           // A_DENSE : a = [batch][M][lda] K-major matrix, lda % 4 == 0
                           // A_GATHER: gather_x = NHWC input with gather_c (% 4 == 0) channels, flat k
  const float* a;
  int64_t lda;
  int64_t a_k;             // A_DENSE: extent of A's k dimension (elements beyond it read as zero)
  const float* gather_x;
  int gather_c;
  const float* bt_hi;      // [batch][npad][kpad] K-major, zero padded (TF32 hi in 3xTF32 mode)
  const float* bt_lo;      // same layout, lo parts (3xTF32 only)
  int64_t kpad, npad;
  float* d;                // [batch][M][ldd]
  int64_t ldd, d_batch_stride;
  float* partial;          // [splits][batch][M][ldd] when splits > 1
  int64_t M, N;
  int batch, splits, block_n;
  bool three_x;
  int hp, wp;              // A_ROWSEG: padded input extent
  bool epi_stg;            // epilogue: smem-staged coalesced STG instead of TMA stores
  bool b_mn;               // B read straight from b_w, a row-major b_rows x N matrix (the HWCF filter,
  const float* b_w;        // k = row): MN-major operand, no filter_prep; needs N % 32 == 0, batch 1
  int64_t b_rows;          // (bt_hi / bt_lo unused; 3xTF32 lo halves are split in smem by the kernel)
  bool bstat;              // B-stationary schedule where B-resident applies with several N tiles
  bool rsplit;             // remainder split of a partial last wave (needs `partial` with
                           // gemm2_rsplit_factor(tiles, nkb) planes of M x ldd floats)
};

cudaError_t launch_gemm2(const Problem& p, const Gemm2Args& g, cudaStream_t s);
// rank-2..5 fp32 tiled tensor map (strides in bytes for dims 1..rank-1), L2 promotion 256 B, OOB -> 0
bool gemm2_encode_tiled(CUtensorMap* m, int rank, const void* base, const uint64_t* dims, const uint64_t* strides,
                        const uint32_t* box, bool swizzle128);

// gemm_halo.cu: 3x3 stride-1 convolution with C % 32 == 0 as a halo-tile implicit GEMM (see file header)
bool halo_ok(const Problem& p);
// space-to-depth stem (gemm_halo.cu): K x K / stride 2, K in {7, 8}, C <= 4, F <= 128
bool s2d_ok(const Problem& p);
bool c4_ok(const Problem& p);
size_t c4_workspace(const Problem& p, int block_n, bool three_x);
cudaError_t launch_gemm_c4(const Problem& p, const float* in, const float* filt, int block_n, bool three_x, void* ws,
                           float* out, cudaStream_t s);
size_t s2d_workspace(const Problem& p, int block_n, bool three_x);
cudaError_t launch_gemm_s2d(const Problem& p, const float* in, const float* filt, int block_n, bool three_x,
                            void* ws, float* out, cudaStream_t s);
// bmn: B straight from the HWCF filter `filt` (MN-major, F % 32 == 0; bt_hi / bt_lo unused), else from the
// K-major Bt hi [/ lo] filter_prep2 wrote
cudaError_t launch_gemm_halo(const Problem& p, const float* in, const float* bt_hi, const float* bt_lo, int64_t kpad,
                             int64_t npad, int block_n, float* out, cudaStream_t s, const float* filt, bool bmn,
                             bool three_x);
bool gemm2_encode_tiled_sw(CUtensorMap* m, int rank, const void* base, const uint64_t* dims, const uint64_t* strides,
                           const uint32_t* box, int swizzle);  // swizzle: a CUtensorMapSwizzle value
// same with TMA traversal strides (elem_strides[i] in [1, 8]; dimension i then loads ceil(box[i] / stride) elements)
bool gemm2_encode_tiled_es(CUtensorMap* m, int rank, const void* base, const uint64_t* dims, const uint64_t* strides,
                           const uint32_t* box, const uint32_t* elem_strides, int swizzle);
int gemm2_choose_block_n(int64_t N);
// remainder-split factor for `tiles` pair tiles of nkb k-blocks (0 = not applicable)
int gemm2_rsplit_factor(int64_t tiles, int nkb);
// K-split count of least modelled time for fewer than 74 pair tiles (1 = no split)
int gemm2_balanced_splits(int64_t tiles, int nkb);
cudaError_t launch_rsplit_reduce(const float* partial, float* d, int64_t M, int64_t N, int64_t ldd, int first_tile,
                                 int ntiles, int nt, int block_n, int splits, cudaStream_t s);
// debug: enable (1) / disable (0) / keep (-1) per-CTA globaltimer stamps of the GEMM kernels (records of
// 148 CTAs x 8 stamps, one per launch, ring of 256) and optionally copy them to `host` (synchronous);
// returns values copied.  gemm2_trace_record(): the next launch's record, or null when disabled.
int gemm2_trace(int enable, unsigned long long* host, int n);
unsigned long long* gemm2_trace_record();
int gemm2_choose_splits(int64_t M, int64_t N, int nkb, int batch, int block_n);
bool gemm2_im2col_ok(const Problem& p);
bool gemm2_narrow_ok(const Problem& p);
bool gemm2_rowseg_ok(const Problem& p);
bool gemm2_stem_ok(const Problem& p, int block_n, bool three_x);

// gemm_common.cu
// Bt[n][tap*cstride + c] = w[tap][c][n] (HWCF viewed as taps x C x F) for c < C, n < F, tap < taps;
// zero elsewhere in the npad x kpad matrix.  bt_lo != null: split into TF32 hi / lo.
// Bt[n][k] with k -> (r = k / rowstride, s = (k % rowstride) / cstride, c = k % cstride); zero padded
cudaError_t launch_filter_prep2(const float* w, int KH, int KW, int C, int F, int cstride, int rowstride,
                                int64_t kpad, int64_t npad, float* bt_hi, float* bt_lo, cudaStream_t s);
cudaError_t launch_pad_spatial(const float* x, int N, int H, int W, int C, int Hp, int Wp, int Cp, int pt, int pl,
                               float* xp, cudaStream_t s);
// NHWC with C channels -> NHWC with Cp >= C channels (zeros in the new channels)
cudaError_t launch_pad_channels(const float* x, int64_t pixels, int C, int Cp, float* xp, cudaStream_t s);

}  // namespace conv2d
