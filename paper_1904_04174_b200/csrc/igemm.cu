// igemm.cu -- CONV2D_ALGO_IMPLICIT_GEMM and CONV2D_ALGO_MATMUL_1X1 launchers.
//
// Both lower the convolution to  Out[M x F] = A[M x K] * W[K x F]  with
// M = N*Ho*Wo, K = Kh*Kw*C (SPEC.md:231-248 im2col; SPEC.md:249-257 1x1 = matmul), but
// neither materialises A: the GEMM core (gemm2sm.cu) loads A tiles straight from the NHWC
// input with TMA im2col boxes (C % 32 == 0), as a dense (N*H*W) x C matrix (1x1/stride 1),
// or with 16-byte gathers (other C; C % 4 != 0 is first padded to a multiple of 4).
//
// Launch sequence (stream-ordered):
//   [pad_channels]  only when C % 4 != 0 (e.g. the C=3 stems R1/V1)
//   [filter_prep2]  W (HWCF) -> Bt (Fpad x Kpad, K-major), TF32 hi/lo split in FP32 mode; skipped on the
//                   im2col / dense paths with F % 32 == 0, where the GEMM reads W itself (MN-major B)
//   gemm2sm         persistent 2-CTA tcgen05 GEMM
//   [split_reduce]  when the pair-tile count is below one wave
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "gemm2sm.h"

namespace conv2d {

namespace {
inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

struct Plan {
  int a_mode;
  bool three_x, pad;
  int block_n, splits, cstride, cg, rowstride, hp, wp;
  bool b_mn;  // B straight from the HWCF filter (no filter_prep launch)
  bool rsplit;  // remainder split (variant bit 4)
  int64_t kpad, npad;
  size_t bt_bytes, pad_bytes, partial_bytes, total;
};

// Per-layer algorithm parameters chosen by the auto-selector ("different parameters
// for each algorithm"): bit 0 selects the alternative A-operand path (implicit_gemm: halo <-> im2col;
// matmul_1x1: dense <-> im2col), bit 1 halves the N tile (256 -> 128: 3xTF32 lo halves then fit in
// TMEM next to the accumulators, deeper TMA ring), bit 2 stores the output through the LSU
// (smem-staged coalesced STG) instead of TMA bulk stores (frees the TMA engine for loads), bit 3 (3xTF32
// only) routes B through filter_prep's K-major hi/lo copies instead of reading the HWCF filter directly
// (the direct path saves a launch but splits B's lo halves in smem inside the GEMM: a win for short
// layers, ~5-8% slower on long tensor-bound ones where smem bandwidth is the limit), bit 5 (3xTF32, the 3x3
// halo path, F % 32 == 0) reads the halo path's B straight from the filter too (MN-major boxes + four
// lo-split warps; in TF32 the halo path always does, no split needed).
using VKey = std::tuple<int, int, int, int, int, int, int, int, int, int, int, bool>;
std::mutex g_vmu;
std::map<VKey, int> g_variant;
VKey vkey(const Problem& p, bool is_1x1) {
  return VKey(p.N, p.H, p.W, p.C, p.F, p.KH, p.KW, p.SH, p.SW, p.pad_top * 64 + p.pad_left, (int)p.math, is_1x1);
}
int variant_of(const Problem& p, bool is_1x1) {
  if (const char* f = getenv("CONV2D_FORCE_VARIANT")) return atoi(f) & 63;  // parity-test hook
  std::lock_guard<std::mutex> lk(g_vmu);
  auto it = g_variant.find(vkey(p, is_1x1));
  return it == g_variant.end() ? 0 : it->second;
}

Plan make_plan(const Problem& p, bool is_1x1, int variant) {
  Plan pl{};
  pl.three_x = p.math == CONV2D_MATH_FP32;
  pl.block_n = gemm2_choose_block_n(p.F);
  if ((variant & 2) && pl.block_n == 256) pl.block_n = 128;
  pl.npad = round_up(p.F, pl.block_n);
  pl.pad = false;
  pl.cg = p.C;
  if (is_1x1 && p.C % 4 == 0 && p.C >= 32 && !((variant & 1) && gemm2_im2col_ok(p))) {
    pl.a_mode = A_DENSE;
    pl.cstride = p.C;
  } else if (!is_1x1 && s2d_ok(p) && !(variant & 1) && getenv("CONV2D_NO_S2D") == nullptr) {
    pl.a_mode = A_S2D;  // 7x7/8x8 stride-2 stems, C <= 4: space-to-depth + 4x4 halo views (gemm_halo.cu)
    pl.cstride = p.C;
  } else if (!is_1x1 && c4_ok(p) && !(variant & 1) && getenv("CONV2D_NO_C4") == nullptr) {
    pl.a_mode = A_C4;  // 3x3 s1, C <= 4 (VGG conv1_1): 4-channel halo, two taps per K=8 step (gemm_halo.cu)
    pl.cstride = p.C;
  } else if (!is_1x1 && halo_ok(p) && !(variant & 1) && getenv("CONV2D_NO_HALO") == nullptr) {
    pl.a_mode = A_HALO;  // 3x3 s1, small N: halo-tile reuse (gemm_halo.cu)
    pl.cstride = p.C;
  } else if (gemm2_im2col_ok(p)) {
    pl.a_mode = A_IM2COL;
    pl.cstride = p.C;  // C % 32 == 0: one tap = C/32 whole k-blocks
  } else if (gemm2_rowseg_ok(p)) {
    // small C, narrow windows (the C=3 stems): A_ROWSEG (one overlapping-stride TMA box per kernel
    // row) by default, A_STEM (halo + transform-built rows) as the tunable alternative
    // (for s2d- and c4-eligible layers bit 0 selects this path over A_S2D / A_C4)
    pl.a_mode = ((variant & 1) && !s2d_ok(p) && !(c4_ok(p) && getenv("CONV2D_NO_C4") == nullptr) &&
                 gemm2_stem_ok(p, pl.block_n, pl.three_x))
                    ? A_STEM
                    : A_ROWSEG;
    pl.cg = (int)round_up(p.C, 4);
    pl.pad = true;         // spatial + channel padding pass
    pl.cstride = pl.cg;
    pl.rowstride = 32;
    pl.hp = (p.HO - 1) * p.SH + p.KH;
    pl.wp = (p.WO - 1) * p.SW + p.KW;
  } else if (p.C <= 32 && gemm2_narrow_ok(p)) {
    pl.a_mode = A_NARROW;  // small C (e.g. the C=3 stems): 4-channel im2col boxes, flat k
    pl.cg = (int)round_up(p.C, 4);
    pl.pad = pl.cg != p.C;
    pl.cstride = pl.cg;
  } else {
    pl.a_mode = A_GATHER;
    pl.cg = (int)round_up(p.C, 4);
    pl.pad = pl.cg != p.C;
    pl.cstride = pl.cg;
  }
  if (const char* f = getenv("CONV2D_FORCE_AMODE")) {  // experiments: force the A-operand path
    const int m = atoi(f);
    if (m == A_GATHER) {
      pl.a_mode = A_GATHER;
      pl.cg = (int)round_up(p.C, 4);
      pl.pad = pl.cg != p.C;
      pl.cstride = pl.cg;
    }
  }
  if (pl.a_mode == A_S2D) {
    if (pl.block_n == 256) pl.block_n = 128;
    pl.kpad = 256;
    pl.npad = round_up(p.F, pl.block_n);
    pl.splits = 1;
    pl.b_mn = false;
    pl.total = s2d_workspace(p, pl.block_n, pl.three_x);
    return pl;
  }
  if (pl.a_mode == A_C4) {
    if (pl.block_n == 256) pl.block_n = 128;
    pl.kpad = 64;
    pl.npad = round_up(p.F, pl.block_n);
    pl.splits = 1;
    pl.b_mn = false;
    pl.total = c4_workspace(p, pl.block_n, pl.three_x);
    return pl;
  }
  const bool rowk = pl.a_mode == A_ROWSEG || pl.a_mode == A_STEM;  // k = (kernel row, 32 floats)
  if (!rowk) pl.rowstride = p.KW * pl.cstride;
  pl.kpad = rowk ? (int64_t)p.KH * 32 : round_up((int64_t)p.KH * p.KW * pl.cstride, 32);
  pl.splits = (p.F % 4 == 0 && !rowk && pl.a_mode != A_HALO)
                  ? gemm2_choose_splits(p.M(), p.F, (int)(pl.kpad / 32), 1, pl.block_n) : 1;
  // HWCF rows are exactly the GEMM's k order for the im2col (C % 32 == 0: k = tap*C + c) and dense 1x1
  // (k = c) paths, so the GEMM reads W as an MN-major B operand -- no filter_prep launch, no Bt copy
  // the halo path reads B straight from the filter always in TF32 and on variant bit 5 in 3xTF32 (there it
  // needs four lo-split warps and loses on R4 / V2 at b32-b256; it wins at b1 and on R10-like layers)
  pl.b_mn = (pl.a_mode == A_HALO ? (!pl.three_x || (variant & 32))
                                 : (pl.a_mode == A_IM2COL || pl.a_mode == A_DENSE) && !((variant & 8) && pl.three_x)) &&
            p.F % 32 == 0 && getenv("CONV2D_NO_BMN") == nullptr;
  pl.bt_bytes = pl.b_mn ? 0 : round_up((int64_t)pl.npad * pl.kpad * 4, 256);
  pl.pad_bytes = !pl.pad ? 0
                 : rowk ? round_up((int64_t)p.N * pl.hp * pl.wp * pl.cg * 4, 256)
                                         : round_up((int64_t)p.N * p.H * p.W * pl.cg * 4, 256);
  pl.partial_bytes = pl.splits > 1 ? (size_t)pl.splits * p.M() * p.F * 4 : 0;
  // bit 4: balanced K split -- fewer pair tiles than pairs: the modelled-best split count instead of
  // 74 / tiles; else a remainder split of the partial last wave (partials for those tiles only, summed
  // by a small kernel)
  pl.rsplit = false;
  const int64_t tiles = ((p.M() + 255) / 256) * ((p.F + pl.block_n - 1) / pl.block_n);
  if ((variant & 16) && tiles < 74 && p.F % 4 == 0 && !rowk && pl.a_mode != A_HALO) {
    pl.splits = gemm2_balanced_splits(tiles, (int)(pl.kpad / 32));
    pl.partial_bytes = pl.splits > 1 ? (size_t)pl.splits * p.M() * p.F * 4 : 0;
  } else if ((variant & 16) && pl.splits == 1 && p.F % 4 == 0 && !rowk && pl.a_mode != A_HALO) {
    const int rs = gemm2_rsplit_factor(tiles, (int)(pl.kpad / 32));
    if (rs >= 2) {
      pl.rsplit = true;
      pl.partial_bytes = (size_t)rs * p.M() * p.F * 4;
    }
  }
  pl.total = pl.bt_bytes * (pl.three_x ? 2 : 1) + pl.pad_bytes + pl.partial_bytes;
  return pl;
}
}  // namespace

int igemm_variants(const Problem& p, bool is_1x1, int* masks) {
  const bool alt_a = is_1x1 ? (p.C % 4 == 0 && p.C >= 32 && gemm2_im2col_ok(p))
                            : ((halo_ok(p) && gemm2_im2col_ok(p)) || (s2d_ok(p) && gemm2_rowseg_ok(p)) ||
                               (c4_ok(p) && gemm2_rowseg_ok(p)) ||
                               (gemm2_rowseg_ok(p) && gemm2_stem_ok(p, gemm2_choose_block_n(p.F), p.math == 0)));
  const bool alt_n = gemm2_choose_block_n(p.F) == 256;
  // bit 3 matters only where some A path reads B directly (im2col / dense, F % 32 == 0) in 3xTF32 mode
  const bool alt_b = p.math == CONV2D_MATH_FP32 && p.F % 32 == 0 &&
                     ((is_1x1 && p.C % 4 == 0 && p.C >= 32) || gemm2_im2col_ok(p));
  // bit 4: balanced K split (fewer pair tiles than pairs, where it differs from the default 74 / tiles)
  // or remainder split (a partial last wave)
  auto rs_ok = [&](int m) {
    const int bn = (m & 2) && gemm2_choose_block_n(p.F) == 256 ? 128 : gemm2_choose_block_n(p.F);
    const int64_t tiles = ((p.M() + 255) / 256) * ((p.F + bn - 1) / bn);
    const int nkb = (int)(((int64_t)p.KH * p.KW * p.C + 31) / 32);
    if (p.F % 4 != 0) return false;
    if (tiles < 74) return gemm2_balanced_splits(tiles, nkb) != gemm2_choose_splits(p.M(), p.F, nkb, 1, bn);
    return gemm2_rsplit_factor(tiles, nkb) >= 2;
  };
  int n = 0;
  // bit 0: A path, bit 1: N tile, bit 3: B path.  Bit 2 (LSU-staged epilogue) is not enumerated: it
  // measured slower than TMA stores on every paper layer (reachable through CONV2D_FORCE_VARIANT).
  // bit 5: the halo path's direct (MN-major) B in 3xTF32 -- only with bit 0 clear (the halo path itself)
  const bool alt_h = !is_1x1 && p.math == CONV2D_MATH_FP32 && p.F % 32 == 0 && halo_ok(p);
  for (int m = 0; m < 64; ++m) {
    if (m & 4) continue;
    if ((m & 32) && (!alt_h || (m & 1) || (m & 8))) continue;
    if ((m & 1) && !alt_a) continue;
    if ((m & 2) && !alt_n) continue;
    if ((m & 8) && !alt_b) continue;
    if ((m & 16) && !rs_ok(m)) continue;
    if (masks) masks[n] = m;
    ++n;
  }
  return n;
}

bool igemm_get_variant(const Problem& p, bool is_1x1, int* v) {
  std::lock_guard<std::mutex> lk(g_vmu);
  auto it = g_variant.find(vkey(p, is_1x1));
  if (it == g_variant.end()) return false;
  *v = it->second;
  return true;
}

void igemm_set_variant(const Problem& p, bool is_1x1, int v) {
  std::lock_guard<std::mutex> lk(g_vmu);
  g_variant[vkey(p, is_1x1)] = v;
}

size_t igemm_workspace(const Problem& p, bool is_1x1) {
  size_t w = 0;
  int masks[32];
  const int n = igemm_variants(p, is_1x1, masks);
  for (int i = 0; i < n; ++i) w = std::max(w, make_plan(p, is_1x1, masks[i]).total);
  return w;
}

int igemm_launches(const Problem& p, bool is_1x1) {
  const Plan pl = make_plan(p, is_1x1, variant_of(p, is_1x1));
  if (pl.a_mode == A_S2D) return (p.C <= 3 && ((int64_t)p.W * p.C) % 4 == 0) ? 2 : 3;  // [s2d input,] filter, GEMM
  if (pl.a_mode == A_C4) return 1;  // the GEMM builds B from the filter itself
  return (pl.b_mn ? 1 : 2) + (pl.pad ? 1 : 0) + (pl.splits > 1 || pl.rsplit ? 1 : 0);
}

int igemm_split_desc(const Problem& p, bool is_1x1) {
  const Plan pl = make_plan(p, is_1x1, variant_of(p, is_1x1));
  if (pl.a_mode == A_S2D || pl.a_mode == A_C4) return 1;
  return pl.rsplit ? -gemm2_rsplit_factor(((p.M() + 255) / 256) * ((p.F + pl.block_n - 1) / pl.block_n),
                                          (int)(pl.kpad / 32))
                   : pl.splits;
}

cudaError_t launch_igemm(const Problem& p, bool is_1x1, const float* in, const float* filt, float* out, void* ws,
                         cudaStream_t s) {
  const Plan pl = make_plan(p, is_1x1, variant_of(p, is_1x1));
  static const bool debug = getenv("CONV2D_DEBUG") != nullptr;
  if (pl.a_mode == A_S2D) return launch_gemm_s2d(p, in, filt, pl.block_n, pl.three_x, ws, out, s);
  if (pl.a_mode == A_C4) return launch_gemm_c4(p, in, filt, pl.block_n, pl.three_x, ws, out, s);
  if (debug)
    fprintf(stderr, "[conv2d] igemm N=%d H=%d W=%d C=%d F=%d K=%dx%d S=%d: a_mode=%d bn=%d splits=%d kpad=%lld 3x=%d\n",
            p.N, p.H, p.W, p.C, p.F, p.KH, p.KW, p.SH, pl.a_mode, pl.block_n, pl.splits, (long long)pl.kpad,
            (int)pl.three_x);
  uint8_t* w8 = static_cast<uint8_t*>(ws);
  float* bt_hi = reinterpret_cast<float*>(w8);
  w8 += pl.bt_bytes;
  float* bt_lo = nullptr;
  if (pl.three_x) {
    bt_lo = reinterpret_cast<float*>(w8);
    w8 += pl.bt_bytes;
  }
  const float* xg = in;
  if (pl.pad) {
    float* xp = reinterpret_cast<float*>(w8);
    w8 += pl.pad_bytes;
    const bool rowk = pl.a_mode == A_ROWSEG || pl.a_mode == A_STEM;
    cudaError_t e = rowk
                        ? launch_pad_spatial(in, p.N, p.H, p.W, p.C, pl.hp, pl.wp, pl.cg, p.pad_top, p.pad_left, xp, s)
                        : launch_pad_channels(in, (int64_t)p.N * p.H * p.W, p.C, pl.cg, xp, s);
    if (e != cudaSuccess) return e;
    xg = xp;
  }
  float* partial = (pl.splits > 1 || pl.rsplit) ? reinterpret_cast<float*>(w8) : nullptr;
  if (!pl.b_mn) {
    cudaError_t e =
        launch_filter_prep2(filt, p.KH, p.KW, p.C, p.F, pl.cstride, pl.rowstride, pl.kpad, pl.npad, bt_hi, bt_lo, s);
    if (e != cudaSuccess) return e;
  }
  if (pl.a_mode == A_HALO)
    return launch_gemm_halo(p, in, bt_hi, bt_lo, pl.kpad, pl.npad, pl.block_n, out, s, filt, pl.b_mn, pl.three_x);
  Gemm2Args g{};
  g.a_mode = pl.a_mode;
  g.a = in;
  g.lda = p.C;
  g.a_k = p.C;
  g.gather_x = xg;
  g.gather_c = pl.cg;
  g.bt_hi = bt_hi;
  g.bt_lo = bt_lo;
  g.kpad = pl.kpad;
  g.npad = pl.npad;
  g.d = out;
  g.ldd = p.F;
  g.d_batch_stride = 0;
  g.partial = partial;
  g.M = p.M();
  g.N = p.F;
  g.batch = 1;
  g.splits = pl.splits;
  g.block_n = pl.block_n;
  g.three_x = pl.three_x;
  g.hp = pl.hp;
  g.wp = pl.wp;
  g.epi_stg = (variant_of(p, is_1x1) & 4) != 0;
  g.b_mn = pl.b_mn;
  g.rsplit = pl.rsplit;
  g.b_w = filt;
  g.b_rows = (int64_t)p.KH * p.KW * p.C;
  return launch_gemm2(p, g, s);
}

}  // namespace conv2d
