// tiled.cu -- CONV2D_ALGO_TILED: tiled direct convolution on CUDA cores
// ("tiled algorithm", SPEC.md:210-230 tile_rows x tile_cols x
// feature_block).  B200 design (round 2):
//   * CTA = 128 threads = 4 warps (three CTAs per SM) over one image x (TH x TW) output tile x FB features.  A warp owns a
//     (32/CG) x (CG*4) pixel block and 16 features; lane (r, g) computes 4 consecutive output pixels of row
//     r x 16 features (64 fp32 accumulators, 32 packed FFMA2 per input value pair).  WFG = FB/16 warps share
//     a pixel block (the others stack vertically), so a warp's filter reads are shared-memory broadcasts.
//   * Per channel chunk (CC <= 16) the input halo ((TH-1)S+KH) x ((TW-1)S+KW) is staged channel-major
//     xs[c][row][col] (NHWC float4 global loads of 4 channels where C % 4 == 0; zero padding) and the filter
//     chunk ws[kh][kw][c][FB] (float4 loads); each thread then reads its input row segment for (c, kh)
//     once into registers -- (4-1)*S+KW floats, 16-byte LDS -- and reuses it for every kw (templated on the
//     common (KW, S); a generic path reads per tap).
//   * FFMA2 (fma.rn.f32x2, sm_100): each instruction does two independent fp32 FMAs, so every output
//     element still sees exactly one RN fp32 FMA per tap: exact-fp32 results, (c-chunk, c, kh, kw) order.
//   * Single-chunk layers (all C channels in one chunk: the small-C layers such as VGG conv1_1, C = 3) run a
//     persistent form instead: each CTA stages its filter block once, keeps its halo element map (smem slot,
//     relative input offset) in registers, and loads the NEXT tile's halo into registers while it computes the
//     current one -- the per-tile staging latency that dominated these layers (ncu: 25% of warp samples
//     waiting on halo loads, 14% in FFMA2) is hidden behind the FMAs.  Same arithmetic, same order.
// Bound: FFMA pipe (74.4 TF/s at 1965 MHz) when the 16-feature x 4-pixel register tile is full; input
// and filter shared-memory reads are ~1 wavefront per 32..64 FMAs per warp.
#include <cstdlib>
#include <type_traits>

#include "internal.h"
#include "launch.cuh"

namespace conv2d {
namespace {

constexpr int NT = 128, NW = NT / 32, PX = 4, FV = 16, CCMAX = 16;
constexpr int SMEM_BUDGET = 72 * 1024;  // three CTAs per SM (registers allow three 128-thread CTAs)
constexpr int PFMAX = 8;                // persistent form: halo elements per thread per tile (floats; float4: 4)

struct TGeo {
  int cg, wfg, th, tw, fb, cc, ih, iw, iwp;
  int64_t ntiles;
  int pf;     // persistent form: halo elements per thread (0 = not applicable)
  size_t smem_pipe;  // persistent form: halo + filter
  bool vec;   // persistent form: float4 elements (C % 4 == 0)
  size_t smem;
  bool ok;
};

TGeo geometry(const Problem& p) {
  TGeo g{};
  g.cg = p.WO >= 32 ? 8 : p.WO >= 16 ? 4 : 2;
  g.wfg = p.F > 32 ? 4 : p.F > 16 ? 2 : 1;
  g.fb = FV * g.wfg;
  g.th = (32 / g.cg) * (NW / g.wfg);
  g.tw = g.cg * PX;
  g.ih = (g.th - 1) * p.SH + p.KH;
  g.iw = (g.tw - 1) * p.SW + p.KW;
  g.iwp = (g.iw + 3) & ~3;
  const size_t per_c = sizeof(float) * ((size_t)g.ih * g.iwp + (size_t)p.KH * p.KW * g.fb);
  const int cc = (int)(SMEM_BUDGET / per_c);
  g.cc = cc < CCMAX ? cc : CCMAX;
  if (g.cc > p.C) g.cc = p.C;
  if (g.cc >= 4) g.cc &= ~3;  // whole channel quads per chunk (float4 staging)
  g.smem = per_c * (size_t)(g.cc > 0 ? g.cc : 1);
  g.ntiles = (int64_t)((p.WO + g.tw - 1) / g.tw) * ((p.HO + g.th - 1) / g.th) * p.N * ((p.F + g.fb - 1) / g.fb);
  g.ok = g.cc >= 1 && g.ntiles <= 0x7FFFFFFFLL;
  // persistent form: the whole C in one chunk, the halo within PFMAX elements per thread, halo coordinates
  // within the 16-bit (row, col) packing
  g.vec = p.C % 4 == 0;
  const int64_t elems = (int64_t)g.ih * g.iw * (g.vec ? p.C / 4 : p.C);
  const int pfmax = g.vec ? PFMAX / 2 : PFMAX;
  g.smem_pipe = per_c * (size_t)p.C;
  g.pf = (g.cc >= p.C && elems <= (int64_t)pfmax * NT && g.iw < 65536 && g.ih < 2048 && g.smem_pipe <= SMEM_BUDGET)
             ? (int)((elems + NT - 1) / NT) : 0;
  return g;
}

__device__ __forceinline__ void fma_tile(float2 (&acc)[PX][FV / 2], const float (&xv)[PX], const float4 (&w4)[FV / 4]) {
#pragma unroll
  for (int i = 0; i < PX; ++i) {
    const float2 xx = make_float2(xv[i], xv[i]);
#pragma unroll
    for (int j = 0; j < FV / 4; ++j) {
      acc[i][2 * j] = __ffma2_rn(xx, make_float2(w4[j].x, w4[j].y), acc[i][2 * j]);
      acc[i][2 * j + 1] = __ffma2_rn(xx, make_float2(w4[j].z, w4[j].w), acc[i][2 * j + 1]);
    }
  }
}

// acc += the staged chunk: x = xs[c][IH][IWP] (this thread's row segment per (c, kh)), w = ws[tap][cc_max][FB];
// (c, kh, kw) order.  KW_, SW_ > 0: compile-time window width / stride (segment cached in registers).
template <int KW_, int SW_>
__device__ __forceinline__ void chunk_mac(float2 (&acc)[PX][FV / 2], const float* xs, const float* ws, int cc,
                                          int cc_max, int IH, int IWP, int KH, int KWr, int SH, int SWr, int row,
                                          int colg, int fg, int FB) {
  const int KW = KW_ ? KW_ : KWr;
  const int SW = SW_ ? SW_ : SWr;
  for (int c = 0; c < cc; ++c) {
    for (int kh = 0; kh < KH; ++kh) {
      const float* xr = xs + ((size_t)c * IH + row * SH + kh) * IWP + colg * PX * SW;
      const float* wr = ws + ((size_t)(kh * KW) * cc_max + c) * FB + fg * FV;
      if constexpr (KW_ > 0) {
        constexpr int L = (PX - 1) * SW_ + KW_;
        constexpr int L4 = L / 4;
        float seg[L4 * 4 + 4];
#pragma unroll
        for (int q = 0; q < L4; ++q) {
          const float4 v = *reinterpret_cast<const float4*>(xr + 4 * q);
          seg[4 * q] = v.x;
          seg[4 * q + 1] = v.y;
          seg[4 * q + 2] = v.z;
          seg[4 * q + 3] = v.w;
        }
#pragma unroll
        for (int q = L4 * 4; q < L; ++q) seg[q] = xr[q];
#pragma unroll
        for (int kw = 0; kw < KW_; ++kw) {
          float4 w4[FV / 4];
          const float4* wp = reinterpret_cast<const float4*>(wr + (size_t)kw * cc_max * FB);
#pragma unroll
          for (int j = 0; j < FV / 4; ++j) w4[j] = wp[j];
          float xv[PX];
#pragma unroll
          for (int i = 0; i < PX; ++i) xv[i] = seg[i * SW_ + kw];
          fma_tile(acc, xv, w4);
        }
      } else {
        for (int kw = 0; kw < KW; ++kw) {
          float4 w4[FV / 4];
          const float4* wp = reinterpret_cast<const float4*>(wr + (size_t)kw * cc_max * FB);
#pragma unroll
          for (int j = 0; j < FV / 4; ++j) w4[j] = wp[j];
          float xv[PX];
#pragma unroll
          for (int i = 0; i < PX; ++i) xv[i] = xr[i * SW + kw];
          fma_tile(acc, xv, w4);
        }
      }
    }
  }
}

// filter chunk (channels [c0, c0 + cc) of feature block fb0): ws[(tap * cc_max + c) * FB + f], features
// fastest (float4 where F % 4 == 0); loads unrolled so each thread's issue back to back
__device__ __forceinline__ void stage_filter(float* ws, const float* __restrict__ filt, int C, int F, int KH, int KW,
                                             int c0, int cc, int cc_max, int fb0, int FB, int t) {
  if ((F & 3) == 0) {
    const int fq = FB >> 2;
#pragma unroll 4
    for (int e = t; e < KH * KW * cc * fq; e += NT) {
      const int q = e % fq;
      const int c = (e / fq) % cc;
      const int tap = e / (fq * cc);
      const int f = fb0 + 4 * q;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (f < F) v = __ldg(reinterpret_cast<const float4*>(filt + ((int64_t)tap * C + c0 + c) * F + f));
      *reinterpret_cast<float4*>(ws + ((size_t)tap * cc_max + c) * FB + 4 * q) = v;
    }
  } else {
    for (int e = t; e < KH * KW * cc * FB; e += NT) {
      const int fl = e % FB;
      const int c = (e / FB) % cc;
      const int tap = e / (FB * cc);
      const int f = fb0 + fl;
      ws[((size_t)tap * cc_max + c) * FB + fl] = (f < F) ? __ldg(filt + ((int64_t)tap * C + c0 + c) * F + f) : 0.f;
    }
  }
}

__device__ __forceinline__ void store_tile(const float2 (&acc)[PX][FV / 2], float* __restrict__ out, int n, int HO,
                                           int WO, int F, int ho, int wo0, int f0) {
  if (ho >= HO) return;
#pragma unroll
  for (int i = 0; i < PX; ++i) {
    const int wo = wo0 + i;
    if (wo >= WO) continue;
    float* o = out + (((int64_t)n * HO + ho) * WO + wo) * F + f0;
    if ((F & 3) == 0 && f0 + FV <= F) {
#pragma unroll
      for (int j = 0; j < FV / 4; ++j)
        reinterpret_cast<float4*>(o)[j] = make_float4(acc[i][2 * j].x, acc[i][2 * j].y, acc[i][2 * j + 1].x,
                                                      acc[i][2 * j + 1].y);
    } else {
#pragma unroll
      for (int j = 0; j < FV / 2; ++j) {
        if (f0 + 2 * j < F) o[2 * j] = acc[i][j].x;
        if (f0 + 2 * j + 1 < F) o[2 * j + 1] = acc[i][j].y;
      }
    }
  }
}

// tile id -> (image, feature block, output tile): x = ((n * fblocks + fb) * htiles + ht) * wtiles + wt
struct TTile {
  int n, fb0, ho0, wo0;
};
__device__ __forceinline__ TTile tdecode(int64_t id, int wtiles, int htiles, int fblocks, int FB, int TH, int TW) {
  TTile r;
  const int wt = (int)(id % wtiles);
  const int ht = (int)((id / wtiles) % htiles);
  const int64_t nf = id / ((int64_t)wtiles * htiles);
  r.n = (int)(nf / fblocks);
  r.fb0 = (int)(nf % fblocks) * FB;
  r.ho0 = ht * TH;
  r.wo0 = wt * TW;
  return r;
}

// One CTA per tile, channel chunks staged in turn (multi-chunk layers).
template <int KW_, int SW_>
__global__ void __launch_bounds__(NT, 3) tiled_kernel(const float* __restrict__ in, const float* __restrict__ filt,
                                                      float* __restrict__ out, int H, int W, int C, int F, int KH,
                                                      int KWr, int SH, int SWr, int HO, int WO, int PT, int PL,
                                                      int cg, int wfg, int cc_max, int wtiles, int htiles,
                                                      int fblocks) {
  pdl_trigger();
  pdl_wait();
  const int KW = KW_ ? KW_ : KWr;
  const int SW = SW_ ? SW_ : SWr;
  extern __shared__ float4 smem4[];
  float* smem = reinterpret_cast<float*>(smem4);
  const int FB = FV * wfg;
  const int rows_w = 32 / cg;                 // pixel rows per warp block
  const int TH = rows_w * (NW / wfg), TW = cg * PX;
  const int IH = (TH - 1) * SH + KH, IW = (TW - 1) * SW + KW, IWP = (IW + 3) & ~3;
  const TTile tl = tdecode(blockIdx.x, wtiles, htiles, fblocks, FB, TH, TW);
  const int ih0 = tl.ho0 * SH - PT, iw0 = tl.wo0 * SW - PL;

  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int fg = warp % wfg, pb = warp / wfg;
  const int row = pb * rows_w + lane / cg;     // output row within the tile
  const int colg = lane % cg;                  // 4-pixel column group

  float* xs = smem;                                        // [cc][IH][IWP]
  float* ws = smem + (size_t)cc_max * IH * IWP;             // [KH*KW][cc][FB]

  float2 acc[PX][FV / 2];
#pragma unroll
  for (int i = 0; i < PX; ++i)
#pragma unroll
    for (int j = 0; j < FV / 2; ++j) acc[i][j] = make_float2(0.f, 0.f);

  const float* xin = in + (int64_t)tl.n * H * W * C;
  const bool vec_c = (C & 3) == 0 && (cc_max & 3) == 0;
  for (int c0 = 0; c0 < C; c0 += cc_max) {
    const int cc = (C - c0) < cc_max ? (C - c0) : cc_max;
    __syncthreads();  // previous chunk fully consumed
    // staging loops are unrolled so each thread's global loads issue back to back
    if (vec_c) {  // 4 channels per float4 load; cc is a multiple of 4 (host rounds cc_max; C % 4 == 0)
      const int cq = cc >> 2;
#pragma unroll 4
      for (int e = t; e < IH * IW * cq; e += NT) {
        const int q = e % cq;
        const int pix = e / cq;
        const int col = pix % IW, r = pix / IW;
        const int ih = ih0 + r, iw = iw0 + col;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (ih >= 0 && ih < H && iw >= 0 && iw < W)
          v = __ldg(reinterpret_cast<const float4*>(xin + ((int64_t)ih * W + iw) * C + c0) + q);
        float* d = xs + ((size_t)(4 * q) * IH + r) * IWP + col;
        d[0] = v.x;
        d[(size_t)IH * IWP] = v.y;
        d[(size_t)2 * IH * IWP] = v.z;
        d[(size_t)3 * IH * IWP] = v.w;
      }
    } else {
#pragma unroll 8
      for (int e = t; e < IH * IW * cc; e += NT) {
        const int c = e % cc;
        const int pix = e / cc;
        const int col = pix % IW, r = pix / IW;
        const int ih = ih0 + r, iw = iw0 + col;
        float v = 0.f;
        if (ih >= 0 && ih < H && iw >= 0 && iw < W) v = __ldg(xin + ((int64_t)ih * W + iw) * C + c0 + c);
        xs[((size_t)c * IH + r) * IWP + col] = v;
      }
    }
    stage_filter(ws, filt, C, F, KH, KW, c0, cc, cc_max, tl.fb0, FB, t);
    __syncthreads();
    chunk_mac<KW_, SW_>(acc, xs, ws, cc, cc_max, IH, IWP, KH, KW, SH, SW, row, colg, fg, FB);
  }
  store_tile(acc, out, tl.n, HO, WO, F, tl.ho0 + row, tl.wo0 + colg * PX, tl.fb0 + fg * FV);
}

// Persistent form for single-chunk layers (C <= the chunk): grid-stride over tiles; each thread owns PF halo
// elements (element e = t + k*NT of the channel-major halo, or of its channel quads when VEC) whose smem slot and
// relative input offset are computed once; the next tile's elements are loaded into registers before the
// current tile's FMAs, so their latency overlaps them.  The filter block is staged once per feature block
// (a CTA's consecutive tiles change it only when fblocks > 1).
template <int KW_, int SW_, bool VEC>
__global__ void __launch_bounds__(NT, 3) tiled_pipe_kernel(const float* __restrict__ in, const float* __restrict__ filt,
                                                           float* __restrict__ out, int H, int W, int C, int F,
                                                           int KH, int KWr, int SH, int SWr, int HO, int WO, int PT,
                                                           int PL, int cg, int wfg, int wtiles, int htiles,
                                                           int fblocks, int64_t ntiles, int pf) {
  pdl_trigger();
  pdl_wait();
  const int KW = KW_ ? KW_ : KWr;
  const int SW = SW_ ? SW_ : SWr;
  extern __shared__ float4 smem4[];
  float* smem = reinterpret_cast<float*>(smem4);
  const int FB = FV * wfg;
  const int rows_w = 32 / cg;
  const int TH = rows_w * (NW / wfg), TW = cg * PX;
  const int IH = (TH - 1) * SH + KH, IW = (TW - 1) * SW + KW, IWP = (IW + 3) & ~3;
  const int cc = C;  // one chunk
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int fg = warp % wfg, pb = warp / wfg;
  const int row = pb * rows_w + lane / cg;
  const int colg = lane % cg;
  float* xs = smem;                                   // [C][IH][IWP]
  float* ws = smem + (size_t)cc * IH * IWP;           // [KH*KW][C][FB]

  // this thread's halo elements e = t + k*NT, packed once as (r << 20 | col << 4 | q), or -1 past the halo:
  // channel (quad) q of halo pixel (r, col); smem slot and input offset are recomputed from it on use
  constexpr int KP = VEC ? PFMAX / 2 : PFMAX;
  const int per = VEC ? C / 4 : C;                    // elements per halo pixel (<= 16: one chunk)
  const int nel = IH * IW * per;
  int el[KP];
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    const int e = t + k * NT;
    const int q = e % per, pix = e / per;
    el[k] = e < nel ? ((pix / IW) << 20 | (pix % IW) << 4 | q) : -1;
  }
  using V = typename std::conditional<VEC, float4, float>::type;
  V pv[KP];
  auto prefetch = [&](int64_t id) {
    const TTile tl = tdecode(id, wtiles, htiles, fblocks, FB, TH, TW);
    const int ih0 = tl.ho0 * SH - PT, iw0 = tl.wo0 * SW - PL;
    const float* base = in + (int64_t)tl.n * H * W * C;
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      if (k < pf) {
        const int r = el[k] >> 20, col = (el[k] >> 4) & 0xFFFF, q = el[k] & 15;
        const int ih = ih0 + r, iw = iw0 + col;
        const bool in_img = el[k] >= 0 && ih >= 0 && ih < H && iw >= 0 && iw < W;
        const float* src = base + ((int64_t)ih * W + iw) * C + (VEC ? 4 * q : q);
        if constexpr (VEC)
          pv[k] = in_img ? __ldg(reinterpret_cast<const float4*>(src)) : make_float4(0.f, 0.f, 0.f, 0.f);
        else
          pv[k] = in_img ? __ldg(src) : 0.f;
      }
    }
  };
  int cur_fb = -1;
  int64_t id = blockIdx.x;
  if (id < ntiles) prefetch(id);
  for (; id < ntiles; id += gridDim.x) {
    const TTile tl = tdecode(id, wtiles, htiles, fblocks, FB, TH, TW);
    __syncthreads();  // the previous tile's FMAs are done with xs (and ws)
    if (tl.fb0 != cur_fb) {
      stage_filter(ws, filt, C, F, KH, KW, 0, cc, cc, tl.fb0, FB, t);
      cur_fb = tl.fb0;
    }
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      if (k < pf && el[k] >= 0) {
        const int r = el[k] >> 20, col = (el[k] >> 4) & 0xFFFF, q = el[k] & 15;
        const int slot = ((VEC ? 4 * q : q) * IH + r) * IWP + col;
        if constexpr (VEC) {
          float* d = xs + slot;
          d[0] = pv[k].x;
          d[(size_t)IH * IWP] = pv[k].y;
          d[(size_t)2 * IH * IWP] = pv[k].z;
          d[(size_t)3 * IH * IWP] = pv[k].w;
        } else {
          xs[slot] = pv[k];
        }
      }
    }
    __syncthreads();
    if (id + gridDim.x < ntiles) prefetch(id + gridDim.x);  // in flight during the FMAs below
    float2 acc[PX][FV / 2];
#pragma unroll
    for (int i = 0; i < PX; ++i)
#pragma unroll
      for (int j = 0; j < FV / 2; ++j) acc[i][j] = make_float2(0.f, 0.f);
    chunk_mac<KW_, SW_>(acc, xs, ws, cc, cc, IH, IWP, KH, KW, SH, SW, row, colg, fg, FB);
    store_tile(acc, out, tl.n, HO, WO, F, tl.ho0 + row, tl.wo0 + colg * PX, tl.fb0 + fg * FV);
  }
}

template <int KW_, int SW_>
cudaError_t launch_t(const Problem& p, const TGeo& g, const float* in, const float* filt, float* out, cudaStream_t s) {
  const int fblocks = (p.F + g.fb - 1) / g.fb;
  const int wtiles = (p.WO + g.tw - 1) / g.tw, htiles = (p.HO + g.th - 1) / g.th;
  static const bool nopipe = getenv("CONV2D_TILED_NOPIPE") != nullptr;  // A/B: the per-tile form only
  if (g.pf > 0 && !nopipe) {
    auto kern = g.vec ? tiled_pipe_kernel<KW_, SW_, true> : tiled_pipe_kernel<KW_, SW_, false>;
    const cudaError_t e = g.vec ? smem_attr_once<tiled_pipe_kernel<KW_, SW_, true>>(SMEM_BUDGET)
                                : smem_attr_once<tiled_pipe_kernel<KW_, SW_, false>>(SMEM_BUDGET);
    if (e != cudaSuccess) return e;
    const int64_t grid = g.ntiles < 148 * 3 ? g.ntiles : 148 * 3;  // three CTAs per SM, persistent
    return launch_k(kern, dim3((unsigned)grid), dim3(NT), g.smem_pipe, s, in, filt, out, p.H, p.W, p.C, p.F, p.KH,
                    p.KW, p.SH, p.SW, p.HO, p.WO, p.pad_top, p.pad_left, g.cg, g.wfg, wtiles, htiles, fblocks,
                    g.ntiles, g.pf);
  }
  const cudaError_t e = smem_attr_once<tiled_kernel<KW_, SW_>>(SMEM_BUDGET);
  if (e != cudaSuccess) return e;
  return launch_k(tiled_kernel<KW_, SW_>, dim3((unsigned)g.ntiles), dim3(NT), g.smem, s, in, filt, out, p.H, p.W,
                  p.C, p.F, p.KH, p.KW, p.SH, p.SW, p.HO, p.WO, p.pad_top, p.pad_left, g.cg, g.wfg, g.cc, wtiles,
                  htiles, fblocks);
}

}  // namespace

bool tiled_supported(const Problem& p) { return geometry(p).ok; }

cudaError_t launch_tiled(const Problem& p, const float* in, const float* filt, float* out, cudaStream_t s) {
  const TGeo g = geometry(p);
  if (!g.ok) return cudaErrorInvalidConfiguration;  // algo_supports(TILED) == tiled_supported() rejects these
  if (p.KW == 1 && p.SW == 1) return launch_t<1, 1>(p, g, in, filt, out, s);
  if (p.KW == 1 && p.SW == 2) return launch_t<1, 2>(p, g, in, filt, out, s);
  if (p.KW == 3 && p.SW == 1) return launch_t<3, 1>(p, g, in, filt, out, s);
  if (p.KW == 3 && p.SW == 2) return launch_t<3, 2>(p, g, in, filt, out, s);
  if (p.KW == 5 && p.SW == 1) return launch_t<5, 1>(p, g, in, filt, out, s);
  if (p.KW == 7 && p.SW == 2) return launch_t<7, 2>(p, g, in, filt, out, s);
  return launch_t<0, 0>(p, g, in, filt, out, s);
}

}  // namespace conv2d
