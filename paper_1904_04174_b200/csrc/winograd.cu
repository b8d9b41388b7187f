// winograd.cu -- CONV2D_ALGO_WINOGRAD_F2X2_3X3 and CONV2D_ALGO_WINOGRAD_F4X4_3X3 (the
// "Winograd large" variant; same pipeline with 6x6 tiles, 36 batched GEMMs, 4x fewer multiplies than
// direct; FP32 math only -- DESIGN.md reading R21): "a tiled Winograd operation which uses
// data transforms to convert the convolution into a number of small matrix multiplies,
// reducing the total number of floating point operations" (
// SPEC.md:258-266; Lavin & Gray F(2x2,3x3), correlation form, reading R12):
//
//   U  = G g G^T          per (c, f)                      (filter transform)
//   V  = B^T d B          per (4x4 input tile, c)          (input transform, tiles overlap by 2)
//   M_xi = sum_c U_xi[c,f] V_xi[t,c]   for the 16 xi       (16 batched tcgen05 GEMMs)
//   Y  = A^T M A          per (tile, f) -> 2x2 outputs     (output transform)
//
//   B^T = [[1,0,-1,0],[0,1,1,0],[0,-1,1,0],[0,1,0,-1]]
//   G   = [[1,0,0],[1/2,1/2,1/2],[1/2,-1/2,1/2],[0,0,1]]
//   A^T = [[1,1,1,0],[0,1,-1,-1]]
//
// Tiles: T = N * ceil(Ho/2) * ceil(Wo/2); odd Ho/Wo extend the grid with zero input and
// the surplus outputs are discarded.  Multiplies per 2x2 output tile: 16 vs 36 direct.
// This file: the transforms as separate bandwidth kernels with V and M staged in the workspace and the
// GEMMs on the tensor cores (parameter variant 0).  F(2x2) variant 1 is the fused kernel (wino_fused.cu);
// the auto-selector times both per layer.
// TF32 mode rounds U and V to TF32 with cvt.rna (reading R16); FP32 mode runs the GEMMs
// in 3xTF32.
#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "gemm2sm.h"
#include "launch.cuh"
#include "sm100.cuh"

namespace conv2d {
namespace {

inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// 1-D transforms of one column (applied along both axes).
// F(2x2,3x3) (Lavin-Gray): G g, B^T d, A^T m
__device__ __forceinline__ void g2(const float* g, float* u) {
  u[0] = g[0];
  u[1] = 0.5f * (g[0] + g[1] + g[2]);
  u[2] = 0.5f * (g[0] - g[1] + g[2]);
  u[3] = g[2];
}
__device__ __forceinline__ void bt2(const float* d, float* v) {
  v[0] = d[0] - d[2];
  v[1] = d[1] + d[2];
  v[2] = d[2] - d[1];
  v[3] = d[1] - d[3];
}
__device__ __forceinline__ void at2(const float* m, float* y) {
  y[0] = m[0] + m[1] + m[2];
  y[1] = m[1] - m[2] - m[3];
}
// F(4x4,3x3) (Lavin-Gray, points 0, +-1, +-2, inf):
//   G   = [[1/4,0,0],[-1/6,-1/6,-1/6],[-1/6,1/6,-1/6],[1/24,1/12,1/6],[1/24,-1/12,1/6],[0,0,1]]
//   B^T = [[4,0,-5,0,1,0],[0,-4,-4,1,1,0],[0,4,-4,-1,1,0],[0,-2,-1,2,1,0],[0,2,-1,-2,1,0],[0,4,0,-5,0,1]]
//   A^T = [[1,1,1,1,1,0],[0,1,-1,2,-2,0],[0,1,1,4,4,0],[0,1,-1,8,-8,1]]
__device__ __forceinline__ void g4(const float* g, float* u) {
  u[0] = 0.25f * g[0];
  u[1] = -(g[0] + g[1] + g[2]) * (1.f / 6.f);
  u[2] = -(g[0] - g[1] + g[2]) * (1.f / 6.f);
  u[3] = g[0] * (1.f / 24.f) + g[1] * (1.f / 12.f) + g[2] * (1.f / 6.f);
  u[4] = g[0] * (1.f / 24.f) - g[1] * (1.f / 12.f) + g[2] * (1.f / 6.f);
  u[5] = g[2];
}
__device__ __forceinline__ void bt4(const float* d, float* v) {
  v[0] = 4.f * d[0] - 5.f * d[2] + d[4];
  v[1] = -4.f * d[1] - 4.f * d[2] + d[3] + d[4];
  v[2] = 4.f * d[1] - 4.f * d[2] - d[3] + d[4];
  v[3] = -2.f * d[1] - d[2] + 2.f * d[3] + d[4];
  v[4] = 2.f * d[1] - d[2] - 2.f * d[3] + d[4];
  v[5] = 4.f * d[1] - 5.f * d[3] + d[5];
}
__device__ __forceinline__ void at4(const float* m, float* y) {
  y[0] = m[0] + m[1] + m[2] + m[3] + m[4];
  y[1] = m[1] - m[2] + 2.f * m[3] - 2.f * m[4];
  y[2] = m[1] + m[2] + 4.f * m[3] + 4.f * m[4];
  y[3] = m[1] - m[2] + 8.f * m[3] - 8.f * m[4] + m[5];
}
template <int MT> __device__ __forceinline__ void gT(const float* g, float* u) { if (MT == 2) g2(g, u); else g4(g, u); }
template <int MT> __device__ __forceinline__ void bT(const float* d, float* v) { if (MT == 2) bt2(d, v); else bt4(d, v); }
template <int MT> __device__ __forceinline__ void aT(const float* m, float* y) { if (MT == 2) at2(m, y); else at4(m, y); }

// U_xi stored K-major per xi: Ut[xi][f][c], Fpad rows x Cpad cols; U = G g G^T (ALPHA x ALPHA).
// One block per 32 (c) x 8 (f) tile (one (c, f) per thread): the nine HWCF taps are read f-fastest into
// smem, then each thread transforms its (c, f) with c fastest so the Ut stores are coalesced too.
template <int MT>
__device__ __forceinline__ void wino_filter_tile(const float* __restrict__ w, int C, int F, int64_t cpad, int64_t fpad,
                                                 float* __restrict__ ut_hi, float* __restrict__ ut_lo, int mode,
                                                 int bx, int by) {
  constexpr int AL = MT + 2;
  __shared__ float g_s[9][8][33];  // [tap][f][c]
  const int c0 = bx * 32, f0 = by * 8;
  for (int q = threadIdx.x; q < 9 * 32 * 8; q += blockDim.x) {  // q = (tap, c, f), f fastest
    const int fl = q % 8, cl = (q / 8) % 32, tap = q / 256;
    const int c = c0 + cl, f = f0 + fl;
    g_s[tap][fl][cl] = (c < C && f < F) ? w[((int64_t)tap * C + c) * F + f] : 0.f;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < 32 * 8; q += blockDim.x) {  // q = (f, c), c fastest
    const int cl = q % 32, fl = q / 32;
    const int c = c0 + cl, f = f0 + fl;
    if (c >= cpad || f >= fpad) continue;
    float u[AL][AL];
    float t[AL][3];  // G g, column by column
#pragma unroll
    for (int sc = 0; sc < 3; ++sc) {
      float col[3], out[AL];
#pragma unroll
      for (int r = 0; r < 3; ++r) col[r] = g_s[r * 3 + sc][fl][cl];
      gT<MT>(col, out);
#pragma unroll
      for (int r = 0; r < AL; ++r) t[r][sc] = out[r];
    }
#pragma unroll
    for (int r = 0; r < AL; ++r) gT<MT>(t[r], u[r]);  // (G g) G^T
#pragma unroll
    for (int xi = 0; xi < AL * AL; ++xi) {
      const float v = u[xi / AL][xi % AL];
      const int64_t o = ((int64_t)xi * fpad + f) * cpad + c;
      if (mode == 0) {
        const float h = sm100::tf32_hi(v);
        ut_hi[o] = h;
        ut_lo[o] = v - h;
      } else {
        ut_hi[o] = tf32_rna(v);
      }
    }
  }
}

// V[xi][t][c] (row stride cpad), t = (n, th, tw); V = B^T d B over the ALPHA x ALPHA input tile at
// (MT*th - PT, MT*tw - PL) (tiles overlap by 2).  VEC: four consecutive channels per thread (float4 loads
// and stores; C % 4 == 0), channel groups fastest so a warp's accesses are contiguous.
template <int MT, int NV>
__device__ __forceinline__ void wino_input_body(const float* __restrict__ x, int H, int W, int C, int TH, int TW,
                                                int PT, int PL, int64_t T, int64_t cpad, float* __restrict__ V,
                                                int round_rna, int64_t blk, int64_t nblk) {
  constexpr int AL = MT + 2;
  const int64_t cg_n = cpad / NV;
  const int64_t total = T * cg_n;
  for (int64_t i = blk * blockDim.x + threadIdx.x; i < total; i += nblk * blockDim.x) {
    const int c0 = (int)(i % cg_n) * NV;
    const int64_t t = i / cg_n;
    const int tw = (int)(t % TW);
    const int th = (int)((t / TW) % TH);
    const int64_t n = t / ((int64_t)TW * TH);
    float d[NV][AL][AL];
    const int h0 = MT * th - PT, w0 = MT * tw - PL;
#pragma unroll
    for (int a = 0; a < AL; ++a)
#pragma unroll
      for (int b = 0; b < AL; ++b) {
        const int ih = h0 + a, iw = w0 + b;
        const bool in = c0 < C && ih >= 0 && ih < H && iw >= 0 && iw < W;
        const float* src = x + ((n * H + ih) * W + iw) * C + c0;
        if constexpr (NV == 4) {
          const float4 v = in ? __ldg(reinterpret_cast<const float4*>(src)) : make_float4(0.f, 0.f, 0.f, 0.f);
          d[0][a][b] = v.x;
          d[1][a][b] = v.y;
          d[2][a][b] = v.z;
          d[3][a][b] = v.w;
        } else if constexpr (NV == 2) {
          const float2 v = in ? __ldg(reinterpret_cast<const float2*>(src)) : make_float2(0.f, 0.f);
          d[0][a][b] = v.x;
          d[1][a][b] = v.y;
        } else {
          d[0][a][b] = in ? src[0] : 0.f;
        }
      }
    float out[NV][AL][AL];
#pragma unroll
    for (int e = 0; e < NV; ++e) {
      float q[AL][AL];  // B^T d, column by column
#pragma unroll
      for (int b = 0; b < AL; ++b) {
        float col[AL], o[AL];
#pragma unroll
        for (int a = 0; a < AL; ++a) col[a] = d[e][a][b];
        bT<MT>(col, o);
#pragma unroll
        for (int a = 0; a < AL; ++a) q[a][b] = o[a];
      }
#pragma unroll
      for (int a = 0; a < AL; ++a) bT<MT>(q[a], out[e][a]);  // (B^T d) B
    }
#pragma unroll
    for (int a = 0; a < AL; ++a)
#pragma unroll
      for (int b = 0; b < AL; ++b) {
        float* dst = V + ((int64_t)(a * AL + b) * T + t) * cpad + c0;
        if constexpr (NV == 4) {
          float4 v = make_float4(out[0][a][b], out[1][a][b], out[2][a][b], out[3][a][b]);
          if (round_rna) v = make_float4(tf32_rna(v.x), tf32_rna(v.y), tf32_rna(v.z), tf32_rna(v.w));
          *reinterpret_cast<float4*>(dst) = v;
        } else if constexpr (NV == 2) {
          float2 v = make_float2(out[0][a][b], out[1][a][b]);
          if (round_rna) v = make_float2(tf32_rna(v.x), tf32_rna(v.y));
          *reinterpret_cast<float2*>(dst) = v;
        } else {
          dst[0] = round_rna ? tf32_rna(out[0][a][b]) : out[0][a][b];
        }
      }
  }
}

// One launch for both operand transforms (they are independent): blocks [0, nfx*nfy) transform 32x8
// filter tiles, the rest run the input transform grid-stride -- one kernel boundary fewer per Winograd
// conv, and the filter work overlaps the input transform.
template <int MT, int NV>
__global__ void __launch_bounds__(256) wino_prep_kernel(const float* __restrict__ w, int C, int F, int64_t cpad,
                                                        int64_t fpad, float* __restrict__ ut_hi,
                                                        float* __restrict__ ut_lo, int mode, int nfx, int nfy,
                                                        const float* __restrict__ x, int H, int W, int TH, int TW,
                                                        int PT, int PL, int64_t T, float* __restrict__ V) {
  pdl_trigger();
  pdl_wait();
  const int nf = nfx * nfy;
  if ((int)blockIdx.x < nf)
    wino_filter_tile<MT>(w, C, F, cpad, fpad, ut_hi, ut_lo, mode, (int)blockIdx.x % nfx, (int)blockIdx.x / nfx);
  else
    wino_input_body<MT, NV>(x, H, W, C, TH, TW, PT, PL, T, cpad, V, mode, (int64_t)blockIdx.x - nf,
                            (int64_t)gridDim.x - nf);
}

// Y tile (MT x MT) = A^T M A, M[xi][t][f] (row stride ldm).  VEC: four consecutive features per thread
// (float4; F % 4 == 0), feature groups fastest.
template <int MT, bool VEC>
__global__ void wino_output_kernel(const float* __restrict__ Mw, int64_t T, int64_t ldm, int F, int HO, int WO,
                                   int TH, int TW, float* __restrict__ y) {
  pdl_trigger();
  pdl_wait();
  constexpr int AL = MT + 2;
  constexpr int NV = VEC ? 4 : 1;
  const int64_t fg_n = F / NV;
  const int64_t total = T * fg_n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int f0 = (int)(i % fg_n) * NV;
    const int64_t t = i / fg_n;
    float m[NV][AL][AL];
#pragma unroll
    for (int xi = 0; xi < AL * AL; ++xi) {
      const float* src = Mw + ((int64_t)xi * T + t) * ldm + f0;
      if constexpr (VEC) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(src));
        m[0][xi / AL][xi % AL] = v.x;
        m[1][xi / AL][xi % AL] = v.y;
        m[2][xi / AL][xi % AL] = v.z;
        m[3][xi / AL][xi % AL] = v.w;
      } else {
        m[0][xi / AL][xi % AL] = src[0];
      }
    }
    const int tw = (int)(t % TW);
    const int th = (int)((t / TW) % TH);
    const int64_t n = t / ((int64_t)TW * TH);
    float yy[NV][MT][MT];
#pragma unroll
    for (int e = 0; e < NV; ++e) {
      float r[MT][AL];  // A^T M, column by column
#pragma unroll
      for (int b = 0; b < AL; ++b) {
        float col[AL], o[MT];
#pragma unroll
        for (int a = 0; a < AL; ++a) col[a] = m[e][a][b];
        aT<MT>(col, o);
#pragma unroll
        for (int a = 0; a < MT; ++a) r[a][b] = o[a];
      }
#pragma unroll
      for (int a = 0; a < MT; ++a) aT<MT>(r[a], yy[e][a]);  // (A^T M) A
    }
#pragma unroll
    for (int a = 0; a < MT; ++a) {
      const int ho = MT * th + a;
      if (ho >= HO) continue;
#pragma unroll
      for (int b = 0; b < MT; ++b) {
        const int wo = MT * tw + b;
        if (wo >= WO) continue;
        float* dst = y + ((n * HO + ho) * WO + wo) * F + f0;
        if constexpr (VEC) *reinterpret_cast<float4*>(dst) = make_float4(yy[0][a][b], yy[1][a][b], yy[2][a][b], yy[3][a][b]);
        else dst[0] = yy[0][a][b];
      }
    }
  }
}

struct WPlan {
  int mt, xi;  // output tile MT x MT, XI = (MT + 2)^2 transformed points = batched GEMMs
  bool three_x;
  int block_n, splits;
  int TH, TW;
  int64_t T, cpad, fpad, ldm;
  size_t ut_bytes, v_bytes, m_bytes, partial_bytes, total;
};

WPlan make_wplan(const Problem& p, int mt) {
  WPlan w{};
  w.mt = mt;
  w.xi = (mt + 2) * (mt + 2);
  w.three_x = p.math == CONV2D_MATH_FP32;
  w.TH = (p.HO + mt - 1) / mt;
  w.TW = (p.WO + mt - 1) / mt;
  w.T = (int64_t)p.N * w.TH * w.TW;
  w.cpad = round_up(p.C, 32);
  w.block_n = gemm2_choose_block_n(p.F);
  w.fpad = round_up(p.F, w.block_n);
  w.ldm = round_up(p.F, 4);
  w.splits = gemm2_choose_splits(w.T, p.F, (int)(w.cpad / 32), w.xi, w.block_n);
  if (w.ldm != p.F) w.splits = 1;
  w.ut_bytes = round_up(w.xi * w.fpad * w.cpad * 4, 256);
  w.v_bytes = round_up(w.xi * w.T * w.cpad * 4, 256);
  w.m_bytes = round_up(w.xi * w.T * w.ldm * 4, 256);
  w.partial_bytes = w.splits > 1 ? (size_t)w.splits * w.m_bytes : 0;
  w.total = w.ut_bytes * (w.three_x ? 2 : 1) + w.v_bytes + w.m_bytes + w.partial_bytes;
  return w;
}

unsigned grid_for(int64_t total) {
  int64_t b = (total + 255) / 256;
  if (b > 148 * 32) b = 148 * 32;
  return (unsigned)(b < 1 ? 1 : b);
}

// filter transform alone (the fused F(2x2) path, wino_fused.cu): one 128-thread block per 32 (c) x 8 (f) tile
template <int MT>
__global__ void __launch_bounds__(128) wino_filter_kernel(const float* __restrict__ w, int C, int F, int64_t cpad,
                                                          int64_t fpad, float* __restrict__ ut_hi,
                                                          float* __restrict__ ut_lo, int mode, int nfx) {
  pdl_trigger();
  pdl_wait();
  wino_filter_tile<MT>(w, C, F, cpad, fpad, ut_hi, ut_lo, mode, (int)blockIdx.x % nfx, (int)blockIdx.x / nfx);
}

// F(2x2) parameter variant (the auto-selector times both): 0 = the transform kernels +
// batched GEMM below, 1 = the fused kernel (wino_fused.cu).  Default 0: the fused kernel is shared-memory-port
// bound with 32-feature MMAs, so it wins only on some shapes.
using WVKey = std::tuple<int, int, int, int, int, int, int, int, int, int, int>;
std::mutex g_wvmu;
std::map<WVKey, int> g_wvariant;
WVKey wvkey(const Problem& p) {
  return WVKey(p.N, p.H, p.W, p.C, p.F, p.KH, p.KW, p.SH, p.SW, p.pad_top * 64 + p.pad_left, (int)p.math);
}
int wvariant_of(const Problem& p) {
  if (const char* f = getenv("CONV2D_FORCE_WINO_VARIANT")) return atoi(f) & 1;  // parity-test hook
  std::lock_guard<std::mutex> lk(g_wvmu);
  auto it = g_wvariant.find(wvkey(p));
  return it == g_wvariant.end() ? 0 : it->second;
}
bool use_fused(const Problem& p, int mt) { return mt == 2 && wvariant_of(p) == 1 && wino_fused_ok(p); }

}  // namespace

int winograd_variants(const Problem& p, int* masks) {
  masks[0] = 0;
  if (!wino_fused_ok(p)) return 1;
  masks[1] = 1;
  return 2;
}
bool winograd_get_variant(const Problem& p, int* v) {
  std::lock_guard<std::mutex> lk(g_wvmu);
  auto it = g_wvariant.find(wvkey(p));
  if (it == g_wvariant.end()) return false;
  *v = it->second;
  return true;
}
void winograd_set_variant(const Problem& p, int v) {
  std::lock_guard<std::mutex> lk(g_wvmu);
  g_wvariant[wvkey(p)] = v;
}

cudaError_t launch_wino_filter(int mt, const float* w, int C, int F, int64_t cpad, int64_t fpad, float* ut_hi,
                               float* ut_lo, bool three_x, cudaStream_t s) {
  const int nfx = (int)(cpad / 32), nfy = (int)((fpad + 7) / 8);
  return launch_k(mt == 2 ? wino_filter_kernel<2> : wino_filter_kernel<4>, dim3((unsigned)(nfx * nfy)), dim3(128), 0,
                  s, w, C, F, cpad, fpad, ut_hi, ut_lo, three_x ? 0 : 1, nfx);
}

size_t winograd_workspace(const Problem& p, int mt) {
  const size_t unfused = make_wplan(p, mt).total;
  return mt == 2 ? std::max(unfused, wino_fused_workspace(p)) : unfused;
}
int winograd_launches(const Problem& p, int mt) {
  if (use_fused(p, mt)) return 2;
  return 3 + (make_wplan(p, mt).splits > 1 ? 1 : 0);
}
int winograd_splits(const Problem& p, int mt) { return use_fused(p, mt) ? 1 : make_wplan(p, mt).splits; }

cudaError_t launch_winograd(const Problem& p, int mt, const float* in, const float* filt, float* out, void* ws,
                            cudaStream_t s) {
  // F(2x2) variant 1: the fused kernel (wino_fused.cu), when the pointers are TMA-aligned
  if (use_fused(p, mt) && ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0)
    return launch_wino_fused(p, in, filt, out, ws, s);
  const WPlan w = make_wplan(p, mt);
  uint8_t* b = static_cast<uint8_t*>(ws);
  float* ut_hi = reinterpret_cast<float*>(b);
  b += w.ut_bytes;
  float* ut_lo = nullptr;
  if (w.three_x) {
    ut_lo = reinterpret_cast<float*>(b);
    b += w.ut_bytes;
  }
  float* V = reinterpret_cast<float*>(b);
  b += w.v_bytes;
  float* Mw = reinterpret_cast<float*>(b);
  b += w.m_bytes;
  float* partial = w.splits > 1 ? reinterpret_cast<float*>(b) : nullptr;

  // input transform: F(2x2) moves 4 channels per thread; F(4x4) 2 (its 6x6 tiles would otherwise need ~190
  // registers per thread and run at 12% occupancy)
  const int nvin = (p.C % 4 == 0 && (reinterpret_cast<uintptr_t>(in) & 15) == 0) ? (mt == 2 ? 4 : 2)
                   : (p.C % 2 == 0 && (reinterpret_cast<uintptr_t>(in) & 7) == 0) ? 2 : 1;  // cpad % 32 == 0
  const bool vout = p.F % 4 == 0 && w.ldm % 4 == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  auto kp = mt == 2 ? (nvin == 4 ? wino_prep_kernel<2, 4> : nvin == 2 ? wino_prep_kernel<2, 2> : wino_prep_kernel<2, 1>)
                    : (nvin == 4 ? wino_prep_kernel<4, 4> : nvin == 2 ? wino_prep_kernel<4, 2> : wino_prep_kernel<4, 1>);
  auto ko = mt == 2 ? (vout ? wino_output_kernel<2, true> : wino_output_kernel<2, false>)
                    : (vout ? wino_output_kernel<4, true> : wino_output_kernel<4, false>);
  const int nfx = (int)(w.cpad / 32), nfy = (int)((w.fpad + 7) / 8);
  // 128-thread blocks: the 128-register input transform fits 4 per SM instead of 2 x 256 (same warps, half the
  // tail granularity; measured R10 / R24 +1-1.5%).  The filter tiles loop over their 256 (c, f) items.
  static const int pt = getenv("CONV2D_WINO_PREP_THREADS") ? atoi(getenv("CONV2D_WINO_PREP_THREADS")) : 128;
  const int64_t in_blocks = std::min<int64_t>((w.T * w.cpad / nvin + pt - 1) / pt, 148LL * 32 * 256 / pt);
  cudaError_t e = launch_k(kp, dim3((unsigned)(nfx * nfy + in_blocks)), dim3(pt), 0, s, filt, p.C,
                           p.F, w.cpad, w.fpad, ut_hi, ut_lo, w.three_x ? 0 : 1, nfx, nfy, in, p.H, p.W, w.TH, w.TW,
                           p.pad_top, p.pad_left, w.T, V);
  if (e != cudaSuccess) return e;
  Gemm2Args g{};
  g.a_mode = A_DENSE;
  g.a = V;
  g.lda = w.cpad;
  g.a_k = w.cpad;
  g.bt_hi = ut_hi;
  g.bt_lo = ut_lo;
  g.kpad = w.cpad;
  g.npad = w.fpad;
  g.d = Mw;
  g.ldd = w.ldm;
  g.d_batch_stride = w.T * w.ldm;
  g.partial = partial;
  g.M = w.T;
  g.N = p.F;
  g.batch = w.xi;
  g.splits = w.splits;
  g.three_x = w.three_x;
  g.block_n = w.block_n;
  e = launch_gemm2(p, g, s);
  if (e != cudaSuccess) return e;
  // 128-thread blocks here too (measured R10 / R17 +2-3% over 256)
  static const int ot = getenv("CONV2D_WINO_OUT_THREADS") ? atoi(getenv("CONV2D_WINO_OUT_THREADS")) : 128;
  const int64_t out_blocks = std::min<int64_t>((w.T * p.F / (vout ? 4 : 1) + ot - 1) / ot, 148LL * 32 * 256 / ot);
  return launch_k(ko, dim3((unsigned)std::max<int64_t>(out_blocks, 1)), dim3(ot), 0, s, Mw, w.T, w.ldm, p.F, p.HO,
                  p.WO, w.TH, w.TW, out);
}

}  // namespace conv2d
