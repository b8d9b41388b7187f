// winograd.cu -- CONV2D_ALGO_WINOGRAD_F2X2_3X3: "a tiled Winograd operation which uses
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
// Round-1 form: transforms are separate CUDA-core kernels with V and M staged in the
// workspace (the GEMMs run on the tensor cores); the fused form is DESIGN.md "Next".
// TF32 mode rounds U and V to TF32 with cvt.rna (reading R16); FP32 mode runs the GEMMs
// in 3xTF32.
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

// U_xi stored K-major per xi: Ut[xi][f][c], Fpad rows x Cpad cols.
__global__ void wino_filter_kernel(const float* __restrict__ w, int C, int F, int64_t cpad, int64_t fpad,
                                   float* __restrict__ ut_hi, float* __restrict__ ut_lo, int mode /*0 3x,1 tf32*/) {
  pdl_trigger();
  pdl_wait();
  const int64_t total = cpad * fpad;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int f = (int)(i % fpad);
    const int c = (int)(i / fpad);
    float u[4][4];
    if (c < C && f < F) {
      float g[3][3];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int s = 0; s < 3; ++s) g[r][s] = w[((int64_t)(r * 3 + s) * C + c) * F + f];
      float t[4][3];  // G g
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        t[0][s] = g[0][s];
        t[1][s] = 0.5f * (g[0][s] + g[1][s] + g[2][s]);
        t[2][s] = 0.5f * (g[0][s] - g[1][s] + g[2][s]);
        t[3][s] = g[2][s];
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) {  // (G g) G^T
        u[r][0] = t[r][0];
        u[r][1] = 0.5f * (t[r][0] + t[r][1] + t[r][2]);
        u[r][2] = 0.5f * (t[r][0] - t[r][1] + t[r][2]);
        u[r][3] = t[r][2];
      }
    } else {
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int s = 0; s < 4; ++s) u[r][s] = 0.f;
    }
#pragma unroll
    for (int xi = 0; xi < 16; ++xi) {
      const float v = u[xi / 4][xi % 4];
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

// V[xi][t][c] (row stride cpad), t = (n, th, tw)
__global__ void wino_input_kernel(const float* __restrict__ x, int H, int W, int C, int TH, int TW, int PT, int PL,
                                  int64_t T, int64_t cpad, float* __restrict__ V, int round_rna) {
  pdl_trigger();
  pdl_wait();
  const int64_t total = T * cpad;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % cpad);
    const int64_t t = i / cpad;
    const int tw = (int)(t % TW);
    const int th = (int)((t / TW) % TH);
    const int64_t n = t / ((int64_t)TW * TH);
    float d[4][4];
    const int h0 = 2 * th - PT, w0 = 2 * tw - PL;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int ih = h0 + a, iw = w0 + b;
        d[a][b] = (c < C && ih >= 0 && ih < H && iw >= 0 && iw < W) ? x[((n * H + ih) * W + iw) * C + c] : 0.f;
      }
    float q[4][4];  // B^T d
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      q[0][b] = d[0][b] - d[2][b];
      q[1][b] = d[1][b] + d[2][b];
      q[2][b] = d[2][b] - d[1][b];
      q[3][b] = d[1][b] - d[3][b];
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {  // (B^T d) B
      const float v0 = q[a][0] - q[a][2];
      const float v1 = q[a][1] + q[a][2];
      const float v2 = q[a][2] - q[a][1];
      const float v3 = q[a][1] - q[a][3];
      const float vv[4] = {v0, v1, v2, v3};
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const float v = round_rna ? tf32_rna(vv[b]) : vv[b];
        V[((int64_t)(a * 4 + b) * T + t) * cpad + c] = v;
      }
    }
  }
}

// Y tile = A^T M A, M[xi][t][f] (row stride ldm)
__global__ void wino_output_kernel(const float* __restrict__ Mw, int64_t T, int64_t ldm, int F, int HO, int WO,
                                   int TH, int TW, float* __restrict__ y) {
  pdl_trigger();
  pdl_wait();
  const int64_t total = T * F;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int f = (int)(i % F);
    const int64_t t = i / F;
    float m[4][4];
#pragma unroll
    for (int xi = 0; xi < 16; ++xi) m[xi / 4][xi % 4] = Mw[((int64_t)xi * T + t) * ldm + f];
    float r[2][4];  // A^T M
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      r[0][b] = m[0][b] + m[1][b] + m[2][b];
      r[1][b] = m[1][b] - m[2][b] - m[3][b];
    }
    const int tw = (int)(t % TW);
    const int th = (int)((t / TW) % TH);
    const int64_t n = t / ((int64_t)TW * TH);
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const float y0 = r[a][0] + r[a][1] + r[a][2];
      const float y1 = r[a][1] - r[a][2] - r[a][3];
      const int ho = 2 * th + a;
      if (ho >= HO) continue;
      const int wo = 2 * tw;
      y[((n * HO + ho) * WO + wo) * F + f] = y0;
      if (wo + 1 < WO) y[((n * HO + ho) * WO + wo + 1) * F + f] = y1;
    }
  }
}

struct WPlan {
  bool three_x;
  int block_n, splits;
  int TH, TW;
  int64_t T, cpad, fpad, ldm;
  size_t ut_bytes, v_bytes, m_bytes, partial_bytes, total;
};

WPlan make_wplan(const Problem& p) {
  WPlan w{};
  w.three_x = p.math == CONV2D_MATH_FP32;
  w.TH = (p.HO + 1) / 2;
  w.TW = (p.WO + 1) / 2;
  w.T = (int64_t)p.N * w.TH * w.TW;
  w.cpad = round_up(p.C, 32);
  w.block_n = gemm2_choose_block_n(p.F);
  w.fpad = round_up(p.F, w.block_n);
  w.ldm = round_up(p.F, 4);
  w.splits = gemm2_choose_splits(w.T, p.F, (int)(w.cpad / 32), 16, w.block_n);
  if (w.ldm != p.F) w.splits = 1;
  w.ut_bytes = round_up(16 * w.fpad * w.cpad * 4, 256);
  w.v_bytes = round_up(16 * w.T * w.cpad * 4, 256);
  w.m_bytes = round_up(16 * w.T * w.ldm * 4, 256);
  w.partial_bytes = w.splits > 1 ? (size_t)w.splits * w.m_bytes : 0;
  w.total = w.ut_bytes * (w.three_x ? 2 : 1) + w.v_bytes + w.m_bytes + w.partial_bytes;
  return w;
}

unsigned grid_for(int64_t total) {
  int64_t b = (total + 255) / 256;
  if (b > 148 * 32) b = 148 * 32;
  return (unsigned)(b < 1 ? 1 : b);
}

}  // namespace

size_t winograd_workspace(const Problem& p) { return make_wplan(p).total; }
int winograd_launches(const Problem& p) { return 4 + (make_wplan(p).splits > 1 ? 1 : 0); }

cudaError_t launch_winograd(const Problem& p, const float* in, const float* filt, float* out, void* ws,
                            cudaStream_t s) {
  const WPlan w = make_wplan(p);
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

  cudaError_t e = launch_k(wino_filter_kernel, dim3(grid_for(w.cpad * w.fpad)), dim3(256), 0, s, filt, p.C, p.F,
                           w.cpad, w.fpad, ut_hi, ut_lo, w.three_x ? 0 : 1);
  if (e != cudaSuccess) return e;
  e = launch_k(wino_input_kernel, dim3(grid_for(w.T * w.cpad)), dim3(256), 0, s, in, p.H, p.W, p.C, w.TH, w.TW,
               p.pad_top, p.pad_left, w.T, w.cpad, V, w.three_x ? 0 : 1);
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
  g.batch = 16;
  g.splits = w.splits;
  g.three_x = w.three_x;
  g.block_n = w.block_n;
  e = launch_gemm2(p, g, s);
  if (e != cudaSuccess) return e;
  return launch_k(wino_output_kernel, dim3(grid_for(w.T * p.F)), dim3(256), 0, s, Mw, w.T, w.ldm, p.F, p.HO, p.WO,
                  w.TH, w.TW, out);
}

}  // namespace conv2d
