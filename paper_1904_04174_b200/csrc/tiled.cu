// tiled.cu -- CONV2D_ALGO_TILED: tiled direct convolution on CUDA cores
// ("tiled algorithm", SPEC.md:210-230 tile_rows x tile_cols x
// feature_block).  B200 design:
//   * CTA = one image x (TH=8) x (TW=16) output tile x (FB=64) features, 256 threads.
//   * Per channel chunk (CC <= 8), the input halo tile ((TH-1)S+KH) x ((TW-1)S+KW) x CC
//     and the filter chunk KH x KW x CC x FB are staged in shared memory (coalesced
//     global loads, zero-filled padding), so each input element is read from L2 once
//     per CTA instead of once per tap.
//   * Each thread keeps a 4-pixel x 8-feature register tile (32 fp32 accumulators):
//     per (c, kh, kw) it does 2 LDS.128 (filter) + 4 LDS (input) for 32 FFMA.
//   * Input rows are padded to CC+1 floats to break the 4-way bank conflict between
//     the four pixel groups of a warp.
// Exact fp32 FFMA, (c-chunk, c, kh, kw) accumulation order.
#include "internal.h"
#include "launch.cuh"

namespace conv2d {
namespace {

constexpr int TH = 8, TW = 16, FB = 64, PX = 4, FV = 8, CCMAX = 8;
constexpr int NTHREADS = (TW / PX) * TH * (FB / FV);  // 256

__global__ void __launch_bounds__(NTHREADS) tiled_kernel(const float* __restrict__ in,
                                                         const float* __restrict__ filt, float* __restrict__ out,
                                                         int H, int W, int C, int F, int KH, int KW, int SH, int SW,
                                                         int HO, int WO, int PT, int PL, int fblocks, int wtiles,
                                                         int htiles) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float smem[];
  const int CC = C < CCMAX ? C : CCMAX;
  const int CCP = CC + 1;
  const int IH = (TH - 1) * SH + KH;
  const int IW = (TW - 1) * SW + KW;
  float* xs = smem;                                  // [IH][IW][CCP]
  float* ws = smem + ((IH * IW * CCP + 3) & ~3);     // [KH][KW][CC][FB], 16-byte aligned for LDS.128

  // 1-D grid (gridDim.z <= 65535 would cap N * fblocks): x = ((n * fblocks + fb) * htiles + ht) * wtiles + wt
  const int64_t bid = blockIdx.x;
  const int wt = (int)(bid % wtiles);
  const int ht = (int)((bid / wtiles) % htiles);
  const int64_t nf = bid / ((int64_t)wtiles * htiles);
  const int n = (int)(nf / fblocks);
  const int fb0 = (int)(nf % fblocks) * FB;
  const int ho0 = ht * TH, wo0 = wt * TW;
  const int ih0 = ho0 * SH - PT, iw0 = wo0 * SW - PL;

  const int t = threadIdx.x;
  const int fv = t % (FB / FV);
  const int tx = (t / (FB / FV)) % (TW / PX);
  const int ty = t / ((FB / FV) * (TW / PX));

  float acc[PX][FV];
#pragma unroll
  for (int i = 0; i < PX; ++i)
#pragma unroll
    for (int j = 0; j < FV; ++j) acc[i][j] = 0.f;

  const float* xin = in + (int64_t)n * H * W * C;
  for (int c0 = 0; c0 < C; c0 += CC) {
    const int cc = (C - c0) < CC ? (C - c0) : CC;
    __syncthreads();  // previous chunk fully consumed
    // stage input halo tile (zero outside the image and beyond cc)
    for (int e = t; e < IH * IW * CC; e += NTHREADS) {
      const int c = e % CC;
      const int col = (e / CC) % IW;
      const int row = e / (CC * IW);
      const int ih = ih0 + row, iw = iw0 + col;
      float v = 0.f;
      if (c < cc && ih >= 0 && ih < H && iw >= 0 && iw < W) v = __ldg(xin + ((int64_t)ih * W + iw) * C + c0 + c);
      xs[(row * IW + col) * CCP + c] = v;
    }
    // stage filter chunk
    for (int e = t; e < KH * KW * CC * FB; e += NTHREADS) {
      const int f = e % FB;
      const int c = (e / FB) % CC;
      const int khw = e / (FB * CC);
      float v = 0.f;
      if (c < cc && fb0 + f < F) v = __ldg(filt + ((int64_t)khw * C + c0 + c) * F + fb0 + f);
      ws[e] = v;
    }
    __syncthreads();
    for (int c = 0; c < cc; ++c) {
      for (int kh = 0; kh < KH; ++kh) {
        const float* xrow = xs + ((ty * SH + kh) * IW) * CCP + c;
        for (int kw = 0; kw < KW; ++kw) {
          const float4* wp = reinterpret_cast<const float4*>(ws + ((kh * KW + kw) * CC + c) * FB + fv * FV);
          const float4 wa = wp[0], wb = wp[1];
          const float wv[FV] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#pragma unroll
          for (int i = 0; i < PX; ++i) {
            const float xv = xrow[((tx * PX + i) * SW + kw) * CCP];
#pragma unroll
            for (int j = 0; j < FV; ++j) acc[i][j] = fmaf(xv, wv[j], acc[i][j]);
          }
        }
      }
    }
  }
  const int ho = ho0 + ty;
  if (ho >= HO) return;
#pragma unroll
  for (int i = 0; i < PX; ++i) {
    const int wo = wo0 + tx * PX + i;
    if (wo >= WO) continue;
    float* o = out + (((int64_t)n * HO + ho) * WO + wo) * F + fb0 + fv * FV;
    const int f = fb0 + fv * FV;
    if ((F % 4) == 0 && f + FV <= F) {
      reinterpret_cast<float4*>(o)[0] = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
      reinterpret_cast<float4*>(o)[1] = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
    } else {
#pragma unroll
      for (int j = 0; j < FV; ++j)
        if (f + j < F) o[j] = acc[i][j];
    }
  }
}

}  // namespace

cudaError_t launch_tiled(const Problem& p, const float* in, const float* filt, float* out, cudaStream_t s) {
  const int CC = p.C < CCMAX ? p.C : CCMAX;
  const int IH = (TH - 1) * p.SH + p.KH, IW = (TW - 1) * p.SW + p.KW;
  const size_t smem = sizeof(float) * ((((size_t)IH * IW * (CC + 1)) + 3) / 4 * 4 + (size_t)p.KH * p.KW * CC * FB);
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  {
    const cudaError_t e = smem_attr_once<tiled_kernel>(227 * 1024);
    if (e != cudaSuccess) return e;
  }
  const int fblocks = (p.F + FB - 1) / FB;
  const int wtiles = (p.WO + TW - 1) / TW, htiles = (p.HO + TH - 1) / TH;
  const int64_t blocks = (int64_t)wtiles * htiles * p.N * fblocks;
  if (blocks > 0x7FFFFFFFLL) return cudaErrorInvalidConfiguration;  // tiled_grid_ok() rejects this in supports()
  return launch_k(tiled_kernel, dim3((unsigned)blocks), dim3(NTHREADS), smem, s, in, filt, out, p.H, p.W, p.C, p.F,
                  p.KH, p.KW, p.SH, p.SW, p.HO, p.WO, p.pad_top, p.pad_left, fblocks, wtiles, htiles);
}

}  // namespace conv2d
