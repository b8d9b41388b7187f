// direct.cu -- CONV2D_ALGO_DIRECT: "a vectorized naive compute kernel which runs a
// single thread per output vector".
//
// One thread per (n, ho, wo, 4-feature chunk).  Threads of a warp share output
// pixels and walk consecutive feature chunks, so filter reads (HWCF: features
// contiguous) are coalesced float4 loads and input reads are warp broadcasts.
// Exact fp32 FFMA accumulation in (kh, kw, c) order.  Bound: FFMA pipe / L1
// (no data reuse beyond L1/L2) -- the baseline the other algorithms beat.
#include "internal.h"

#include "launch.cuh"

namespace conv2d {
namespace {

template <bool VEC>
__global__ void __launch_bounds__(256) direct_kernel(const float* __restrict__ in, const float* __restrict__ filt,
                                                     float* __restrict__ out, int H, int W, int C, int F, int KH,
                                                     int KW, int SH, int SW, int HO, int WO, int PT, int PL,
                                                     int64_t total) {
  pdl_trigger();
  pdl_wait();
  const int FQ = (F + 3) / 4;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int fq = (int)(t % FQ);
    const int64_t pix = t / FQ;
    const int wo = (int)(pix % WO);
    const int ho = (int)((pix / WO) % HO);
    const int64_t n = pix / ((int64_t)WO * HO);
    const int f0 = fq * 4;
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    for (int kh = 0; kh < KH; ++kh) {
      const int ih = ho * SH + kh - PT;
      if (ih < 0 || ih >= H) continue;
      for (int kw = 0; kw < KW; ++kw) {
        const int iw = wo * SW + kw - PL;
        if (iw < 0 || iw >= W) continue;
        const float* xr = in + ((n * H + ih) * W + iw) * (int64_t)C;
        const float* wr = filt + ((int64_t)(kh * KW + kw) * C) * F + f0;
        for (int c = 0; c < C; ++c) {
          const float xv = __ldg(xr + c);
          if (VEC) {
            const float4 w4 = __ldg(reinterpret_cast<const float4*>(wr + (int64_t)c * F));
            a0 = fmaf(xv, w4.x, a0);
            a1 = fmaf(xv, w4.y, a1);
            a2 = fmaf(xv, w4.z, a2);
            a3 = fmaf(xv, w4.w, a3);
          } else {
            const float* w1 = wr + (int64_t)c * F;
            a0 = fmaf(xv, __ldg(w1), a0);
            if (f0 + 1 < F) a1 = fmaf(xv, __ldg(w1 + 1), a1);
            if (f0 + 2 < F) a2 = fmaf(xv, __ldg(w1 + 2), a2);
            if (f0 + 3 < F) a3 = fmaf(xv, __ldg(w1 + 3), a3);
          }
        }
      }
    }
    float* o = out + pix * F + f0;
    if (VEC) {
      *reinterpret_cast<float4*>(o) = make_float4(a0, a1, a2, a3);
    } else {
      o[0] = a0;
      if (f0 + 1 < F) o[1] = a1;
      if (f0 + 2 < F) o[2] = a2;
      if (f0 + 3 < F) o[3] = a3;
    }
  }
}

}  // namespace

cudaError_t launch_direct(const Problem& p, const float* in, const float* filt, float* out, cudaStream_t s) {
  const int64_t total = p.M() * ((p.F + 3) / 4);
  const int threads = 256;
  int64_t blocks = (total + threads - 1) / threads;
  if (blocks > 148LL * 64) blocks = 148LL * 64;  // grid-stride beyond ~64 resident-block waves
  auto kern = p.F % 4 == 0 ? direct_kernel<true> : direct_kernel<false>;
  return launch_k(kern, dim3((unsigned)blocks), dim3(threads), 0, s, in, filt, out, p.H, p.W, p.C, p.F, p.KH, p.KW,
                  p.SH, p.SW, p.HO, p.WO, p.pad_top, p.pad_left, total);
}

}  // namespace conv2d
