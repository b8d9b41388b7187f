// pool.cu -- NHWC max / average pooling (include/pool2d.h).
//
// HBM-bound: one thread per (n, ho, wo, 4-channel group), channels fastest so a warp reads whole
// 16-byte-per-lane runs of a pixel's channel vector (coalesced) and overlapping windows hit L1/L2;
// grid-stride over a multiple of the SM count.  Average accumulates in double in (kh, kw) order and
// divides in double (bit-identical to the definition evaluated in double; FP64 throughput is irrelevant
// at ~1 flop per 4 bytes).
#include <cuda_runtime.h>

#include "internal.h"
#include "launch.cuh"

namespace conv2d {
namespace {

struct PoolArgs {
  int N, H, W, C, KH, KW, SH, SW, HO, WO, PT, PL;
};

// KS > 0: square KS x KS window known at compile time (loads unrolled and issued together);
// KS == 0: generic KH x KW loop.  IDX = int (totals < 2^31) or int64_t.
template <bool AVG, bool VEC, int KS, typename IDX>
__global__ void __launch_bounds__(256) pool_kernel(const float* __restrict__ x, float* __restrict__ y,
                                                   const PoolArgs a, IDX total) {
  pdl_trigger();
  pdl_wait();
  constexpr int V = VEC ? 4 : 1;
  const int KH = KS > 0 ? KS : a.KH, KW = KS > 0 ? KS : a.KW;
  const IDX CG = a.C / V;  // channel groups per pixel
  for (IDX t = blockIdx.x * (IDX)blockDim.x + threadIdx.x; t < total; t += (IDX)gridDim.x * blockDim.x) {
    const int cg = (int)(t % CG);
    IDX q = t / CG;
    const int wo = (int)(q % a.WO);
    q /= a.WO;
    const int ho = (int)(q % a.HO);
    const int n = (int)(q / a.HO);
    const int ih0 = ho * a.SH - a.PT, iw0 = wo * a.SW - a.PL;
    const float* base = x + ((int64_t)n * a.H * a.W) * a.C + (int64_t)cg * V;
    double s[V];
    float m[V];
#pragma unroll
    for (int e = 0; e < V; ++e) {
      s[e] = 0.0;
      m[e] = -__int_as_float(0x7f800000);  // -inf: every window has >= 1 in-bounds element
    }
    int count = 0;
    // KS <= 3: the whole window unrolled (all loads in flight); KS = 7: one unrolled 7-wide row at a
    // time (7 float4 loads in flight without spilling); KS = 0: generic loops
    constexpr int UR = KS > 0 && KS <= 3 ? KS : 1;
#pragma unroll UR
    for (int r = 0; r < KH; ++r) {
      const int ih = ih0 + r;
      if (ih < 0 || ih >= a.H) continue;
#pragma unroll (KS > 0 ? KS : 1)
      for (int cc = 0; cc < KW; ++cc) {
        const int iw = iw0 + cc;
        if (iw < 0 || iw >= a.W) continue;
        const float* src = base + ((int64_t)ih * a.W + iw) * a.C;
        float v[V];
        if constexpr (VEC) {
          const float4 f = __ldg(reinterpret_cast<const float4*>(src));
          v[0] = f.x;
          v[1] = f.y;
          v[2] = f.z;
          v[3] = f.w;
        } else {
          v[0] = __ldg(src);
        }
#pragma unroll
        for (int e = 0; e < V; ++e) {
          if (AVG) s[e] += (double)v[e];
          else m[e] = fmaxf(m[e], v[e]);
        }
        ++count;
      }
    }
    float r[V];
#pragma unroll
    for (int e = 0; e < V; ++e) r[e] = AVG ? (float)(s[e] / (double)count) : m[e];
    float* dst = y + ((((int64_t)n * a.HO + ho) * a.WO + wo) * a.C) + (int64_t)cg * V;
    if constexpr (VEC) *reinterpret_cast<float4*>(dst) = make_float4(r[0], r[1], r[2], r[3]);
    else dst[0] = r[0];
  }
}

template <bool AVG, bool VEC, typename IDX>
cudaError_t launch_ks(const PoolArgs& a, const float* x, float* y, IDX total, dim3 g, dim3 b, cudaStream_t s) {
  if (a.KH == 2 && a.KW == 2) return launch_k(pool_kernel<AVG, VEC, 2, IDX>, g, b, 0, s, x, y, a, total);
  if (a.KH == 3 && a.KW == 3) return launch_k(pool_kernel<AVG, VEC, 3, IDX>, g, b, 0, s, x, y, a, total);
  if (a.KH == 7 && a.KW == 7) return launch_k(pool_kernel<AVG, VEC, 7, IDX>, g, b, 0, s, x, y, a, total);
  return launch_k(pool_kernel<AVG, VEC, 0, IDX>, g, b, 0, s, x, y, a, total);
}

template <bool AVG, bool VEC>
cudaError_t launch_idx(const PoolArgs& a, const float* x, float* y, int64_t total, dim3 g, dim3 b, cudaStream_t s) {
  if (total < (1LL << 31) - (int64_t)g.x * b.x) return launch_ks<AVG, VEC, int>(a, x, y, (int)total, g, b, s);
  return launch_ks<AVG, VEC, int64_t>(a, x, y, total, g, b, s);
}

}  // namespace

cudaError_t launch_pool(const PoolProblem& p, const float* x, float* y, cudaStream_t s) {
  PoolArgs a{p.N, p.H, p.W, p.C, p.KH, p.KW, p.SH, p.SW, p.HO, p.WO, p.PT, p.PL};
  const bool vec = p.C % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(y) & 15) == 0;
  const int64_t total = (int64_t)p.N * p.HO * p.WO * (vec ? p.C / 4 : p.C);
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  const dim3 g((unsigned)blocks), b(256);
  if (p.avg) return vec ? launch_idx<true, true>(a, x, y, total, g, b, s) : launch_idx<true, false>(a, x, y, total, g, b, s);
  return vec ? launch_idx<false, true>(a, x, y, total, g, b, s) : launch_idx<false, false>(a, x, y, total, g, b, s);
}

}  // namespace conv2d
