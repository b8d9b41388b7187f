// gemm_common.cu -- small CUDA-core helpers around the tensor-core GEMM core:
//   filter_prep2   : HWCF filter -> K-major Bt (the B operand), TF32 hi/lo split in 3xTF32 mode
//   pad_channels   : NHWC C -> Cp (zero channels) so 16-byte gathers stay aligned (C=3 stems)
//   split_reduce   : deterministic fixed-order sum of split-K partial tiles
#include "gemm2sm.h"
#include "launch.cuh"
#include "sm100.cuh"

namespace conv2d {
namespace {

// One 32 (k) x 32 (n) destination tile per block.  Source rows of the 32 k's are read
// coalesced (32 consecutive features), written transposed (32 consecutive k's).
// k -> (r = k / rowstride, e = k % rowstride, s = e / cstride, c = e % cstride); valid when
// r < KH, s < KW, c < C.  Tap-major layouts use rowstride = KW * cstride.
__global__ void filter_prep2_kernel(const float* __restrict__ w, int KH, int KW, int C, int F, int cstride,
                                    int rowstride, int64_t kpad, int64_t npad, float* __restrict__ bt_hi,
                                    float* __restrict__ bt_lo) {
  pdl_trigger();
  pdl_wait();
  __shared__ float tile[32][33];
  const int64_t k0 = (int64_t)blockIdx.x * 32, n0 = (int64_t)blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t k = k0 + r;
    const int kr = (int)(k / rowstride), e = (int)(k % rowstride);
    const int ks = e / cstride, c = e % cstride;
    const int64_t n = n0 + threadIdx.x;
    float v = 0.f;
    if (kr < KH && ks < KW && c < C && n < F) v = w[((int64_t)(kr * KW + ks) * C + c) * F + n];
    tile[r][threadIdx.x] = v;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t n = n0 + r, k = k0 + threadIdx.x;
    if (n < npad && k < kpad) {
      const float v = tile[threadIdx.x][r];
      const float h = bt_lo ? sm100::tf32_hi(v) : v;
      bt_hi[n * kpad + k] = h;
      if (bt_lo) bt_lo[n * kpad + k] = v - h;
    }
  }
}

// x (N,H,W,C) -> xp (N,Hp,Wp,Cp): xp[n][i][j][c] = x[n][i-pt][j-pl][c] inside the image and c < C, else 0.
// One thread per padded pixel (32-bit index math), Cp/4 float4 stores each.
__global__ void pad_spatial_kernel(const float* __restrict__ x, int N, int H, int W, int C, int Hp, int Wp, int Cp,
                                   int pt, int pl, float* __restrict__ xp) {
  pdl_trigger();
  pdl_wait();
  const int total = N * Hp * Wp;
  for (int px = blockIdx.x * blockDim.x + threadIdx.x; px < total; px += gridDim.x * blockDim.x) {
    const int j = px % Wp;
    const int q = px / Wp;
    const int ii = q % Hp;
    const int n = q / Hp;
    const int ih = ii - pt, iw = j - pl;
    const bool in = ih >= 0 && ih < H && iw >= 0 && iw < W;
    const float* src = x + (((int64_t)n * H + ih) * W + iw) * C;
    float4* dst = reinterpret_cast<float4*>(xp + (int64_t)px * Cp);
    for (int c4 = 0; c4 < Cp; c4 += 4) {
      float v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = (in && c4 + k < C) ? __ldg(src + c4 + k) : 0.f;
      dst[c4 / 4] = make_float4(v[0], v[1], v[2], v[3]);
    }
  }
}

__global__ void pad_channels_kernel(const float* __restrict__ x, int64_t pixels, int C, int Cp,
                                    float* __restrict__ xp) {
  pdl_trigger();
  pdl_wait();
  const int64_t total = pixels * Cp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t px = i / Cp;
    const int c = (int)(i % Cp);
    xp[i] = c < C ? x[px * C + c] : 0.f;
  }
}

// d[i] = sum_{s=0..splits-1} partial[s][i] over a dense rows x ldd plane (ldd % 4 == 0),
// fixed split order: deterministic.
__global__ void split_reduce_kernel(const float* __restrict__ partial, float* __restrict__ d, int64_t plane4,
                                    int splits) {
  pdl_trigger();
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < plane4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 acc = reinterpret_cast<const float4*>(partial)[i];
    for (int s = 1; s < splits; ++s) {
      const float4 v = reinterpret_cast<const float4*>(partial)[s * plane4 + i];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    reinterpret_cast<float4*>(d)[i] = acc;
  }
}

// remainder split: d[tile rows, tile cols] = sum_{s} partial[s][...] in fixed order, for the pair tiles
// [first_tile, first_tile + ntiles) (tile t: M rows [(t / nt)*256, +256), N cols [(t % nt)*BN, +BN)).
// One thread per float4 of a tile row; ldd % 4 == 0.
__global__ void rsplit_reduce_kernel(const float* __restrict__ partial, float* __restrict__ d, int64_t M, int64_t N,
                                     int64_t ldd, int first_tile, int ntiles, int nt, int block_n, int splits) {
  pdl_trigger();
  pdl_wait();
  const int q4 = block_n / 4;
  const int64_t total = (int64_t)ntiles * 256 * q4;
  const int64_t plane = M * ldd;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c4 = (int)(i % q4);
    const int64_t rr = i / q4;
    const int r = (int)(rr % 256);
    const int t = first_tile + (int)(rr / 256);
    const int64_t m = (int64_t)(t / nt) * 256 + r;
    const int64_t n = (int64_t)(t % nt) * block_n + c4 * 4;
    if (m >= M || n >= N) continue;
    const int64_t o = m * ldd + n;
    float4 acc = *reinterpret_cast<const float4*>(partial + o);
    for (int s2 = 1; s2 < splits; ++s2) {
      const float4 v = *reinterpret_cast<const float4*>(partial + s2 * plane + o);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    if (n + 3 < N) {
      *reinterpret_cast<float4*>(d + o) = acc;
    } else {
      const float a4[4] = {acc.x, acc.y, acc.z, acc.w};
      for (int e = 0; e < 4 && n + e < N; ++e) d[o + e] = a4[e];
    }
  }
}

}  // namespace

cudaError_t launch_rsplit_reduce(const float* partial, float* d, int64_t M, int64_t N, int64_t ldd, int first_tile,
                                 int ntiles, int nt, int block_n, int splits, cudaStream_t s) {
  const int64_t total = (int64_t)ntiles * 256 * (block_n / 4);
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  return launch_k(rsplit_reduce_kernel, dim3((unsigned)blocks), dim3(256), 0, s, partial, d, M, N, ldd, first_tile,
                  ntiles, nt, block_n, splits);
}

cudaError_t launch_filter_prep2(const float* w, int KH, int KW, int C, int F, int cstride, int rowstride,
                                int64_t kpad, int64_t npad, float* bt_hi, float* bt_lo, cudaStream_t s) {
  dim3 grid((unsigned)((kpad + 31) / 32), (unsigned)((npad + 31) / 32));
  return launch_k(filter_prep2_kernel, grid, dim3(32, 8), 0, s, w, KH, KW, C, F, cstride, rowstride, kpad, npad, bt_hi,
                  bt_lo);
}

cudaError_t launch_pad_spatial(const float* x, int N, int H, int W, int C, int Hp, int Wp, int Cp, int pt, int pl,
                               float* xp, cudaStream_t s) {
  const int64_t total = (int64_t)N * Hp * Wp;
  if (total > 0x7FFFFFFF) return cudaErrorInvalidValue;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  return launch_k(pad_spatial_kernel, dim3((unsigned)blocks), dim3(256), 0, s, x, N, H, W, C, Hp, Wp, Cp, pt, pl, xp);
}

cudaError_t launch_pad_channels(const float* x, int64_t pixels, int C, int Cp, float* xp, cudaStream_t s) {
  const int64_t total = pixels * Cp;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  return launch_k(pad_channels_kernel, dim3((unsigned)blocks), dim3(256), 0, s, x, pixels, C, Cp, xp);
}

cudaError_t launch_split_reduce(const float* partial, float* d, int64_t rows, int64_t cols, int64_t ldd, int splits,
                                cudaStream_t s) {
  if (ldd % 4 != 0 || cols != ldd) return cudaErrorInvalidValue;  // callers only split dense, 16B rows
  const int64_t plane4 = rows * ldd / 4;
  int64_t blocks = (plane4 + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  return launch_k(split_reduce_kernel, dim3((unsigned)blocks), dim3(256), 0, s, partial, d, plane4, splits);
}

}  // namespace conv2d
