// gemm_tcgen05.cu -- the tensor-core GEMM core on 5th-gen tensor cores (tcgen05 + TMEM).
//
//   D[b](m, n) = sum_k A[b](m, k) * Bt[b](n, k)         fp32 in, fp32 accumulate in TMEM
//
// It is the contraction behind three of the paper's algorithms:
//   * implicit GEMM (im2col never materialised): A(m,k) is gathered
//     straight from the NHWC input, m = (n,ho,wo), k = (kh,kw,c);
//   * 1x1 as matmul: A is the NHWC input viewed as a (N*H*W) x C matrix;
//   * Winograd's "number of small matrix multiplies": 16 batched
//     GEMMs over transformed tiles (dense A).
// B is the filter, pre-transposed to K-major and TF32-split by filter_prep_kernel.
//
// Kernel structure (one 128 x BN output tile per CTA, warp-specialised):
//   warps 0-3 (128 thr) : producers -- cp.async 16-byte gathers of A (zero-filled padding /
//                         tails) and B into SWIZZLE_128B K-major smem stages; in 3xTF32 mode
//                         they also split A into (hi, lo) in place; then fence.proxy.async +
//                         mbarrier arrive.  After the main loop they are the epilogue:
//                         tcgen05.ld (32 lanes x 32 cols) -> registers -> global.
//   warp 4              : TMEM allocator + single-thread tcgen05.mma issuer
//                         (kind::tf32, M=128, N=BN, K=8; 4 per 32-deep k-block, x3 in 3xTF32:
//                         hi*hi + hi*lo + lo*hi), tcgen05.commit frees each smem stage.
// Split-K: gridDim.z = batch * splits; partial tiles go to a workspace reduced in fixed
// split order by split_reduce_kernel (deterministic, no atomics).
#include <cstdio>

#include "internal.h"
#include "sm100.cuh"

namespace conv2d {
namespace {

using namespace sm100;

constexpr int BM = 128;       // UMMA M (cta_group::1)
constexpr int BK = 32;        // fp32 per 128-byte swizzle row
constexpr int NPROD = 128;    // producer / epilogue threads (warps 0-3)
constexpr int NTHREADS = NPROD + 32;
constexpr int A_TILE = BM * BK * 4;  // 16 KB

enum { A_CONV_VEC4 = 0, A_CONV_SCALAR = 1, A_DENSE = 2 };

struct DevArgs {
  // conv geometry (A_CONV_*)
  int H, W, C, KH, KW, SH, SW, HO, WO, PT, PL;
  // operands
  const float* a;
  int64_t lda, a_bstride;
  const float* bt_hi;
  const float* bt_lo;
  int64_t ldb, b_bstride;
  float* d;
  int64_t ldd, d_bstride;
  float* partial;
  int64_t M, N, K;
  int nkb;     // k-blocks (Kpad / 32)
  int splits;
  int batch;
};

template <int BN, bool THREE_X>
struct Cfg {
  static constexpr int B_TILE = BN * BK * 4;
  static constexpr int STAGE = (THREE_X ? 2 : 1) * (A_TILE + B_TILE);
  static constexpr int BUDGET = 200 * 1024;
  static constexpr int STAGES = (BUDGET / STAGE) > 8 ? 8 : (BUDGET / STAGE);
  static constexpr int SMEM = STAGES * STAGE + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr uint32_t TMEM_COLS = BN < 32 ? 32 : BN;
};

template <int BN, bool THREE_X, int AMODE>
__global__ void __launch_bounds__(NTHREADS, 1) gemm_tcgen05_kernel(const DevArgs args) {
  using C_ = Cfg<BN, THREE_X>;
  constexpr int STAGES = C_::STAGES;
  constexpr int LAG = STAGES - 1;
  static_assert(STAGES >= 2, "need >= 2 stages");

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // stage s: [A_hi | A_lo? | B_hi | B_lo?]
  auto a_hi = [&](int s) { return smem + (size_t)s * C_::STAGE; };
  auto a_lo = [&](int s) { return smem + (size_t)s * C_::STAGE + A_TILE; };
  auto b_hi = [&](int s) { return smem + (size_t)s * C_::STAGE + (THREE_X ? 2 : 1) * A_TILE; };
  auto b_lo = [&](int s) { return smem + (size_t)s * C_::STAGE + 2 * A_TILE + C_::B_TILE; };
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C_::STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;
  const int bz = blockIdx.z / args.splits;
  const int split = blockIdx.z % args.splits;
  const int kb_begin = (int)((int64_t)split * args.nkb / args.splits);
  const int kb_end = (int)((int64_t)(split + 1) * args.nkb / args.splits);
  const int nk = kb_end - kb_begin;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], NPROD);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_mbar_init();
  }
  if (warp == 4) tmem_alloc<C_::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp < 4) {
    // ======================= producers =======================
    const int t = threadIdx.x;
    const int j = t & 7;       // 16-byte chunk within the 128-byte k-row
    const int rb = t >> 3;     // rows rb + 16 i, i = 0..7
    const float* __restrict__ A = args.a + (AMODE == A_DENSE ? (int64_t)bz * args.a_bstride : 0);
    const float* __restrict__ Bh = args.bt_hi + (int64_t)bz * args.b_bstride;
    const float* __restrict__ Bl = THREE_X ? args.bt_lo + (int64_t)bz * args.b_bstride : nullptr;

    // per-row gather state
    int ihb[8], iwb[8];
    int64_t rbase[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t m = m0 + rb + 16 * i;
      if (AMODE == A_DENSE) {
        rbase[i] = m < args.M ? m * args.lda : -1;
        ihb[i] = iwb[i] = 0;
      } else {
        if (m < args.M) {
          const int wo = (int)(m % args.WO);
          const int64_t q = m / args.WO;
          const int ho = (int)(q % args.HO);
          const int64_t n = q / args.HO;
          ihb[i] = ho * args.SH - args.PT;
          iwb[i] = wo * args.SW - args.PL;
          rbase[i] = n * args.H * args.W * args.C;
        } else {
          ihb[i] = -(1 << 28);  // forces out-of-bounds
          iwb[i] = 0;
          rbase[i] = 0;
        }
      }
    }

    auto finalize = [&](int kk) {
      const int s = (kk - kb_begin) % STAGES;
      if (THREE_X) {
        uint8_t* ah = a_hi(s);
        uint8_t* al = a_lo(s);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint32_t off = sw128_offset(rb + 16 * i, j);
          float4 v = *reinterpret_cast<float4*>(ah + off);
          float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
          *reinterpret_cast<float4*>(ah + off) = h;
          *reinterpret_cast<float4*>(al + off) = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
        }
      }
      fence_proxy_async_smem();
      mbar_arrive(&full[s]);
    };

    for (int kb = kb_begin; kb < kb_end; ++kb) {
      const int it = kb - kb_begin;
      const int s = it % STAGES;
      const int use = it / STAGES;
      if (use > 0) mbar_wait(&empty[s], (use - 1) & 1);
      const uint32_t sa = smem_u32(a_hi(s));
      // ---- A
      const int k0 = kb * BK + j * 4;
      if (AMODE == A_DENSE) {
        const bool kv = k0 < args.K;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const bool v = kv && rbase[i] >= 0;
          const float* src = v ? A + rbase[i] + k0 : A;
          cp_async16(sa + sw128_offset(rb + 16 * i, j), src, v ? 16u : 0u);
        }
      } else if (AMODE == A_CONV_VEC4) {
        const int c = k0 % args.C;
        const int rs = k0 / args.C;
        const int sx = rs % args.KW;
        const int r = rs / args.KW;
        const bool kv = k0 < args.K;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int ih = ihb[i] + r, iw = iwb[i] + sx;
          const bool v = kv && ih >= 0 && ih < args.H && iw >= 0 && iw < args.W;
          const float* src = v ? args.a + rbase[i] + ((int64_t)ih * args.W + iw) * args.C + c : args.a;
          cp_async16(sa + sw128_offset(rb + 16 * i, j), src, v ? 16u : 0u);
        }
      } else {  // A_CONV_SCALAR: each of the 4 k's of the chunk decoded separately
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int k = k0 + e;
          const int c = k % args.C;
          const int rs = k / args.C;
          const int sx = rs % args.KW;
          const int r = rs / args.KW;
          const bool kv = k < args.K;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int ih = ihb[i] + r, iw = iwb[i] + sx;
            const bool v = kv && ih >= 0 && ih < args.H && iw >= 0 && iw < args.W;
            const float* src = v ? args.a + rbase[i] + ((int64_t)ih * args.W + iw) * args.C + c : args.a;
            cp_async4(sa + sw128_offset(rb + 16 * i, j) + 4 * e, src, v ? 4u : 0u);
          }
        }
      }
      // ---- B (padded: always in bounds)
      const uint32_t sbh = smem_u32(b_hi(s));
      const uint32_t sbl = THREE_X ? smem_u32(b_lo(s)) : 0u;
#pragma unroll
      for (int q = t; q < BN * 8; q += NPROD) {
        const int row = q >> 3, jj = q & 7;
        const int64_t goff = (int64_t)(n0 + row) * args.ldb + kb * BK + jj * 4;
        cp_async16(sbh + sw128_offset(row, jj), Bh + goff, 16u);
        if (THREE_X) cp_async16(sbl + sw128_offset(row, jj), Bl + goff, 16u);
      }
      cp_async_commit();
      if (it >= LAG) {
        cp_async_wait<LAG>();
        finalize(kb - LAG);
      }
    }
    cp_async_wait<0>();
    for (int kk = (nk > LAG ? kb_end - LAG : kb_begin); kk < kb_end; ++kk) finalize(kk);

    // ======================= epilogue =======================
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    const int64_t m = m0 + warp * 32 + lane;
    float* D;
    if (args.splits == 1) {
      D = args.d + (int64_t)bz * args.d_bstride;
    } else {
      D = args.partial + ((int64_t)split * args.batch + bz) * args.M * args.ldd;
    }
    const bool vec_ok = (args.ldd % 4) == 0;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      float v[32];
      tmem_ld32(tmem_base + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
      if (m < args.M) {
        float* dst = D + m * args.ldd + n0 + c0;
        const int64_t nrem = args.N - (n0 + c0);
        if (vec_ok && nrem >= 32) {
#pragma unroll
          for (int q = 0; q < 8; ++q)
            reinterpret_cast<float4*>(dst)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        } else {
#pragma unroll
          for (int q = 0; q < 32; ++q)
            if (q < nrem) dst[q] = v[q];
        }
      }
    }
  } else {
    // ======================= MMA issuer (warp 4) =======================
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_tf32(BM, BN);
      for (int kb = kb_begin; kb < kb_end; ++kb) {
        const int it = kb - kb_begin;
        const int s = it % STAGES;
        mbar_wait(&full[s], (it / STAGES) & 1);
        tc_fence_after();
        const uint64_t dah = umma_desc_sw128_kmajor(smem_u32(a_hi(s)));
        const uint64_t dbh = umma_desc_sw128_kmajor(smem_u32(b_hi(s)));
        const uint64_t dal = THREE_X ? umma_desc_sw128_kmajor(smem_u32(a_lo(s))) : 0;
        const uint64_t dbl = THREE_X ? umma_desc_sw128_kmajor(smem_u32(b_lo(s))) : 0;
#pragma unroll
        for (int k = 0; k < BK / 8; ++k) {
          const uint64_t adv = (uint64_t)(k * 8 * 4) >> 4;  // 32 bytes per K=8 step
          if (THREE_X) {
            // small terms first, then the dominant hi*hi product
            mma_tf32(tmem_base, dal + adv, dbh + adv, idesc, (it > 0 || k > 0) ? 1u : 0u);
            mma_tf32(tmem_base, dah + adv, dbl + adv, idesc, 1u);
            mma_tf32(tmem_base, dah + adv, dbh + adv, idesc, 1u);
          } else {
            mma_tf32(tmem_base, dah + adv, dbh + adv, idesc, (it > 0 || k > 0) ? 1u : 0u);
          }
        }
        mma_commit(&empty[s]);
      }
      mma_commit(tmem_full);
    }
    __syncwarp();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc<C_::TMEM_COLS>(tmem_base);
  }
}

// ---------------------------------------------------------------- filter prep
// HWCF filter viewed as K x F (row-major)  ->  Bt[n][k] (K-major, Npad x Kpad, zero padded),
// split into TF32 hi (low 13 mantissa bits cleared) and lo = w - hi.  32x32 smem transpose.
__global__ void filter_prep_kernel(const float* __restrict__ w, int64_t K, int64_t F, int64_t kpad, int64_t npad,
                                   float* __restrict__ bt_hi, float* __restrict__ bt_lo) {
  __shared__ float tile[32][33];
  const int64_t k0 = (int64_t)blockIdx.x * 32, f0 = (int64_t)blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t k = k0 + r, f = f0 + threadIdx.x;
    tile[r][threadIdx.x] = (k < K && f < F) ? w[k * F + f] : 0.f;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t f = f0 + r, k = k0 + threadIdx.x;
    if (f < npad && k < kpad) {
      const float v = tile[threadIdx.x][r];
      const float h = bt_lo ? sm100::tf32_hi(v) : v;
      bt_hi[f * kpad + k] = h;
      if (bt_lo) bt_lo[f * kpad + k] = v - h;
    }
  }
}

// d[i] = sum_{s=0..splits-1} partial[s][i] over a dense rows x ldd plane (ldd % 4 == 0),
// fixed split order: deterministic.
__global__ void split_reduce_kernel(const float* __restrict__ partial, float* __restrict__ d, int64_t plane4,
                                    int splits) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < plane4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 acc = reinterpret_cast<const float4*>(partial)[i];
    for (int s = 1; s < splits; ++s) {
      const float4 v = reinterpret_cast<const float4*>(partial)[s * plane4 + i];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    reinterpret_cast<float4*>(d)[i] = acc;
  }
}

template <int BN, bool THREE_X, int AMODE>
cudaError_t launch_t(const DevArgs& a, dim3 grid, cudaStream_t s) {
  using C_ = Cfg<BN, THREE_X>;
  auto kern = gemm_tcgen05_kernel<BN, THREE_X, AMODE>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C_::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  kern<<<grid, NTHREADS, C_::SMEM, s>>>(a);
  return cudaGetLastError();
}

template <bool THREE_X, int AMODE>
cudaError_t launch_bn(int bn, const DevArgs& a, dim3 grid, cudaStream_t s) {
  switch (bn) {
    case 64: return launch_t<64, THREE_X, AMODE>(a, grid, s);
    case 128: return launch_t<128, THREE_X, AMODE>(a, grid, s);
    case 256: return launch_t<256, THREE_X, AMODE>(a, grid, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

int gemm_choose_block_n(int64_t N, bool three_x) {
  if (N <= 64) return 64;
  if (N <= 128) return 128;
  return three_x ? 128 : 256;
}

int gemm_choose_splits(int64_t M, int64_t N, int64_t K, int batch, int block_n) {
  const int64_t tiles = ((M + BM - 1) / BM) * ((N + block_n - 1) / block_n) * batch;
  const int64_t nkb = (K + BK - 1) / BK;
  if (tiles >= 148 || nkb < 8) return 1;
  int64_t s = 148 / tiles;            // fill about one wave
  if (s > nkb / 4) s = nkb / 4;       // keep >= 4 k-blocks per split
  if (s > 16) s = 16;
  return s < 1 ? 1 : (int)s;
}

cudaError_t launch_gemm(const Problem& conv, const GemmArgs& g, cudaStream_t s) {
  DevArgs a{};
  a.H = conv.H; a.W = conv.W; a.C = conv.C; a.KH = conv.KH; a.KW = conv.KW; a.SH = conv.SH; a.SW = conv.SW;
  a.HO = conv.HO; a.WO = conv.WO; a.PT = conv.pad_top; a.PL = conv.pad_left;
  a.a = g.a; a.lda = g.lda; a.a_bstride = g.a_batch_stride;
  a.bt_hi = g.bt_hi; a.bt_lo = g.bt_lo; a.ldb = g.ldb; a.b_bstride = g.b_batch_stride;
  a.d = g.d; a.ldd = g.ldd; a.d_bstride = g.d_batch_stride; a.partial = g.partial;
  a.M = g.M; a.N = g.N; a.K = g.K;
  a.nkb = (int)((g.K + BK - 1) / BK);
  a.splits = g.splits; a.batch = g.batch;
  const int64_t mt = (g.M + BM - 1) / BM;
  const int64_t nt = (g.N + g.block_n - 1) / g.block_n;
  if (mt > 0x7FFFFFFF || nt > 65535 || (int64_t)g.batch * g.splits > 65535) return cudaErrorInvalidConfiguration;
  dim3 grid((unsigned)mt, (unsigned)nt, (unsigned)(g.batch * g.splits));
  int amode;
  if (g.a_mode == 1) amode = A_DENSE;
  else amode = (conv.C % 4 == 0) ? A_CONV_VEC4 : A_CONV_SCALAR;
  cudaError_t e;
  if (g.three_x) {
    if (amode == A_DENSE) e = launch_bn<true, A_DENSE>(g.block_n, a, grid, s);
    else if (amode == A_CONV_VEC4) e = launch_bn<true, A_CONV_VEC4>(g.block_n, a, grid, s);
    else e = launch_bn<true, A_CONV_SCALAR>(g.block_n, a, grid, s);
  } else {
    if (amode == A_DENSE) e = launch_bn<false, A_DENSE>(g.block_n, a, grid, s);
    else if (amode == A_CONV_VEC4) e = launch_bn<false, A_CONV_VEC4>(g.block_n, a, grid, s);
    else e = launch_bn<false, A_CONV_SCALAR>(g.block_n, a, grid, s);
  }
  if (e != cudaSuccess) return e;
  if (g.splits > 1) e = launch_split_reduce(g.partial, g.d, (int64_t)g.batch * g.M, g.N, g.ldd, g.splits, s);
  return e;
}

cudaError_t launch_split_reduce(const float* partial, float* d, int64_t rows, int64_t cols, int64_t ldd, int splits,
                                cudaStream_t s) {
  if (ldd % 4 != 0 || cols != ldd) return cudaErrorInvalidValue;  // callers only split dense, 16B rows
  const int64_t plane4 = rows * ldd / 4;
  int64_t blocks = (plane4 + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  split_reduce_kernel<<<(unsigned)blocks, 256, 0, s>>>(partial, d, plane4, splits);
  return cudaGetLastError();
}

cudaError_t launch_filter_prep(const float* filt, int64_t K, int64_t F, int64_t kpad, int64_t npad, float* bt_hi,
                               float* bt_lo, cudaStream_t s) {
  dim3 grid((unsigned)(kpad / 32), (unsigned)((npad + 31) / 32));
  filter_prep_kernel<<<grid, dim3(32, 8), 0, s>>>(filt, K, F, kpad, npad, bt_hi, bt_lo);
  return cudaGetLastError();
}

}  // namespace conv2d
