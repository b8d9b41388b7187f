// gemm_halo.cu -- 3x3 / stride-1 implicit GEMM with halo-tile reuse (IMPLICIT_GEMM variant for
// small-N layers such as ResNet-50 R4 and VGG conv1_2/conv2_x).
//
// Why: with im2col boxes every input pixel is fetched by TMA once per filter tap (9x), and on
// B200 the TMA engine moves padded/strided 128-byte rows at only ~23-34 B/clk/SM
// (tools/tma_probe.cu, profiles/round1_ncu.md).  For N <= 128 tiles that, not the tensor core,
// bounds the main loop.  Here one 4-D tiled box -- the 16 (w) x 18 (h) input halo of an 8 (wo) x
// 16 (ho) output tile, 32 channels -- is loaded per channel block, and the nine tap-shifted
// A operands are *views* of it: tap (r, s) starts s rows + 16 r rows into the halo, its 8-row
// groups (one output row of 8 pixels each) are 16 halo rows = 2048 B apart (a whole number of
// SWIZZLE_128B periods).  The tensor core applies the 128-byte swizzle on absolute smem address
// bits, so these row-shifted views need no descriptor correction (base offset 0; measured).
// TMA traffic for A drops from 9 x 16 KB to 36 KB per channel block, and the 3xTF32 lo split is
// computed once per halo instead of once per tap.
//
// Same warp roles as gemm2sm.cu (0-3 transform, 4 TMA producer, 5 MMA issuer + TMEM, 6-9
// epilogue), same CTA pair (cta_group::2, M = 256 = two independent 8x16 spatial tiles), two
// rings: halo slots (TMA -> transform -> MMA) and B stages (2-CTA TMA straight to the leader).
#include <cstdlib>

#include "gemm2sm.h"
#include "sm100.cuh"

namespace conv2d {
namespace {

using namespace sm100;

constexpr int BK = 32;
constexpr int NTHREADS = 320;
constexpr int TW = 8, TH = 16;            // CTA output tile (wo x ho) = 128 GEMM rows
constexpr int HWD = 16, HHT = TH + 2;     // halo box: 16 (w) x 18 (h) pixels
constexpr int HALO_ROWS = HWD * HHT;      // 288
constexpr int HALO_BYTES = HALO_ROWS * 128;  // 36 KB (multiple of 1024)

struct HArgs {
  int N, H, W, HO, WO, PT, PL, ncb;
  int tiles_w, tiles_h, cta_tiles, pair_tiles, nt, total;
  int64_t M, F, ldd;
  float* d;
  int tma_store;
};

template <int BN, bool THREE_X>
struct HCfg {
  static constexpr int BHALF = (BN / 2) * BK * 4;
  static constexpr int BFULL = BN * BK * 4;
  static constexpr int HS = THREE_X ? 2 : 3;                           // halo slots
  static constexpr int HSLOT = HALO_BYTES * (THREE_X ? 2 : 1);         // hi (+ lo)
  // CONCAT (3xTF32, BN = 64, where smem operand reads bound the MMA): B stage Z = BN rows (CTA0:
  // B_hi, CTA1: B_lo) for one N'=2BN MMA hi x [B_hi | B_lo] -- A_hi is read once for both products --
  // plus X = BN/2 rows of B_hi (this CTA's half) for lo x B_hi; the epilogue adds the two column halves.
  // Otherwise (BN = 128, TF32): X = B_hi half [+ B_lo half], three / one MMAs per K step.
  static constexpr bool CONCAT = THREE_X && BN == 64;
  static constexpr int BSTAGE = CONCAT ? BFULL + BHALF : (THREE_X ? 2 : 1) * BHALF;
  static constexpr int ACC = CONCAT ? 2 * BN : BN;                     // TMEM columns per accumulator
  static constexpr int EPI = 4 * 2 * 32 * 128;
  static constexpr int BUDGET = 232448 - EPI - 1024 - 512 - HS * HSLOT;
  static constexpr int S = (BUDGET / BSTAGE) > 12 ? 12 : (BUDGET / BSTAGE);
  static constexpr int SMEM = HS * HSLOT + S * BSTAGE + EPI + 1024 + 512;
  static constexpr uint32_t TMEM_COLS = 2 * ACC;
  static_assert(S >= 2, "halo kernel needs >= 2 B stages");
  static_assert(2 * ACC <= 512, "TMEM");
};

struct HTile {
  int ni, n, wo0, ho0;
};

__device__ __forceinline__ HTile hdecode(const HArgs& a, int t, uint32_t rank) {
  HTile r;
  r.ni = t % a.nt;
  const int ct = (t / a.nt) * 2 + (int)rank;  // this CTA's spatial tile (pairs take consecutive tiles)
  r.wo0 = (ct % a.tiles_w) * TW;
  r.ho0 = ((ct / a.tiles_w) % a.tiles_h) * TH;
  r.n = ct / (a.tiles_w * a.tiles_h);         // == N for the dummy tile of an odd count: all OOB
  return r;
}

template <int BN, bool THREE_X>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NTHREADS, 1)
    halo_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmBh,
                const __grid_constant__ CUtensorMap tmBhF, const __grid_constant__ CUtensorMap tmBlF,
                const __grid_constant__ CUtensorMap tmD,
                const __grid_constant__ HArgs args) {
  using C_ = HCfg<BN, THREE_X>;
  constexpr int HS = C_::HS, S = C_::S;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  auto halo_hi = [&](int h) { return smem + (size_t)h * C_::HSLOT; };
  auto halo_lo = [&](int h) { return smem + (size_t)h * C_::HSLOT + HALO_BYTES; };
  auto b_z = [&](int s) { return smem + (size_t)HS * C_::HSLOT + (size_t)s * C_::BSTAGE; };  // CONCAT only
  auto b_x = [&](int s) { return b_z(s) + (C_::CONCAT ? C_::BFULL : 0); };                    // B_hi half
  auto b_lo = [&](int s) { return b_x(s) + C_::BHALF; };                                      // 3x, !CONCAT
  uint8_t* epi_smem = smem + (size_t)HS * C_::HSLOT + (size_t)S * C_::BSTAGE;
  uint64_t* h_ld = reinterpret_cast<uint64_t*>(epi_smem + C_::EPI);
  uint64_t* h_full = h_ld + HS;
  uint64_t* h_empty = h_full + HS;
  uint64_t* b_full = h_empty + HS;
  uint64_t* b_empty = b_full + S;
  uint64_t* tmem_full = b_empty + S;
  uint64_t* tmem_empty = tmem_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int cid = (int)cluster_id_x(), ncl = (int)nclusters_x();
  const int taps = 9;

  if (threadIdx.x == 0) {
    for (int h = 0; h < HS; ++h) {
      mbar_init(&h_ld[h], 1);
      mbar_init(&h_full[h], 2 * 128);
      mbar_init(&h_empty[h], 1);
    }
    for (int s = 0; s < S; ++s) {
      mbar_init(&b_full[s], 1);
      mbar_init(&b_empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], 2 * 128);
    }
    fence_mbar_init();
  }
  if (warp == 4 && lane == 0) {
    tma_prefetch(&tmX);
    tma_prefetch(&tmBh);
    if (THREE_X) {
      tma_prefetch(&tmBhF);
      tma_prefetch(&tmBlF);  // !CONCAT: the B_lo half map
    }
  }
  if (warp == 5) tmem_alloc_2sm<C_::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 4) {
    // ============================ TMA producer ============================
    // Work is a flat sequence of "units" (tile, channel block); the halo of unit u+1 is issued
    // before the nine B loads of unit u so it lands while unit u's MMAs run.
    if (lane == 0) {
      const uint32_t b_full_leader = mapa(smem_u32(b_full), 0);
      const int my_tiles = args.total > cid ? (args.total - cid + ncl - 1) / ncl : 0;
      const int units = my_tiles * args.ncb;
      auto issue_halo = [&](int u) {
        const HTile tl = hdecode(args, cid + (u / args.ncb) * ncl, rank);
        const int cb = u % args.ncb;
        const int h = u % HS;
        if (u >= HS) mbar_wait(&h_empty[h], ((u / HS) - 1) & 1);
        mbar_arrive_expect_tx(&h_ld[h], HALO_BYTES);
        tma_load_4d(&tmX, &h_ld[h], smem_u32(halo_hi(h)), cb * BK, tl.wo0 - args.PL, tl.ho0 - args.PT, tl.n);
      };
      if (units > 0) issue_halo(0);
      uint32_t bit = 0;
      for (int u = 0; u < units; ++u) {
        if (u + 1 < units) issue_halo(u + 1);
        const HTile tl = hdecode(args, cid + (u / args.ncb) * ncl, rank);
        const int cb = u % args.ncb;
        const int nrow = tl.ni * BN + (int)rank * (BN / 2);
        for (int tap = 0; tap < taps; ++tap, ++bit) {
          const int s = bit % S;
          if (bit >= (uint32_t)S) mbar_wait(&b_empty[s], ((bit / S) - 1) & 1);
          if (rank == 0) mbar_arrive_expect_tx(&b_full[s], 2 * C_::BSTAGE);
          const uint32_t fb = b_full_leader + (uint32_t)(s * sizeof(uint64_t));
          const int k0 = (tap * args.ncb + cb) * BK;  // filter prep order: k = tap * C + c
          tma_load_3d_2sm(&tmBh, fb, smem_u32(b_x(s)), k0, nrow, 0);
          if (C_::CONCAT)  // CTA0: B_hi rows [ni*BN, +BN); CTA1: B_lo rows [ni*BN, +BN)
            tma_load_3d_2sm(rank == 0 ? (const void*)&tmBhF : (const void*)&tmBlF, fb, smem_u32(b_z(s)), k0,
                            tl.ni * BN, 0);
          else if (THREE_X)  // B_lo half (tmBlF holds the half-box B_lo map when !CONCAT)
            tma_load_3d_2sm(&tmBlF, fb, smem_u32(b_lo(s)), k0, nrow, 0);
        }
      }
      for (int i = 0; i < S; ++i, ++bit)
        if (bit >= (uint32_t)S) mbar_wait(&b_empty[bit % S], ((bit / S) - 1) & 1);
      for (int i = 0; i < HS; ++i) {
        const int u = units + i;
        if (u >= HS) mbar_wait(&h_empty[u % HS], ((u / HS) - 1) & 1);
      }
    }
  } else if (warp == 5) {
    // ============================ MMA issuer (leader) ============================
    if (rank == 0) {  // whole warp, converged: operands stay warp-uniform
      constexpr uint32_t idesc = idesc_tf32(256, BN);
      constexpr uint32_t idesc2 = idesc_tf32(256, 2 * BN);  // 3x: hi x [B_hi | B_lo]
      uint32_t hit = 0, bit = 0, ai = 0;
      for (int t = cid; t < args.total; t += ncl, ++ai) {
        const int acc = ai & 1;
        if (ai >= 2) mbar_wait(&tmem_empty[acc], ((ai >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem_base + (uint32_t)(acc * C_::ACC);
        for (int cb = 0; cb < args.ncb; ++cb, ++hit) {
          const int h = hit % HS;
          mbar_wait(&h_full[h], (hit / HS) & 1);
          tc_fence_after();
          for (int tap = 0; tap < taps; ++tap, ++bit) {
            const int s = bit % S;
            mbar_wait(&b_full[s], (bit / S) & 1);
            tc_fence_after();
            const int r = tap / 3, c = tap % 3;
            const uint32_t off = (uint32_t)((r * HWD + c) * 128);  // view start: row r*16 + c of the halo
            // base offset stays 0: the tensor core swizzles on absolute smem address bits, so a view
            // starting c rows into a 1024-byte period needs no descriptor correction (measured:
            // setting the base-offset field to c breaks the integer-exact parity tests)
            const uint64_t dah = umma_desc_sw128_kmajor_sbo(smem_u32(halo_hi(h)) + off, HWD * 128, 0u);
            const uint64_t dal =
                THREE_X ? umma_desc_sw128_kmajor_sbo(smem_u32(halo_lo(h)) + off, HWD * 128, 0u) : 0;
            const uint64_t dbx = umma_desc_sw128_kmajor(smem_u32(b_x(s)));
            const uint64_t dbz = C_::CONCAT ? umma_desc_sw128_kmajor(smem_u32(b_z(s))) : 0;
            const uint64_t dbl = (THREE_X && !C_::CONCAT) ? umma_desc_sw128_kmajor(smem_u32(b_lo(s))) : 0;
#pragma unroll
            for (int k = 0; k < BK / 8; ++k) {
              const uint64_t adv = (uint64_t)((k * 8 * 4) >> 4);
              const uint32_t accum = (cb > 0 || tap > 0 || k > 0) ? 1u : 0u;
              if (THREE_X && !C_::CONCAT) {
                mma_tf32_2sm_warp(d, dal + adv, dbx + adv, idesc, accum);
                mma_tf32_2sm_warp(d, dah + adv, dbl + adv, idesc, 1u);
                mma_tf32_2sm_warp(d, dah + adv, dbx + adv, idesc, 1u);
              } else if (C_::CONCAT) {
                // cols [0,BN) += hi*B_hi, cols [BN,2BN) += hi*B_lo   (A_hi read once for both products)
                mma_tf32_2sm_warp(d, dah + adv, dbz + adv, idesc2, accum);
                // cols [0,BN) += lo*B_hi
                mma_tf32_2sm_warp(d, dal + adv, dbx + adv, idesc, 1u);
              } else {
                mma_tf32_2sm_warp(d, dah + adv, dbx + adv, idesc, accum);
              }
            }
            mma_commit_2sm_mc_warp(&b_empty[s], 0x3);
          }
          mma_commit_2sm_mc_warp(&h_empty[h], 0x3);
        }
        mma_commit_2sm_mc_warp(&tmem_full[acc], 0x3);
      }
    }
    __syncwarp();
  } else if (warp < 4) {
    // ============================ halo transform (128 threads) ============================
    const int t = threadIdx.x;
    const uint32_t h_full_leader = mapa(smem_u32(h_full), 0);
    uint32_t hit = 0;
    for (int tt = cid; tt < args.total; tt += ncl) {
      for (int cb = 0; cb < args.ncb; ++cb, ++hit) {
        const int h = hit % HS;
        mbar_wait(&h_ld[h], (hit / HS) & 1);
        if (THREE_X) {
          // elementwise lo = x - trunc_tf32(x) over the whole halo (layout-agnostic: same offsets)
          const uint32_t hi = smem_u32(halo_hi(h)), lo = smem_u32(halo_lo(h));
          for (int q = t; q < HALO_ROWS * 8; q += 128) {
            const float4 v = lds128(hi + q * 16);
            sts128(lo + q * 16, make_float4(v.x - tf32_hi(v.x), v.y - tf32_hi(v.y), v.z - tf32_hi(v.z),
                                             v.w - tf32_hi(v.w)));
          }
          fence_proxy_async_smem();
        }
        mbar_arrive_remote(h_full_leader + (uint32_t)(h * sizeof(uint64_t)));
      }
    }
  } else {
    // ============================ epilogue (warps 6-9) ============================
    // warp q owns TMEM lanes [32q, 32q+32) = output rows ho0 + 4q .. +3, wo0 .. wo0+7
    const int q = warp & 3;
    const uint32_t tmem_empty_leader = mapa(smem_u32(tmem_empty), 0);
    const uint32_t ebuf = smem_u32(epi_smem) + (uint32_t)(q * 2 * 4096);
    if (args.tma_store && lane == 0) tma_prefetch(&tmD);
    uint32_t ai = 0, chunk = 0;
    for (int t = cid; t < args.total; t += ncl, ++ai) {
      const HTile tl = hdecode(args, t, rank);
      const int acc = ai & 1;
      mbar_wait(&tmem_full[acc], (ai >> 1) & 1);
      tc_fence_after();
      const int ho = tl.ho0 + 4 * q + lane / 8, wo = tl.wo0 + lane % 8;
      const bool row_ok = tl.n < args.N && ho < args.HO && wo < args.WO;
      const bool warp_ok = tl.n < args.N && tl.ho0 + 4 * q < args.HO;
      const int n0 = tl.ni * BN;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        float v[32];
        tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * C_::ACC + c0), v);
        if (C_::CONCAT) {  // add the hi*B_lo correction columns
          float w[32];
          tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * C_::ACC + BN + c0), w);
#pragma unroll
          for (int k = 0; k < 32; ++k) v[k] += w[k];
        }
        if (c0 + 32 >= BN) {
          tc_fence_before();
          mbar_arrive_remote(tmem_empty_leader + (uint32_t)(acc * sizeof(uint64_t)));
        }
        if (args.tma_store) {
          if (warp_ok && n0 + c0 < args.F) {
            const uint32_t buf = ebuf + (chunk & 1) * 4096;
            if (lane == 0) bulk_wait_read<1>();
            __syncwarp();
#pragma unroll
            for (int k = 0; k < 8; ++k)
              sts128(buf + sw128_offset(lane, k), make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]));
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_4d(&tmD, buf, n0 + c0, tl.wo0, tl.ho0 + 4 * q, tl.n);
              bulk_commit();
            }
            ++chunk;
          }
        } else if (row_ok) {
          float* dst = args.d + (((int64_t)tl.n * args.HO + ho) * args.WO + wo) * args.ldd + n0 + c0;
          const int64_t nrem = args.F - (n0 + c0);
#pragma unroll
          for (int k = 0; k < 32; ++k)
            if (k < nrem) dst[k] = v[k];
        }
      }
    }
    if (args.tma_store && lane == 0) bulk_wait<0>();
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc_2sm<C_::TMEM_COLS>(tmem_base);
  }
}

template <int BN, bool THREE_X>
cudaError_t launch_h(const CUtensorMap& x, const CUtensorMap& bh, const CUtensorMap& bhf, const CUtensorMap& blf,
                     const CUtensorMap& dm, const HArgs& a, int clusters, cudaStream_t s) {
  using C_ = HCfg<BN, THREE_X>;
  auto kern = halo_kernel<BN, THREE_X>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C_::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  kern<<<dim3(2 * clusters), NTHREADS, C_::SMEM, s>>>(x, bh, bhf, blf, dm, a);
  return cudaGetLastError();
}

}  // namespace

bool halo_ok(const Problem& p) {
  return p.KH == 3 && p.KW == 3 && p.SH == 1 && p.SW == 1 && p.C % 32 == 0 && p.F <= 128 &&
         (int64_t)p.N * ((p.HO + TH - 1) / TH) * ((p.WO + TW - 1) / TW) < (1 << 30);
}

cudaError_t launch_gemm_halo(const Problem& p, const float* in, const float* bt_hi, const float* bt_lo, int64_t kpad,
                             int64_t npad, int block_n, float* out, cudaStream_t s) {
  const bool three_x = bt_lo != nullptr;
  HArgs a{};
  a.N = p.N; a.H = p.H; a.W = p.W; a.HO = p.HO; a.WO = p.WO; a.PT = p.pad_top; a.PL = p.pad_left;
  a.ncb = p.C / 32;
  a.tiles_w = (p.WO + TW - 1) / TW;
  a.tiles_h = (p.HO + TH - 1) / TH;
  a.cta_tiles = p.N * a.tiles_w * a.tiles_h;
  a.pair_tiles = (a.cta_tiles + 1) / 2;
  a.nt = (int)((p.F + block_n - 1) / block_n);
  a.total = a.pair_tiles * a.nt;
  a.M = p.M();
  a.F = p.F;
  a.ldd = p.F;
  a.d = out;
  alignas(64) CUtensorMap tx{}, tbh{}, tbhf{}, tblf{}, td{};
  {  // input halo boxes: {32 ch, 16 w, 18 h, 1 n} over NHWC, OOB (padding) -> 0
    const uint64_t dims[4] = {(uint64_t)p.C, (uint64_t)p.W, (uint64_t)p.H, (uint64_t)p.N};
    const uint64_t st[3] = {(uint64_t)p.C * 4, (uint64_t)p.W * p.C * 4, (uint64_t)p.H * p.W * p.C * 4};
    const uint32_t box[4] = {32, HWD, HHT, 1};
    if (!gemm2_encode_tiled(&tx, 4, in, dims, st, box, true)) return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[3] = {(uint64_t)kpad, (uint64_t)npad, 1};
    const uint64_t st[2] = {(uint64_t)kpad * 4, (uint64_t)kpad * 4 * npad};
    const uint32_t box[3] = {32, (uint32_t)block_n / 2, 1};
    const uint32_t boxf[3] = {32, (uint32_t)block_n, 1};
    if (!gemm2_encode_tiled(&tbh, 3, bt_hi, dims, st, box, true)) return cudaErrorInvalidValue;
    const bool concat = three_x && block_n == 64;
    if (concat && (!gemm2_encode_tiled(&tbhf, 3, bt_hi, dims, st, boxf, true) ||
                   !gemm2_encode_tiled(&tblf, 3, bt_lo, dims, st, boxf, true)))
      return cudaErrorInvalidValue;
    if (three_x && !concat) {  // half-box B_lo map in the tmBlF slot
      if (!gemm2_encode_tiled(&tblf, 3, bt_lo, dims, st, box, true)) return cudaErrorInvalidValue;
      tbhf = tbh;
    }
    if (!three_x) tbhf = tblf = tbh;
  }
  a.tma_store = 0;
  if (p.F % 4 == 0) {  // output boxes {32 f, 8 wo, 4 ho, 1 n}
    const uint64_t dims[4] = {(uint64_t)p.F, (uint64_t)p.WO, (uint64_t)p.HO, (uint64_t)p.N};
    const uint64_t st[3] = {(uint64_t)p.F * 4, (uint64_t)p.F * 4 * p.WO, (uint64_t)p.F * 4 * p.WO * p.HO};
    const uint32_t box[4] = {32, TW, 4, 1};
    a.tma_store = gemm2_encode_tiled(&td, 4, out, dims, st, box, true) ? 1 : 0;
  }
  if (!a.tma_store) td = tbh;
  const int clusters = a.total < 74 ? a.total : 74;
  switch (block_n) {
    case 64: return three_x ? launch_h<64, true>(tx, tbh, tbhf, tblf, td, a, clusters, s)
                            : launch_h<64, false>(tx, tbh, tbhf, tblf, td, a, clusters, s);
    case 128: return three_x ? launch_h<128, true>(tx, tbh, tbhf, tblf, td, a, clusters, s)
                             : launch_h<128, false>(tx, tbh, tbhf, tblf, td, a, clusters, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace conv2d
