// gemm2sm.cu -- persistent 2-CTA tcgen05 GEMM core (the contraction behind implicit GEMM,
// 1x1-as-matmul and Winograd's batched GEMMs).
//
//   D[b](m, n) = sum_k A[b](m, k) * Bt[b](n, k)        fp32 in, fp32 accumulate in TMEM
//
// Design:
//   * a CTA pair (cluster of 2, tcgen05 cta_group::2) owns a 256 x BN output tile: CTA r holds
//     A rows [128r, 128r+128) and B rows (output features) [r*BN/2, (r+1)*BN/2) in its smem;
//     the leader issues M=256 x N=BN x K=8 kind::tf32 MMAs that read both CTAs' smem and
//     accumulate into both CTAs' TMEM (each CTA: its 128 rows x BN fp32 columns);
//   * persistent: grid = min(tiles, 74) pairs, static round-robin tile schedule, two TMEM
//     accumulators so the epilogue of tile i overlaps the main loop of tile i+1;
//   * operands arrive by TMA into SWIZZLE_128B K-major stages:
//       A_IM2COL : cp.async.bulk.tensor.4d.im2col straight from the NHWC input -- the im2col
//                  matrix is never materialised; one box = 128 output
//                  pixels x 32 channels at filter tap (r, s); OOB (padding, tails) -> zeros;
//       A_DENSE  : 3-D tiled TMA of a dense K-major matrix (Winograd V, 1x1 fallbacks);
//       A_GATHER : cp.async 16-byte gathers by the transform warps (C % 32 != 0, e.g. the
//                  C=3 stem after channel padding to 4, flat k = (r, s, c));
//     B (filter, pre-transposed/split by filter_prep) always by 3-D tiled TMA;
//   * 3xTF32 (fp32-faithful mode): the transform warps write lo = a - trunc_tf32(a) next to
//     each A stage (hi = the raw fp32 stage itself: the tensor core reads only its top 19
//     bits); B's split comes from filter_prep; the MMA warp issues lo*hi + hi*lo + hi*hi
//     per K=8 step.
// Warp roles (448 threads): 0-3 transform/gather, 4 TMA producer, 5 MMA issuer + TMEM
// allocator, 6-9 epilogue (TMEM -> registers -> global, 32 columns per tcgen05.ld), 10-13 B-lo split
// (3xTF32 with B streamed straight from the filter: lo = b - trunc(b) of each stage's B half, so
// the transform warps only handle A; idle otherwise).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "gemm2sm.h"
#include "launch.cuh"
#include "sm100.cuh"

namespace conv2d {
namespace {

using namespace sm100;

constexpr int BMC = 128;  // rows per CTA (pair tile = 256)
constexpr int BK = 32;    // fp32 per 128-byte swizzle row
constexpr int NTHREADS = 448;  // 14 warps: see the role list in the header comment
constexpr int A_TILE = BMC * BK * 4;  // 16 KB

struct DevArgs {
  int H, W, C, KH, KW, SH, SW, HO, WO, PT, PL;
  int ncb;
  int Cg;
  const float* xg;
  int64_t Kg;
  int64_t M, N;
  int nkb, mt, nt, splits, batch, total_tiles;
  int wblk, hblk;  // A_ROWSEG: 16-wide / 16-high spatial pair-tile grid
  int a_row_bytes; // A_ROWSEG: bytes TMA writes per 128-B smem row (KW*C4*4); the rest stays zero
  int halo_row_floats, halo_bytes;  // A_STEM: floats per halo row ((15*SW+KW)*C4), bytes per halo
  float* d;
  int64_t ldd, d_bstride;
  float* partial;
  int tma_store;  // 1: epilogue stages 32x32 chunks in smem and writes them with TMA stores
  // remainder split (rs_splits >= 2): units [0, rs_first) are whole tiles; the remaining tiles of the
  // partial last wave are cut into rs_splits K ranges each (units rs_first + i: tile rs_first + i / s, split
  // i % s), stored to the partial planes via tmP and summed by rsplit_reduce_kernel afterwards
  int rs_first, rs_splits;
  alignas(64) CUtensorMap tmP;  // partial planes {N, M, s} (remainder split only)
  int bstat;  // B-stationary schedule (B-resident with several N tiles): pair p owns N tile p % nt
  int b_mn;  // 1: B read straight from the row-major K x F filter (MN-major operand; no filter_prep)
  int early;  // 1: 3xTF32 relay A paths issue the first stages before the cluster barrier completes
  unsigned long long* trace;  // debug (conv2d_debug_trace): TRACE_SLOTS globaltimer stamps per CTA, or null
};

// debug trace slots (per CTA): entry, setup done, first TMA issued, first stage consumed by the MMA
// (leader), first accumulator ready (epilogue), last epilogue store issued, stores drained, exit
constexpr int TRACE_SLOTS = 8;
__device__ __forceinline__ void trace_at(const DevArgs& a, int slot) {
  if (a.trace) a.trace[blockIdx.x * TRACE_SLOTS + slot] = globaltimer_ns();
}

template <int BN, bool THREE_X, bool BRES = false, bool STEMH = false>
struct Cfg {
  static constexpr int BHALF = (BN / 2) * BK * 4;
  // TMA ring stage: [A (raw fp32 = TF32 hi) | B_hi | B_lo (3xTF32)].  3xTF32 keeps A's lo halves in
  // TMEM (LO_TMEM: 32 columns per stage next to the two accumulators; the lo*hi MMA takes A from
  // TMEM) when 2*BN leaves room, else in a separate smem ring (BN = 256).
  // BRES: the CTA's whole B half (all k-blocks, hi [+ lo]) is loaded once per kernel into a 64 KB
  // resident region and stages carry only A -- for single-N-tile, short-K layers where per-k-block
  // B traffic is a third of the TMA engine's work (the C=3 stems, 1x1 layers).
  static constexpr bool LO_TMEM = THREE_X && BN <= 128;
  static constexpr int STAGE = BRES ? A_TILE : A_TILE + (THREE_X ? 2 : 1) * BHALF;
  static constexpr int RES = BRES ? 65536 : 0;
  static constexpr int SL = (THREE_X && !LO_TMEM) ? 3 : 0;
  static constexpr int EPI = 4 * 2 * 32 * 128;  // 4 epilogue warps x 2 buffers x (32 rows x 128 B)
  static constexpr int HALO = STEMH ? 2 * 16384 : 0;  // A_STEM: two input-halo slots
  static constexpr int BUDGET = 232448 - EPI - 1024 - 512 - SL * A_TILE - RES - HALO;
  static constexpr int SMAX = LO_TMEM ? (512 - 2 * BN) / 32 : 12;
  static constexpr int STAGES = (BUDGET / STAGE) > SMAX ? SMAX : (BUDGET / STAGE);
  static constexpr int SMEM = STAGES * STAGE + SL * A_TILE + RES + HALO + EPI + 1024 + 512;
  static constexpr uint32_t TMEM_COLS = LO_TMEM ? 512 : 2 * BN;
  static constexpr uint32_t LO_COL0 = 2 * BN;  // first TMEM column of the lo slots (LO_TMEM)
  static constexpr int RES_KB_MAX = RES / ((THREE_X ? 2 : 1) * BHALF);  // k-blocks that fit resident
};

struct Tile {
  int mi, ni, bz, split, kb0, kb1;
  bool part;  // remainder-split unit: accumulates K range [kb0, kb1) of its tile into partial plane `split`
};

__device__ __forceinline__ Tile decode(const DevArgs& a, int u) {
  int t = u, rs = -1;
  if (a.rs_splits > 1 && u >= a.rs_first) {
    t = a.rs_first + (u - a.rs_first) / a.rs_splits;
    rs = (u - a.rs_first) % a.rs_splits;
  }
  Tile r;
  r.part = rs >= 0;
  r.ni = t % a.nt;
  const int rest = t / a.nt;
  r.mi = rest % a.mt;
  const int z = rest / a.mt;
  r.bz = z / a.splits;
  r.split = z % a.splits;
  r.kb0 = (int)((int64_t)r.split * a.nkb / a.splits);
  r.kb1 = (int)((int64_t)(r.split + 1) * a.nkb / a.splits);
  if (rs >= 0) {
    r.split = rs;
    r.kb0 = (int)((int64_t)rs * a.nkb / a.rs_splits);
    r.kb1 = (int)((int64_t)(rs + 1) * a.nkb / a.rs_splits);
  }
  return r;
}

// The j-th tile of CTA pair `cid` (of ncl), or -1.  Default: static round-robin over all tiles.
// B-stationary (args.bstat): pair cid owns N tile ni = cid % nt and walks that tile column's M tiles
// with stride = the number of pairs owning ni, so the pair's resident B half serves every tile it runs.
__device__ __forceinline__ int tile_at(const DevArgs& a, int cid, int ncl, int j) {
  if (!a.bstat) {
    const int64_t t = (int64_t)cid + (int64_t)j * ncl;
    return t < a.total_tiles ? (int)t : -1;
  }
  const int ni = cid % a.nt;
  const int owners = (ncl - ni + a.nt - 1) / a.nt;
  const int64_t mi = (int64_t)(cid / a.nt) + (int64_t)j * owners;
  return mi < a.mt ? (int)(mi * a.nt + ni) : -1;
}

template <int BN, bool THREE_X, int AMODE, bool BRES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NTHREADS, 1)
    gemm2sm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmBh,
                   const __grid_constant__ CUtensorMap tmBl, const __grid_constant__ CUtensorMap tmD,
                   const __grid_constant__ DevArgs args) {
  using C_ = Cfg<BN, THREE_X, BRES, AMODE == A_STEM>;
  constexpr int S = C_::STAGES;
  constexpr int LAG = S - 1 < 6 ? S - 1 : 6;  // gather pipelining depth (cp.async groups in flight)
  static_assert(S >= 2, "need >= 2 stages");
  // RELAY: A passes through the transform warps (3xTF32 split or cp.async gather), which then
  // signal the leader; otherwise the TMA engines signal the leader's full barrier directly.
  constexpr bool RELAY = THREE_X || AMODE == A_GATHER || AMODE == A_STEM;
  constexpr bool SPATIAL = AMODE == A_ROWSEG || AMODE == A_STEM;  // 16x8 spatial CTA tiles

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int SL = C_::SL;
  auto a_hi = [&](int s) { return smem + (size_t)s * C_::STAGE; };
  auto b_hi = [&](int s) { return smem + (size_t)s * C_::STAGE + A_TILE; };
  auto b_lo = [&](int s) { return smem + (size_t)s * C_::STAGE + A_TILE + C_::BHALF; };
  auto a_lo = [&](int l) { return smem + (size_t)S * C_::STAGE + (size_t)l * A_TILE; };  // lo ring slot
  uint8_t* res = smem + S * C_::STAGE + SL * A_TILE;  // BRES: resident B, hi k-blocks then lo k-blocks
  auto res_hi = [&](int kb) { return res + (size_t)kb * C_::BHALF; };
  auto res_lo = [&](int kb) { return res + (size_t)(C_::RES / 2) + (size_t)kb * C_::BHALF; };
  uint8_t* halo = res + C_::RES;  // A_STEM: two 16 KB input-halo slots
  uint8_t* epi_smem = halo + C_::HALO;  // 1024-aligned (all sizes multiples of 1024)
  uint64_t* ld_full = reinterpret_cast<uint64_t*>(epi_smem + C_::EPI);
  uint64_t* full = ld_full + S;
  uint64_t* empty = full + S;
  uint64_t* lo_empty = empty + S;
  uint64_t* tmem_full = lo_empty + (SL > 0 ? SL : 1);
  uint64_t* tmem_empty = tmem_full + 2;
  uint64_t* b_res = tmem_empty + 2;
  uint64_t* hs_full = b_res + 1;    // A_STEM halo ring: TMA -> transform
  uint64_t* hs_empty = hs_full + 2; //                   transform -> producer
  uint64_t* b_ready = hs_empty + 2; // BRES + b_mn + 3xTF32: both CTAs' resident lo halves written
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(b_ready + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int cid = (int)cluster_id_x();
  const int ncl = (int)nclusters_x();
  if (threadIdx.x == 0) trace_at(args, 0);
  pdl_trigger();  // launch.cuh: the next kernel may start its prologue while this one runs

  const uint32_t full_leader = mapa(smem_u32(full), 0);
  // A_NARROW: k-block kb = 8 (tap, channel-quad) boxes of 128 px x 16 B, box q at +2 KB;
  // taps past Kh*Kw get an out-of-image offset so the TMA zero-fills them.
  const int nq = args.Cg / 4;
  const int taps = args.KH * args.KW;
  auto narrow_box = [&](int kb, int q, int& c, uint16_t& ow, uint16_t& oh) {
    const int idx = kb * 8 + q;
    const int tap = idx / nq;
    c = (idx - tap * nq) * 4;
    if (tap < taps) {
      ow = (uint16_t)(tap % args.KW);
      oh = (uint16_t)(tap / args.KW);
    } else {
      ow = 0xFFFF;
      oh = 0xFFFF;
      c = 0;
    }
  };
  auto narrow_loads = [&](uint64_t* bar, uint32_t dst, int kb, int wb, int hb, int nimg) {
#pragma unroll 1
    for (int q = 0; q < 8; ++q) {
      int c;
      uint16_t ow, oh;
      narrow_box(kb, q, c, ow, oh);
      tma_load_im2col_4d(&tmA, bar, dst + q * 2048, c, wb, hb, nimg, ow, oh);
    }
  };
  auto narrow_loads_2sm = [&](uint32_t bar, uint32_t dst, int kb, int wb, int hb, int nimg) {
#pragma unroll 1
    for (int q = 0; q < 8; ++q) {
      int c;
      uint16_t ow, oh;
      narrow_box(kb, q, c, ow, oh);
      tma_load_im2col_4d_2sm(&tmA, bar, dst + q * 2048, c, wb, hb, nimg, ow, oh);
    }
  };
  // b_mn: B box = {32 n, 32 k, BN/64 n-chunks} of the 3-D view {n % 32, k, n / 32} of the HWCF
  // filter; only hi (= the raw fp32) comes by TMA, the transform warps derive lo in smem.
  const bool bmn = args.b_mn != 0;
  const int b_copies = (THREE_X && !bmn) ? 2 : 1;
  // A_ROWSEG boxes are exactly KW*C4 floats wide (no OOB elements -> TMA fast path): fewer bytes
  const uint32_t a_bytes = AMODE == A_GATHER ? 0u : AMODE == A_ROWSEG ? (uint32_t)args.a_row_bytes * 128u : A_TILE;
  const uint32_t bytes = a_bytes + (BRES ? 0u : (uint32_t)(b_copies * C_::BHALF));
  // tile -> TMA coordinates of this CTA's A rows (m_cta / image window) and B half (nrow)
  auto coords = [&](const Tile& tl, int64_t& m_cta, int& wb, int& hb, int& nimg, int& nrow) {
    m_cta = (int64_t)tl.mi * 2 * BMC + rank * BMC;
    wb = hb = nimg = 0;
    if (SPATIAL) {
      wb = (tl.mi % args.wblk) * 16;
      hb = ((tl.mi / args.wblk) % args.hblk) * 16 + (int)rank * 8;
      nimg = tl.mi / (args.wblk * args.hblk);
    } else if (AMODE == A_IM2COL || AMODE == A_NARROW) {
      const int64_t hw = (int64_t)args.HO * args.WO;
      nimg = (int)(m_cta / hw);
      const int rem = (int)(m_cta % hw);
      wb = (rem % args.WO) * args.SW - args.PL;
      hb = (rem / args.WO) * args.SH - args.PT;
    }
    nrow = tl.ni * BN + (int)rank * (BN / 2);
  };
  // RELAY stage s <- k-block kb: A (and the per-stage B) into this CTA's smem, on its own ld_full[s]
  auto relay_load = [&](int s, int kb, const Tile& tl, int64_t m_cta, int wb, int hb, int nimg, int nrow) {
    const int tap = AMODE == A_IM2COL ? kb / args.ncb : 0;
    const int cb = AMODE == A_IM2COL ? kb - tap * args.ncb : 0;
    mbar_arrive_expect_tx(&ld_full[s], bytes);
    if (AMODE == A_IM2COL)
      tma_load_im2col_4d(&tmA, &ld_full[s], smem_u32(a_hi(s)), cb * BK, wb, hb, nimg, (uint16_t)(tap % args.KW),
                         (uint16_t)(tap / args.KW));
    else if (AMODE == A_NARROW)
      narrow_loads(&ld_full[s], smem_u32(a_hi(s)), kb, wb, hb, nimg);
    else if (AMODE == A_ROWSEG)
      tma_load_5d(&tmA, &ld_full[s], smem_u32(a_hi(s)), 0, wb, hb, nimg, kb);
    else if (AMODE == A_DENSE)
      tma_load_3d(&tmA, &ld_full[s], smem_u32(a_hi(s)), kb * BK, (int)m_cta, tl.bz);
    if (!BRES && bmn) {
      tma_load_3d(&tmBh, &ld_full[s], smem_u32(b_hi(s)), 0, kb * BK, nrow / 32);
    } else if (!BRES) {
      tma_load_3d(&tmBh, &ld_full[s], smem_u32(b_hi(s)), kb * BK, nrow, tl.bz);
      if (THREE_X) tma_load_3d(&tmBl, &ld_full[s], smem_u32(b_lo(s)), kb * BK, nrow, tl.bz);
    }
  };
  // 3xTF32 relay loads signal only this CTA's own ld_full barriers, so the producer thread initialises
  // the barriers itself and issues the first tile's first S k-blocks after its cluster-barrier arrival,
  // before the barrier completes: the first loads' latency hides behind the CTA-pair setup (excluded:
  // A paths whose stages are zero-filled first, the gather and the stem halo)
  const bool early = THREE_X && args.early && (AMODE == A_IM2COL || AMODE == A_DENSE || AMODE == A_NARROW ||
                                 (AMODE == A_ROWSEG && args.a_row_bytes == 128));
  uint32_t pre = 0;  // producer: k-block iterations already issued
  if (warp == 4 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&ld_full[s], 1);
      // RELAY: both CTAs' 128 transform threads (+ 128 B-split threads each when they run) arrive
      mbar_init(&full[s], RELAY ? 2 * 128 * ((THREE_X && !BRES && args.b_mn) ? 2 : 1) : 1);
      mbar_init(&empty[s], 1);
    }
    for (int l = 0; l < SL; ++l) mbar_init(&lo_empty[l], 1);
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], 2 * 128);
    }
    mbar_init(b_res, 1);
    mbar_init(b_ready, 2 * 128);
    for (int h = 0; h < 2; ++h) {
      mbar_init(&hs_full[h], 1);
      mbar_init(&hs_empty[h], 128);
    }
    fence_mbar_init();
    if (AMODE != A_GATHER) tma_prefetch(&tmA);
    tma_prefetch(&tmBh);
    if (THREE_X) tma_prefetch(&tmBl);
  }
  if ((AMODE == A_ROWSEG && args.a_row_bytes < 128) || AMODE == A_STEM) {
    // TMA writes only the first a_row_bytes of each 128-byte row; the tail must read as 0.0 for the
    // (zero-weight) padding k's, so clear every A stage once before any TMA traffic.
    for (int i = threadIdx.x; i < S * (A_TILE / 16); i += NTHREADS)
      sts128(smem_u32(a_hi(i / (A_TILE / 16))) + (uint32_t)(i % (A_TILE / 16)) * 16u, make_float4(0.f, 0.f, 0.f, 0.f));
    fence_proxy_async_smem();
  }
  if (warp == 5) tmem_alloc_2sm<C_::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  cluster_arrive();
  // between this CTA's arrival and the cluster barrier's completion (no thread waits on the producer)
  if (early && warp == 4 && lane == 0) {
    const int t0 = tile_at(args, cid, ncl, 0);
    if (t0 >= 0) {
      pdl_wait();
      const Tile tl = decode(args, t0);
      int64_t m_cta;
      int wb, hb, nimg, nrow;
      coords(tl, m_cta, wb, hb, nimg, nrow);
      trace_at(args, 2);
      for (int kb = tl.kb0; kb < tl.kb1 && pre < (uint32_t)S; ++kb, ++pre)
        relay_load((int)pre, kb, tl, m_cta, wb, hb, nimg, nrow);
    }
  }
  __syncwarp();
  cluster_wait();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // first global-memory access below: the previous kernel has completed
  if (threadIdx.x == 0) trace_at(args, 1);

  if (warp == 4) {
    // ============================ TMA producer ============================
    if (lane == 0) {
      uint32_t it = 0;
      // BRES: this CTA's B half of the pair's N tile (tile ni: rows [ni*BN + rank*BN/2, +BN/2)), once
      const int res_row = (args.bstat ? (cid % args.nt) * BN : 0) + (int)rank * (BN / 2);
      if (BRES && bmn && THREE_X) {  // own B half into own smem; the transform warps split it, then signal
        mbar_arrive_expect_tx(b_res, (uint32_t)(args.nkb * C_::BHALF));
        for (int kb = 0; kb < args.nkb; ++kb)
          tma_load_3d(&tmBh, b_res, smem_u32(res_hi(kb)), 0, kb * BK, res_row / 32);
      } else if (BRES) {  // to the leader's barrier
        const uint32_t rb = mapa(smem_u32(b_res), 0);
        if (rank == 0) mbar_arrive_expect_tx(b_res, 2u * (uint32_t)(args.nkb * b_copies * C_::BHALF));
        for (int kb = 0; kb < args.nkb; ++kb) {
          if (bmn) {
            tma_load_3d_2sm(&tmBh, rb, smem_u32(res_hi(kb)), 0, kb * BK, res_row / 32);
          } else {
            tma_load_3d_2sm(&tmBh, rb, smem_u32(res_hi(kb)), kb * BK, res_row, 0);
            if (THREE_X) tma_load_3d_2sm(&tmBl, rb, smem_u32(res_lo(kb)), kb * BK, res_row, 0);
          }
        }
      }
      if (AMODE == A_STEM) {
        uint32_t u = 0;
        for (int t, jj = 0; (t = tile_at(args, cid, ncl, jj)) >= 0; ++jj, ++u) {
          const Tile tl = decode(args, t);
          const int wo0 = (tl.mi % args.wblk) * 16;
          const int ho0 = ((tl.mi / args.wblk) % args.hblk) * 16 + (int)rank * 8;
          const int h = u & 1;
          if (u >= 2) mbar_wait(&hs_empty[h], ((u >> 1) - 1) & 1);
          mbar_arrive_expect_tx(&hs_full[h], (uint32_t)args.halo_bytes);
          tma_load_3d(&tmA, &hs_full[h], smem_u32(halo + h * 16384), wo0 * args.SW * args.Cg, ho0 * args.SH,
                      tl.mi / (args.wblk * args.hblk));
        }
      }
      for (int t, jj = 0; AMODE != A_STEM && (t = tile_at(args, cid, ncl, jj)) >= 0; ++jj) {
        const Tile tl = decode(args, t);
        int64_t m_cta;
        int wb, hb, nimg, nrow;
        coords(tl, m_cta, wb, hb, nimg, nrow);
        for (int kb = tl.kb0; kb < tl.kb1; ++kb, ++it) {
          if (it < pre) continue;  // issued before the cluster barrier
          const int s = it % S;
          const uint32_t u = it / S;
          if (u > 0) mbar_wait(&empty[s], (u - 1) & 1);
          if (it == 0) trace_at(args, 2);
          const int tap = AMODE == A_IM2COL ? kb / args.ncb : 0;
          const int cb = AMODE == A_IM2COL ? kb - tap * args.ncb : 0;
          if (RELAY) {
            relay_load(s, kb, tl, m_cta, wb, hb, nimg, nrow);
          } else {
            // both CTAs' bytes land on the leader's full[s]; only the leader arms it
            if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * bytes);
            const uint32_t fb = full_leader + (uint32_t)(s * sizeof(uint64_t));
            if (AMODE == A_IM2COL)
              tma_load_im2col_4d_2sm(&tmA, fb, smem_u32(a_hi(s)), cb * BK, wb, hb, nimg, (uint16_t)(tap % args.KW),
                                     (uint16_t)(tap / args.KW));
            else if (AMODE == A_NARROW)
              narrow_loads_2sm(fb, smem_u32(a_hi(s)), kb, wb, hb, nimg);
            else if (AMODE == A_ROWSEG)
              tma_load_5d_2sm(&tmA, fb, smem_u32(a_hi(s)), 0, wb, hb, nimg, kb);
            else
              tma_load_3d_2sm(&tmA, fb, smem_u32(a_hi(s)), kb * BK, (int)m_cta, tl.bz);
            if (!BRES && bmn) tma_load_3d_2sm(&tmBh, fb, smem_u32(b_hi(s)), 0, kb * BK, nrow / 32);
            else if (!BRES) tma_load_3d_2sm(&tmBh, fb, smem_u32(b_hi(s)), kb * BK, nrow, tl.bz);
          }
        }
      }
      // drain: every stage must be released before the CTA may exit (multicast commits target us);
      // in A_STEM mode the transform warps own the stages and drain them
      for (int i = 0; i < S && AMODE != A_STEM; ++i, ++it) {
        const uint32_t u = it / S;
        if (u > 0) mbar_wait(&empty[it % S], (u - 1) & 1);
      }
    }
  } else if (warp == 5) {
    // ============================ MMA issuer (leader CTA) ============================
    if (rank == 0) {  // whole warp, converged: operands stay warp-uniform
      const bool bmn = args.b_mn != 0;
      const uint32_t idesc = idesc_tf32(2 * BMC, BN) | (bmn ? IDESC_B_MN : 0u);
      // B descriptors: K-major SW128 (filter_prep's Bt) or MN-major SW128_BASE32B (b_mn: 32 k-rows x 128 B
      // per 32-wide n chunk -> LBO 4 KB; 4-row atoms -> SBO 512 B; K=8 step = 1 KB)
      auto bdesc = [&](const uint8_t* ptr) {
        return bmn ? umma_desc_sw128b32_mn(smem_u32(ptr), BK * 128, 512) : umma_desc_sw128_kmajor(smem_u32(ptr));
      };
      uint32_t it = 0, ai = 0;
      if (BRES) {
        mbar_wait((THREE_X && bmn) ? b_ready : b_res, 0);
        tc_fence_after();
      }
      for (int t, jj = 0; (t = tile_at(args, cid, ncl, jj)) >= 0; ++jj, ++ai) {
        const Tile tl = decode(args, t);
        const int acc = ai & 1;
        const uint32_t ua = ai >> 1;
        if (ua > 0) mbar_wait(&tmem_empty[acc], (ua - 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem_base + (uint32_t)(acc * BN);
        for (int kb = tl.kb0; kb < tl.kb1; ++kb, ++it) {
          const int s = it % S;
          mbar_wait(&full[s], (it / S) & 1);
          tc_fence_after();
          if (it == 0 && lane == 0) trace_at(args, 3);
          const uint64_t dah = AMODE == A_NARROW ? umma_desc_interleave_kmajor(smem_u32(a_hi(s)), 2048, 128)
                                                 : umma_desc_sw128_kmajor(smem_u32(a_hi(s)));
          const uint64_t dbh = bdesc(BRES ? res_hi(kb) : b_hi(s));
          const int l = (THREE_X && !C_::LO_TMEM) ? (int)(it % SL) : 0;
          const uint32_t lo_t = tmem_base + C_::LO_COL0 + (uint32_t)(s * BK);  // LO_TMEM: stage s's lo columns
          const uint64_t dal = (!THREE_X || C_::LO_TMEM) ? 0
                               : AMODE == A_NARROW ? umma_desc_interleave_kmajor(smem_u32(a_lo(l)), 2048, 128)
                                                   : umma_desc_sw128_kmajor(smem_u32(a_lo(l)));
          const uint64_t dbl = THREE_X ? bdesc(BRES ? res_lo(kb) : b_lo(s)) : 0;
          // the k-block's four K=8 steps from one asm block (sm100.cuh mma2_kblock_*): descriptors advance 32 B
          // per step (MN-major B: 1 KB; narrow A: two 16-byte core-matrix columns = 2 boxes = 4 KB)
          static_assert(BK == 32, "mma2_kblock_* issue four K=8 steps");
          const uint64_t a_step = AMODE == A_NARROW ? (uint64_t)(4096 >> 4) : (uint64_t)(32 >> 4);
          const uint64_t b_step = bmn ? (uint64_t)(1024 >> 4) : (uint64_t)(32 >> 4);
          const uint32_t acc0 = kb > tl.kb0 ? 1u : 0u;
          if (THREE_X && C_::LO_TMEM)
            mma2_kblock_3x_ts(d, lo_t, dah, dbh, dbl, a_step, b_step, idesc, acc0);
          else if (THREE_X)
            mma2_kblock_3x_ss(d, dah, dal, dbh, dbl, a_step, b_step, idesc, acc0);
          else
            mma2_kblock_1x_ss(d, dah, dbh, a_step, b_step, idesc, acc0);
          mma_commit_2sm_mc_warp(&empty[s], 0x3);
          if (THREE_X && !C_::LO_TMEM) mma_commit_2sm_mc_warp(&lo_empty[l], 0x3);
        }
        mma_commit_2sm_mc_warp(&tmem_full[acc], 0x3);
      }
    }
    __syncwarp();
  } else if (warp < 4) {
    // ============================ transform / gather (128 threads) ============================
    const int t = threadIdx.x;
    const int j = t & 7;    // 16-byte chunk within the 128-byte k-row
    const int rb = t >> 3;  // rows rb + 16 i
    const uint32_t full_leader = mapa(smem_u32(full), 0);  // full[0] in the leader CTA
    const bool bmn_lo = THREE_X && args.b_mn != 0;

    // lo = x - trunc_tf32(x) over `bytes` of B hi at `hi`, written at the same offsets from `lo_dst`
    // (elementwise: the swizzled MN-major layout carries over)
    auto split_b = [&](const uint8_t* hi, uint8_t* lo_dst, int nbytes) {
      const uint32_t h = smem_u32(hi), l = smem_u32(lo_dst);
      for (int i = t * 16; i < nbytes; i += 128 * 16) {
        const float4 v = lds128(h + (uint32_t)i);
        sts128(l + (uint32_t)i, make_float4(v.x - tf32_hi(v.x), v.y - tf32_hi(v.y), v.z - tf32_hi(v.z),
                                            v.w - tf32_hi(v.w)));
      }
    };
    if (BRES && bmn_lo) {  // resident B: split every k-block once, then tell the leader's MMA warp
      mbar_wait(b_res, 0);
      split_b(res_hi(0), res_lo(0), args.nkb * C_::BHALF);
      fence_proxy_async_smem();
      mbar_arrive_remote(mapa(smem_u32(b_ready), 0));
    }

    auto finalize = [&](uint32_t jt) {
      const int s = jt % S;
      if (AMODE != A_STEM) mbar_wait(&ld_full[s], (jt / S) & 1);
      if (THREE_X && C_::LO_TMEM) {
        // thread t owns A row t: read its 32 k's, write lo = x - trunc_tf32(x) to TMEM lane t, stage s's
        // 32 lo columns (the lo*hi MMA reads A from there).  hi stays in smem as raw fp32.
        const uint32_t ah = smem_u32(a_hi(s));
        float lo[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint32_t off = AMODE == A_NARROW ? (uint32_t)(c * 2048 + t * 16) : sw128_offset(t, c);
          const float4 v = lds128(ah + off);
          lo[4 * c] = v.x - tf32_hi(v.x);
          lo[4 * c + 1] = v.y - tf32_hi(v.y);
          lo[4 * c + 2] = v.z - tf32_hi(v.z);
          lo[4 * c + 3] = v.w - tf32_hi(v.w);
        }
        tmem_st32(tmem_base + ((uint32_t)(warp * 32) << 16) + C_::LO_COL0 + (uint32_t)(s * BK), lo);
        tmem_st_wait();
        tc_fence_before();
      } else if (THREE_X) {
        const int l = jt % SL;
        const uint32_t ul = jt / SL;
        if (ul > 0) mbar_wait(&lo_empty[l], (ul - 1) & 1);  // the MMA has finished reading this lo slot
        const uint32_t ah = smem_u32(a_hi(s));
        const uint32_t al = smem_u32(a_lo(l));
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint32_t off = AMODE == A_NARROW ? (uint32_t)(t * 16 + i * 2048) : sw128_offset(rb + 16 * i, j);
          // hi stays in place as raw fp32: kind::tf32 MMAs read only the top 19 bits (truncation,
          // pinned by tests/test_gpu_parity.py::test_tf32_mma_reads_truncated_operands)
          const float4 v = lds128(ah + off);
          sts128(al + off, make_float4(v.x - tf32_hi(v.x), v.y - tf32_hi(v.y), v.z - tf32_hi(v.z),
                                       v.w - tf32_hi(v.w)));
        }
      }
      fence_proxy_async_smem();
      mbar_arrive_remote(full_leader + (uint32_t)(s * sizeof(uint64_t)));
    };

    uint32_t it = 0;
    for (int tt, jj = 0; (tt = tile_at(args, cid, ncl, jj)) >= 0; ++jj) {
      const Tile tl = decode(args, tt);
      if (AMODE == A_GATHER) {
        int ihb[8], iwb[8];
        int64_t rbase[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int64_t m = (int64_t)tl.mi * 2 * BMC + rank * BMC + rb + 16 * i;
          if (m < args.M) {
            const int wo = (int)(m % args.WO);
            const int64_t q = m / args.WO;
            const int ho = (int)(q % args.HO);
            const int64_t n = q / args.HO;
            ihb[i] = ho * args.SH - args.PT;
            iwb[i] = wo * args.SW - args.PL;
            rbase[i] = n * args.H * args.W * args.Cg;
          } else {
            ihb[i] = -(1 << 28);
            iwb[i] = 0;
            rbase[i] = 0;
          }
        }
        for (int kb = tl.kb0; kb < tl.kb1; ++kb, ++it) {
          const int s = it % S;
          const uint32_t u = it / S;
          if (u > 0) mbar_wait(&empty[s], (u - 1) & 1);
          const uint32_t sa = smem_u32(a_hi(s));
          const int k0 = kb * BK + j * 4;
          const int c = k0 % args.Cg;
          const int rs = k0 / args.Cg;
          const int sx = rs % args.KW;
          const int r = rs / args.KW;
          const bool kv = k0 < args.Kg;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int ih = ihb[i] + r, iw = iwb[i] + sx;
            const bool v = kv && ih >= 0 && ih < args.H && iw >= 0 && iw < args.W;
            const float* src = v ? args.xg + rbase[i] + ((int64_t)ih * args.W + iw) * args.Cg + c : args.xg;
            cp_async16(sa + sw128_offset(rb + 16 * i, j), src, v ? 16u : 0u);
          }
          cp_async_commit();
          if (it >= (uint32_t)LAG) {
            cp_async_wait<LAG>();
            // finalize reads whole A rows (LO_TMEM: thread t <- row t), gathered by other threads' cp.asyncs:
            // every transform thread's groups for that stage must have landed (named barrier, warps 0-3)
            named_bar_sync(1, 128);
            finalize(it - LAG);
          }
        }
      } else if (AMODE == A_STEM) {
        // thread t builds A row t = (ho_l, wo_l) = (t / 16, t % 16) of this CTA's 16x8 tile: for kernel
        // row r, the KW*C4 contiguous halo floats at halo row ho_l*SH + r, column wo_l*SW*C4; the
        // remaining chunks of the 128-B row stay zero (cleared at kernel start).
        const uint32_t uh = (uint32_t)jj;
        const int h = uh & 1;
        mbar_wait(&hs_full[h], (uh >> 1) & 1);
        const uint32_t hbase = smem_u32(halo + h * 16384) +
                               (uint32_t)(((t / 16) * args.SH * args.halo_row_floats + (t % 16) * args.SW * args.Cg) * 4);
        const int nchunk = args.a_row_bytes / 16;
        for (int kb = tl.kb0; kb < tl.kb1; ++kb, ++it) {
          const int s = it % S;
          const uint32_t u = it / S;
          if (u > 0) mbar_wait(&empty[s], (u - 1) & 1);
          const uint32_t src = hbase + (uint32_t)(kb * args.halo_row_floats * 4);
          const uint32_t sa = smem_u32(a_hi(s));
          float lo[32];
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (c < nchunk) {
              v = lds128(src + c * 16);
              sts128(sa + sw128_offset(t, c), v);
            }
            lo[4 * c] = v.x - tf32_hi(v.x);
            lo[4 * c + 1] = v.y - tf32_hi(v.y);
            lo[4 * c + 2] = v.z - tf32_hi(v.z);
            lo[4 * c + 3] = v.w - tf32_hi(v.w);
          }
          if (THREE_X && C_::LO_TMEM) {  // lo straight from registers (no read-back)
            tmem_st32(tmem_base + ((uint32_t)(warp * 32) << 16) + C_::LO_COL0 + (uint32_t)(s * BK), lo);
            tmem_st_wait();
            tc_fence_before();
          }
          fence_proxy_async_smem();
          mbar_arrive_remote(full_leader + (uint32_t)(s * sizeof(uint64_t)));
        }
        mbar_arrive(&hs_empty[h]);
      } else if (RELAY) {
        for (int kb = tl.kb0; kb < tl.kb1; ++kb, ++it) finalize(it);
      }
    }
    if (AMODE == A_STEM) {  // drain the stage ring (multicast commits from the MMA target this CTA)
      for (int i = 0; i < S; ++i, ++it) {
        const uint32_t u = it / S;
        if (u > 0) mbar_wait(&empty[it % S], (u - 1) & 1);
      }
    }
    if (AMODE == A_GATHER) {
      cp_async_wait<0>();
      named_bar_sync(1, 128);  // all transform threads' gathers landed (see above)
      for (uint32_t jt = (it > (uint32_t)LAG ? it - LAG : 0); jt < it; ++jt) finalize(jt);
    }
    if (THREE_X && !C_::LO_TMEM) {  // drain: every lo slot released before exit (multicast commits target us)
      for (int i = 0; i < SL; ++i, ++it) {
        const uint32_t ul = it / SL;
        if (ul > 0) mbar_wait(&lo_empty[it % SL], (ul - 1) & 1);
      }
    }
  } else if (warp >= 10) {
    // ============================ B-lo split (warps 10-13) ============================
    if (THREE_X && !BRES && args.b_mn) {
      const int t2 = threadIdx.x - 320;
      const uint32_t full_leader = mapa(smem_u32(full), 0);
      uint32_t it = 0;
      for (int tt, jj = 0; (tt = tile_at(args, cid, ncl, jj)) >= 0; ++jj) {
        const Tile tl = decode(args, tt);
        for (int kb = tl.kb0; kb < tl.kb1; ++kb, ++it) {
          const int s = it % S;
          mbar_wait(&ld_full[s], (it / S) & 1);
          const uint32_t h = smem_u32(b_hi(s)), l = smem_u32(b_lo(s));
          // lo = b - trunc_tf32(b), elementwise: the swizzled MN-major layout carries over
#pragma unroll 4
          for (int i = t2 * 16; i < C_::BHALF; i += 128 * 16) {
            const float4 v = lds128(h + (uint32_t)i);
            sts128(l + (uint32_t)i, make_float4(v.x - tf32_hi(v.x), v.y - tf32_hi(v.y), v.z - tf32_hi(v.z),
                                                v.w - tf32_hi(v.w)));
          }
          fence_proxy_async_smem();
          mbar_arrive_remote(full_leader + (uint32_t)(s * sizeof(uint64_t)));
        }
      }
    }
  } else {
    // ============================ epilogue (warps 6-9) ============================
    // Each warp owns TMEM lanes [32q, 32q+32) = 32 output rows.  Per 32-column chunk:
    // tcgen05.ld (thread i <- row i, 32 columns) -> either a SWIZZLE_128B smem chunk stored by
    // TMA (coalesced, asynchronous; double-buffered per warp) or direct 16-byte stores.
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const uint32_t tmem_empty_leader = mapa(smem_u32(tmem_empty), 0);
    const bool vec_ok = (args.ldd % 4) == 0;
    const uint32_t ebuf = smem_u32(epi_smem) + (uint32_t)(q * 2 * 4096);
    if (args.tma_store == 1 && lane == 0) tma_prefetch(&tmD);
    if (args.rs_splits > 1 && lane == 0) tma_prefetch(&args.tmP);
    uint32_t ai = 0, chunk = 0;
    for (int t, jj = 0; (t = tile_at(args, cid, ncl, jj)) >= 0; ++jj, ++ai) {
      const Tile tl = decode(args, t);
      const int acc = ai & 1;
      mbar_wait(&tmem_full[acc], (ai >> 1) & 1);
      tc_fence_after();
      if (ai == 0 && q == 2 && lane == 0) trace_at(args, 4);
      int64_t row0 = (int64_t)tl.mi * 2 * BMC + rank * BMC + q * 32;
      int64_t m = row0 + lane;
      int sw0 = 0, sh0 = 0, sn = 0;  // A_ROWSEG / A_STEM: this warp's 16 x 2 spatial block
      if (SPATIAL) {
        sw0 = (tl.mi % args.wblk) * 16;
        sh0 = ((tl.mi / args.wblk) % args.hblk) * 16 + (int)rank * 8 + 2 * q;
        sn = tl.mi / (args.wblk * args.hblk);
        const int ho = sh0 + lane / 16, wo = sw0 + lane % 16;
        m = (ho < args.HO && wo < args.WO) ? ((int64_t)sn * args.HO + ho) * args.WO + wo : args.M;
        row0 = (sh0 < args.HO && sw0 < args.WO) ? 0 : args.M;  // warp-uniform "any row valid"
      }
      const int z = args.splits == 1 ? tl.bz : tl.split * args.batch + tl.bz;
      float* D = args.splits == 1 ? args.d + (int64_t)tl.bz * args.d_bstride
                                  : args.partial + ((int64_t)tl.split * args.batch + tl.bz) * args.M * args.ldd;
      const int n0 = tl.ni * BN;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        float v[32];
        tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c0), v);
        if (c0 + 32 >= BN) {  // last TMEM read of this accumulator: hand it back to the MMA warp
          tc_fence_before();
          mbar_arrive_remote(tmem_empty_leader + (uint32_t)(acc * sizeof(uint64_t)));
        }
        if (args.tma_store == 2) {
          // smem-staged coalesced stores through the LSU (keeps the TMA engine free for loads):
          // STS the 32x32 chunk swizzled, then each lane stores 16 B of row (i/8), column group (i%8)
          if (row0 < args.M && n0 + c0 < args.N) {
            const uint32_t buf = ebuf;
            __syncwarp();
#pragma unroll
            for (int k = 0; k < 8; ++k)
              sts128(buf + sw128_offset(lane, k), make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]));
            __syncwarp();
            const int cq = lane & 7;
            const int64_t col = n0 + c0 + cq * 4;
#pragma unroll
            for (int r4 = 0; r4 < 32; r4 += 4) {
              const int rr = r4 + (lane >> 3);
              const float4 val = lds128(buf + sw128_offset(rr, cq));
              int64_t mrow;
              if (SPATIAL) {
                const int ho = sh0 + rr / 16, wo = sw0 + rr % 16;
                mrow = (ho < args.HO && wo < args.WO) ? ((int64_t)sn * args.HO + ho) * args.WO + wo : args.M;
              } else {
                mrow = row0 + rr;
              }
              if (mrow < args.M && col + 3 < args.N)
                *reinterpret_cast<float4*>(D + mrow * args.ldd + col) = val;
              else if (mrow < args.M)
                for (int e = 0; e < 4; ++e)
                  if (col + e < args.N) D[mrow * args.ldd + col + e] = (&val.x)[e];
            }
          }
        } else if (args.tma_store) {
          if (row0 < args.M && n0 + c0 < args.N) {
            const uint32_t buf = ebuf + (chunk & 1) * 4096;
            if (lane == 0) bulk_wait_read<1>();  // the store issued two chunks ago has read `buf`
            __syncwarp();
#pragma unroll
            for (int k = 0; k < 8; ++k)
              sts128(buf + sw128_offset(lane, k), make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]));
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              if (SPATIAL) tma_store_4d(&tmD, buf, n0 + c0, sw0, sh0, sn);
              else if (tl.part) tma_store_3d(&args.tmP, buf, n0 + c0, (int)row0, tl.split);
              else tma_store_3d(&tmD, buf, n0 + c0, (int)row0, z);
              bulk_commit();
            }
            ++chunk;
          }
        } else if (m < args.M) {
          float* dst = D + m * args.ldd + n0 + c0;
          const int64_t nrem = args.N - (n0 + c0);
          if (vec_ok && nrem >= 32) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
              reinterpret_cast<float4*>(dst)[k] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
          } else {
#pragma unroll
            for (int k = 0; k < 32; ++k)
              if (k < nrem) dst[k] = v[k];
          }
        }
      }
    }
    if (q == 2 && lane == 0) trace_at(args, 5);
    if (args.tma_store == 1 && lane == 0) bulk_wait<0>();
    if (q == 2 && lane == 0) trace_at(args, 6);
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc_2sm<C_::TMEM_COLS>(tmem_base);
  }
  if (threadIdx.x == 0) trace_at(args, 7);
}

// ------------------------------------------------------------------ host: debug trace
constexpr int TRACE_LAUNCHES = 256;           // ring of launch records
constexpr int TRACE_RECORD = 148 * TRACE_SLOTS;  // one record: 148 CTAs x TRACE_SLOTS stamps
unsigned long long* g_trace_buf = nullptr;       // TRACE_LAUNCHES records, device
bool g_trace_on = false;
int g_trace_next = 0;

// ------------------------------------------------------------------ host: tensor maps
PFN_cuTensorMapEncodeTiled_v12000 g_encode_tiled = nullptr;
PFN_cuTensorMapEncodeIm2col_v12000 g_encode_im2col = nullptr;
int g_driver_version = 0;
std::once_flag g_once;

cudaError_t load_driver_fns() {
  cudaError_t err = cudaSuccess;
  std::call_once(g_once, [&]() {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode_tiled = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode_im2col = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(p);
    cudaDriverGetVersion(&g_driver_version);
  });
  if (!g_encode_tiled || !g_encode_im2col) err = cudaErrorSymbolNotFound;
  return err;
}

// 3-D tiled map over a K-major matrix stack [d2][d1][d0], box {32, box1, 1}, SWIZZLE_128B
bool make_tiled_3d(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t row_stride_elems,
                   uint32_t box1) {
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {row_stride_elems * 4, row_stride_elems * 4 * d1};
  cuuint32_t box[3] = {32, box1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return g_encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_im2col(CUtensorMap* m, const Problem& p, const float* x) {
  cuuint64_t dims[4] = {(cuuint64_t)p.C, (cuuint64_t)p.W, (cuuint64_t)p.H, (cuuint64_t)p.N};
  cuuint64_t strides[3] = {(cuuint64_t)p.C * 4, (cuuint64_t)p.W * p.C * 4, (cuuint64_t)p.H * p.W * p.C * 4};
  const int pb = (p.HO - 1) * p.SH + p.KH - p.H - p.pad_top;
  const int pr = (p.WO - 1) * p.SW + p.KW - p.W - p.pad_left;
  int lower[2] = {-p.pad_left, -p.pad_top};
  int upper[2] = {pr - (p.KW - 1), pb - (p.KH - 1)};
  cuuint32_t es[4] = {1, (cuuint32_t)p.SW, (cuuint32_t)p.SH, 1};
  if (g_encode_im2col(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(x), dims, strides, lower, upper, 32,
                      BMC, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  // Same driver workaround CUTLASS applies to im2col descriptors of tensors < 128 KiB on drivers <= 13.1.
  if (g_driver_version <= 13010 && (uint64_t)p.in_elems() * 4 < 131072)
    reinterpret_cast<uint64_t*>(m)[1] &= ~(1ull << 21);
  return true;
}

bool make_im2col_narrow(CUtensorMap* m, const Problem& p, const float* x, int cg) {
  cuuint64_t dims[4] = {(cuuint64_t)cg, (cuuint64_t)p.W, (cuuint64_t)p.H, (cuuint64_t)p.N};
  cuuint64_t strides[3] = {(cuuint64_t)cg * 4, (cuuint64_t)p.W * cg * 4, (cuuint64_t)p.H * p.W * cg * 4};
  const int pb = (p.HO - 1) * p.SH + p.KH - p.H - p.pad_top;
  const int pr = (p.WO - 1) * p.SW + p.KW - p.W - p.pad_left;
  int lower[2] = {-p.pad_left, -p.pad_top};
  int upper[2] = {pr - (p.KW - 1), pb - (p.KH - 1)};
  cuuint32_t es[4] = {1, (cuuint32_t)p.SW, (cuuint32_t)p.SH, 1};
  if (g_encode_im2col(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(x), dims, strides, lower, upper, 4,
                      BMC, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  if (g_driver_version <= 13010 && (uint64_t)p.N * p.H * p.W * cg * 4 < 131072)
    reinterpret_cast<uint64_t*>(m)[1] &= ~(1ull << 21);
  return true;
}

// A_ROWSEG: 5-D view {e, wo, ho, n, r} of the padded input xp (N, Hp, Wp, cg) with OVERLAPPING strides:
// element (e, wo, ho, n, r) = xp[n][ho*SH + r][wo*SW + e / cg][e % cg]; e < KW*cg, box {32, 16, 8, 1, 1}.
bool make_rowseg(CUtensorMap* m, const Problem& p, const float* xp, int cg, int hp, int wp) {
  cuuint64_t dims[5] = {(cuuint64_t)p.KW * cg, (cuuint64_t)p.WO, (cuuint64_t)p.HO, (cuuint64_t)p.N,
                        (cuuint64_t)p.KH};
  cuuint64_t strides[4] = {(cuuint64_t)p.SW * cg * 4, (cuuint64_t)p.SH * wp * cg * 4, (cuuint64_t)hp * wp * cg * 4,
                           (cuuint64_t)wp * cg * 4};
  cuuint32_t box[5] = {(cuuint32_t)(p.KW * cg), 16, 8, 1, 1};  // exactly the segment: no OOB elements
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  return g_encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(xp), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, bool THREE_X, int AMODE, bool BRES>
cudaError_t launch_t(const CUtensorMap& a, const CUtensorMap& bh, const CUtensorMap& bl, const CUtensorMap& dm,
                     const DevArgs& args, int clusters, cudaStream_t s) {
  using C_ = Cfg<BN, THREE_X, BRES, AMODE == A_STEM>;
  auto kern = gemm2sm_kernel<BN, THREE_X, AMODE, BRES>;
  const cudaError_t e = smem_attr_once<gemm2sm_kernel<BN, THREE_X, AMODE, BRES>>(C_::SMEM);
  if (e != cudaSuccess) return e;
  return launch_k(kern, dim3(2 * clusters), dim3(NTHREADS), C_::SMEM, s, a, bh, bl, dm, args);
}

template <bool THREE_X, int AMODE>
cudaError_t launch_bn(int bn, const CUtensorMap& a, const CUtensorMap& bh, const CUtensorMap& bl,
                      const CUtensorMap& dm, const DevArgs& args, int clusters, cudaStream_t s) {
  // BRES: no split-K / batching, every k-block of this CTA's B half fits the region, and one N tile --
  // or several with the B-stationary schedule (args.bstat, set by the caller when every N tile gets a
  // pair: tiles >= 74 pairs)
  const bool bres = AMODE == A_STEM ||
                    ((args.nt == 1 || args.bstat) && args.splits == 1 && args.batch == 1 &&
                     getenv("CONV2D_NO_BRES") == nullptr &&
                     (AMODE == A_ROWSEG || AMODE == A_DENSE || AMODE == A_IM2COL));
  if (AMODE == A_STEM) {  // always B-resident; only instantiated where it fits (host checks gemm2_stem_ok)
    if (bn == 64) return launch_t<64, THREE_X, AMODE, true>(a, bh, bl, dm, args, clusters, s);
    if (bn == 128) return launch_t<128, THREE_X, AMODE, true>(a, bh, bl, dm, args, clusters, s);
    return cudaErrorInvalidValue;
  }
  switch (bn) {
    case 64:
      if (bres && args.nkb <= Cfg<64, THREE_X, true>::RES_KB_MAX)
        return launch_t<64, THREE_X, AMODE, true>(a, bh, bl, dm, args, clusters, s);
      return launch_t<64, THREE_X, AMODE, false>(a, bh, bl, dm, args, clusters, s);
    case 128:
      if (bres && args.nkb <= Cfg<128, THREE_X, true>::RES_KB_MAX)
        return launch_t<128, THREE_X, AMODE, true>(a, bh, bl, dm, args, clusters, s);
      return launch_t<128, THREE_X, AMODE, false>(a, bh, bl, dm, args, clusters, s);
    case 256:
      if (bres && args.nkb <= Cfg<256, THREE_X, true>::RES_KB_MAX)
        return launch_t<256, THREE_X, AMODE, true>(a, bh, bl, dm, args, clusters, s);
      return launch_t<256, THREE_X, AMODE, false>(a, bh, bl, dm, args, clusters, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

bool gemm2_encode_tiled(CUtensorMap* m, int rank, const void* base, const uint64_t* dims, const uint64_t* strides,
                        const uint32_t* box, bool swizzle128) {
  return gemm2_encode_tiled_sw(m, rank, base, dims, strides, box,
                               swizzle128 ? (int)CU_TENSOR_MAP_SWIZZLE_128B : (int)CU_TENSOR_MAP_SWIZZLE_NONE);
}

bool gemm2_encode_tiled_sw(CUtensorMap* m, int rank, const void* base, const uint64_t* dims, const uint64_t* strides,
                           const uint32_t* box, int swizzle) {
  return gemm2_encode_tiled_es(m, rank, base, dims, strides, box, nullptr, swizzle);
}

bool gemm2_encode_tiled_es(CUtensorMap* m, int rank, const void* base, const uint64_t* dims, const uint64_t* strides,
                           const uint32_t* box, const uint32_t* elem_strides, int swizzle) {
  if (load_driver_fns() != cudaSuccess) return false;
  cuuint64_t d[5], st[4];
  cuuint32_t b[5], es[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    es[i] = elem_strides ? elem_strides[i] : 1;
    if (i < rank - 1) st[i] = strides[i];
  }
  return g_encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<void*>(base), d, st, b, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, (CUtensorMapSwizzle)swizzle,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

unsigned long long* gemm2_trace_record() {
  if (!g_trace_on || !g_trace_buf) return nullptr;
  return g_trace_buf + (size_t)(g_trace_next++ % TRACE_LAUNCHES) * TRACE_RECORD;
}

int gemm2_trace(int enable, unsigned long long* host, int n) {
  const size_t total = (size_t)TRACE_LAUNCHES * TRACE_RECORD;
  if (enable >= 0) {
    if (enable && !g_trace_buf && cudaMalloc(&g_trace_buf, total * sizeof(unsigned long long)) != cudaSuccess)
      return -1;
    if (enable && g_trace_buf) cudaMemset(g_trace_buf, 0, total * sizeof(unsigned long long));
    if (enable) g_trace_next = 0;
    g_trace_on = enable != 0;
  }
  if (host && g_trace_buf) {
    const int m = (size_t)n < total ? n : (int)total;
    if (cudaMemcpy(host, g_trace_buf, (size_t)m * sizeof(unsigned long long), cudaMemcpyDeviceToHost) != cudaSuccess)
      return -1;
    return m;
  }
  return 0;
}

int gemm2_choose_block_n(int64_t N) {
  if (N <= 64) return 64;
  if (N <= 128) return 128;
  return 256;
}

int gemm2_choose_splits(int64_t M, int64_t N, int nkb, int batch, int block_n) {
  const int64_t tiles = ((M + 255) / 256) * ((N + block_n - 1) / block_n) * batch;
  if (tiles >= 74 || nkb < 8) return 1;
  int64_t s = 74 / tiles;             // fill one wave of CTA pairs
  if (s > nkb / 4) s = nkb / 4;       // keep >= 4 k-blocks per split
  if (s > 16) s = 16;
  return s < 1 ? 1 : (int)s;
}

static bool corners_ok(const Problem& p) {
  const int pb = (p.HO - 1) * p.SH + p.KH - p.H - p.pad_top;
  const int pr = (p.WO - 1) * p.SW + p.KW - p.W - p.pad_left;
  const int lo[2] = {-p.pad_left, -p.pad_top}, up[2] = {pr - (p.KW - 1), pb - (p.KH - 1)};
  for (int i = 0; i < 2; ++i)
    if (lo[i] < -128 || lo[i] > 127 || up[i] < -128 || up[i] > 127) return false;
  return p.SH <= 8 && p.SW <= 8 && p.W < 60000 && p.H < 60000;
}

bool gemm2_narrow_ok(const Problem& p) { return corners_ok(p); }

bool gemm2_stem_ok(const Problem& p, int block_n, bool three_x) {
  const int cg = (p.C + 3) / 4 * 4;
  const int row_floats = (15 * p.SW + p.KW) * cg;
  const int halo = (7 * p.SH + p.KH) * row_floats * 4;
  const int res_kb = three_x ? Cfg<64, true, true, true>::RES_KB_MAX * 64 / block_n
                             : Cfg<64, false, true, true>::RES_KB_MAX * 64 / block_n;
  return gemm2_rowseg_ok(p) && p.F <= block_n && block_n <= 128 && row_floats <= 256 && halo <= 16384 &&
         p.KH <= res_kb && p.SH <= 8;
}

bool gemm2_rowseg_ok(const Problem& p) {
  const int cg = (p.C + 3) / 4 * 4;
  return p.KW * cg <= 32 && p.C < 32 && p.KH <= 64;
}

bool gemm2_im2col_ok(const Problem& p) {
  const int pb = (p.HO - 1) * p.SH + p.KH - p.H - p.pad_top;
  const int pr = (p.WO - 1) * p.SW + p.KW - p.W - p.pad_left;
  const int lo[2] = {-p.pad_left, -p.pad_top}, up[2] = {pr - (p.KW - 1), pb - (p.KH - 1)};
  for (int i = 0; i < 2; ++i)
    if (lo[i] < -128 || lo[i] > 127 || up[i] < -128 || up[i] > 127) return false;
  return p.C % 32 == 0 && p.SH <= 8 && p.SW <= 8 && p.KH <= 65535 && p.KW <= 65535;
}

cudaError_t launch_gemm2(const Problem& p, const Gemm2Args& g, cudaStream_t s) {
  cudaError_t e = load_driver_fns();
  if (e != cudaSuccess) return e;
  DevArgs a{};
  a.H = p.H; a.W = p.W; a.C = p.C; a.KH = p.KH; a.KW = p.KW; a.SH = p.SH; a.SW = p.SW;
  a.HO = p.HO; a.WO = p.WO; a.PT = p.pad_top; a.PL = p.pad_left;
  a.ncb = (p.C + 31) / 32;
  a.Cg = g.gather_c;
  a.xg = g.gather_x;
  a.Kg = (int64_t)p.KH * p.KW * g.gather_c;
  a.M = g.M; a.N = g.N;
  a.nkb = (int)(g.kpad / 32);
  a.mt = (int)((g.M + 255) / 256);
  if (g.a_mode == A_ROWSEG || g.a_mode == A_STEM) {
    a.a_row_bytes = p.KW * g.gather_c * 4;
    a.halo_row_floats = (15 * p.SW + p.KW) * g.gather_c;
    a.halo_bytes = (7 * p.SH + p.KH) * a.halo_row_floats * 4;
    a.wblk = (p.WO + 15) / 16;
    a.hblk = (p.HO + 15) / 16;
    a.mt = p.N * a.wblk * a.hblk;
  }
  a.nt = (int)((g.N + g.block_n - 1) / g.block_n);
  a.splits = g.splits;
  a.batch = g.batch;
  int64_t tiles = (int64_t)a.mt * a.nt * g.batch * g.splits;
  if (tiles > 0x7FFFFFFF) return cudaErrorInvalidConfiguration;
  a.total_tiles = (int)tiles;
  a.rs_first = a.rs_splits = 0;
  const int rs = g.rsplit ? gemm2_rsplit_factor(tiles, a.nkb) : 0;
  const bool rs_ok = rs >= 2 && g.splits == 1 && g.batch == 1 && g.partial && g.ldd % 4 == 0 &&
                     g.a_mode != A_ROWSEG && g.a_mode != A_STEM;
  a.d = g.d; a.ldd = g.ldd; a.d_bstride = g.d_batch_stride; a.partial = g.partial;
  a.trace = gemm2_trace_record();
  a.b_mn = g.b_mn ? 1 : 0;
  static const bool no_early = getenv("CONV2D_NO_EARLY_TMA") != nullptr;  // A/B switch (DESIGN.md env hooks)
  a.early = no_early ? 0 : 1;
  {  // B-stationary: several N tiles, each owned by >= 1 pair, B half resident (short K)
    const int kbmax = g.block_n == 64 ? (g.three_x ? Cfg<64, true, true>::RES_KB_MAX : Cfg<64, false, true>::RES_KB_MAX)
                      : g.block_n == 128 ? (g.three_x ? Cfg<128, true, true>::RES_KB_MAX : Cfg<128, false, true>::RES_KB_MAX)
                                         : (g.three_x ? Cfg<256, true, true>::RES_KB_MAX : Cfg<256, false, true>::RES_KB_MAX);
    static const bool bstat_env = getenv("CONV2D_BSTAT") != nullptr;
    a.bstat = (bstat_env || g.bstat) && a.nt > 1 && g.splits == 1 && g.batch == 1 && tiles >= 74 &&
              a.nkb <= kbmax && (g.a_mode == A_DENSE || g.a_mode == A_IM2COL) ? 1 : 0;
  }

  alignas(64) CUtensorMap ta{}, tbh{}, tbl{};
  bool ok = true;
  if (g.a_mode == A_IM2COL) ok = make_im2col(&ta, p, g.a);
  else if (g.a_mode == A_NARROW) ok = make_im2col_narrow(&ta, p, g.gather_x, g.gather_c);
  else if (g.a_mode == A_ROWSEG) ok = make_rowseg(&ta, p, g.gather_x, g.gather_c, g.hp, g.wp);
  else if (g.a_mode == A_STEM) {  // halo boxes over the padded input viewed as {Wp*C4 floats, Hp, N}
    const uint64_t dims[3] = {(uint64_t)g.wp * g.gather_c, (uint64_t)g.hp, (uint64_t)p.N};
    const uint64_t st[2] = {(uint64_t)g.wp * g.gather_c * 4, (uint64_t)g.hp * g.wp * g.gather_c * 4};
    const uint32_t box[3] = {(uint32_t)a.halo_row_floats, (uint32_t)(7 * p.SH + p.KH), 1};
    ok = gemm2_encode_tiled(&ta, 3, g.gather_x, dims, st, box, false);
  }
  else if (g.a_mode == A_DENSE) ok = make_tiled_3d(&ta, g.a, g.a_k, g.M, g.batch, g.lda, BMC);
  if (g.b_mn) {
    // B straight from the row-major (b_rows x N) filter: 3-D view {n % 32, k, n / 32}; box {32, 32, BN/64}
    if (g.N % 32 != 0 || g.batch != 1 || !g.b_w) return cudaErrorInvalidValue;
    const uint64_t dims[3] = {32, (uint64_t)g.b_rows, (uint64_t)(g.N / 32)};
    const uint64_t st[2] = {(uint64_t)g.N * 4, 128};
    const uint32_t box[3] = {32, 32, (uint32_t)(g.block_n / 64)};
    ok = ok && gemm2_encode_tiled_sw(&tbh, 3, g.b_w, dims, st, box, (int)CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    tbl = tbh;
  } else {
    ok = ok && make_tiled_3d(&tbh, g.bt_hi, g.kpad, g.npad, g.batch, g.kpad, g.block_n / 2);
    if (g.three_x) ok = ok && make_tiled_3d(&tbl, g.bt_lo, g.kpad, g.npad, g.batch, g.kpad, g.block_n / 2);
  }
  // output tensor map: dims {N, M, planes} with row stride ldd; box 32 x 32, SWIZZLE_128B
  alignas(64) CUtensorMap td{};
  a.tma_store = 0;
  if (ok && g.ldd % 4 == 0) {
    float* dbase = g.splits == 1 ? g.d : g.partial;
    const uint64_t planes = (uint64_t)g.batch * (g.splits == 1 ? 1 : g.splits);
    const bool dense_batch = g.splits > 1 || g.batch == 1 || g.d_batch_stride == g.M * g.ldd;
    if (g.a_mode == A_ROWSEG || g.a_mode == A_STEM) {
      cuuint64_t dims[4] = {(cuuint64_t)g.N, (cuuint64_t)p.WO, (cuuint64_t)p.HO, (cuuint64_t)p.N};
      cuuint64_t strides[3] = {(cuuint64_t)g.ldd * 4, (cuuint64_t)g.ldd * 4 * p.WO,
                               (cuuint64_t)g.ldd * 4 * p.WO * p.HO};
      cuuint32_t box[4] = {32, 16, 2, 1};
      cuuint32_t es[4] = {1, 1, 1, 1};
      a.tma_store = g_encode_tiled(&td, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, g.d, dims, strides, box, es,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    } else if (dense_batch) {
      cuuint64_t dims[3] = {(cuuint64_t)g.N, (cuuint64_t)g.M, planes};
      cuuint64_t strides[2] = {(cuuint64_t)g.ldd * 4, (cuuint64_t)g.ldd * 4 * g.M};
      cuuint32_t box[3] = {32, 32, 1};
      cuuint32_t es[3] = {1, 1, 1};
      a.tma_store = g_encode_tiled(&td, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, dbase, dims, strides, box, es,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
  }
  if (!ok) return cudaErrorInvalidValue;
  if (rs_ok && a.tma_store == 1 && !g.epi_stg && !a.bstat) {
    cuuint64_t dims[3] = {(cuuint64_t)g.N, (cuuint64_t)g.M, (cuuint64_t)rs};
    cuuint64_t strides[2] = {(cuuint64_t)g.ldd * 4, (cuuint64_t)g.ldd * 4 * g.M};
    cuuint32_t box[3] = {32, 32, 1};
    cuuint32_t es[3] = {1, 1, 1};
    if (g_encode_tiled(&a.tmP, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, g.partial, dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS) {
      const int64_t rem = tiles % 74;
      a.rs_first = (int)(tiles - rem);
      a.rs_splits = rs;
      tiles = a.rs_first + rem * rs;  // work units
      a.total_tiles = (int)tiles;
    }
  }
  if (g.epi_stg && a.tma_store && g.ldd % 4 == 0) a.tma_store = 2;  // tuned variant: LSU-staged stores
  if (a.tma_store != 1) td = tbh;  // unused slot
  if (g.a_mode == A_GATHER) ta = tbh;  // unused operand slot
  if (!g.three_x || g.b_mn) tbl = tbh;

  const int clusters = (int)(tiles < 74 ? tiles : 74);
  if (g.three_x) {
    switch (g.a_mode) {
      case A_IM2COL: e = launch_bn<true, A_IM2COL>(g.block_n, ta, tbh, tbl, td, a, clusters, s); break;
      case A_DENSE: e = launch_bn<true, A_DENSE>(g.block_n, ta, tbh, tbl, td, a, clusters, s); break;
      case A_NARROW: e = launch_bn<true, A_NARROW>(g.block_n, ta, tbh, tbl, td, a, clusters, s); break;
      case A_ROWSEG: e = launch_bn<true, A_ROWSEG>(g.block_n, ta, tbh, tbl, td, a, clusters, s); break;
      case A_STEM: e = launch_bn<true, A_STEM>(g.block_n, ta, tbh, tbl, td, a, clusters, s); break;
      default: e = launch_bn<true, A_GATHER>(g.block_n, ta, tbh, tbl, td, a, clusters, s); break;
    }
  } else {
    switch (g.a_mode) {
      case A_IM2COL: e = launch_bn<false, A_IM2COL>(g.block_n, ta, tbh, tbl, td, a, clusters, s); break;
      case A_DENSE: e = launch_bn<false, A_DENSE>(g.block_n, ta, tbh, tbl, td, a, clusters, s); break;
      case A_NARROW: e = launch_bn<false, A_NARROW>(g.block_n, ta, tbh, tbl, td, a, clusters, s); break;
      case A_ROWSEG: e = launch_bn<false, A_ROWSEG>(g.block_n, ta, tbh, tbl, td, a, clusters, s); break;
      case A_STEM: e = launch_bn<false, A_STEM>(g.block_n, ta, tbh, tbl, td, a, clusters, s); break;
      default: e = launch_bn<false, A_GATHER>(g.block_n, ta, tbh, tbl, td, a, clusters, s); break;
    }
  }
  if (e != cudaSuccess) return e;
  if (g.splits > 1) e = launch_split_reduce(g.partial, g.d, (int64_t)g.batch * g.M, g.N, g.ldd, g.splits, s);
  if (a.rs_splits > 1)
    e = launch_rsplit_reduce(g.partial, g.d, g.M, g.N, g.ldd, a.rs_first, a.mt * a.nt - a.rs_first, a.nt,
                             g.block_n, a.rs_splits, s);
  return e;
}

// Modelled time, in k-block units, of `tiles` pair tiles of nkb k-blocks on the 74 CTA pairs when the
// last r tiles are cut into s K ranges (r == tiles: every tile): each wave of units costs its k-blocks
// plus a pipeline fill/drain of ~2 k-blocks; any split adds the partial planes' write + reduce (~4).
static int64_t split_cost(int64_t tiles, int64_t r, int s, int nkb) {
  const int64_t waves_whole = (tiles - r) / 74;
  const int64_t waves_split = (r * s + 73) / 74;
  return waves_whole * (nkb + 2) + waves_split * ((nkb + s - 1) / s + 2) + (s > 1 ? 4 : 0);
}

int gemm2_balanced_splits(int64_t tiles, int nkb) {
  // fewer pair tiles than pairs: the K-split count (<= 16, >= 4 k-blocks each) of least modelled time
  if (tiles <= 0 || tiles >= 74) return 1;
  int best = 1;
  for (int s = 2; s <= 16 && s <= nkb / 4; ++s)
    if (split_cost(tiles, tiles, s, nkb) < split_cost(tiles, tiles, best, nkb)) best = s;
  return best;
}

int gemm2_rsplit_factor(int64_t tiles, int nkb) {
  // remainder split: the tiles fill >= 1 wave of the 74 CTA pairs; the r = tiles % 74 tiles of the
  // partial last wave are cut into s <= 8 K ranges (>= 4 k-blocks each) of least modelled time
  if (tiles < 74) return 0;
  const int64_t r = tiles % 74;
  if (r == 0) return 0;
  int best = 1;
  for (int s = 2; s <= 8 && s <= nkb / 4; ++s)
    if (split_cost(tiles, r, s, nkb) < split_cost(tiles, r, best, nkb)) best = s;
  return best >= 2 ? best : 0;
}

}  // namespace conv2d
