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
// epilogue; G3C4: 6-13), same CTA pair (cta_group::2, M = 256 = two independent 8x16 spatial tiles),
// two rings: halo slots (TMA -> transform -> MMA) and B stages (2-CTA TMA straight to the leader).
// Four geometries share the kernel (see Geo): G3X3 (C % 32 == 0), GS2D / GS2P (the space-to-depth stem,
// 64-byte SW64 pixels / packed 16-byte chunk planes) and G3C4 (3x3 with C <= 4: 16-byte pixels, two taps
// per K=8 step, B built in the kernel).
#include <cstdlib>

#include "gemm2sm.h"
#include "launch.cuh"
#include "sm100.cuh"

namespace conv2d {
namespace {

using namespace sm100;

constexpr int BK = 32;
constexpr int TW = 8, TH = 16;            // CTA output tile (wo x ho) = 128 GEMM rows
constexpr int HWD = 16;                   // halo box width (pixels) = 8-row group pitch

// Halo geometries:
//   G3X3 (0): 3x3 / stride 1, C % 32 == 0: halo box {32 ch, 16 w, 18 h} SWIZZLE_128B (128-byte pixel
//             rows), one k-block (32 channels) per tap, nine k-blocks per channel block;
//   GS2D (1): the space-to-depth stem: a 4x4 / stride-1 VALID conv over X' = s2d(x) with 16 channels
//             (64-byte pixel rows, SWIZZLE_64B): halo box {16 ch, 16 w, 19 h}, two taps per 32-wide
//             k-block, eight k-blocks.  (7x7 or 8x8 / stride 2 with C <= 4 maps onto it exactly.)
//   G3C4 (2): 3x3 / stride 1 with C <= 4 (VGG conv1_1): a halo of 4-channel pixels (16-byte rows, built by the
//             transform warps from a raw TMA patch, zero channels past C).  A K=8 step covers two horizontally
//             adjacent taps: the view of tap (r, s) is a no-swizzle K-major operand whose second 16-byte core
//             matrix column (channels of tap s+1) starts ONE pixel later (LBO = 16 B; SBO = 16 halo pixels =
//             one output row) -- overlapping views, no data replicated.  Six steps (r, s in {0, 2}; the s = 3
//             half has zero B) = two k-blocks, against 16 for a 32-channel-padded tap.
//   GS2P (3): the space-to-depth stem with the s2d pixel split into C planes of 16-byte chunks (plane q =
//             slots 4q..4q+3 of every X' pixel; the all-zero 16-byte chunks of C = 3 are not stored).  A K=8
//             step pairs ANY two (tap, plane) chunks that carry a real (tap, slot): its A view is a
//             no-swizzle K-major descriptor at the first chunk with LBO = the distance to the second, so the
//             step list packs the real chunks densely: C = 3, 7x7 -> 43 chunks = 22 steps (176 K-slots)
//             against GS2D's 28 steps (224) -- a 0.835 instead of 0.656 ceiling on the 147 real MACs.
enum { G3X3 = 0, GS2D = 1, G3C4 = 2, GS2P = 3 };
template <int GEOM>
struct Geo {
  static constexpr bool S2D = GEOM == GS2D || GEOM == GS2P;  // stride-2 stems over s2d halos
  static constexpr int TAPW = S2D ? 4 : 3;              // taps per filter row
  static constexpr int HHT = TH + TAPW - 1;             // halo box height
  static constexpr int ROWB = GEOM == GS2D ? 64 : (GEOM == G3C4 || GEOM == GS2P) ? 16 : 128;  // bytes per halo pixel
  static constexpr int HALO_ROWS = HWD * HHT;
  static constexpr int PLANE_BYTES = HALO_ROWS * ROWB;  // GS2P: one 16-byte-chunk plane
  static constexpr int HALO_BYTES = ((GEOM == GS2P ? 3 : 1) * HALO_ROWS * ROWB + 1023) / 1024 * 1024;
  static constexpr int KB_PER_UNIT = GEOM == GS2D ? 8 : GEOM == GS2P ? 6 : GEOM == G3C4 ? 2 : 9;  // k-blocks per unit
  static constexpr bool RAWG = GEOM != G3X3;           // halo built from raw patches, K steps from a table
  // epilogue warps: G3C4 tiles are short (six K=8 steps), so the per-tile epilogue chain (TMEM load ->
  // smem stage -> proxy fence -> TMA store) is the critical path; two warps per TMEM lane quarter, each
  // owning half the accumulator columns, halve it (measured on VGG conv1_1: the MMA warp waited on
  // tmem_empty, the epilogue never on tmem_full)
  static constexpr int EW = GEOM == G3C4 ? 8 : 4;
  static constexpr int NT = (6 + EW) * 32;
};

struct HArgs {
  int N, H, W, HO, WO, PT, PL, ncb;  // GS2D: H, W, PT, PL describe X' (padding already applied: 0)
  int tiles_w, tiles_h, cta_tiles, pair_tiles, nt, total;
  int64_t M, F, ldd;
  float* d;
  int tma_store;
  unsigned long long* trace;  // debug: conv2d_debug_trace record (stamps 0, 1, 7), or null
  // GS2D raw mode: tmX boxes are raw input patches (RAW_ROWS rows x 32 pixels x rc channels of x, origin
  // (2*ho0 - rpt, 2*wo0 - rpl)) and the transform warps build the swizzled s2d halo from them
  int raw, rc, rpt, rpl;
  // GS2D: the K=8 steps that touch a real (tap, slot), in B's k order: code = tap*2 + half (half = slots
  // 8h..8h+7 of the tap's 16); kbu = ceil(steps / 4) k-blocks (all-padding steps are never issued -- with
  // C = 3 the second half of the a = 3 taps of a 7x7 stem; the list is padded with zero-B steps)
  // per k-block kb: the four steps' A-view offsets from the halo base, in 16-byte descriptor units (u16 x 4)
  uint64_t soff[8];
  uint64_t slbo[8];  // GS2P: per step, the LBO (16-byte units) from the step's first chunk to its second
  int kbu;
  // G3C4: the transform warps build the resident B stages straight from the HWCF filter at kernel start
  // (no filter-prep launch, no workspace); wc / wf = the filter's C and F
  const float* w;
  int wc, wf;
  int wbulk;  // 1: the producer bulk-copies the filter (16-byte aligned, 9 C F % 4 == 0) in one cp.async.bulk
};

struct S2DSteps {
  uint8_t code[32];  // tap*2 + half per issued K=8 step
  int n;             // issued (non-padding) steps
};

// GS2P step list: step i multiplies chunks c1[i] (k = 8i..8i+3) and c2[i] (k = 8i+4..8i+7), chunk code =
// tap*4 + plane (tap = a*4 + e); c2 = 0xFF: the second half of the step is zero B (odd chunk count)
struct S2PSteps {
  uint8_t c1[32], c2[32];
  int n;
};

constexpr int RAW_ROWS = 2 * (TH + 3);  // 38 input rows behind a 19-row s2d halo
// a patch row = 32 pixels x C floats plus 4 floats of slack: the TMA needs the innermost box
// coordinate 16-byte aligned, so the load starts at the aligned float below the patch origin
__host__ __device__ constexpr int raw_row_floats(int c) { return 32 * c + 4; }
constexpr int RAW_BYTES_MAX = RAW_ROWS * raw_row_floats(3) * 4;  // C <= 3: 15200 B
// G3C4: 18 rows x 11 pixels (the views reach pixel wo_l + 3 + 7 = 10) x C floats, + up to 3 floats of
// alignment slack, rounded to whole 16-byte TMA units
constexpr int RAW_ROWS_C4 = TH + 2;
__host__ __device__ constexpr int raw_row_floats_c4(int c) { return (11 * c + 3 + 3) / 4 * 4; }
template <int GEOM> __host__ __device__ constexpr int raw_rows() { return GEOM == G3C4 ? RAW_ROWS_C4 : RAW_ROWS; }
template <int GEOM> __host__ __device__ constexpr int raw_floats(int c) {
  return GEOM == G3C4 ? raw_row_floats_c4(c) : raw_row_floats(c);
}

template <int BN, bool THREE_X, int GEOM, bool BMN = false>
struct HCfg {
  static constexpr int HALO_BYTES = Geo<GEOM>::HALO_BYTES;
  static constexpr int BHALF = (BN / 2) * BK * 4;
  static constexpr int BFULL = BN * BK * 4;
  // ATM (3xTF32, G3X3): the transform warps copy every tap's A rows out of the halo into TMEM, hi and lo
  // (a 64-column slot per tap: hi | lo), and the MMAs take A from TMEM -- shared memory then only feeds B
  // to the tensor core (fact 12: with A_hi and the halo lo read from smem by every MMA, R4 was bound by
  // shared-memory bandwidth at ~0.67 of the tensor peak).  The halo slots hold hi only.
  static constexpr bool ATM = THREE_X && GEOM == G3X3;
  static constexpr int HS = (THREE_X && !ATM) ? 2 : 3;                 // halo slots
  static constexpr int HSLOT = HALO_BYTES * ((THREE_X && !ATM) ? 2 : 1);  // hi (+ lo)
  // CONCAT (3xTF32, BN = 64, where smem operand reads bound the MMA): B stage Z = BN rows (CTA0:
  // B_hi, CTA1: B_lo) for one N'=2BN MMA hi x [B_hi | B_lo] -- A_hi is read once for both products --
  // plus X = BN/2 rows of B_hi (this CTA's half) for lo x B_hi; the epilogue adds the two column halves.
  // Otherwise (BN = 128, TF32): X = B_hi half [+ B_lo half], three / one MMAs per K step.
  // BMN (G3X3, F % 32 == 0): B streams straight from the HWCF filter as an MN-major operand (no filter-prep
  // launch); 3xTF32 then splits B_lo in smem (warps 6+EW .. 9+EW) and uses the plain three-MMA form
  static constexpr bool CONCAT = THREE_X && BN == 64 && !BMN;
  static constexpr bool BSPLIT = BMN && THREE_X;
  static constexpr int NT = Geo<GEOM>::NT + (BSPLIT ? 128 : 0);
  static constexpr int BSTAGE = CONCAT ? BFULL + BHALF : (THREE_X ? 2 : 1) * BHALF;
  static constexpr int ACC = CONCAT ? 2 * BN : BN;                     // TMEM columns per accumulator
  static constexpr int EPI = Geo<GEOM>::EW * 2 * 32 * 128;
  static_assert(GEOM != G3C4 || EPI >= 9 * 4 * 128 * 4, "G3C4 stages the filter in the epilogue buffers");
  // raw-patch ring: G3C4 patches are small (18 rows x 48 floats at most), so four are in flight -- a single
  // slot serialises every tile behind one TMA round trip (measured: 1.6 us per tile on VGG conv1_1); GS2P's
  // smaller halo leaves room for two stem patches
  static constexpr int NR = GEOM == G3C4 ? 4 : GEOM == GS2P ? 2 : 1;
  static constexpr int RAW_SLOT = GEOM == G3C4   ? (RAW_ROWS_C4 * raw_row_floats_c4(4) * 4 + 127) / 128 * 128
                                  : GEOM == GS2P ? (RAW_BYTES_MAX + 127) / 128 * 128
                                                 : 0;
  static constexpr int RAWB = !Geo<GEOM>::RAWG ? 0 : (NR * RAW_SLOT > RAW_BYTES_MAX ? NR * RAW_SLOT : RAW_BYTES_MAX);
  static_assert(NR * RAW_SLOT <= RAWB, "raw ring");
  static constexpr int BUDGET = 232448 - EPI - RAWB - 1024 - 1024 - HS * HSLOT;
  // BRES (GS2D with CONCAT or TF32): the whole B (8 k-blocks, K = 256) stays resident -- stage kb holds
  // k-block kb for the kernel's lifetime; otherwise B streams through an S-stage ring per unit.
  static constexpr bool BRES = Geo<GEOM>::RAWG && (CONCAT || !THREE_X || GEOM == G3C4);
  static constexpr int S = BRES ? Geo<GEOM>::KB_PER_UNIT : ((BUDGET / BSTAGE) > 12 ? 12 : (BUDGET / BSTAGE));
  static_assert(!BRES || S * BSTAGE <= BUDGET, "resident B does not fit");
  static constexpr int SMEM = HS * HSLOT + S * BSTAGE + EPI + RAWB + 1024 + 1024;
  static constexpr int AS = ATM ? (512 - 2 * ACC) / 64 : 0;            // ATM: TMEM tap slots
  static constexpr uint32_t A_COL0 = 2 * ACC;                            // first column of the tap slots
  // accumulator buffers: G3C4 (short tiles) keeps four in TMEM so the epilogue of tile i overlaps the
  // MMAs of tiles i+1 .. i+3; the others double-buffer
  static constexpr int NACC = GEOM == G3C4 ? 4 : 2;
  static constexpr uint32_t TMEM_COLS = ATM ? 512 : NACC * ACC;
  static_assert(S >= 2, "halo kernel needs >= 2 B stages");
  static_assert(!ATM || (AS >= 2 && AS <= 8), "ATM needs 2..8 TMEM tap slots");
  static_assert(NACC * ACC <= 512, "TMEM");
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

template <int BN, bool THREE_X, int GEOM, bool BMN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(HCfg<BN, THREE_X, GEOM, BMN>::NT, 1)
    halo_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmBh,
                const __grid_constant__ CUtensorMap tmBhF, const __grid_constant__ CUtensorMap tmBlF,
                const __grid_constant__ CUtensorMap tmD,
                const __grid_constant__ HArgs args) {
  using C_ = HCfg<BN, THREE_X, GEOM, BMN>;
  using G_ = Geo<GEOM>;
  constexpr int HALO_BYTES = G_::HALO_BYTES;
  constexpr int HS = C_::HS, S = C_::S;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  auto halo_hi = [&](int h) { return smem + (size_t)h * C_::HSLOT; };
  auto halo_lo = [&](int h) { return smem + (size_t)h * C_::HSLOT + HALO_BYTES; };
  auto b_z = [&](int s) { return smem + (size_t)HS * C_::HSLOT + (size_t)s * C_::BSTAGE; };  // CONCAT only
  auto b_x = [&](int s) { return b_z(s) + (C_::CONCAT ? C_::BFULL : 0); };                    // B_hi half
  auto b_lo = [&](int s) { return b_x(s) + C_::BHALF; };                                      // 3x, !CONCAT
  uint8_t* epi_smem = smem + (size_t)HS * C_::HSLOT + (size_t)S * C_::BSTAGE;
  uint8_t* raw = epi_smem + C_::EPI;  // GS2D raw mode
  uint64_t* h_ld = reinterpret_cast<uint64_t*>(raw + C_::RAWB);
  uint64_t* h_full = h_ld + HS;
  uint64_t* h_empty = h_full + HS;
  uint64_t* b_full = h_empty + HS;
  uint64_t* b_empty = b_full + S;
  uint64_t* tmem_full = b_empty + S;
  uint64_t* tmem_empty = tmem_full + C_::NACC;
  uint64_t* raw_ld = tmem_empty + C_::NACC;     // raw patch landed (TMA -> transform), per ring slot
  uint64_t* raw_empty = raw_ld + 4;      // raw patch consumed (transform -> producer), per ring slot
  uint64_t* a_full = raw_empty + 4;      // ATM: tap slot written (both CTAs' transform warps -> leader MMA)
  uint64_t* a_empty = a_full + 8;        // ATM: tap slot read by the MMAs (commit -> transform warps)
  uint64_t* w_ld = a_empty + 8;         // G3C4: the filter's bulk copy into the epilogue buffers landed
  uint64_t* b_ld = w_ld + 1;            // BSPLIT: this CTA's B_hi half landed (TMA -> B-split warps), per stage
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(b_ld + S);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int cid = (int)cluster_id_x(), ncl = (int)nclusters_x();
  const int KBU = G_::RAWG ? args.kbu : G_::KB_PER_UNIT;
  pdl_trigger();  // launch.cuh
  if (threadIdx.x == 0 && args.trace) args.trace[blockIdx.x * 8 + 0] = globaltimer_ns();

  if (threadIdx.x == 0) {
    for (int h = 0; h < HS; ++h) {
      mbar_init(&h_ld[h], 1);
      mbar_init(&h_full[h], 2 * 128);
      mbar_init(&h_empty[h], C_::ATM ? 128 : 1);  // ATM: this CTA's transform threads release the halo
    }
    for (int i = 0; i < 8; ++i) {
      mbar_init(&a_full[i], 2 * 128);
      mbar_init(&a_empty[i], 1);
    }
    for (int s = 0; s < S; ++s) {
      // G3C4: both CTAs' epilogue threads build B; BSPLIT: both CTAs' B-split threads relay their stage
      mbar_init(&b_full[s], GEOM == G3C4 ? 2 * 32 * G_::EW : C_::BSPLIT ? 2 * 128 : 1);
      mbar_init(&b_empty[s], 1);
      mbar_init(&b_ld[s], 1);
    }
    for (int a = 0; a < C_::NACC; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], 2 * 32 * G_::EW);
    }
    for (int r = 0; r < 4; ++r) {
      mbar_init(&raw_ld[r], 1);
      if (r == 0) mbar_init(w_ld, 1);
      mbar_init(&raw_empty[r], 128);
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
  pdl_wait();  // first global-memory access below
  if (threadIdx.x == 0 && args.trace) args.trace[blockIdx.x * 8 + 1] = globaltimer_ns();

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
        if (G_::RAWG && args.raw) {  // raw patch into ring slot u % NR; the transform warps write the halo slot
          const int r = u % C_::NR;
          if (u >= C_::NR) mbar_wait(&raw_empty[r], ((u / C_::NR) - 1) & 1);
          mbar_arrive_expect_tx(&raw_ld[r], (uint32_t)(raw_rows<GEOM>() * raw_floats<GEOM>(args.rc) * 4));
          const int sc = G_::S2D ? 2 : 1;  // input pixels per output pixel
          const int col0 = (sc * tl.wo0 - args.rpl) * args.rc;
          tma_load_3d(&tmX, &raw_ld[r], smem_u32(raw + r * C_::RAW_SLOT), col0 - (col0 & 3), sc * tl.ho0 - args.rpt,
                      tl.n);
          return;
        }
        if (u >= HS) mbar_wait(&h_empty[h], ((u / HS) - 1) & 1);
        mbar_arrive_expect_tx(&h_ld[h], (uint32_t)(G_::HALO_ROWS * G_::ROWB));  // box bytes
        tma_load_4d(&tmX, &h_ld[h], smem_u32(halo_hi(h)), cb * BK, tl.wo0 - args.PL, tl.ho0 - args.PT, tl.n);
      };
      if (C_::BRES && GEOM != G3C4 && units > 0) {  // all of B once (single N tile: F <= BN), to the leader's b_full[0]
        if (rank == 0) mbar_arrive_expect_tx(&b_full[0], 2 * KBU * C_::BSTAGE);
        for (int kb = 0; kb < KBU; ++kb) {
          tma_load_3d_2sm(&tmBh, b_full_leader, smem_u32(b_x(kb)), kb * BK, (int)rank * (BN / 2), 0);
          if (C_::CONCAT)
            tma_load_3d_2sm(rank == 0 ? (const void*)&tmBhF : (const void*)&tmBlF, b_full_leader, smem_u32(b_z(kb)),
                            kb * BK, 0, 0);
          else if (THREE_X)  // G3C4, BN = 128: the B_lo half
            tma_load_3d_2sm(&tmBlF, b_full_leader, smem_u32(b_lo(kb)), kb * BK, (int)rank * (BN / 2), 0);
        }
      }
      if (GEOM == G3C4 && args.wbulk && units > 0) {  // the filter, in flight with the first raw patches
        const uint32_t bytes = (uint32_t)(9 * args.wc * args.wf * 4);
        mbar_arrive_expect_tx(w_ld, bytes);
        bulk_load(smem_u32(epi_smem), args.w, bytes, w_ld);
      }
      if (units > 0) issue_halo(0);
      uint32_t bit = 0;
      for (int u = 0; u < units; ++u) {
        if (u + 1 < units) issue_halo(u + 1);
        if (C_::BRES) continue;
        const HTile tl = hdecode(args, cid + (u / args.ncb) * ncl, rank);
        const int cb = u % args.ncb;
        const int nrow = tl.ni * BN + (int)rank * (BN / 2);
        for (int kb = 0; kb < KBU; ++kb, ++bit) {
          const int s = bit % S;
          if (bit >= (uint32_t)S) mbar_wait(&b_empty[s], ((bit / S) - 1) & 1);
          if constexpr (BMN) {
            // MN-major B_hi half straight from the HWCF filter: rows k = tap*C + cb*32 .. +31, this CTA's
            // 32-column chunks of the pair's N tile ({n % 32, k, n / 32} view, box {32, 32, BN/64})
            const int krow = (kb * args.ncb + cb) * BK;
            if constexpr (C_::BSPLIT) {  // to this CTA's barrier: the B-split warps derive lo, then relay
              mbar_arrive_expect_tx(&b_ld[s], (uint32_t)C_::BHALF);
              tma_load_3d(&tmBh, &b_ld[s], smem_u32(b_x(s)), 0, krow, nrow / 32);
            } else {
              if (rank == 0) mbar_arrive_expect_tx(&b_full[s], 2 * C_::BHALF);
              tma_load_3d_2sm(&tmBh, b_full_leader + (uint32_t)(s * sizeof(uint64_t)), smem_u32(b_x(s)), 0, krow,
                              nrow / 32);
            }
            continue;
          }
          if (rank == 0) mbar_arrive_expect_tx(&b_full[s], 2 * C_::BSTAGE);
          const uint32_t fb = b_full_leader + (uint32_t)(s * sizeof(uint64_t));
          // filter prep order k = tap * C + c: G3X3 k-block kb = tap kb, channel block cb; GS2D k-block
          // kb = taps 2kb, 2kb+1 (16 channels each)
          const int k0 = G_::RAWG ? kb * BK : (kb * args.ncb + cb) * BK;
          tma_load_3d_2sm(&tmBh, fb, smem_u32(b_x(s)), k0, nrow, 0);
          if (C_::CONCAT)  // CTA0: B_hi rows [ni*BN, +BN); CTA1: B_lo rows [ni*BN, +BN)
            tma_load_3d_2sm(rank == 0 ? (const void*)&tmBhF : (const void*)&tmBlF, fb, smem_u32(b_z(s)), k0,
                            tl.ni * BN, 0);
          else if (THREE_X)  // B_lo half (tmBlF holds the half-box B_lo map when !CONCAT)
            tma_load_3d_2sm(&tmBlF, fb, smem_u32(b_lo(s)), k0, nrow, 0);
        }
      }
      for (int i = 0; i < S && !C_::BRES; ++i, ++bit)
        if (bit >= (uint32_t)S) mbar_wait(&b_empty[bit % S], ((bit / S) - 1) & 1);
      for (int i = 0; i < HS; ++i) {
        const int u = units + i;
        if (u >= HS) mbar_wait(&h_empty[u % HS], ((u / HS) - 1) & 1);
      }
    }
  } else if (warp == 5) {
    // ============================ MMA issuer (leader) ============================
    if (rank == 0) {  // whole warp, converged: operands stay warp-uniform
      constexpr uint32_t idesc = idesc_tf32(256, BN) | (BMN ? IDESC_B_MN : 0u);
      constexpr uint32_t idesc2 = idesc_tf32(256, 2 * BN);  // 3x: hi x [B_hi | B_lo]
      uint32_t hit = 0, bit = 0, ai = 0, ait = 0;
      if (C_::BRES && cid < args.total) {
        mbar_wait(&b_full[0], 0);
        tc_fence_after();
      }
      for (int t = cid; t < args.total; t += ncl, ++ai) {
        const int acc = (int)(ai % C_::NACC);
        uint64_t soff_next = G_::RAWG ? args.soff[0] : 0;  // GS2D / G3C4: next k-block's view offsets, a step ahead
        uint64_t slbo_next = GEOM == GS2P ? args.slbo[0] : 0;
        if (ai >= (uint32_t)C_::NACC) mbar_wait(&tmem_empty[acc], ((ai / C_::NACC) - 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem_base + (uint32_t)(acc * C_::ACC);
        for (int cb = 0; cb < args.ncb; ++cb, ++hit) {
          const int h = hit % HS;
          if (!C_::ATM) {
            mbar_wait(&h_full[h], (hit / HS) & 1);
            tc_fence_after();
          }
          if constexpr (GEOM == G3C4) {  // B resident (stages 0, 1): the whole tile from one asm block
            static_assert(C_::BRES, "G3C4 keeps B resident");
            const uint64_t ah = umma_desc_interleave_kmajor(smem_u32(halo_hi(h)), 16u, HWD * G_::ROWB);
            const uint64_t al = THREE_X ? umma_desc_interleave_kmajor(smem_u32(halo_lo(h)), 16u, HWD * G_::ROWB) : 0;
            if (C_::CONCAT)
              mma2_c4_tile_concat(d, ah, al, umma_desc_sw128_kmajor(smem_u32(b_z(0))),
                                  umma_desc_sw128_kmajor(smem_u32(b_z(1))), umma_desc_sw128_kmajor(smem_u32(b_x(0))),
                                  umma_desc_sw128_kmajor(smem_u32(b_x(1))), idesc2, idesc);
            else if (THREE_X)
              mma2_c4_tile_3x(d, ah, al, umma_desc_sw128_kmajor(smem_u32(b_x(0))),
                              umma_desc_sw128_kmajor(smem_u32(b_x(1))), umma_desc_sw128_kmajor(smem_u32(b_lo(0))),
                              umma_desc_sw128_kmajor(smem_u32(b_lo(1))), idesc);
            else
              mma2_c4_tile_1x(d, ah, umma_desc_sw128_kmajor(smem_u32(b_x(0))),
                              umma_desc_sw128_kmajor(smem_u32(b_x(1))), idesc);
            mma_commit_2sm_mc_warp(&h_empty[h], 0x3);
            continue;
          }
          for (int kb = 0; kb < KBU; ++kb, ++bit) {
            const uint64_t soff = soff_next, slbo = slbo_next;
            if constexpr (G_::RAWG) soff_next = args.soff[kb + 1 < 8 ? kb + 1 : 7];
            if constexpr (GEOM == GS2P) slbo_next = args.slbo[kb + 1 < 8 ? kb + 1 : 7];
            const int s = C_::BRES ? kb : (int)(bit % S);
            if (!C_::BRES) {
              mbar_wait(&b_full[s], (bit / S) & 1);
              tc_fence_after();
            }
            // A view of tap (r, c): starts r*16 + c pixel rows into the halo; 8-row groups (one output
            // row of 8 pixels) are 16 pixel rows apart.  Base offset stays 0: the tensor core swizzles
            // on absolute smem address bits, so a view starting c rows into a swizzle period needs no
            // descriptor correction (measured: setting the base-offset field breaks the exact parity).
            auto view = [&](uint32_t base, int tap) {
              const int r = tap / G_::TAPW, c = tap % G_::TAPW;
              const uint32_t a = base + (uint32_t)((r * HWD + c) * G_::ROWB);
              return GEOM == GS2D   ? umma_desc_sw64_kmajor_sbo(a, HWD * G_::ROWB)
                     : GEOM == G3C4 ? umma_desc_interleave_kmajor(a, 16u, HWD * G_::ROWB)  // LBO: next pixel
                     : GEOM == GS2P ? umma_desc_interleave_kmajor(a, 0u, HWD * G_::ROWB)   // LBO per step
                                    : umma_desc_sw128_kmajor_sbo(a, HWD * G_::ROWB, 0u);
            };
            if constexpr (C_::ATM) {  // A from the TMEM tap slot the transform warps filled
              const int slot = (int)(ait % C_::AS);
              mbar_wait(&a_full[slot], (ait / C_::AS) & 1);
              tc_fence_after();
              const uint32_t ahi = tmem_base + C_::A_COL0 + (uint32_t)(slot * 64), alo = ahi + 32;
              // BMN: MN-major SW128_BASE32B B (32 k-rows x 128 B per 32-wide n chunk: LBO 4 KB, SBO 512 B,
              // K=8 step = 1 KB = 64 descriptor units)
              auto bd = [&](const uint8_t* ptr) {
                return BMN ? umma_desc_sw128b32_mn(smem_u32(ptr), BK * 128, 512) : umma_desc_sw128_kmajor(smem_u32(ptr));
              };
              const uint64_t dbx = bd(b_x(s));
              const uint64_t dbz = C_::CONCAT ? umma_desc_sw128_kmajor(smem_u32(b_z(s))) : 0;
              const uint64_t dbl = C_::CONCAT ? 0 : bd(b_lo(s));
              // the tap's four K=8 steps from one asm block (sm100.cuh mma2_kblock_tt_*)
              const uint32_t acc0 = (cb > 0 || kb > 0) ? 1u : 0u;
              if (C_::CONCAT)
                mma2_kblock_tt_concat(d, ahi, alo, dbz, dbx, idesc2, idesc, acc0);
              else
                mma2_kblock_tt_3x(d, ahi, alo, dbx, dbl, idesc, acc0, BMN ? 64u : 2u);
              if (!C_::BRES) mma_commit_2sm_mc_warp(&b_empty[s], 0x3);
              mma_commit_2sm_mc_warp(&a_empty[slot], 0x3);
              ++ait;
              continue;
            }
            const int tap0 = G_::RAWG ? 0 : kb;
            const uint64_t dah0 = view(smem_u32(halo_hi(h)), tap0);
            const uint64_t dal0 = THREE_X ? view(smem_u32(halo_lo(h)), tap0) : 0;
            const uint64_t dbx = umma_desc_sw128_kmajor(smem_u32(b_x(s)));
            const uint64_t dbz = C_::CONCAT ? umma_desc_sw128_kmajor(smem_u32(b_z(s))) : 0;
            const uint64_t dbl = (THREE_X && !C_::CONCAT) ? umma_desc_sw128_kmajor(smem_u32(b_lo(s))) : 0;
            if constexpr (GEOM == G3X3 && !THREE_X) {  // TF32 3x3: one asm block per k-block (sm100.cuh)
              const uint64_t dbm = BMN ? umma_desc_sw128b32_mn(smem_u32(b_x(s)), BK * 128, 512) : dbx;
              mma2_kblock_1x_ss(d, dah0, dbm, 2, BMN ? 64 : 2, idesc, (cb > 0 || kb > 0) ? 1u : 0u);
              if (!C_::BRES) mma_commit_2sm_mc_warp(&b_empty[s], 0x3);
              continue;
            }
#pragma unroll
            for (int k = 0; k < BK / 8; ++k) {
              const uint64_t adv = (uint64_t)((k * 8 * 4) >> 4);  // B: 32 bytes per K=8 step
              // A: G3X3 steps through the tap's 128-byte row; GS2D step 4kb+k is (tap, half) from the step
              // table: the tap's view plus 32 bytes for the second 8 slots (uniform arithmetic, no branch)
              uint64_t dah, dal;
              if constexpr (G_::RAWG) {
                uint64_t off = (soff >> (16 * k)) & 0xFFFFu;
                if constexpr (GEOM == GS2P) off += ((slbo >> (16 * k)) & 0xFFFFu) << 16;  // LBO field
                dah = dah0 + off;
                dal = dal0 + off;
              } else {
                dah = dah0 + adv;
                dal = dal0 + adv;
              }
              const uint32_t accum = (cb > 0 || kb > 0 || k > 0) ? 1u : 0u;
              if (THREE_X && !C_::CONCAT) {
                mma_tf32_2sm_warp(d, dal, dbx + adv, idesc, accum);
                mma_tf32_2sm_warp(d, dah, dbl + adv, idesc, 1u);
                mma_tf32_2sm_warp(d, dah, dbx + adv, idesc, 1u);
              } else if (C_::CONCAT) {
                // cols [0,BN) += hi*B_hi, cols [BN,2BN) += hi*B_lo   (A_hi read once for both products)
                mma_tf32_2sm_warp(d, dah, dbz + adv, idesc2, accum);
                // cols [0,BN) += lo*B_hi
                mma_tf32_2sm_warp(d, dal, dbx + adv, idesc, 1u);
              } else {
                mma_tf32_2sm_warp(d, dah, dbx + adv, idesc, accum);
              }
            }
            if (!C_::BRES) mma_commit_2sm_mc_warp(&b_empty[s], 0x3);
          }
          if (!C_::ATM) mma_commit_2sm_mc_warp(&h_empty[h], 0x3);
        }
        mma_commit_2sm_mc_warp(&tmem_full[acc], 0x3);
      }
    }
    __syncwarp();
  } else if (warp < 4) {
    // ============================ halo transform (128 threads) ============================
    const int t = threadIdx.x;
    const uint32_t h_full_leader = mapa(smem_u32(h_full), 0);
    const uint32_t a_full_leader = mapa(smem_u32(a_full), 0);
    uint32_t hit = 0, ait = 0;
    for (int tt = cid; tt < args.total; tt += ncl) {
      for (int cb = 0; cb < args.ncb; ++cb, ++hit) {
        const int h = hit % HS;
        if constexpr (C_::ATM) {
          // thread t = A row t = output pixel (ho0 + t / 8, wo0 + t % 8); tap (r, c) reads halo pixel
          // (t / 8 + r) * 16 + (t % 8 + c): its 32 channels (one 128-byte SWIZZLE_128B row) -> TMEM lane t,
          // hi = raw fp32 (the MMA reads its top 19 bits) in slot columns [0, 32), lo = x - trunc_tf32(x) in [32, 64)
          mbar_wait(&h_ld[h], (hit / HS) & 1);
          const uint32_t hb = smem_u32(halo_hi(h));
          const uint32_t lane_addr = tmem_base + ((uint32_t)(warp * 32) << 16) + C_::A_COL0;
          for (int tap = 0; tap < 9; ++tap, ++ait) {
            const int p = (t / TW + tap / 3) * HWD + (t % TW + tap % 3);
            float hi[32], lo[32];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float4 v = lds128(hb + sw128_offset((uint32_t)p, (uint32_t)j));
              hi[4 * j] = v.x;
              hi[4 * j + 1] = v.y;
              hi[4 * j + 2] = v.z;
              hi[4 * j + 3] = v.w;
              lo[4 * j] = v.x - tf32_hi(v.x);
              lo[4 * j + 1] = v.y - tf32_hi(v.y);
              lo[4 * j + 2] = v.z - tf32_hi(v.z);
              lo[4 * j + 3] = v.w - tf32_hi(v.w);
            }
            const int slot = (int)(ait % C_::AS);
            if (ait >= (uint32_t)C_::AS) mbar_wait(&a_empty[slot], ((ait / C_::AS) - 1) & 1);
            tc_fence_after();
            tmem_st32(lane_addr + (uint32_t)(slot * 64), hi);
            tmem_st32(lane_addr + (uint32_t)(slot * 64 + 32), lo);
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive_remote(a_full_leader + (uint32_t)(slot * sizeof(uint64_t)));
          }
          mbar_arrive(&h_empty[h]);  // every tap of this halo is in TMEM: the producer may refill the slot
          continue;
        }
        if (GEOM == G3C4 && args.raw) {
          // build the 4-channel halo: pixel p = (hr, wc) of the 18 x 16 halo is one 16-byte row, slot
          // c <- raw[hr][wc][c] for c < C, zero past C (and for the columns wc > 10 no view reaches)
          const int rs = (int)(hit % C_::NR);
          mbar_wait(&raw_ld[rs], (hit / C_::NR) & 1);
          if (hit >= (uint32_t)HS) mbar_wait(&h_empty[h], ((hit / HS) - 1) & 1);  // the MMAs released the slot
          const HTile tl = hdecode(args, tt, rank);
          const int C = args.rc, rowf = raw_row_floats_c4(C);
          const int shift = ((tl.wo0 - args.rpl) * C) & 3;  // patch origin within the aligned load
          const uint32_t rb = smem_u32(raw + rs * C_::RAW_SLOT), hh = smem_u32(halo_hi(h)), hl = smem_u32(halo_lo(h));
          const int wc = t & (HWD - 1);  // fixed per thread: p advances by 128 = 8 halo rows
          int soff[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) soff[e] = (e < C && wc <= 10) ? shift + wc * C + e : -1;
          for (int p = t; p < G_::HALO_ROWS; p += 128) {
            const uint32_t rrow = rb + 4u * (uint32_t)((p / HWD) * rowf);
            float v[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) v[e] = soff[e] >= 0 ? lds32(rrow + 4u * (uint32_t)soff[e]) : 0.f;
            sts128(hh + (uint32_t)(p * 16), make_float4(v[0], v[1], v[2], v[3]));
            if (THREE_X)
              sts128(hl + (uint32_t)(p * 16), make_float4(v[0] - tf32_hi(v[0]), v[1] - tf32_hi(v[1]),
                                                          v[2] - tf32_hi(v[2]), v[3] - tf32_hi(v[3])));
          }
          mbar_arrive(&raw_empty[rs]);
          fence_proxy_async_smem();
          mbar_arrive_remote(h_full_leader + (uint32_t)(h * sizeof(uint64_t)));
          continue;
        }
        if (G_::S2D && args.raw) {
          // build the s2d halo: pixel p = (hi, wi) of the 19 x 16 halo, 16-byte chunk k = slots 4k..4k+3,
          // slot = (b*2 + d)*C + c <- raw[2*hi + b][2*wi + d][c]; GS2D: SWIZZLE_64B placement (chunk k of the
          // 64-byte pixel row goes to k ^ ((p >> 1) & 3)), as the TMA would have written X'; GS2P: chunk k
          // is pixel p of plane k (planes k < C only)
          const int rs = (int)(hit % C_::NR);
          mbar_wait(&raw_ld[rs], (hit / C_::NR) & 1);
          if (hit >= (uint32_t)HS) mbar_wait(&h_empty[h], ((hit / HS) - 1) & 1);  // the MMAs released the slot
          const HTile tl = hdecode(args, tt, rank);
          const int C = args.rc, rowf = raw_row_floats(C);
          const int shift = ((2 * tl.wo0 - args.rpl) * C) & 3;  // patch origin within the aligned load
          const uint32_t rb = smem_u32(raw + rs * C_::RAW_SLOT), hh = smem_u32(halo_hi(h)), hl = smem_u32(halo_lo(h));
          // thread t always handles chunk k = t & 3 of pixels p = (t >> 2) + 32 j: column wc and the swizzle
          // phase are fixed, the halo row advances by 2 per step -- all index math hoisted
          const int k = t & 3, p0 = t >> 2;
          const int wc = p0 % HWD;
          int soff[4];  // raw float offset of slot 4k+e relative to (2*hr rows, 2*wc pixels), -1 = zero
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int slot = 4 * k + e;
            const int bd = slot / C, c = slot - bd * C;
            soff[e] = bd < 4 ? (bd >> 1) * rowf + shift + (2 * wc + (bd & 1)) * C + c : -1;
          }
          const uint32_t chunk_off = (uint32_t)((k ^ ((p0 >> 1) & 3)) << 4);
          const bool skip = GEOM == GS2P && k >= C;  // C planes only
          for (int p = p0; p < G_::HALO_ROWS && !skip; p += 32) {
            const int hr = p / HWD;
            const uint32_t rrow = rb + 4u * (uint32_t)(2 * hr * rowf);
            float v[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) v[e] = soff[e] >= 0 ? lds32(rrow + 4u * (uint32_t)soff[e]) : 0.f;
            const uint32_t off = GEOM == GS2P ? (uint32_t)(k * G_::PLANE_BYTES + p * 16) : (uint32_t)(p * 64) + chunk_off;
            sts128(hh + off, make_float4(v[0], v[1], v[2], v[3]));
            if (THREE_X)
              sts128(hl + off, make_float4(v[0] - tf32_hi(v[0]), v[1] - tf32_hi(v[1]), v[2] - tf32_hi(v[2]),
                                           v[3] - tf32_hi(v[3])));
          }
          mbar_arrive(&raw_empty[rs]);
          fence_proxy_async_smem();
          mbar_arrive_remote(h_full_leader + (uint32_t)(h * sizeof(uint64_t)));
          continue;
        }
        mbar_wait(&h_ld[h], (hit / HS) & 1);
        if (THREE_X) {
          // elementwise lo = x - trunc_tf32(x) over the whole halo (layout-agnostic: same offsets)
          const uint32_t hi = smem_u32(halo_hi(h)), lo = smem_u32(halo_lo(h));
          for (int q = t; q < HALO_BYTES / 16; q += 128) {
            const float4 v = lds128(hi + q * 16);
            sts128(lo + q * 16, make_float4(v.x - tf32_hi(v.x), v.y - tf32_hi(v.y), v.z - tf32_hi(v.z),
                                             v.w - tf32_hi(v.w)));
          }
          fence_proxy_async_smem();
        }
        mbar_arrive_remote(h_full_leader + (uint32_t)(h * sizeof(uint64_t)));
      }
    }
  } else if (C_::BSPLIT && warp >= 6 + G_::EW) {
    // ============================ B-lo split (BSPLIT: warps 6+EW .. 9+EW) ============================
    // lo = b - trunc_tf32(b) elementwise over this CTA's B_hi half (the swizzled MN-major layout carries
    // over), then relay the stage to the leader's b_full -- same k-block order as the producer
    const int t2 = (int)threadIdx.x - (6 + G_::EW) * 32;
    const uint32_t b_full_leader = mapa(smem_u32(b_full), 0);
    uint32_t bit = 0;
    const int my_tiles = args.total > cid ? (args.total - cid + ncl - 1) / ncl : 0;
    for (int u = 0; u < my_tiles * args.ncb; ++u)
      for (int kb = 0; kb < KBU; ++kb, ++bit) {
        const int s = (int)(bit % S);
        mbar_wait(&b_ld[s], (bit / S) & 1);
        const uint32_t hb = smem_u32(b_x(s)), lb = smem_u32(b_lo(s));
#pragma unroll
        for (int i = t2 * 16; i < C_::BHALF; i += 128 * 16) {
          const float4 v = lds128(hb + (uint32_t)i);
          sts128(lb + (uint32_t)i, make_float4(v.x - tf32_hi(v.x), v.y - tf32_hi(v.y), v.z - tf32_hi(v.z),
                                               v.w - tf32_hi(v.w)));
        }
        fence_proxy_async_smem();
        mbar_arrive_remote(b_full_leader + (uint32_t)(s * sizeof(uint64_t)));
      }
  } else {
    // ============================ epilogue (warps 6 .. 6 + EW) ============================
    // warp q = warp % 4 owns TMEM lanes [32q, 32q+32) = output rows ho0 + 4q .. +3, wo0 .. wo0+7; with
    // EW = 8 the two warps of a quarter take alternate 32-column chunks
    const int q = warp & 3;
    constexpr int CSTEP = 32 * (G_::EW / 4);
    const int cfirst = 32 * ((warp - 6) / 4);
    const uint32_t tmem_empty_leader = mapa(smem_u32(tmem_empty), 0);
    const uint32_t ebuf = smem_u32(epi_smem) + (uint32_t)((warp - 6) * 2 * 4096);
    if (args.tma_store && lane == 0) tma_prefetch(&tmD);
    if constexpr (GEOM == G3C4) {
      const int et = (int)threadIdx.x - 6 * 32;
      // resident B, K-major SWIZZLE_128B (row n: 128 bytes = k-block kb's 32 k; 16-byte chunk j at j ^ (n & 7)),
      // k = 8 * step + j: step (r, q) = (step / 2, step % 2) < 6, tap s = 2q + j / 4, channel c = j % 4.
      // CONCAT: b_z = B_hi (CTA0) / B_lo (CTA1), all BN rows; b_x = B_hi, this CTA's BN/2 rows.
      // !CONCAT: b_x = B_hi [+ b_lo = B_lo], this CTA's BN/2 rows.  TF32: b_x = raw B.
      // built by the epilogue warps, idle until the first accumulator (which needs this B) while the transform
      // warps turn the first raw patches into halos; the filter (9 C F <= 4608 floats) is first staged in
      // the epilogue's own smem: coalesced loads, all in flight together
      float* wsm = reinterpret_cast<float*>(epi_smem);
      const int nw = 9 * args.wc * args.wf;
      const bool has_units = args.total > cid;
      if (args.wbulk && has_units) {
        mbar_wait(w_ld, 0);
      } else {
#pragma unroll 8
        for (int i = et; i < nw; i += 256) wsm[i] = __ldg(args.w + i);
        named_bar_sync(1, 256);
      }
      auto bval = [&](int f, int k, bool lo) {
        const int step = k >> 3, j = k & 7, r = step >> 1, sc = 2 * (step & 1) + (j >> 2), c = j & 3;
        float v = 0.f;
        if (step < 6 && sc < 3 && c < args.wc && f < args.wf) v = wsm[((r * 3 + sc) * args.wc + c) * args.wf + f];
        if (!THREE_X) return v;
        const float hi = tf32_hi(v);
        return lo ? v - hi : hi;
      };
      auto put = [&](uint8_t* base, int n, int k, float v) {
        sts32(smem_u32(base) + (uint32_t)(n * 128 + ((((k & 31) >> 2) ^ (n & 7)) << 4) + (k & 3) * 4), v);
      };
      for (int kb = 0; kb < 2; ++kb) {
        if (C_::CONCAT)
          for (int i = et; i < BN * 32; i += 256) {
            const int n = i >> 5, k = kb * 32 + (i & 31);
            put(b_z(kb), n, k, bval(n, k, rank == 1));
          }
        for (int i = et; i < (BN / 2) * 32; i += 256) {
          const int n = i >> 5, k = kb * 32 + (i & 31), f = (int)rank * (BN / 2) + n;
          put(b_x(kb), n, k, bval(f, k, false));
          if (THREE_X && !C_::CONCAT) put(b_lo(kb), n, k, bval(f, k, true));
        }
      }
      fence_proxy_async_smem();
      mbar_arrive_remote(mapa(smem_u32(b_full), 0));
    }
    uint32_t ai = 0, chunk = 0;
    for (int t = cid; t < args.total; t += ncl, ++ai) {
      const HTile tl = hdecode(args, t, rank);
      const int acc = (int)(ai % C_::NACC);
      mbar_wait(&tmem_full[acc], (ai / C_::NACC) & 1);
      tc_fence_after();
      const int ho = tl.ho0 + 4 * q + lane / 8, wo = tl.wo0 + lane % 8;
      const bool row_ok = tl.n < args.N && ho < args.HO && wo < args.WO;
      const bool warp_ok = tl.n < args.N && tl.ho0 + 4 * q < args.HO;
      const int n0 = tl.ni * BN;
#pragma unroll 1
      for (int c0 = cfirst; c0 < BN; c0 += CSTEP) {
        float v[32];
        tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * C_::ACC + c0), v);
        if (C_::CONCAT) {  // add the hi*B_lo correction columns
          float w[32];
          tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * C_::ACC + BN + c0), w);
#pragma unroll
          for (int k = 0; k < 32; ++k) v[k] += w[k];
        }
        if (c0 + CSTEP >= BN) {
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
  if (threadIdx.x == 0 && args.trace) args.trace[blockIdx.x * 8 + 7] = globaltimer_ns();
}

template <int BN, bool THREE_X, int GEOM, bool BMN = false>
cudaError_t launch_h(const CUtensorMap& x, const CUtensorMap& bh, const CUtensorMap& bhf, const CUtensorMap& blf,
                     const CUtensorMap& dm, const HArgs& a, int clusters, cudaStream_t s) {
  using C_ = HCfg<BN, THREE_X, GEOM, BMN>;
  auto kern = halo_kernel<BN, THREE_X, GEOM, BMN>;
  const cudaError_t e = smem_attr_once<halo_kernel<BN, THREE_X, GEOM, BMN>>(C_::SMEM);
  if (e != cudaSuccess) return e;
  return launch_k(kern, dim3(2 * clusters), dim3(C_::NT), C_::SMEM, s, x, bh, bhf, blf, dm, a);
}

}  // namespace

bool halo_ok(const Problem& p) {
  return p.KH == 3 && p.KW == 3 && p.SH == 1 && p.SW == 1 && p.C % 32 == 0 && p.F <= 128 &&
         (int64_t)p.N * ((p.HO + TH - 1) / TH) * ((p.WO + TW - 1) / TW) < (1 << 30);
}

// Space-to-depth stem (GS2D): a K x K / stride-2 conv with K in {7, 8} and C <= 4 equals a 4x4 /
// stride-1 VALID conv over X'[n][i][j][(b*2 + d)*C + c] = x[n][2i + b - PT][2j + d - PL][c] (16 channel
// slots, zero outside the image / past 4C) with W'[a][e][(b*2 + d)*C + c][f] = w[2a + b][2e + d][c][f]
// (zero past K).  X' is (N, HO + 3, WO + 3, 16).
bool s2d_ok(const Problem& p) {
  return p.SH == 2 && p.SW == 2 && (p.KH == 7 || p.KH == 8) && (p.KW == 7 || p.KW == 8) && p.C <= 4 &&
         p.F <= 128 && (int64_t)p.N * ((p.HO + TH - 1) / TH) * ((p.WO + TW - 1) / TW) < (1 << 30) &&
         (int64_t)p.N * (p.HO + 3) * (p.WO + 3) * 16 < (1LL << 31);
}

namespace {
// Shared host path: tensor maps for the halo boxes (geometry GEOM), B (K-major Bt hi/lo, kpad x npad)
// and the output, then the launch.  x = the NHWC tensor the halo boxes read (X' for GS2D) with dims
// (n, h, w, cx).
template <int GEOM>
cudaError_t launch_halo_geo(const Problem& p, const float* x, int h, int w, int cx, int pt, int pl, int ncb,
                            const float* bt_hi, const float* bt_lo, int64_t kpad, int64_t npad, int block_n,
                            float* out, cudaStream_t s, bool raw = false, const void* s2d_steps = nullptr,
                            const float* c4_filt = nullptr, bool c4_three_x = false, bool bmn = false) {
  using G_ = Geo<GEOM>;
  // G3C4 and BMN read the filter itself (c4_filt): the math mode comes from the caller
  const bool three_x = (GEOM == G3C4 || bmn) ? c4_three_x : bt_lo != nullptr;
  HArgs a{};
  a.trace = gemm2_trace_record();
  a.kbu = Geo<GEOM>::KB_PER_UNIT;
  if (GEOM == GS2D && s2d_steps) {  // issued steps, in B's k order
    const auto* st = static_cast<const S2DSteps*>(s2d_steps);
    for (int i = 0; i < 32; ++i) {
      const int tap = st->code[i] >> 1, half = st->code[i] & 1;
      const uint64_t off = (uint64_t)(((tap / Geo<GS2D>::TAPW) * HWD + tap % Geo<GS2D>::TAPW) * Geo<GS2D>::ROWB +
                                      half * 32) >> 4;
      a.soff[i / 4] |= off << (16 * (i % 4));
    }
    a.kbu = (st->n + 3) / 4;
  }
  if (GEOM == GS2P && s2d_steps) {  // chunk pairs: view at the first chunk, LBO to the second
    const auto* st = static_cast<const S2PSteps*>(s2d_steps);
    auto addr16 = [](int code) {  // chunk address in 16-byte units from the halo base
      const int tap = code >> 2, plane = code & 3;
      return (plane * Geo<GS2P>::PLANE_BYTES + ((tap >> 2) * HWD + (tap & 3)) * 16) >> 4;
    };
    for (int i = 0; i < 32; ++i) {
      const int o1 = addr16(st->c1[i]);
      const int lbo = st->c2[i] == 0xFF ? 0 : addr16(st->c2[i]) - o1;
      a.soff[i / 4] |= (uint64_t)o1 << (16 * (i % 4));
      a.slbo[i / 4] |= (uint64_t)lbo << (16 * (i % 4));
    }
    a.kbu = (st->n + 3) / 4;
  }
  a.N = p.N; a.H = h; a.W = w; a.HO = p.HO; a.WO = p.WO; a.PT = pt; a.PL = pl;
  a.ncb = ncb;
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
  if (GEOM == G3C4) {  // six steps (r, q): taps (r, 2q) and (r, 2q + 1); steps 6, 7 have zero B rows
    for (int i = 0; i < 6; ++i) a.soff[i / 4] |= (uint64_t)((i / 2) * HWD + 2 * (i % 2)) << (16 * (i % 4));
    a.kbu = 2;
  }
  if (raw) {  // raw mode: patches {raw floats, raw rows, 1} of x viewed as (N, H, W*C)
    a.raw = 1;
    a.rc = p.C;
    a.rpt = p.pad_top;
    a.rpl = p.pad_left;
    const uint64_t dims[3] = {(uint64_t)p.W * p.C, (uint64_t)p.H, (uint64_t)p.N};
    const uint64_t st[2] = {(uint64_t)p.W * p.C * 4, (uint64_t)p.H * p.W * p.C * 4};
    const uint32_t box[3] = {(uint32_t)raw_floats<GEOM>(p.C), (uint32_t)raw_rows<GEOM>(), 1};
    if (!gemm2_encode_tiled(&tx, 3, x, dims, st, box, false)) return cudaErrorInvalidValue;
  } else {  // input halo boxes {32 | 16 ch, 16 w, HHT h, 1 n} over NHWC, OOB (padding) -> 0
    const uint64_t dims[4] = {(uint64_t)cx, (uint64_t)w, (uint64_t)h, (uint64_t)p.N};
    const uint64_t st[3] = {(uint64_t)cx * 4, (uint64_t)w * cx * 4, (uint64_t)h * w * cx * 4};
    const uint32_t box[4] = {(uint32_t)(G_::ROWB / 4), HWD, G_::HHT, 1};
    if (!gemm2_encode_tiled_sw(&tx, 4, x, dims, st, box,
                               GEOM == GS2D ? (int)CU_TENSOR_MAP_SWIZZLE_64B : (int)CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  }
  if (GEOM == G3C4) {  // B is built in the kernel from the filter: no B maps (the slots hold the X map)
    a.w = c4_filt;
    a.wc = p.C;
    a.wf = (int)p.F;
    a.wbulk = (reinterpret_cast<uintptr_t>(c4_filt) & 15) == 0 && (9 * p.C * p.F) % 4 == 0 &&
              getenv("CONV2D_C4_NO_WBULK") == nullptr;
    tbh = tbhf = tblf = tx;
  } else if (bmn) {  // MN-major B from the row-major (9C x F) filter: view {n % 32, k, n / 32}, box {32, 32, BN/64}
    if (p.F % 32 != 0 || !c4_filt) return cudaErrorInvalidValue;
    const uint64_t dims[3] = {32, (uint64_t)p.KH * p.KW * p.C, (uint64_t)(p.F / 32)};
    const uint64_t st[2] = {(uint64_t)p.F * 4, 128};
    const uint32_t box[3] = {32, 32, (uint32_t)(block_n / 64)};
    if (!gemm2_encode_tiled_sw(&tbh, 3, c4_filt, dims, st, box, (int)CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
      return cudaErrorInvalidValue;
    tbhf = tblf = tbh;
  } else {
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
  if constexpr (GEOM == G3X3) {
    if (bmn) {
      switch (block_n) {
        case 64: return three_x ? launch_h<64, true, GEOM, true>(tx, tbh, tbhf, tblf, td, a, clusters, s)
                                : launch_h<64, false, GEOM, true>(tx, tbh, tbhf, tblf, td, a, clusters, s);
        case 128: return three_x ? launch_h<128, true, GEOM, true>(tx, tbh, tbhf, tblf, td, a, clusters, s)
                                 : launch_h<128, false, GEOM, true>(tx, tbh, tbhf, tblf, td, a, clusters, s);
      }
      return cudaErrorInvalidValue;
    }
  }
  switch (block_n) {
    case 64: return three_x ? launch_h<64, true, GEOM>(tx, tbh, tbhf, tblf, td, a, clusters, s)
                            : launch_h<64, false, GEOM>(tx, tbh, tbhf, tblf, td, a, clusters, s);
    case 128: return three_x ? launch_h<128, true, GEOM>(tx, tbh, tbhf, tblf, td, a, clusters, s)
                             : launch_h<128, false, GEOM>(tx, tbh, tbhf, tblf, td, a, clusters, s);
  }
  return cudaErrorInvalidValue;
}

// X' = s2d(x): block row blockIdx.y = one X' row (n, i); four threads per X' pixel, thread q writes
// slots 4q..4q+3 (one float4) so a warp stores 512 contiguous bytes; no index divisions beyond / 4;
// C static so the slot -> (b, d, c) map folds
template <int C>
__global__ void s2d_input_kernel(const float* __restrict__ x, int N, int H, int W, int PT, int PL, int Hs, int Ws,
                                 float* __restrict__ xs) {
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.y + blockIdx.z * 65535;  // n * Hs + i
  if (row >= N * Hs) return;
  const int n = row / Hs, i = row - n * Hs;
  const int g = blockIdx.x * blockDim.x + threadIdx.x;  // j * 4 + q
  if (g >= Ws * 4) return;
  const int j = g >> 2, qd = g & 3;
  float v[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int slot = 4 * qd + e;
    const int bd = slot / C, c = slot % C;
    const int ih = 2 * i + (bd >> 1) - PT, iw = 2 * j + (bd & 1) - PL;
    v[e] = (bd < 4 && ih >= 0 && ih < H && iw >= 0 && iw < W) ? __ldg(x + (((int64_t)n * H + ih) * W + iw) * C + c)
                                                               : 0.f;
  }
  reinterpret_cast<float4*>(xs + (int64_t)row * Ws * 16)[g] = make_float4(v[0], v[1], v[2], v[3]);
}

// Bt'[f][k] (npad x 256, K-major), k = (a*4 + e)*16 + (b*2 + d)*C + c  <-  w[2a+b][2e+d][c][f]; 3xTF32: hi/lo
__global__ void s2d_filter_kernel(const float* __restrict__ w, int KH, int KW, int C, int F, int64_t npad,
                                  float* __restrict__ bt_hi, float* __restrict__ bt_lo, const S2DSteps st) {
  pdl_trigger();
  pdl_wait();
  const int64_t total = npad * 256;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i % 256);
    const int f = (int)(i / 256);
    // k = 8 * step + j: step -> (tap, half) from the table; steps past st.n are zero rows
    const int step = k / 8, j = k % 8;
    if (step >= st.n) {
      bt_hi[i] = 0.f;
      if (bt_lo) bt_lo[i] = 0.f;
      continue;
    }
    const int tap = st.code[step] >> 1, slot = (st.code[step] & 1) * 8 + j;
    const int a = tap / 4, e = tap % 4;
    const int bd = C > 0 ? slot / C : 0, c = C > 0 ? slot % C : 0;
    const int r = 2 * a + (bd >> 1), sc = 2 * e + (bd & 1);
    float v = 0.f;
    if (bd < 4 && r < KH && sc < KW && f < F) v = w[((int64_t)(r * KW + sc) * C + c) * F + f];
    const float h = bt_lo ? tf32_hi(v) : v;
    bt_hi[i] = h;
    if (bt_lo) bt_lo[i] = v - h;
  }
}
// Bt'[f][k] (npad x 192, K-major) for GS2P: k = 8 * step + j, chunk = j < 4 ? c1 : c2 (tap (a, e), plane q),
// slot = 4q + j % 4 = (b*2 + d)*C + c  <-  w[2a+b][2e+d][c][f] (zero past K, past 4C slots, for c2 = 0xFF and
// for steps past st.n); 3xTF32: hi/lo
__global__ void s2p_filter_kernel(const float* __restrict__ w, int KH, int KW, int C, int F, int64_t npad,
                                  float* __restrict__ bt_hi, float* __restrict__ bt_lo, const S2PSteps st) {
  pdl_trigger();
  pdl_wait();
  constexpr int KP = Geo<GS2P>::KB_PER_UNIT * 32;
  const int64_t total = npad * KP;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i % KP);
    const int f = (int)(i / KP);
    const int step = k / 8, j = k % 8;
    const int code = step < st.n ? (j < 4 ? st.c1[step] : st.c2[step]) : 0xFF;
    float v = 0.f;
    if (code != 0xFF && f < F) {
      const int tap = code >> 2, plane = code & 3, a = tap >> 2, e = tap & 3;
      const int slot = 4 * plane + (j & 3), bd = slot / C, c = slot % C;
      const int r = 2 * a + (bd >> 1), sc = 2 * e + (bd & 1);
      if (bd < 4 && r < KH && sc < KW) v = w[((int64_t)(r * KW + sc) * C + c) * F + f];
    }
    const float h = bt_lo ? tf32_hi(v) : v;
    bt_hi[i] = h;
    if (bt_lo) bt_lo[i] = v - h;
  }
}
}  // namespace

cudaError_t launch_gemm_halo(const Problem& p, const float* in, const float* bt_hi, const float* bt_lo, int64_t kpad,
                             int64_t npad, int block_n, float* out, cudaStream_t s, const float* filt, bool bmn,
                             bool three_x) {
  return launch_halo_geo<G3X3>(p, in, p.H, p.W, p.C, p.pad_top, p.pad_left, p.C / 32, bt_hi, bt_lo, kpad, npad,
                               block_n, out, s, false, nullptr, filt, three_x, bmn);
}

// G3C4: 3x3 / stride 1 with C <= 4, raw patches straight from x (16-byte rows of W*C floats)
bool c4_ok(const Problem& p) {
  return p.KH == 3 && p.KW == 3 && p.SH == 1 && p.SW == 1 && p.C <= 4 && p.F <= 128 &&
         ((int64_t)p.W * p.C) % 4 == 0 && (int64_t)p.W * p.C < (1LL << 31) &&
         (int64_t)p.N * ((p.HO + TH - 1) / TH) * ((p.WO + TW - 1) / TW) < (1 << 30);
}

size_t c4_workspace(const Problem&, int, bool) { return 0; }  // B is built inside the kernel

cudaError_t launch_gemm_c4(const Problem& p, const float* in, const float* filt, int block_n, bool three_x, void*,
                           float* out, cudaStream_t s) {
  const int64_t npad = (p.F + block_n - 1) / block_n * block_n;
  return launch_halo_geo<G3C4>(p, in, p.H, p.W, 4, p.pad_top, p.pad_left, 1, nullptr, nullptr, 64, npad, block_n, out,
                               s, true, nullptr, filt, three_x);
}

size_t s2d_workspace(const Problem& p, int block_n, bool three_x) {
  const int64_t npad = (p.F + block_n - 1) / block_n * block_n;
  const size_t bt = (size_t)((npad * 256 * 4 + 255) / 256 * 256);
  const size_t xs = (size_t)(((int64_t)p.N * (p.HO + 3) * (p.WO + 3) * 16 * 4 + 255) / 256 * 256);
  return bt * (three_x ? 2 : 1) + xs;
}

cudaError_t launch_gemm_s2d(const Problem& p, const float* in, const float* filt, int block_n, bool three_x,
                            void* ws, float* out, cudaStream_t s) {
  const int64_t npad = (p.F + block_n - 1) / block_n * block_n;
  const size_t bt = (size_t)((npad * 256 * 4 + 255) / 256 * 256);
  uint8_t* w8 = static_cast<uint8_t*>(ws);
  float* bt_hi = reinterpret_cast<float*>(w8);
  w8 += bt;
  float* bt_lo = nullptr;
  if (three_x) {
    bt_lo = reinterpret_cast<float*>(w8);
    w8 += bt;
  }
  float* xs = reinterpret_cast<float*>(w8);
  const int hs = p.HO + 3, wsd = p.WO + 3;
  // the K=8 steps with any real (tap, slot) (slot = (b*2 + d)*C + c, tap = (a, e)): issued in this order
  S2DSteps st{};
  for (int code = 0; code < 32; ++code) {
    const int tap = code >> 1, a_ = tap / 4, e_ = tap % 4;
    bool any = false;
    for (int slot = (code & 1) * 8; slot < (code & 1) * 8 + 8 && !any; ++slot) {
      const int bd = slot / p.C;
      any = bd < 4 && 2 * a_ + (bd >> 1) < p.KH && 2 * e_ + (bd & 1) < p.KW;
    }
    if (any) st.code[st.n++] = (uint8_t)code;
  }
  for (int c = st.n; c < 32; ++c) st.code[c] = st.code[0];  // padding steps: any view, zero B rows
  // raw mode (C <= 3, 16-byte input rows): the GEMM builds s2d halos from raw input patches itself
  const bool raw = p.C <= 3 && ((int64_t)p.W * p.C) % 4 == 0 && getenv("CONV2D_S2D_PREPASS") == nullptr;
  if (raw && getenv("CONV2D_S2D_SW64") == nullptr) {
    // GS2P: the (tap, plane) chunks with a real (tap, slot), in halo-address order, paired into K=8 steps
    S2PSteps sp{};
    int chunks[64], nc = 0;
    for (int plane = 0; plane < p.C; ++plane)
      for (int tap = 0; tap < 16; ++tap) {
        const int a_ = tap >> 2, e_ = tap & 3;
        bool any = false;
        for (int j = 0; j < 4 && !any; ++j) {
          const int slot = 4 * plane + j, bd = slot / p.C;
          any = bd < 4 && 2 * a_ + (bd >> 1) < p.KH && 2 * e_ + (bd & 1) < p.KW;
        }
        if (any) chunks[nc++] = tap * 4 + plane;
      }
    // address order = (plane, a, e): already ascending by construction (plane-major, tap = a*4 + e)
    for (int i = 0; i < nc; i += 2) {
      sp.c1[sp.n] = (uint8_t)chunks[i];
      sp.c2[sp.n] = i + 1 < nc ? (uint8_t)chunks[i + 1] : (uint8_t)0xFF;
      ++sp.n;
    }
    for (int i = sp.n; i < 32; ++i) {  // padding steps: any view, zero B rows
      sp.c1[i] = sp.c1[0];
      sp.c2[i] = 0xFF;
    }
    if (sp.n > 4 * Geo<GS2P>::KB_PER_UNIT) return cudaErrorInvalidValue;
    constexpr int KP = Geo<GS2P>::KB_PER_UNIT * 32;
    const int64_t fb = (npad * KP + 255) / 256;
    cudaError_t e = launch_k(s2p_filter_kernel, dim3((unsigned)fb), dim3(256), 0, s, filt, p.KH, p.KW, p.C, p.F,
                             npad, bt_hi, bt_lo, sp);
    if (e != cudaSuccess) return e;
    return launch_halo_geo<GS2P>(p, in, hs, wsd, 16, 0, 0, 1, bt_hi, bt_lo, KP, npad, block_n, out, s, true, &sp);
  }
  if (raw) {
    int64_t fb = (npad * 256 + 255) / 256;
    cudaError_t e = launch_k(s2d_filter_kernel, dim3((unsigned)fb), dim3(256), 0, s, filt, p.KH, p.KW, p.C, p.F,
                             npad, bt_hi, bt_lo, st);
    if (e != cudaSuccess) return e;
    return launch_halo_geo<GS2D>(p, in, hs, wsd, 16, 0, 0, 1, bt_hi, bt_lo, 256, npad, block_n, out, s, true, &st);
  }
  const int rows = p.N * hs;
  auto kin = p.C == 1 ? s2d_input_kernel<1> : p.C == 2 ? s2d_input_kernel<2> : p.C == 3 ? s2d_input_kernel<3>
                                                                                         : s2d_input_kernel<4>;
  const dim3 grid((unsigned)((wsd * 4 + 255) / 256), (unsigned)(rows < 65535 ? rows : 65535),
                  (unsigned)((rows + 65534) / 65535));
  cudaError_t e = launch_k(kin, grid, dim3(256), 0, s, in, p.N, p.H, p.W, p.pad_top, p.pad_left, hs, wsd, xs);
  if (e != cudaSuccess) return e;
  int64_t fb = (npad * 256 + 255) / 256;
  e = launch_k(s2d_filter_kernel, dim3((unsigned)fb), dim3(256), 0, s, filt, p.KH, p.KW, p.C, p.F, npad, bt_hi,
               bt_lo, st);
  if (e != cudaSuccess) return e;
  return launch_halo_geo<GS2D>(p, xs, hs, wsd, 16, 0, 0, 1, bt_hi, bt_lo, 256, npad, block_n, out, s, false, &st);
}

}  // namespace conv2d
