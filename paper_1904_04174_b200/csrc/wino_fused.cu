// wino_fused.cu -- CONV2D_ALGO_WINOGRAD_F2X2_3X3 in fused form: "a tiled Winograd operation which uses data
// transforms to convert the convolution into a number of small matrix multiplies" (
// SPEC.md:258-266; Lavin-Gray F(2x2,3x3), correlation form, reading R12), with the input transform,
// the 16 per-coordinate GEMMs and the output transform in ONE kernel: V and M never leave the SM pair.
//
//   V_kl = (B^T d B)_kl   per 4x4 input patch d of a 2x2 output tile, per channel
//   M_kl = sum_c V_kl[t, c] U_kl[c, f]                       (16 GEMMs, k, l in 0..3)
//   Y    = A^T M A  =>  Y[i][j] = sum_k A^T[i][k] z_k[j],  z_k[j] = sum_l M_kl A[l][j]
//   B^T = [[1,0,-1,0],[0,1,1,0],[0,-1,1,0],[0,1,0,-1]]      A^T = [[1,1,1,0],[0,1,-1,-1]]
//
// Work split.  A cluster of two CTAs owns a unit = (block of up to 128 tiles, 32 features).  CTA r computes the
// coordinate rows k = 2r, 2r+1 (eight of the 16 GEMMs) for all 128 tiles: its accumulators are 8 x 32 TMEM
// columns, one TMEM lane per tile.  Row k of B^T has two non-zeros, so CTA r reads only input patch rows
// r .. r+2 (rows 0-2 for r = 0, 1-3 for r = 1).  Output rows: A^T[0] = (1,1,1,0) and A^T[1] = (0,1,-1,-1), so
//   CTA 0 holds  P0[0] = z0 + z1  and  P0[1] = z1,      CTA 1 holds  P1[0] = z2  and  P1[1] = -z2 - z3;
// CTA 0 finishes output row i = 0 (Y0 = P0[0] + P1[0]) and CTA 1 row i = 1 (Y1 = P0[1] + P1[1]): each sends
// the other ONE partial row (2 values per tile and feature) through distributed shared memory (st.async),
// adds the one it receives in fixed order, and TMA-stores its output row.  Deterministic: no atomics, every
// sum in a fixed order.
//
// Pipeline per CTA (warp roles, 320 threads):
//   warp 4      TMA producer: per 16-channel stage, one half of the input halo (multicast to both CTAs) and
//               this CTA's 8 coordinates x 32 features x 16 channels of U (hi, + lo in 3xTF32);
//   warps 0-3   transform: thread = tile = TMEM lane; reads 3 patch rows x 4 columns x 8 channels from the
//               swizzled halo, forms V for its 8 coordinates and writes them (hi | lo) into a TMEM staging
//               slot (tcgen05.st) -- the MMAs take A from TMEM, shared memory only feeds them U;
//   warp 5      MMA issuer: per K=8 step and coordinate, lo*U_hi + hi*U_lo + hi*U_hi (3xTF32) or hi*U_hi
//               (TF32; V and U rounded with cvt.rna, reading R16), M=128 x N=32 x K=8, cta_group::1;
//   warps 6-9   epilogue: tcgen05.ld of the 8 accumulators, z and the partial rows, the DSMEM exchange, the
//               final add, TMA store of one output row per tile.  The accumulator columns are released
//               coordinate by coordinate, so the next unit's MMAs start while the exchange runs.
// The filter transform U = G g G^T (per (c, f), shared by every tile) runs once per call in a small
// preceding launch (launch_wino_filter, winograd.cu).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>

#include "gemm2sm.h"
#include "launch.cuh"
#include "sm100.cuh"

namespace conv2d {
namespace {

using namespace sm100;

constexpr int NTHREADS = 448;  // 14 warps: 0-7 transform (two groups), 8 producer, 9 MMA, 10-13 epilogue
constexpr int BN = 32;         // features per unit
constexpr int CH = 16;         // channels per pipeline stage (64-byte halo pixel rows, SWIZZLE_64B)
constexpr int NCO = 8;         // GEMM coordinates per CTA (two rows of the 4 x 4 grid)
constexpr int NVS = 2;         // TMEM staging slots for V: slot g = K step g of every stage, transform group g
constexpr int MAXS = 4;        // pipeline stages (halo + U), as many as shared memory allows
constexpr uint32_t ACC_COLS = NCO * BN;   // 256 accumulator columns: coordinate c at [32c, 32c + 32)
constexpr uint32_t VS_COLS = NCO * 16;    // per staging slot: coordinate c hi at +16c, lo at +16c + 8
constexpr uint32_t V_COL0 = ACC_COLS;
constexpr uint32_t U_BYTES = NCO * BN * CH * 4;   // 16 KB: [8 coords][32 f][16 c], SWIZZLE_64B rows
constexpr uint32_t RECV_BYTES = 128 * 2 * BN * 4; // 32 KB: [tile][j][32 f], SWIZZLE_128B rows (= the store box)
constexpr uint32_t BAR_BYTES = 512;
constexpr int SMEM_LIMIT = 232448;

struct WFArgs {
  int HO, WO, PT, PL;
  int NB, BH, BW, HWB, HH2;  // tile block: NB images x BH x BW tiles; halo box HWB wide, HH2 = half its height
  int blocks_w, blocks_h, nfb, units, ncs, S;
  // The halo of a stage is four TMA boxes: rows [h*HH2, (h+1)*HH2) (h = the issuing CTA) x pixel parity p (W
  // traversal stride 2: the BW + 1 even or odd pixels), each in its own 1024-aligned region (h, p)
  uint32_t q_bytes;      // smem bytes of one (half, parity) region
  uint32_t box_bytes;    // TMA bytes of one (half, parity) box
  uint32_t stage_bytes;  // 4 * q_bytes + U (hi [, lo])
  unsigned long long* trace;
  int dbg;  // CONV2D_WF_DEBUG bit mask (timing experiments only; results are garbage when set)
  unsigned long long* prof;  // CONV2D_WF_PROF: per-role clock64 counters of CTA 0 and 1 (32 per CTA)
};

struct WUnit {
  int n0, th0, tw0, f0;
};

__device__ __forceinline__ WUnit wdecode(const WFArgs& a, int u) {
  WUnit r;
  const int fb = u % a.nfb;  // feature blocks fastest: concurrent clusters share the halo in L2
  int tb = u / a.nfb;
  const int bwi = tb % a.blocks_w;
  tb /= a.blocks_w;
  const int bhi = tb % a.blocks_h;
  r.n0 = (tb / a.blocks_h) * a.NB;
  r.th0 = bhi * a.BH;
  r.tw0 = bwi * a.BW;
  r.f0 = fb * BN;
  return r;
}

__device__ __forceinline__ long long clk() { return clock64(); }
#define WCOUNT(slot) do { if (a.prof && blockIdx.x < 2) atomicAdd(&a.prof[blockIdx.x * 32 + (slot)], 1ull); } while (0)
#define WPROF(slot, t0) do { if (a.prof && blockIdx.x < 2) { const long long _t = clk(); atomicAdd(&a.prof[blockIdx.x * 32 + (slot)], (unsigned long long)(_t - (t0))); t0 = _t; } } while (0)

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// Packed fp32 pairs (two consecutive channels in one 64-bit register): FADD2 does both lanes in one
// instruction (sm_100), halving the transform's adds.
__device__ __forceinline__ uint64_t f2add(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t f2sub(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ void f2split(uint64_t v, float& x, float& y) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(v));
}

// One coordinate row of V for 8 channels (4 pairs): t[b][p] (4 patch columns) -> V_l = (t B)_l, l = 0..3,
// written as [l][hi 8 | lo 8] into two 32-column TMEM stores at `taddr` (coordinates 0,1) and taddr + 32 (2,3).
template <bool THREE_X>
__device__ __forceinline__ void v_row_store(const uint64_t (&t)[4][4], uint32_t taddr) {
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    float o[32];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int l = 2 * g + h;
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        // B^T column transform (same expressions as the unfused input transform, winograd.cu bt2)
        const uint64_t v = l == 0 ? f2sub(t[0][p], t[2][p]) : l == 1 ? f2add(t[1][p], t[2][p])
                           : l == 2 ? f2sub(t[2][p], t[1][p]) : f2sub(t[1][p], t[3][p]);
        float x, y;
        f2split(v, x, y);
        if (THREE_X) {
          // hi = raw fp32 (the MMA reads its top 19 bits, reading R16), lo = v - trunc_tf32(v), exact
          const uint64_t hv = v & 0xFFFFE000FFFFE000ull;
          float lx, ly;
          f2split(f2sub(v, hv), lx, ly);
          o[16 * h + 2 * p] = x;
          o[16 * h + 2 * p + 1] = y;
          o[16 * h + 8 + 2 * p] = lx;
          o[16 * h + 8 + 2 * p + 1] = ly;
        } else {
          o[16 * h + 2 * p] = tf32_rna(x);
          o[16 * h + 2 * p + 1] = tf32_rna(y);
          o[16 * h + 8 + 2 * p] = 0.f;
          o[16 * h + 8 + 2 * p + 1] = 0.f;
        }
      }
    }
    tmem_st32(taddr + (uint32_t)(32 * g), o);
  }
}

// the 8 channels (16-byte chunks 2ks, 2ks+1 of the 64-byte pixel row) of the four patch pixels of one halo row
// (TMA SWIZZLE_64B: chunk j of a pixel row sits at j ^ address bits [7,9)).  Even and odd pixels live in separate
// regions, so consecutive lanes (tiles) read consecutive 64-byte rows: the 8-lane phases of each 128-bit load
// hit 8 different bank groups (with interleaved pixels, tiles two pixels apart conflicted 2-way).
__device__ __forceinline__ void load_row(uint32_t hb, uint32_t oe, uint32_t oo, int ks, bool valid,
                                         uint64_t (&d)[4][4]) {
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const uint32_t off = ((b & 1) ? oo : oe) + (uint32_t)(64 * (b >> 1));  // pixel 2*bw + b
    const uint32_t sw = (off >> 7) & 3u;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t j = (uint32_t)(2 * ks + h);
      uint64_t lo = 0, hi = 0;
      if (valid) asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "r"(hb + off + ((j ^ sw) << 4)));
      d[b][2 * h] = lo;
      d[b][2 * h + 1] = hi;
    }
  }
}

// ---- one K=8 step of the fused Winograd MMAs (wino_fused.cu): 8 coordinates c (accumulator d0 + 32c, A hi at
// a0 + 16c and lo at a0 + 16c + 8 in TMEM, B = U_c at descriptor + 128c (2048 bytes)), issued from ONE asm block
// with a single elect: per-MMA wrappers cost an ELECT / R2UR / VOTEU chain each (~70 cycles per MMA, measured),
// which bounded the N = 32 MMAs.  Coordinate order: rank 0 issues row 1 (4..7) first (its epilogue frees
// those first), rank 1 row 0.
__device__ __forceinline__ void wf_mma_kstep_r0_3x(uint32_t d0, uint32_t a0, uint64_t bh0, uint64_t bl0, uint32_t idesc,
                                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred e, p, t;\n\t.reg .b32 d, ah, al;\n\t.reg .b64 bh, bl;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "setp.eq.u32 t, 0, 0;\n\t"
      "add.u32 d, %0, 128;\n\tadd.u32 ah, %1, 64;\n\tadd.u64 bh, %2, 512;\n\t"
      "add.u32 al, %1, 72;\n\tadd.u64 bl, %3, 512;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [al], bh, %4, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bl, %4, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, t;\n\t"
      "add.u32 d, %0, 160;\n\tadd.u32 ah, %1, 80;\n\tadd.u64 bh, %2, 640;\n\t"
      "add.u32 al, %1, 88;\n\tadd.u64 bl, %3, 640;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [al], bh, %4, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bl, %4, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, t;\n\t"
      "add.u32 d, %0, 192;\n\tadd.u32 ah, %1, 96;\n\tadd.u64 bh, %2, 768;\n\t"
      "add.u32 al, %1, 104;\n\tadd.u64 bl, %3, 768;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [al], bh, %4, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bl, %4, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, t;\n\t"
      "add.u32 d, %0, 224;\n\tadd.u32 ah, %1, 112;\n\tadd.u64 bh, %2, 896;\n\t"
      "add.u32 al, %1, 120;\n\tadd.u64 bl, %3, 896;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [al], bh, %4, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bl, %4, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, t;\n\t"
      "add.u32 d, %0, 0;\n\tadd.u32 ah, %1, 0;\n\tadd.u64 bh, %2, 0;\n\t"
      "add.u32 al, %1, 8;\n\tadd.u64 bl, %3, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [al], bh, %4, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bl, %4, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, t;\n\t"
      "add.u32 d, %0, 32;\n\tadd.u32 ah, %1, 16;\n\tadd.u64 bh, %2, 128;\n\t"
      "add.u32 al, %1, 24;\n\tadd.u64 bl, %3, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [al], bh, %4, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bl, %4, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, t;\n\t"
      "add.u32 d, %0, 64;\n\tadd.u32 ah, %1, 32;\n\tadd.u64 bh, %2, 256;\n\t"
      "add.u32 al, %1, 40;\n\tadd.u64 bl, %3, 256;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [al], bh, %4, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bl, %4, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, t;\n\t"
      "add.u32 d, %0, 96;\n\tadd.u32 ah, %1, 48;\n\tadd.u64 bh, %2, 384;\n\t"
      "add.u32 al, %1, 56;\n\tadd.u64 bl, %3, 384;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [al], bh, %4, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bl, %4, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, t;\n\t"
      "}"
      ::"r"(d0), "r"(a0), "l"(bh0), "l"(bl0), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void wf_mma_kstep_r0_1x(uint32_t d0, uint32_t a0, uint64_t bh0, uint64_t bl0, uint32_t idesc,
                                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred e, p, t;\n\t.reg .b32 d, ah, al;\n\t.reg .b64 bh, bl;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "setp.eq.u32 t, 0, 0;\n\t"
      "add.u32 d, %0, 128;\n\tadd.u32 ah, %1, 64;\n\tadd.u64 bh, %2, 512;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, p;\n\t"
      "add.u32 d, %0, 160;\n\tadd.u32 ah, %1, 80;\n\tadd.u64 bh, %2, 640;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, p;\n\t"
      "add.u32 d, %0, 192;\n\tadd.u32 ah, %1, 96;\n\tadd.u64 bh, %2, 768;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, p;\n\t"
      "add.u32 d, %0, 224;\n\tadd.u32 ah, %1, 112;\n\tadd.u64 bh, %2, 896;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, p;\n\t"
      "add.u32 d, %0, 0;\n\tadd.u32 ah, %1, 0;\n\tadd.u64 bh, %2, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, p;\n\t"
      "add.u32 d, %0, 32;\n\tadd.u32 ah, %1, 16;\n\tadd.u64 bh, %2, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, p;\n\t"
      "add.u32 d, %0, 64;\n\tadd.u32 ah, %1, 32;\n\tadd.u64 bh, %2, 256;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, p;\n\t"
      "add.u32 d, %0, 96;\n\tadd.u32 ah, %1, 48;\n\tadd.u64 bh, %2, 384;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, p;\n\t"
      "}"
      ::"r"(d0), "r"(a0), "l"(bh0), "l"(bl0), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void wf_mma_kstep_r1_3x(uint32_t d0, uint32_t a0, uint64_t bh0, uint64_t bl0, uint32_t idesc,
                                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred e, p, t;\n\t.reg .b32 d, ah, al;\n\t.reg .b64 bh, bl;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "setp.eq.u32 t, 0, 0;\n\t"
      "add.u32 d, %0, 0;\n\tadd.u32 ah, %1, 0;\n\tadd.u64 bh, %2, 0;\n\t"
      "add.u32 al, %1, 8;\n\tadd.u64 bl, %3, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [al], bh, %4, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bl, %4, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, t;\n\t"
      "add.u32 d, %0, 32;\n\tadd.u32 ah, %1, 16;\n\tadd.u64 bh, %2, 128;\n\t"
      "add.u32 al, %1, 24;\n\tadd.u64 bl, %3, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [al], bh, %4, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bl, %4, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, t;\n\t"
      "add.u32 d, %0, 64;\n\tadd.u32 ah, %1, 32;\n\tadd.u64 bh, %2, 256;\n\t"
      "add.u32 al, %1, 40;\n\tadd.u64 bl, %3, 256;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [al], bh, %4, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bl, %4, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, t;\n\t"
      "add.u32 d, %0, 96;\n\tadd.u32 ah, %1, 48;\n\tadd.u64 bh, %2, 384;\n\t"
      "add.u32 al, %1, 56;\n\tadd.u64 bl, %3, 384;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [al], bh, %4, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bl, %4, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, t;\n\t"
      "add.u32 d, %0, 128;\n\tadd.u32 ah, %1, 64;\n\tadd.u64 bh, %2, 512;\n\t"
      "add.u32 al, %1, 72;\n\tadd.u64 bl, %3, 512;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [al], bh, %4, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bl, %4, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, t;\n\t"
      "add.u32 d, %0, 160;\n\tadd.u32 ah, %1, 80;\n\tadd.u64 bh, %2, 640;\n\t"
      "add.u32 al, %1, 88;\n\tadd.u64 bl, %3, 640;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [al], bh, %4, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bl, %4, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, t;\n\t"
      "add.u32 d, %0, 192;\n\tadd.u32 ah, %1, 96;\n\tadd.u64 bh, %2, 768;\n\t"
      "add.u32 al, %1, 104;\n\tadd.u64 bl, %3, 768;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [al], bh, %4, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bl, %4, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, t;\n\t"
      "add.u32 d, %0, 224;\n\tadd.u32 ah, %1, 112;\n\tadd.u64 bh, %2, 896;\n\t"
      "add.u32 al, %1, 120;\n\tadd.u64 bl, %3, 896;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [al], bh, %4, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bl, %4, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, t;\n\t"
      "}"
      ::"r"(d0), "r"(a0), "l"(bh0), "l"(bl0), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void wf_mma_kstep_r1_1x(uint32_t d0, uint32_t a0, uint64_t bh0, uint64_t bl0, uint32_t idesc,
                                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred e, p, t;\n\t.reg .b32 d, ah, al;\n\t.reg .b64 bh, bl;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "setp.eq.u32 t, 0, 0;\n\t"
      "add.u32 d, %0, 0;\n\tadd.u32 ah, %1, 0;\n\tadd.u64 bh, %2, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, p;\n\t"
      "add.u32 d, %0, 32;\n\tadd.u32 ah, %1, 16;\n\tadd.u64 bh, %2, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, p;\n\t"
      "add.u32 d, %0, 64;\n\tadd.u32 ah, %1, 32;\n\tadd.u64 bh, %2, 256;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, p;\n\t"
      "add.u32 d, %0, 96;\n\tadd.u32 ah, %1, 48;\n\tadd.u64 bh, %2, 384;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, p;\n\t"
      "add.u32 d, %0, 128;\n\tadd.u32 ah, %1, 64;\n\tadd.u64 bh, %2, 512;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, p;\n\t"
      "add.u32 d, %0, 160;\n\tadd.u32 ah, %1, 80;\n\tadd.u64 bh, %2, 640;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, p;\n\t"
      "add.u32 d, %0, 192;\n\tadd.u32 ah, %1, 96;\n\tadd.u64 bh, %2, 768;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, p;\n\t"
      "add.u32 d, %0, 224;\n\tadd.u32 ah, %1, 112;\n\tadd.u64 bh, %2, 896;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah], bh, %4, p;\n\t"
      "}"
      ::"r"(d0), "r"(a0), "l"(bh0), "l"(bl0), "r"(idesc), "r"(accumulate)
      : "memory");
}

// ---------------------------------------------------------------- input transform (warps 0-7)
// Two groups of four warps; group g transforms K step g (channels 8g .. 8g+7) of every 16-channel stage into
// TMEM slot g, so one group computes while the MMAs consume the other's slot.
// Thread = tile = TMEM lane.  Rank R computes coordinate rows k = 2R, 2R+1 from patch rows R .. R+2:
//   R = 0: t0 = d0 - d2, t1 = d1 + d2   (shared row d2, first d0, second d1)
//   R = 1: t2 = d2 - d1, t3 = d1 - d3   (shared row d1, first d2, second d3)
// (the expressions of the unfused input transform, winograd.cu bt2, so both paths form identical V).
template <int R, bool THREE_X>
__device__ __forceinline__ void transform_role(const WFArgs& a, uint8_t* halo0, uint64_t* full, uint64_t* v_empty,
                                               uint64_t* v_full, uint64_t* h_empty, uint32_t tmem, int my_units) {
  const int g = threadIdx.x >> 7, l = threadIdx.x & 127, warp = l >> 5;
  const int S = a.S;
  const bool valid = l < a.NB * a.BH * a.BW;
  int nb = 0, bh = 0, bw = 0;
  if (valid) {
    nb = l / (a.BH * a.BW);
    bh = (l / a.BW) % a.BH;
    bw = l % a.BW;
  }
  // halo byte offsets of the four pixels of patch row pa: halo row hh = 2*bh + pa lies in half hh / HH2
  // (each half 1024-aligned, so the swizzle phase is a function of the offset within the stage)
  auto row_offset = [&](int pa, int par) {  // pixel 2*bw + par of patch row pa (region (half, par), row-major)
    const int hh = 2 * bh + pa;
    const int half = hh / a.HH2, hr = hh - half * a.HH2;
    return (uint32_t)(2 * half + par) * a.q_bytes + (uint32_t)(((nb * a.HH2 + hr) * (a.BW + 1) + bw) * 64);
  };
  const uint32_t o_she = row_offset(R == 0 ? 2 : 1, 0), o_sho = row_offset(R == 0 ? 2 : 1, 1);
  const uint32_t o_fe = row_offset(R == 0 ? 0 : 2, 0), o_fo = row_offset(R == 0 ? 0 : 2, 1);
  const uint32_t o_ge = row_offset(R == 0 ? 1 : 3, 0), o_go = row_offset(R == 0 ? 1 : 3, 1);
  const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16) + V_COL0;
  const uint32_t h_empty_peer = mapa(smem_u32(h_empty), (uint32_t)(R ^ 1));
  uint32_t it = 0;
  const bool pr = threadIdx.x == 0;
  long long t0 = clk();
  const uint32_t ta = lane_base + (uint32_t)g * VS_COLS;
  const int ks = g;
  for (int ui = 0; ui < my_units; ++ui) {
    for (int cs = 0; cs < a.ncs; ++cs, ++it) {
      const int s = (int)(it % (uint32_t)S);
      mbar_wait(&full[s], (it / (uint32_t)S) & 1);
      if (pr) WPROF(0, t0);
      const uint32_t hb = smem_u32(halo0) + (uint32_t)s * a.stage_bytes;
      {
        uint64_t sh[4][4], t[4][4];
        const bool ld = valid && !(a.dbg & 1);
        load_row(hb, o_she, o_sho, ks, ld, sh);
        load_row(hb, o_fe, o_fo, ks, ld, t);
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
          for (int p = 0; p < 4; ++p) t[b][p] = f2sub(t[b][p], sh[b][p]);
        if (pr) WPROF(1, t0);
        if (it > 0) mbar_wait(&v_empty[g], (it - 1) & 1);
        tc_fence_after();
        if (pr) WPROF(2, t0);
        v_row_store<THREE_X>(t, ta);
        load_row(hb, o_ge, o_go, ks, ld, t);
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
          for (int p = 0; p < 4; ++p) t[b][p] = R == 0 ? f2add(t[b][p], sh[b][p]) : f2sub(sh[b][p], t[b][p]);
        v_row_store<THREE_X>(t, ta + 64);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&v_full[g]);
        if (pr) {
          WPROF(3, t0);
          WCOUNT(5);
        }
      }
      // every tile of this stage is transformed: release the halo slot in both CTAs (the peer multicasts
      // into this CTA's copy too)
      named_bar_sync(1 + 2 * g, 128);  // ids 1, 3 (2 is the epilogue's)
      if (l == 0) {
        mbar_arrive(&h_empty[s]);
        mbar_arrive_remote(h_empty_peer + (uint32_t)(s * sizeof(uint64_t)));
      }
      if (pr) WPROF(4, t0);
    }
  }
}

// ---------------------------------------------------------------- epilogue (warps 6-9)
// Partial output rows from A^T rows (1,1,1,0) and (0,1,-1,-1):
//   R = 0 keeps P0[0] = z0 + z1 and sends P0[1] = z1;   R = 1 sends P1[0] = z2 and keeps P1[1] = -z2 - z3.
// Y_R = P0[R] + P1[R] (rank 0's partial first), TMA-stored as output row i = R of every tile.
template <int R>
__device__ __forceinline__ void epilogue_role(const WFArgs& a, uint8_t* recv, uint64_t* tmem_full,
                                              uint64_t* tmem_empty, uint64_t* recv_full, uint64_t* recv_free,
                                              const CUtensorMap* tmY, uint32_t tmem, int cid, int ncl,
                                              int my_units) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3;  // TMEM lane quadrant
  const int l = q * 32 + lane;
  const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
  const uint32_t slot = smem_u32(recv) + (uint32_t)(l * 256);  // rows 2l + j, 128 B each, SWIZZLE_128B
  const uint32_t slot_peer = mapa(slot, (uint32_t)(R ^ 1));
  const uint32_t recv_full_peer = mapa(smem_u32(recv_full), (uint32_t)(R ^ 1));
  const uint32_t recv_free_peer = mapa(smem_u32(recv_free), (uint32_t)(R ^ 1));
  if (l == 0) tma_prefetch(tmY);
  auto chunk_off = [&](int j, int c) {
    const uint32_t row = (uint32_t)(2 * l + j);
    return (uint32_t)(j * 128) + (((uint32_t)c ^ (row & 7u)) << 4);
  };
  const bool pr = l == 0;
  long long t0 = clk();
  for (int ui = 0; ui < my_units; ++ui) {
    const WUnit w = wdecode(a, cid + ui * ncl);
    mbar_wait(tmem_full, ui & 1);
    tc_fence_after();
    if (pr) WPROF(24, t0);
    // the coordinate row whose z is sent first (R = 0: z1 = P0[1]; R = 1: z2 = P1[0]), then the kept partial
    // accumulated onto it from the other row's four accumulators:
    //   R = 0: keep[j] = z1[j] + z0[j]          = ((z1[0] + M00) + M01) + M02,  ((z1[1] + M01) - M02) - M03
    //   R = 1: keep[j] = -z2[j] - z3[j]         = ((-z2[0] - M30) - M31) - M32,  ((-z2[1] - M31) + M32) + M33
    // z_k[0] = (Mk0 + Mk1) + Mk2,  z_k[1] = (Mk1 - Mk2) - Mk3   (A columns (1,1,1,0), (0,1,-1,-1))
    constexpr int KF = R == 0 ? 1 : 0;  // coordinate row (local) read first
    float zp[2][BN];
#pragma unroll
    for (int li = 0; li < 4; ++li) {
      float m[BN];
      tmem_ld32(tl + (uint32_t)((4 * KF + li) * BN), m);
      tc_fence_before();
      mbar_arrive(&tmem_empty[4 * KF + li]);
#pragma unroll
      for (int f = 0; f < BN; ++f) {
        if (li == 0) {
          zp[0][f] = m[f];
        } else if (li == 1) {
          zp[0][f] += m[f];
          zp[1][f] = m[f];
        } else if (li == 2) {
          zp[0][f] += m[f];
          zp[1][f] -= m[f];
        } else {
          zp[1][f] -= m[f];
        }
      }
    }
    if (pr) WPROF(25, t0);
    if (ui > 0) mbar_wait(recv_free, (ui - 1) & 1);  // the peer has stored what we sent before
    if (pr) WPROF(26, t0);
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int c = 0; c < BN / 4; ++c)
        st_async_v4(slot_peer + chunk_off(j, c), zp[j][4 * c], zp[j][4 * c + 1], zp[j][4 * c + 2], zp[j][4 * c + 3],
                    recv_full_peer);
    if (R == 1) {
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int f = 0; f < BN; ++f) zp[j][f] = -zp[j][f];
    }
#pragma unroll
    for (int li = 0; li < 4; ++li) {
      float m[BN];
      tmem_ld32(tl + (uint32_t)((4 * (1 - KF) + li) * BN), m);
      tc_fence_before();
      mbar_arrive(&tmem_empty[4 * (1 - KF) + li]);
      // R = 0 adds z0 (signs +), R = 1 subtracts z3 (signs -)
      constexpr float sg = R == 0 ? 1.f : -1.f;
#pragma unroll
      for (int f = 0; f < BN; ++f) {
        if (li == 0) {
          zp[0][f] += sg * m[f];
        } else if (li == 1) {
          zp[0][f] += sg * m[f];
          zp[1][f] += sg * m[f];
        } else if (li == 2) {
          zp[0][f] += sg * m[f];
          zp[1][f] -= sg * m[f];
        } else {
          zp[1][f] -= sg * m[f];
        }
      }
    }
    if (pr) WPROF(27, t0);
    mbar_wait(recv_full, ui & 1);
    if (pr) WPROF(28, t0);
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int c = 0; c < BN / 4; ++c) {
        const uint32_t o = slot + chunk_off(j, c);
        const float4 r = lds128(o);
        const float* k = &zp[j][4 * c];
        const float4 y = R == 0 ? make_float4(k[0] + r.x, k[1] + r.y, k[2] + r.z, k[3] + r.w)
                                : make_float4(r.x + k[0], r.y + k[1], r.z + k[2], r.w + k[3]);
        sts128(o, y);
      }
    fence_proxy_async_smem();
    named_bar_sync(2, 128);
    if (l == 0) {
      // output row i = R of every tile: box {32 f, 2*BW w, BH tile rows, NB images} of the parity-R view
      tma_store_4d(tmY, smem_u32(recv), w.f0, 2 * w.tw0, w.th0, w.n0);
      bulk_commit();
      bulk_wait_read<0>();
      mbar_arrive_expect_tx(recv_full, RECV_BYTES);  // next phase: the peer's next partial row
      mbar_arrive_remote(recv_free_peer);  // the peer may overwrite our buffer
    }
    if (pr) {
      WPROF(29, t0);
      WCOUNT(30);
    }
  }
  if (l == 0) bulk_wait<0>();
}

template <bool THREE_X>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NTHREADS, 1)
    wino_fused_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmUh,
                      const __grid_constant__ CUtensorMap tmUl, const __grid_constant__ CUtensorMap tmY0,
                      const __grid_constant__ CUtensorMap tmY1, const __grid_constant__ WFArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = a.S;
  auto halo = [&](int s) { return smem + (size_t)s * a.stage_bytes; };
  auto u_hi = [&](int s) { return halo(s) + 4 * a.q_bytes; };
  auto u_lo = [&](int s) { return u_hi(s) + U_BYTES; };
  uint8_t* recv = smem + (size_t)S * a.stage_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(recv + RECV_BYTES);
  uint64_t* h_empty = full + MAXS;     // halo slot consumed by both transform groups of BOTH CTAs (count 4)
  uint64_t* u_empty = h_empty + MAXS;  // U slot read by this CTA's MMAs
  uint64_t* v_full = u_empty + MAXS;   // TMEM V slot written (128 transform threads)
  uint64_t* v_empty = v_full + NVS;    // TMEM V slot read by the MMAs
  uint64_t* tmem_full = v_empty + NVS;
  uint64_t* tmem_empty = tmem_full + 1;     // per coordinate: accumulator read by the epilogue
  uint64_t* recv_full = tmem_empty + NCO;   // the peer's partial row landed (st.async bytes)
  uint64_t* recv_free = recv_full + 1;      // the peer has consumed what this CTA sent it
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(recv_free + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int cid = (int)cluster_id_x(), ncl = (int)nclusters_x();
  pdl_trigger();
  if (threadIdx.x == 0 && a.trace && blockIdx.x < 148) a.trace[blockIdx.x * 8 + 0] = globaltimer_ns();

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&h_empty[s], 4);  // 2 transform groups x 2 CTAs
      mbar_init(&u_empty[s], 1);
    }
    for (int v = 0; v < NVS; ++v) {
      mbar_init(&v_full[v], 128);
      mbar_init(&v_empty[v], 1);
    }
    mbar_init(tmem_full, 1);
    for (int c = 0; c < NCO; ++c) mbar_init(&tmem_empty[c], 128);
    mbar_init(recv_full, 1);
    mbar_init(recv_free, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(recv_full, RECV_BYTES);  // phase 0: the peer's first partial row
  }
  if (warp == 8 && lane == 0) {
    tma_prefetch(&tmX);
    tma_prefetch(&tmUh);
    if (THREE_X) tma_prefetch(&tmUl);
  }
  if (warp == 9) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // first global-memory access below
  if (threadIdx.x == 0 && a.trace && blockIdx.x < 148) a.trace[blockIdx.x * 8 + 1] = globaltimer_ns();
  const int my_units = cid < a.units ? (a.units - cid + ncl - 1) / ncl : 0;

  if (warp == 8) {
    // ============================ TMA producer ============================
    if (lane == 0) {
      const uint32_t tx = ((a.dbg & 8) ? 0 : 4 * a.box_bytes) + ((a.dbg & 4) ? 0 : (THREE_X ? 2 : 1) * U_BYTES);
      uint32_t it = 0;
      long long t0 = clk();
      for (int ui = 0; ui < my_units; ++ui) {
        const WUnit w = wdecode(a, cid + ui * ncl);
        for (int cs = 0; cs < a.ncs; ++cs, ++it) {
          const int s = (int)(it % (uint32_t)S);
          const uint32_t ph = it / (uint32_t)S;
          if (ph > 0) {
            mbar_wait(&h_empty[s], (ph - 1) & 1);  // both CTAs' copies of the halo slot are free
            WPROF(16, t0);
            mbar_wait(&u_empty[s], (ph - 1) & 1);
            WPROF(17, t0);
          }
          mbar_arrive_expect_tx(&full[s], tx);
          // this CTA's half of the halo rows, into both CTAs (rows [r*HH2, (r+1)*HH2) of the 2*HH2-row box)
          if (!(a.dbg & 8))
            for (int par = 0; par < 2; ++par)
              tma_load_4d_mc(&tmX, &full[s], smem_u32(halo(s)) + (2 * rank + par) * a.q_bytes, cs * CH,
                             2 * w.tw0 - a.PL + par, 2 * w.th0 - a.PT + (int)rank * a.HH2, w.n0, (uint16_t)0x3);
          if (!(a.dbg & 4)) {
            tma_load_3d(&tmUh, &full[s], smem_u32(u_hi(s)), cs * CH, w.f0, NCO * (int)rank);
            if (THREE_X) tma_load_3d(&tmUl, &full[s], smem_u32(u_lo(s)), cs * CH, w.f0, NCO * (int)rank);
          }
          WPROF(18, t0);
          WCOUNT(19);
        }
      }
    }
  } else if (warp == 9) {
    // ============================ MMA issuer (whole warp, converged) ============================
    constexpr uint32_t idesc = idesc_tf32(128, BN);
    uint32_t it = 0;
    const bool pr = lane == 0;
    long long t0 = clk();
    for (int ui = 0; ui < my_units; ++ui) {
      for (int cs = 0; cs < a.ncs; ++cs, ++it) {
        const int s = (int)(it % (uint32_t)S);
        mbar_wait(&full[s], (it / (uint32_t)S) & 1);
        tc_fence_after();
        if (pr) WPROF(8, t0);
        const uint32_t ubh = smem_u32(u_hi(s)), ubl = smem_u32(u_lo(s));
#pragma unroll
        for (int ks = 0; ks < CH / 8; ++ks) {
          const int vs = ks;  // transform group ks's slot, written once per stage
          mbar_wait(&v_full[vs], it & 1);
          tc_fence_after();
          if (pr) WPROF(9, t0);
          const uint32_t va = tmem + V_COL0 + (uint32_t)vs * VS_COLS;
          const uint32_t acc = (cs > 0 || ks > 0) ? 1u : 0u;
          if (ui > 0 && cs == 0 && ks == 0) {  // the epilogue has read the previous unit's accumulators
            if (pr) WPROF(10, t0);
            for (int c = 0; c < NCO; ++c) mbar_wait(&tmem_empty[c], (ui - 1) & 1);
            tc_fence_after();
            if (pr) WPROF(11, t0);
          }
          // U for coordinate c: 32 K-major rows of 64 bytes (SWIZZLE_64B, 8-row groups 512 B apart) at + 2048 c;
          // K step ks = +32 bytes inside the row
          const uint64_t bh = umma_desc_sw64_kmajor_sbo(ubh, 512) + (uint64_t)(2 * ks);
          const uint64_t bl = umma_desc_sw64_kmajor_sbo(ubl, 512) + (uint64_t)(2 * ks);
          if (!(a.dbg & 2)) {
            if (rank == 0) {
              if (THREE_X) wf_mma_kstep_r0_3x(tmem, va, bh, bl, idesc, acc);
              else wf_mma_kstep_r0_1x(tmem, va, bh, bl, idesc, acc);
            } else {
              if (THREE_X) wf_mma_kstep_r1_3x(tmem, va, bh, bl, idesc, acc);
              else wf_mma_kstep_r1_1x(tmem, va, bh, bl, idesc, acc);
            }
          }
          mma_commit_warp(&v_empty[vs]);
          if (pr) {
            WPROF(10, t0);
            WCOUNT(12);
          }
        }
        mma_commit_warp(&u_empty[s]);
      }
      mma_commit_warp(tmem_full);
    }
    __syncwarp();
  } else if (warp < 8) {
    if (rank == 0)
      transform_role<0, THREE_X>(a, halo(0), full, v_empty, v_full, h_empty, tmem, my_units);
    else
      transform_role<1, THREE_X>(a, halo(0), full, v_empty, v_full, h_empty, tmem, my_units);
  } else {
    const CUtensorMap* tmY = rank == 0 ? &tmY0 : &tmY1;
    if (rank == 0)
      epilogue_role<0>(a, recv, tmem_full, tmem_empty, recv_full, recv_free, tmY, tmem, cid, ncl, my_units);
    else
      epilogue_role<1>(a, recv, tmem_full, tmem_empty, recv_full, recv_free, tmY, tmem, cid, ncl, my_units);
  }

  tc_fence_before();
  cluster_sync();  // no CTA leaves while its peer may still touch its shared memory
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
  if (threadIdx.x == 0 && a.trace && blockIdx.x < 148) a.trace[blockIdx.x * 8 + 7] = globaltimer_ns();
}

struct WFPlan {
  bool ok = false;
  bool three_x = false;
  WFArgs a{};
  int64_t cpad = 0, fpad = 0;
  size_t smem = 0, ut_bytes = 0;
};

WFPlan wf_plan(const Problem& p) {
  WFPlan w;
  if (!(p.KH == 3 && p.KW == 3 && p.SH == 1 && p.SW == 1 && p.C >= 32 && p.C % 4 == 0 && p.F % 4 == 0 &&
        p.HO >= 2))
    return w;
  w.three_x = p.math == CONV2D_MATH_FP32;
  const int tht = (p.HO + 1) / 2, twt = (p.WO + 1) / 2;
  const uint32_t ub = (w.three_x ? 2u : 1u) * U_BYTES;
  double best = 1e300;
  // tile block: fewest 128-lane units first (each runs the full MMA work), then the least halo traffic
  for (int bw = 1; bw <= std::min(twt, 63); ++bw)
    for (int bh = 1; bh <= std::min(tht, 128 / bw); ++bh) {
      const bool whole = bh >= tht && bw >= twt;
      const int nb = whole ? std::max(1, std::min(p.N, 128 / (bh * bw))) : 1;
      const int hwb = 2 * bw + 2, hh2 = bh + 1;
      const uint32_t box = (uint32_t)(bw + 1) * hh2 * nb * 64;  // one (half, parity) box
      const uint32_t qb = (box + 1023) / 1024 * 1024;
      const int S = std::min<int>(MAXS, (int)((SMEM_LIMIT - 1024 - RECV_BYTES - BAR_BYTES) / (4 * qb + ub)));
      if (S < 2) continue;
      const int64_t blocks = (int64_t)((p.N + nb - 1) / nb) * ((tht + bh - 1) / bh) * ((twt + bw - 1) / bw);
      const double cost = (double)blocks * (1.0 + 4.0 * box / 64.0 / 1700.0);
      if (cost < best) {
        best = cost;
        w.a.NB = nb;
        w.a.BH = bh;
        w.a.BW = bw;
        w.a.HWB = hwb;
        w.a.HH2 = hh2;
        w.a.S = S;
        w.a.box_bytes = box;
        w.a.q_bytes = qb;
        w.a.stage_bytes = 4 * qb + ub;
        w.a.blocks_w = (twt + bw - 1) / bw;
        w.a.blocks_h = (tht + bh - 1) / bh;
      }
    }
  if (best >= 1e299) return w;
  const int64_t blocks_n = (p.N + w.a.NB - 1) / w.a.NB;
  w.a.nfb = (p.F + BN - 1) / BN;
  const int64_t units = blocks_n * w.a.blocks_h * w.a.blocks_w * w.a.nfb;
  if (units >= (int64_t(1) << 31)) return w;
  w.a.units = (int)units;
  w.cpad = (p.C + 31) / 32 * 32;
  w.fpad = (p.F + BN - 1) / BN * BN;
  w.a.ncs = (int)(w.cpad / CH);
  w.a.HO = p.HO;
  w.a.WO = p.WO;
  w.a.PT = p.pad_top;
  w.a.PL = p.pad_left;
  w.smem = (size_t)w.a.S * w.a.stage_bytes + RECV_BYTES + BAR_BYTES + 1024;
  w.ut_bytes = (size_t)((16 * w.fpad * w.cpad * 4 + 255) / 256 * 256);
  w.ok = true;
  return w;
}

template <bool THREE_X>
int max_clusters(size_t smem) {  // co-resident clusters of 2 at this footprint (1 CTA per SM), per device
  static std::mutex mu;
  static std::map<int, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * 74);
  cfg.blockDim = dim3(NTHREADS);
  cfg.dynamicSmemBytes = smem;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, wino_fused_kernel<THREE_X>, &cfg) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    n = 74;
  }
  cache[dev] = n;
  return n;
}

}  // namespace

bool wino_fused_ok(const Problem& p) { return wf_plan(p).ok; }

size_t wino_fused_workspace(const Problem& p) {
  const WFPlan w = wf_plan(p);
  return w.ok ? w.ut_bytes * (w.three_x ? 2 : 1) : 0;
}

cudaError_t launch_wino_fused(const Problem& p, const float* in, const float* filt, float* out, void* ws,
                              cudaStream_t s) {
  WFPlan w = wf_plan(p);
  if (!w.ok) return cudaErrorInvalidValue;
  float* ut_hi = static_cast<float*>(ws);
  float* ut_lo = w.three_x ? reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + w.ut_bytes) : nullptr;
  cudaError_t e = launch_wino_filter(2, filt, p.C, p.F, w.cpad, w.fpad, ut_hi, ut_lo, w.three_x, s);
  if (e != cudaSuccess) return e;
  alignas(64) CUtensorMap tx{}, tuh{}, tul{}, ty0{}, ty1{};
  {  // input halo boxes {16 ch, HWB w (every other pixel), HH2 h, NB n} over NHWC, SWIZZLE_64B (load_row);
     // OOB (padding) -> 0
    const uint64_t dims[4] = {(uint64_t)p.C, (uint64_t)p.W, (uint64_t)p.H, (uint64_t)p.N};
    const uint64_t st[3] = {(uint64_t)p.C * 4, (uint64_t)p.W * p.C * 4, (uint64_t)p.H * p.W * p.C * 4};
    const uint32_t box[4] = {(uint32_t)CH, (uint32_t)w.a.HWB, (uint32_t)w.a.HH2, (uint32_t)w.a.NB};
    const uint32_t es[4] = {1, 2, 1, 1};
    if (!gemm2_encode_tiled_es(&tx, 4, in, dims, st, box, es, (int)CU_TENSOR_MAP_SWIZZLE_64B))
      return cudaErrorInvalidValue;
  }
  {  // Ut[xi][fpad][cpad]: boxes {16 c, 32 f, 8 coordinates}
    const uint64_t dims[3] = {(uint64_t)w.cpad, (uint64_t)w.fpad, 16};
    const uint64_t st[2] = {(uint64_t)w.cpad * 4, (uint64_t)w.fpad * w.cpad * 4};
    const uint32_t box[3] = {(uint32_t)CH, (uint32_t)BN, (uint32_t)NCO};
    if (!gemm2_encode_tiled_sw(&tuh, 3, ut_hi, dims, st, box, (int)CU_TENSOR_MAP_SWIZZLE_64B))
      return cudaErrorInvalidValue;
    if (w.three_x) {
      if (!gemm2_encode_tiled_sw(&tul, 3, ut_lo, dims, st, box, (int)CU_TENSOR_MAP_SWIZZLE_64B))
        return cudaErrorInvalidValue;
    } else {
      tul = tuh;
    }
  }
  for (int r = 0; r < 2; ++r) {  // output rows of parity r: {F, WO, ceil((HO - r) / 2), N}, rows 2 apart
    const uint64_t dims[4] = {(uint64_t)p.F, (uint64_t)p.WO, (uint64_t)((p.HO - r + 1) / 2), (uint64_t)p.N};
    const uint64_t st[3] = {(uint64_t)p.F * 4, (uint64_t)p.F * 4 * p.WO * 2, (uint64_t)p.F * 4 * p.WO * p.HO};
    const uint32_t box[4] = {(uint32_t)BN, (uint32_t)(2 * w.a.BW), (uint32_t)w.a.BH, (uint32_t)w.a.NB};
    if (!gemm2_encode_tiled_sw(r ? &ty1 : &ty0, 4, out + (size_t)r * p.WO * p.F, dims, st, box,
                               (int)CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  }
  w.a.trace = gemm2_trace_record();
  static const int dbg = getenv("CONV2D_WF_DEBUG") ? atoi(getenv("CONV2D_WF_DEBUG")) : 0;
  w.a.dbg = dbg;
  auto kern = w.three_x ? wino_fused_kernel<true> : wino_fused_kernel<false>;
  e = w.three_x ? smem_attr_once<wino_fused_kernel<true>>(SMEM_LIMIT)
                : smem_attr_once<wino_fused_kernel<false>>(SMEM_LIMIT);
  if (e != cudaSuccess) return e;
  const int maxc = w.three_x ? max_clusters<true>(SMEM_LIMIT) : max_clusters<false>(SMEM_LIMIT);
  const int ncl = std::max(1, std::min(w.a.units, maxc));
  static const bool prof = getenv("CONV2D_WF_PROF") != nullptr;  // diagnostics: synchronous, prints to stderr
  static unsigned long long* prof_buf = nullptr;
  if (prof) {
    if (!prof_buf && cudaMalloc(&prof_buf, 64 * sizeof(unsigned long long)) != cudaSuccess) prof_buf = nullptr;
    if (prof_buf) cudaMemsetAsync(prof_buf, 0, 64 * sizeof(unsigned long long), s);
    w.a.prof = prof_buf;
  }
  e = launch_k(kern, dim3((unsigned)(2 * ncl)), dim3(NTHREADS), w.smem, s, tx, tuh, tul, ty0, ty1, w.a);
  if (e == cudaSuccess && prof && prof_buf) {
    unsigned long long h[64];
    cudaStreamSynchronize(s);
    cudaMemcpy(h, prof_buf, sizeof(h), cudaMemcpyDeviceToHost);
    for (int c = 0; c < 2; ++c) {
      const unsigned long long* q = h + 32 * c;
      const double nk = q[5] ? (double)q[5] : 1.0, nm = q[12] ? (double)q[12] : 1.0, np = q[19] ? (double)q[19] : 1.0,
                   nu = q[30] ? (double)q[30] : 1.0;
      fprintf(stderr,
              "[wf prof cta %d] units %d ncs %d S %d | transform/kstep: full %.0f ldmath %.0f vempty %.0f store %.0f "
              "stagebar %.0f (n %llu) | mma/kstep: full %.0f vfull %.0f issue %.0f tmem_empty %.0f (n %llu) | "
              "producer/stage: hempty %.0f uempty %.0f issue %.0f (n %llu) | epi/unit: tmemfull %.0f drain %.0f "
              "recvfree %.0f send %.0f recvfull %.0f store %.0f (n %llu)\n",
              c, w.a.units, w.a.ncs, w.a.S, q[0] / nk, q[1] / nk, q[2] / nk, q[3] / nk, q[4] / nk, q[5], q[8] / nm,
              q[9] / nm, q[10] / nm, q[11] / nm, q[12], q[16] / np, q[17] / np, q[18] / np, q[19], q[24] / nu,
              q[25] / nu, q[26] / nu, q[27] / nu, q[28] / nu, q[29] / nu, q[30]);
    }
  }
  return e;
}

}  // namespace conv2d
