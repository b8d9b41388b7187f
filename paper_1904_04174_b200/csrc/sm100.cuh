// sm100.cuh -- thin inline-PTX wrappers for the Blackwell (sm_100a) features the
// tensor-core kernels use: mbarriers, cp.async, async-proxy fences, tcgen05
// (TMEM alloc / MMA / commit / ld) and UMMA shared-memory + instruction descriptors.
//
// Descriptor bit layouts follow the PTX ISA "tcgen05 matrix descriptors" and
// "instruction descriptor" tables (kind::tf32):
//   smem desc: [0,14) start>>4 | [16,30) LBO>>4 | [32,46) SBO>>4 | [46,48) version=1 |
//              [49,52) base offset | [52] LBO mode | [61,64) layout (2 = SWIZZLE_128B)
//   idesc    : [4,6) D fmt (1=f32) | [7,10) A fmt (2=tf32) | [10,13) B fmt (2=tf32) |
//              [15] A major | [16] B major (0=K) | [17,23) N>>3 | [24,29) M>>4
#pragma once
#include <cstdint>

namespace sm100 {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ------------------------------------------------------------------ mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// ------------------------------------------------------------------ cp.async (LDGSTS)
// 16-byte global->shared copy; src_bytes = 0 zero-fills the destination (padding / tails).
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// generic-proxy smem writes -> visible to the async proxy (tcgen05.mma operand reads)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ------------------------------------------------------------------ tcgen05 / TMEM
template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem) {  // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {  // whole warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, both K-major, kind::tf32, issued by ONE thread.
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive on an mbarrier when all previously issued tcgen05.mma of this thread complete.
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// 32 lanes x 32 columns of 32-bit: thread i of the warp gets lane (base+i), columns [col, col+32)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// ------------------------------------------------------------------ descriptors
// K-major operand tile, rows of 128 bytes (32 fp32), SWIZZLE_128B, 8-row atoms 1024 B apart.
__device__ __forceinline__ uint64_t umma_desc_sw128_kmajor(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;             // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024u >> 4) << 32;   // SBO: 8 rows * 128 B
  d |= (uint64_t)1u << 46;             // version = 1 (sm_100)
  d |= (uint64_t)2u << 61;             // SWIZZLE_128B
  return d;
}

// MN-major tf32 operand (e.g. B read straight from a row-major K x N matrix).  For 32-bit MN-major
// operands the only smem layout is SWIZZLE_128B_BASE32B (descriptor layout type 1; TMA's
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B): 128-byte rows = one k each, 32 consecutive n; 32-byte chunks
// swizzled over a 4-row (512 B) atom.  LBO = byte stride between 32-wide n chunks, SBO = byte stride
// between 4-row k groups.
__device__ __forceinline__ uint64_t umma_desc_sw128b32_mn(uint32_t smem_addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;  // version = 1 (sm_100)
  d |= (uint64_t)1u << 61;  // SWIZZLE_128B_BASE32B
  return d;
}
constexpr uint32_t IDESC_B_MN = 1u << 16;  // instruction descriptor: B operand MN-major

__host__ __device__ constexpr uint32_t idesc_tf32(uint32_t M, uint32_t N) {
  return (1u << 4)            // D = f32
         | (2u << 7)          // A = tf32
         | (2u << 10)         // B = tf32
         | ((N >> 3) << 17)   // N
         | ((M >> 4) << 24);  // M
}

// byte offset of 16-byte chunk j of row r inside a SWIZZLE_128B K-major tile (1024 B aligned)
__host__ __device__ __forceinline__ uint32_t sw128_offset(uint32_t r, uint32_t j) {
  return r * 128u + ((j ^ (r & 7u)) << 4);
}

// TF32 split: hi = fp32 with the low 13 mantissa bits cleared (what the tensor core reads),
// lo = x - hi (exact in fp32).
__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

}  // namespace sm100

// ====================================================================== cluster / 2-CTA extensions
namespace sm100 {

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t nclusters_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
// shared::cta address of this CTA -> shared::cluster address of the same offset in CTA `rank`
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// arrive (release, cluster scope) on an mbarrier given by its shared::cluster address
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait_cluster(bar, parity)) {
  }
}
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---- TMA (tensor maps are __grid_constant__ kernel parameters)
__device__ __forceinline__ void tma_prefetch(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}
__device__ __forceinline__ void tma_load_3d(const void* tmap, uint64_t* bar, uint32_t dst, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// plain (non-tensor) bulk copy global -> own smem, completing on an mbarrier (16-byte aligned, size % 16 == 0)
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tma_load_im2col_4d(const void* tmap, uint64_t* bar, uint32_t dst, int c, int w, int h,
                                                   int n, uint16_t off_w, uint16_t off_h) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, "
      "%6}], [%2], {%7, %8};" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c), "r"(w), "r"(h), "r"(n), "h"(off_w),
      "h"(off_h)
      : "memory");
}

// ---- 2-CTA tcgen05
template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_alloc_2sm(uint32_t* dst_smem) {  // one warp in EACH CTA of the pair
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_dealloc_2sm(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS) : "memory");
}
// issued by ONE thread of the leader CTA: D (both CTAs' TMEM) += A (both CTAs' smem) * B (both halves)
__device__ __forceinline__ void mma_tf32_2sm(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on the mbarrier at the same smem offset in every CTA of `mask` when prior MMAs complete
__device__ __forceinline__ void mma_commit_2sm_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

}  // namespace sm100

namespace sm100 {
// default-semantics remote arrive (what CUTLASS's 2-SM pipelines use; no GPU-scope fence)
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ float lds32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts32(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void sts128(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
// TMA loads whose completion is signalled on an mbarrier of either CTA of the pair (cluster address)
__device__ __forceinline__ void tma_load_3d_2sm(const void* tmap, uint32_t bar_cluster, uint32_t dst, int c0, int c1,
                                                int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_load_im2col_4d_2sm(const void* tmap, uint32_t bar_cluster, uint32_t dst, int c,
                                                       int w, int h, int n, uint16_t off_w, uint16_t off_h) {
  asm volatile(
      "cp.async.bulk.tensor.4d.im2col.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
      "{%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar_cluster), "r"(c), "r"(w), "r"(h), "r"(n), "h"(off_w),
      "h"(off_h)
      : "memory");
}
}  // namespace sm100

namespace sm100 {
// ---- TMA bulk tensor store (smem -> global), bulk async-groups
__device__ __forceinline__ void tma_store_3d(const void* tmap, uint32_t src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(tmap)),
               "r"(src), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
}  // namespace sm100

namespace sm100 {
// K-major operand tile in the no-swizzle ("interleave") canonical layout: core matrices of
// 8 rows x 16 B (128 B contiguous); lbo = byte stride between core matrices along K,
// sbo = byte stride between 8-row groups along M/N.
__device__ __forceinline__ uint64_t umma_desc_interleave_kmajor(uint32_t smem_addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;  // version = 1 (sm_100); layout type 0 = SWIZZLE_NONE
  return d;
}
}  // namespace sm100

namespace sm100 {
__device__ __forceinline__ void tma_load_5d(const void* tmap, uint64_t* bar, uint32_t dst, int c0, int c1, int c2,
                                            int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, "
      "%7}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
__device__ __forceinline__ void tma_load_5d_2sm(const void* tmap, uint32_t bar_cluster, uint32_t dst, int c0, int c1,
                                                int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5, %6, %7}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
__device__ __forceinline__ void tma_store_4d(const void* tmap, uint32_t src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(tmap)),
               "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
}  // namespace sm100

namespace sm100 {
// SWIZZLE_128B K-major tile whose 8-row groups are `sbo` bytes apart and whose start row sits
// `phase` rows into the 1024-byte swizzle period (matrix base offset, bits [49,52)).
// K-major SWIZZLE_64B operand (64-byte rows, 8-row / 512-byte atoms; descriptor layout type 4),
// SBO = byte stride between 8-row groups
__device__ __forceinline__ uint64_t umma_desc_sw64_kmajor_sbo(uint32_t smem_addr, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)4u << 61;
  return d;
}
__device__ __forceinline__ uint64_t umma_desc_sw128_kmajor_sbo(uint32_t smem_addr, uint32_t sbo, uint32_t phase) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)(phase & 7u) << 49;
  d |= (uint64_t)2u << 61;
  return d;
}
__device__ __forceinline__ void tma_load_4d(const void* tmap, uint64_t* bar, uint32_t dst, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, "
      "%6}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
}  // namespace sm100

namespace sm100 {
// Warp-collective variants: call with the WHOLE warp converged and warp-uniform operands; one
// elected lane issues.  Keeping the warp converged lets ptxas hold descriptors in uniform
// registers -- with a `lane == 0` guard it wraps every UTCHMMA in an ELECT/R2UR waterfall loop
// (~10 extra instructions per MMA, which bounds N=64 tiles; profiles/round1_ncu.md).
__device__ __forceinline__ void mma_tf32_2sm_warp(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                                  uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit_2sm_mc_warp(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
}  // namespace sm100

namespace sm100 {
// 32 lanes x 32 columns of 32-bit into TMEM (thread i of the warp -> lane base+i)
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]),
      "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]),
      "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// single-CTA (cta_group::1) forms, warp-collective issue: D[tmem] (+)= A[tmem] * B[smem]
__device__ __forceinline__ void mma_tf32_ts_warp(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                                 uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit_warp(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
// 4-D tiled TMA load multicast to every CTA of `mask`: the box lands at the same smem offset in each, and
// each destination's mbarrier (same offset) receives complete_tx for its copy
__device__ __forceinline__ void tma_load_4d_mc(const void* tmap, uint64_t* bar, uint32_t dst, int c0, int c1, int c2,
                                               int c3, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster [%0], "
      "[%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "h"(mask)
      : "memory");
}
// asynchronous 16-byte store into a peer CTA's shared memory; completion is counted (complete_tx, bytes) on the
// peer's mbarrier.  Both addresses are shared::cluster addresses (mapa).
__device__ __forceinline__ void st_async_v4(uint32_t remote_addr, float a, float b, float c, float d,
                                            uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                   remote_addr),
               "f"(a), "f"(b), "f"(c), "f"(d), "r"(remote_bar)
               : "memory");
}
// A operand from TMEM (this CTA's 128 rows in lanes, K in columns), B from smem; warp-collective issue
__device__ __forceinline__ void mma_tf32_2sm_ts_warp(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                                     uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
}  // namespace sm100

namespace sm100 {
// ---- one 32-wide k-block (four K=8 steps) of cta_group::2 MMAs issued from ONE asm block with a single elect.
// Per-MMA warp-collective wrappers each cost an ELECT / R2UR / VOTEU dependency chain of ~60-70 cycles
// (measured with clock64 in wino_fused.cu); an M=256 x N<=128 x K=8 MMA executes in 32-64 cycles per SM, so
// issue, not the tensor pipe, bounded N <= 128 tiles (R4 halo: tensor pipe 61% active, transform warps
// waiting on the MMA warp, profiles/round2_ncu.md).  Descriptors advance by a_step / b_step (16-byte units)
// per K step; the first MMA of the block accumulates iff acc0, all later ones always do.
__device__ __forceinline__ void mma2_kblock_3x_ss(uint32_t d, uint64_t ah, uint64_t al, uint64_t bh, uint64_t bl,
                                                  uint64_t a_step, uint64_t b_step, uint32_t idesc, uint32_t acc0) {
  asm volatile(
      "{\n\t.reg .pred e, p, t;\n\t.reg .b64 ah, al, bh, bl;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %8, 0;\n\tsetp.eq.u32 t, 0, 0;\n\t"
      "mov.b64 ah, %1;\n\tmov.b64 al, %2;\n\tmov.b64 bh, %3;\n\tmov.b64 bl, %4;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], al, bh, %7, p;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], ah, bl, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], ah, bh, %7, t;\n\t"
      "add.u64 ah, ah, %5;\n\tadd.u64 al, al, %5;\n\tadd.u64 bh, bh, %6;\n\tadd.u64 bl, bl, %6;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], al, bh, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], ah, bl, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], ah, bh, %7, t;\n\t"
      "add.u64 ah, ah, %5;\n\tadd.u64 al, al, %5;\n\tadd.u64 bh, bh, %6;\n\tadd.u64 bl, bl, %6;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], al, bh, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], ah, bl, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], ah, bh, %7, t;\n\t"
      "add.u64 ah, ah, %5;\n\tadd.u64 al, al, %5;\n\tadd.u64 bh, bh, %6;\n\tadd.u64 bl, bl, %6;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], al, bh, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], ah, bl, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], ah, bh, %7, t;\n\t"
      "}" ::"r"(d), "l"(ah), "l"(al), "l"(bh), "l"(bl), "l"(a_step), "l"(b_step), "r"(idesc), "r"(acc0)
      : "memory");
}
__device__ __forceinline__ void mma2_kblock_3x_ts(uint32_t d, uint32_t alo_tmem, uint64_t ah, uint64_t bh, uint64_t bl,
                                                  uint64_t a_step, uint64_t b_step, uint32_t idesc, uint32_t acc0) {
  asm volatile(
      "{\n\t.reg .pred e, p, t;\n\t.reg .b64 ah, bh, bl;\n\t.reg .b32 lt;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %8, 0;\n\tsetp.eq.u32 t, 0, 0;\n\t"
      "mov.b32 lt, %1;\n\tmov.b64 ah, %2;\n\tmov.b64 bh, %3;\n\tmov.b64 bl, %4;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [lt], bh, %7, p;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], ah, bl, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], ah, bh, %7, t;\n\t"
      "add.u32 lt, lt, 8;\n\tadd.u64 ah, ah, %5;\n\tadd.u64 bh, bh, %6;\n\tadd.u64 bl, bl, %6;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [lt], bh, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], ah, bl, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], ah, bh, %7, t;\n\t"
      "add.u32 lt, lt, 8;\n\tadd.u64 ah, ah, %5;\n\tadd.u64 bh, bh, %6;\n\tadd.u64 bl, bl, %6;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [lt], bh, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], ah, bl, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], ah, bh, %7, t;\n\t"
      "add.u32 lt, lt, 8;\n\tadd.u64 ah, ah, %5;\n\tadd.u64 bh, bh, %6;\n\tadd.u64 bl, bl, %6;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [lt], bh, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], ah, bl, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], ah, bh, %7, t;\n\t"
      "}" ::"r"(d), "r"(alo_tmem), "l"(ah), "l"(bh), "l"(bl), "l"(a_step), "l"(b_step), "r"(idesc), "r"(acc0)
      : "memory");
}
__device__ __forceinline__ void mma2_kblock_1x_ss(uint32_t d, uint64_t ah, uint64_t bh, uint64_t a_step,
                                                  uint64_t b_step, uint32_t idesc, uint32_t acc0) {
  asm volatile(
      "{\n\t.reg .pred e, p, t;\n\t.reg .b64 ah, bh;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %6, 0;\n\tsetp.eq.u32 t, 0, 0;\n\t"
      "mov.b64 ah, %1;\n\tmov.b64 bh, %2;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], ah, bh, %5, p;\n\t"
      "add.u64 ah, ah, %3;\n\tadd.u64 bh, bh, %4;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], ah, bh, %5, t;\n\t"
      "add.u64 ah, ah, %3;\n\tadd.u64 bh, bh, %4;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], ah, bh, %5, t;\n\t"
      "add.u64 ah, ah, %3;\n\tadd.u64 bh, bh, %4;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], ah, bh, %5, t;\n\t"
      "}" ::"r"(d), "l"(ah), "l"(bh), "l"(a_step), "l"(b_step), "r"(idesc), "r"(acc0)
      : "memory");
}
// halo kernel, A (hi | lo) from TMEM: hi x [B_hi | B_lo] (N = 2 BN, idesc2, bz) then lo x B_hi (idesc, bx)
__device__ __forceinline__ void mma2_kblock_tt_concat(uint32_t d, uint32_t ahi_tmem, uint32_t alo_tmem, uint64_t bz,
                                                      uint64_t bx, uint32_t idesc2, uint32_t idesc, uint32_t acc0) {
  asm volatile(
      "{\n\t.reg .pred e, p, t;\n\t.reg .b64 bz, bx;\n\t.reg .b32 ah, al;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %7, 0;\n\tsetp.eq.u32 t, 0, 0;\n\t"
      "mov.b32 ah, %1;\n\tmov.b32 al, %2;\n\tmov.b64 bz, %3;\n\tmov.b64 bx, %4;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [ah], bz, %5, p;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [al], bx, %6, t;\n\t"
      "add.u32 ah, ah, 8;\n\tadd.u32 al, al, 8;\n\tadd.u64 bz, bz, 2;\n\tadd.u64 bx, bx, 2;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [ah], bz, %5, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [al], bx, %6, t;\n\t"
      "add.u32 ah, ah, 8;\n\tadd.u32 al, al, 8;\n\tadd.u64 bz, bz, 2;\n\tadd.u64 bx, bx, 2;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [ah], bz, %5, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [al], bx, %6, t;\n\t"
      "add.u32 ah, ah, 8;\n\tadd.u32 al, al, 8;\n\tadd.u64 bz, bz, 2;\n\tadd.u64 bx, bx, 2;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [ah], bz, %5, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [al], bx, %6, t;\n\t"
      "}" ::"r"(d), "r"(ahi_tmem), "r"(alo_tmem), "l"(bz), "l"(bx), "r"(idesc2), "r"(idesc), "r"(acc0)
      : "memory");
}
// halo kernel, A (hi | lo) from TMEM, BN = 128: lo x B_hi, hi x B_lo, hi x B_hi
__device__ __forceinline__ void mma2_kblock_tt_3x(uint32_t d, uint32_t ahi_tmem, uint32_t alo_tmem, uint64_t bx,
                                                  uint64_t bl, uint32_t idesc, uint32_t acc0, uint32_t b_step = 2) {
  const uint64_t bs = b_step;  // descriptor units per K=8 step: 2 (K-major SW128), 64 (MN-major, 1 KB)
  asm volatile(
      "{\n\t.reg .pred e, p, t;\n\t.reg .b64 bx, bl;\n\t.reg .b32 ah, al;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %6, 0;\n\tsetp.eq.u32 t, 0, 0;\n\t"
      "mov.b32 ah, %1;\n\tmov.b32 al, %2;\n\tmov.b64 bx, %3;\n\tmov.b64 bl, %4;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [al], bx, %5, p;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [ah], bl, %5, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [ah], bx, %5, t;\n\t"
      "add.u32 ah, ah, 8;\n\tadd.u32 al, al, 8;\n\tadd.u64 bx, bx, %7;\n\tadd.u64 bl, bl, %7;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [al], bx, %5, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [ah], bl, %5, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [ah], bx, %5, t;\n\t"
      "add.u32 ah, ah, 8;\n\tadd.u32 al, al, 8;\n\tadd.u64 bx, bx, %7;\n\tadd.u64 bl, bl, %7;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [al], bx, %5, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [ah], bl, %5, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [ah], bx, %5, t;\n\t"
      "add.u32 ah, ah, 8;\n\tadd.u32 al, al, 8;\n\tadd.u64 bx, bx, %7;\n\tadd.u64 bl, bl, %7;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [al], bx, %5, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [ah], bl, %5, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [ah], bx, %5, t;\n\t"
      "}" ::"r"(d), "r"(ahi_tmem), "r"(alo_tmem), "l"(bx), "l"(bl), "r"(idesc), "r"(acc0), "l"(bs)
      : "memory");
}
}  // namespace sm100

namespace sm100 {
// halo kernel G3C4 (gemm_halo.cu): a whole tile's six K=8 steps from one asm block (one elect).  Step i
// reads the A view at halo offset {0, 2, 16, 18, 32, 34}[i] (16-byte units: tap row r = i / 2, tap pair
// q = i % 2) and B k-block i / 4 (resident stages: descriptors *0 / *1) at 32 * (i % 4) bytes.  The first
// MMA overwrites the accumulator.
__device__ __forceinline__ void mma2_c4_tile_concat(uint32_t d, uint64_t ah, uint64_t al, uint64_t bz0, uint64_t bz1, uint64_t bx0, uint64_t bx1, uint32_t idesc2,
    uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred e, p, t;\n\t.reg .b64 a, b, c;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, 0, 0;\n\tsetp.eq.u32 t, 0, 0;\n\t"
      "add.u64 a, %1, 0;\n\tadd.u64 b, %3, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, b, %7, p;\n\t"
      "add.u64 a, %2, 0;\n\tadd.u64 c, %5, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, c, %8, t;\n\t"
      "add.u64 a, %1, 2;\n\tadd.u64 b, %3, 2;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, b, %7, t;\n\t"
      "add.u64 a, %2, 2;\n\tadd.u64 c, %5, 2;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, c, %8, t;\n\t"
      "add.u64 a, %1, 16;\n\tadd.u64 b, %3, 4;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, b, %7, t;\n\t"
      "add.u64 a, %2, 16;\n\tadd.u64 c, %5, 4;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, c, %8, t;\n\t"
      "add.u64 a, %1, 18;\n\tadd.u64 b, %3, 6;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, b, %7, t;\n\t"
      "add.u64 a, %2, 18;\n\tadd.u64 c, %5, 6;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, c, %8, t;\n\t"
      "add.u64 a, %1, 32;\n\tadd.u64 b, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, b, %7, t;\n\t"
      "add.u64 a, %2, 32;\n\tadd.u64 c, %6, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, c, %8, t;\n\t"
      "add.u64 a, %1, 34;\n\tadd.u64 b, %4, 2;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, b, %7, t;\n\t"
      "add.u64 a, %2, 34;\n\tadd.u64 c, %6, 2;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, c, %8, t;\n\t"
      "}" ::"r"(d), "l"(ah), "l"(al), "l"(bz0), "l"(bz1), "l"(bx0), "l"(bx1), "r"(idesc2), "r"(idesc)
      : "memory");
}
__device__ __forceinline__ void mma2_c4_tile_3x(uint32_t d, uint64_t ah, uint64_t al, uint64_t bx0, uint64_t bx1, uint64_t bl0, uint64_t bl1,
    uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred e, p, t;\n\t.reg .b64 a, b, c;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, 0, 0;\n\tsetp.eq.u32 t, 0, 0;\n\t"
      "add.u64 a, %2, 0;\n\tadd.u64 b, %3, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, b, %7, p;\n\t"
      "add.u64 a, %1, 0;\n\tadd.u64 c, %5, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, c, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, b, %7, t;\n\t"
      "add.u64 a, %2, 2;\n\tadd.u64 b, %3, 2;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, b, %7, t;\n\t"
      "add.u64 a, %1, 2;\n\tadd.u64 c, %5, 2;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, c, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, b, %7, t;\n\t"
      "add.u64 a, %2, 16;\n\tadd.u64 b, %3, 4;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, b, %7, t;\n\t"
      "add.u64 a, %1, 16;\n\tadd.u64 c, %5, 4;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, c, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, b, %7, t;\n\t"
      "add.u64 a, %2, 18;\n\tadd.u64 b, %3, 6;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, b, %7, t;\n\t"
      "add.u64 a, %1, 18;\n\tadd.u64 c, %5, 6;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, c, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, b, %7, t;\n\t"
      "add.u64 a, %2, 32;\n\tadd.u64 b, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, b, %7, t;\n\t"
      "add.u64 a, %1, 32;\n\tadd.u64 c, %6, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, c, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, b, %7, t;\n\t"
      "add.u64 a, %2, 34;\n\tadd.u64 b, %4, 2;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, b, %7, t;\n\t"
      "add.u64 a, %1, 34;\n\tadd.u64 c, %6, 2;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, c, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, b, %7, t;\n\t"
      "}" ::"r"(d), "l"(ah), "l"(al), "l"(bx0), "l"(bx1), "l"(bl0), "l"(bl1), "r"(idesc)
      : "memory");
}
__device__ __forceinline__ void mma2_c4_tile_1x(uint32_t d, uint64_t ah, uint64_t bx0, uint64_t bx1, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred e, p, t;\n\t.reg .b64 a, b;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, 0, 0;\n\tsetp.eq.u32 t, 0, 0;\n\t"
      "add.u64 a, %1, 0;\n\tadd.u64 b, %2, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, b, %4, p;\n\t"
      "add.u64 a, %1, 2;\n\tadd.u64 b, %2, 2;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, b, %4, t;\n\t"
      "add.u64 a, %1, 16;\n\tadd.u64 b, %2, 4;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, b, %4, t;\n\t"
      "add.u64 a, %1, 18;\n\tadd.u64 b, %2, 6;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, b, %4, t;\n\t"
      "add.u64 a, %1, 32;\n\tadd.u64 b, %3, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, b, %4, t;\n\t"
      "add.u64 a, %1, 34;\n\tadd.u64 b, %3, 2;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, b, %4, t;\n\t"
      "}" ::"r"(d), "l"(ah), "l"(bx0), "l"(bx1), "r"(idesc)
      : "memory");
}
}  // namespace sm100
