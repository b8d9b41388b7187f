// tma_probe.cu -- microbenchmark: per-SM throughput of TMA box loads on B200 (not part of the library).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe tools/tma_probe.cu -lcuda
// Modes: 0 = tiled 3-D box {32 fp32, 128 rows, 1} (16 KB, SWIZZLE_128B) over a dense matrix
//        1 = im2col 4-D box (128 px x 32 ch) over an NHWC tensor, 3x3 window taps cycling
//        2 = tiled 4-D box {32 ch, 16 w, 8 h, 1} over the same NHWC tensor (spatial tile, tap-shifted)
// Each CTA keeps `depth` boxes in flight (ring of mbarriers), loads `iters` boxes, reports B/clk/SM.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void probe(const __grid_constant__ CUtensorMap tm, int iters, int depth, int W, int H, int N,
                      unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* buf = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(buf + depth * 16384);
  if (threadIdx.x == 0) {
    for (int i = 0; i < depth; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters + depth; ++it) {
    const int s = it % depth;
    if (it >= depth) {  // wait for the load issued `depth` iterations ago
      const uint32_t par = ((it - depth) / depth) & 1;
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}"
                     : "=r"(ok)
                     : "r"(su32(&bars[s])), "r"(par));
    }
    if (it < iters) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bars[s])), "r"(16384));
      const uint32_t dst = su32(buf + s * 16384);
      const int g = blockIdx.x * iters + it;
      if (MODE == 0 || MODE == 3) {
        const int row = (g * 128) % (MODE == 0 ? (1 << 20) : (1 << 14));
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
            "%5}], [%2];" ::"r"(dst),
            "l"((uint64_t)&tm), "r"(su32(&bars[s])), "r"(0), "r"(row), "r"(0));
      } else if (MODE == 1) {
        const int tap = it % 9;
        const int pix = (g / 9 * 128) % (W * H * N);
        const int n = pix / (W * H), w = pix % W, h = (pix / W) % H;
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
            "%5, %6}], [%2], {%7, %8};" ::"r"(dst),
            "l"((uint64_t)&tm), "r"(su32(&bars[s])), "r"(0), "r"(w - 1), "r"(h - 1), "r"(n), "h"((uint16_t)(tap % 3)),
            "h"((uint16_t)(tap / 3)));
      } else if (MODE == 4) {
        const int blk = g % (3 * 6 * N);
        const int wb = blk % 3, hb = (blk / 3) % 6, n = blk / 18;
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
            "%5, %6}], [%2];" ::"r"(dst),
            "l"((uint64_t)&tm), "r"(su32(&bars[s])), "r"(0), "r"(wb * 16 + 1), "r"(hb * 8 + 1), "r"(n));
      } else if (MODE == 5) {
        const int tap = it % 9;
        const int pix = (g / 9 * 128) % (54 * 54 * N);
        const int n = pix / (54 * 54), w = pix % 54, h = (pix / 54) % 54;
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
            "%5, %6}], [%2], {%7, %8};" ::"r"(dst),
            "l"((uint64_t)&tm), "r"(su32(&bars[s])), "r"(0), "r"(w), "r"(h), "r"(n), "h"((uint16_t)(tap % 3)),
            "h"((uint16_t)(tap / 3)));
      } else {
        const int tap = it % 9;
        const int blk = (g / 9) % ((W / 16) * (H / 8) * N);
        const int wb = blk % (W / 16), hb = (blk / (W / 16)) % (H / 8), n = blk / ((W / 16) * (H / 8));
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
            "%5, %6}], [%2];" ::"r"(dst),
            "l"((uint64_t)&tm), "r"(su32(&bars[s])), "r"(0), "r"(wb * 16 + tap % 3 - 1), "r"(hb * 8 + tap / 3 - 1),
            "r"(n));
      }
    }
  }
  cycles[blockIdx.x] = clock64() - t0;
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  const int depth = argc > 2 ? atoi(argv[2]) : 6;
  const int ctas = argc > 3 ? atoi(argv[3]) : 148;
  const int C = 64, W = 56, H = 56, N = 64, iters = 2000;
  const int stride_b = argc > 4 ? atoi(argv[4]) : 256;  // mode 3: row stride in bytes
  PFN_cuTensorMapEncodeTiled_v12000 enc_t;
  PFN_cuTensorMapEncodeIm2col_v12000 enc_i;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc_t, cudaEnableDefault, &q));
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", (void**)&enc_i, cudaEnableDefault, &q));
  float* x;
  const size_t elems = (size_t)N * H * W * C;  // 51 MB: L2-resident after the first touch
  const size_t bytes_alloc = std::max(std::max(elems * 4, (size_t)(1 << 20) * 128), (size_t)(1 << 14) * 16384);
  CK(cudaMalloc(&x, bytes_alloc));
  CK(cudaMemset(x, 0, bytes_alloc));
  alignas(64) CUtensorMap tm;
  CUresult r;
  if (mode == 0) {
    cuuint64_t dims[3] = {32, 1 << 20, 1}, str[2] = {128, 128ull << 20};
    cuuint32_t box[3] = {32, 128, 1}, es[3] = {1, 1, 1};
    r = enc_t(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, x, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (mode == 3) {
    cuuint64_t dims[3] = {32, 1 << 14, 1}, str[2] = {(cuuint64_t)stride_b, (cuuint64_t)stride_b << 14};
    cuuint32_t box[3] = {32, 128, 1}, es[3] = {1, 1, 1};
    r = enc_t(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, x, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (mode == 5) {
    cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
    cuuint64_t str[3] = {(cuuint64_t)C * 4, (cuuint64_t)W * C * 4, (cuuint64_t)H * W * C * 4};
    int lo[2] = {0, 0}, up[2] = {-2, -2};
    cuuint32_t es[4] = {1, 1, 1, 1};
    r = enc_i(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, x, dims, str, lo, up, 32, 128, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (mode == 1) {
    cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
    cuuint64_t str[3] = {(cuuint64_t)C * 4, (cuuint64_t)W * C * 4, (cuuint64_t)H * W * C * 4};
    int lo[2] = {-1, -1}, up[2] = {-1, -1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    r = enc_i(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, x, dims, str, lo, up, 32, 128, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {  // modes 2 and 4
    cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
    cuuint64_t str[3] = {(cuuint64_t)C * 4, (cuuint64_t)W * C * 4, (cuuint64_t)H * W * C * 4};
    cuuint32_t box[4] = {32, 16, 8, 1}, es[4] = {1, 1, 1, 1};
    r = enc_t(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, x, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", (int)r);
    return 1;
  }
  unsigned long long* cyc;
  CK(cudaMalloc(&cyc, ctas * 8));
  const int smem = depth * 16384 + 1024 + 256;
  void (*k)(const CUtensorMap, int, int, int, int, int, unsigned long long*) =
      mode == 0 ? probe<0> : mode == 1 ? probe<1> : mode == 2 ? probe<2> : mode == 3 ? probe<3> : mode == 4 ? probe<4>
                                                                                                 : probe<5>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<ctas, 32, smem>>>(tm, iters, depth, W, H, N, cyc);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> h(ctas);
    CK(cudaMemcpy(h.data(), cyc, ctas * 8, cudaMemcpyDeviceToHost));
    unsigned long long mx = 0;
    for (auto v : h) mx = v > mx ? v : mx;
    const double bytes = (double)ctas * iters * 16384;
    printf("mode=%d depth=%d ctas=%d: %.1f B/clk/SM (max cycles %llu), chip %.2f TB/s\n", mode, depth, ctas,
           (double)iters * 16384 / mx, mx, bytes / (ms * 1e-3) / 1e12);
  }
  return 0;
}
