// synth.cu -- device twin of paper_1904_04174_b200/synth.py (counter-based splitmix64).
// Not part of the convolution: it only fills bench inputs.  Element i of stream `key`:
//   u = sm64(key + offset + i) >> 40;  uniform: u * 2^-23 - 1;  int5: (u mod 5) - 2.
#include "internal.h"

namespace conv2d {
namespace {

__device__ __forceinline__ uint64_t sm64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void synth_kernel(float* __restrict__ dst, uint64_t count, uint64_t key, uint64_t offset, int dist) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t u = sm64(key + offset + i) >> 40;
    dst[i] = dist == 0 ? (float)((int64_t)u - (1 << 23)) * (1.0f / 8388608.0f) : (float)((int)(u % 5) - 2);
  }
}

}  // namespace

cudaError_t launch_synth_fill(float* dst, uint64_t count, uint64_t key, uint64_t offset, int dist, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  uint64_t blocks = (count + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  synth_kernel<<<(unsigned)blocks, 256, 0, s>>>(dst, count, key, offset, dist);
  return cudaGetLastError();
}

}  // namespace conv2d
