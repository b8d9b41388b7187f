// launch.cuh -- kernel launches with programmatic dependent launch (PDL).
//
// Every kernel of the library is launched with cudaLaunchAttributeProgrammaticStreamSerialization, so
// its CTAs may start (prologue: barrier init, TMEM allocation, tensor-map prefetch) while the previous
// kernel on the stream is still finishing.  The contract each kernel keeps:
//   * pdl_trigger() first: lets the next kernel be scheduled as soon as all CTAs of this one run;
//   * pdl_wait() before its first global-memory read or write: returns once the previous grid has
//     completed and its writes are visible.  Since every kernel waits before it can complete, kernel
//     i+1 completing implies kernel i completed -- stream order stays transitive.
// Size-gated (pdl_enabled below): small convs only.  The wait releases only after the previous grid's
// completion flush, so the gain is the launch + prologue of CTAs that land on SMs the previous grid's
// tail has already freed.  Without the attribute griddepcontrol.* are no-ops.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <utility>

namespace conv2d {

__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Set by run_algo around the launches of one conv2d_forward: the conv is small (<= 8 GFLOP and <= 2048
// pair tiles, i.e. a few waves), so its launch + prologue are worth overlapping with the previous tail.
inline thread_local bool t_pdl_hint = false;

// PDL on a launch: CONV2D_PDL=1 always, CONV2D_PDL=0 never, unset: for small convs (t_pdl_hint).
// Measured (same box, fixed selection): on every launch b32 -1.3%, b256 +1.1%; size-gated b32 -1.3%, b256 0.
inline bool pdl_enabled() {
  static const int mode = getenv("CONV2D_PDL") ? atoi(getenv("CONV2D_PDL")) : -1;
  return mode >= 0 ? mode == 1 : t_pdl_hint;
}

// cudaFuncAttributeMaxDynamicSharedMemorySize for kernel KERN, set once per device (the attribute is a
// per-device property, so a process driving several GPUs needs it on each); thread-safe.
template <auto KERN>
cudaError_t smem_attr_once(int bytes) {
  static std::atomic<uint64_t> done{0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = dev < 64 ? (uint64_t{1} << dev) : 0;
  if (bit && (done.load(std::memory_order_acquire) & bit)) return cudaSuccess;
  e = cudaFuncSetAttribute(KERN, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace conv2d
