// Kernel launches with Programmatic Dependent Launch (PDL): each hot-path kernel is launched with
// programmatic stream serialization, so its launch and prologue (TMEM allocation, barrier init,
// descriptor prefetch) overlap the tail of the previous kernel in the stream; the kernel executes
// griddep_wait() before it reads anything the previous kernel wrote. W4A16_NO_PDL=1 disables it.
#pragma once
#include <atomic>
#include <cstdlib>
#include <cuda_runtime.h>

namespace w4 {

#ifndef W4A16_EARLY_PDL
#define W4A16_EARLY_PDL 0
#endif
// After its own wait a kernel lets the next kernel in the stream launch (-DW4A16_EARLY_PDL=1):
// without the explicit trigger the dependent launches only as this grid's blocks exit. Safe because
// every kernel here waits (griddep_wait) before it reads or writes anything another kernel touches.
// Let the next kernel in the stream launch now (PDL) rather than as this grid's blocks exit: its
// CTAs become resident and run their prologue (the grouped GEMM's TMEM allocation and barrier init)
// while this kernel finishes; everything it reads from this kernel still waits in its own
// griddep_wait. Called by the small routing / permutation / gather / combine kernels right after
// their own wait, for grids of at most kSmallTriggerBlocks blocks (decode sizes: with the tens of
// thousands of blocks of a prefill gather the dependent GEMM's CTAs would only contend with its
// tail). Measured, same box (DS-R1 / Qwen3 / Mixtral layers): T=1 -1.3 / -5 / -3 %, T=16 -0.2 /
// -2.6 / -1.5 %, DS-R1 T=64 -0.6 %; prefill +1 % without the grid limit. -DW4A16_SMALL_TRIGGER=0
// disables it.
#ifndef W4A16_SMALL_TRIGGER
#define W4A16_SMALL_TRIGGER 1
#endif
constexpr unsigned kSmallTriggerBlocks = 4096;
__device__ __forceinline__ void griddep_launch_dependents() {
#if W4A16_SMALL_TRIGGER
  if (gridDim.x * gridDim.y * gridDim.z <= kSmallTriggerBlocks) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

__device__ __forceinline__ void griddep_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
#if W4A16_EARLY_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("W4A16_NO_PDL");
    return !(e && atoi(e) != 0);
  }();
  return on;
}

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device property of a kernel: `done` holds one
// bit per device ordinal (< 64) for which it has been set. Setting it twice is harmless, so the racy
// first use from two threads only costs a repeated (cheap) call.
template <typename Kern>
bool ensure_smem_attr(Kern kernel, int bytes, std::atomic<unsigned long long>& done) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  const unsigned long long bit = dev < 64 ? 1ull << dev : 0ull;
  if (bit && (done.load(std::memory_order_relaxed) & bit)) return true;
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) return false;
  if (bit) done.fetch_or(bit, std::memory_order_relaxed);
  return true;
}

template <typename Kern, typename... Args>
cudaError_t launch_pdl(Kern kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

}  // namespace w4
