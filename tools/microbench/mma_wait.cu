// Microbenchmark: after one thread issues 16 tcgen05.mma (M128 x N128 x K16, A in TMEM), how long
// does the SAME warp take to pass (a) an mbarrier try_wait on an already-completed phase, (b) a
// named barrier with only itself, (c) an mbarrier arrive seen by another warp? And does another
// warp's try_wait right after see any delay?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2504_16214_b200/csrc
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace w4;

template <int N, int kMode>
__global__ void mma_wait(long long* out) {
  __shared__ __align__(1024) uint8_t smem[16384];
  __shared__ uint32_t holder;
  __shared__ __align__(8) uint64_t done, bar2, bar3;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (warp == 0) tmem_alloc<512>(&holder);
  if (threadIdx.x == 32) {
    mbar_init(&done, 1);
    mbar_init(&bar2, 1);
    mbar_init(&bar3, 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) mbar_arrive(&bar2);  // bar2 phase 0 completes now
  __syncthreads();
  const uint32_t tb = holder;
  if (warp == 1) {
    constexpr uint32_t idesc = make_idesc_f16(128, N, false);
    const uint64_t bdesc = make_sdesc_sw128(smem_u32(smem));
    long long t0 = clock64();
#pragma unroll
    for (int k = 0; k < 16; ++k) umma_ts_f16_warp(tb + (k & 1) * 128, tb + 256 + (k & 7) * 8, bdesc + (k & 3) * 2, idesc, 1);
    long long t1 = clock64();
    if (kMode == 0) mbar_wait_warp(&bar2, 0);           // completed long ago
    if (kMode == 1) named_bar_sync(3, 32);               // only this warp
    if (kMode == 2 && lane == 0) mbar_arrive(&bar3);     // seen by warp 2
    if (kMode == 3) { uint32_t x; asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(x) : "r"(smem_u32(smem))); if (x == 7) out[7] = x; }
    long long t2 = clock64();
    umma_commit_warp(&done);
    mbar_wait(&done, 0);
    long long t3 = clock64();
    if (lane == 0) { out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t0; out[4] = t1; }
  } else if (warp == 2) {
    if (kMode == 2) {
      mbar_wait(&bar3, 0);
      long long t = clock64();
      if (lane == 0) out[3] = t;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (kMode == 2 && threadIdx.x == 0) out[3] -= out[4];
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tb); }
}

template <int kMode>
void run(long long* d, const char* what) {
  cudaMemset(d, 0, 64);
  mma_wait<128, kMode><<<1, 96>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[5];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%-44s issue 16 MMAs %5lld cyc; then op %5lld cyc; all MMAs done %5lld cyc%s%s\n", what, h[0], h[1], h[2],
         kMode == 2 ? "; arrive seen by warp 2 after (cyc): " : "", e == cudaSuccess ? "" : cudaGetErrorString(e));
  if (kMode == 2) printf("    %lld\n", h[3]);
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  for (int r = 0; r < 2; ++r) {
    run<0>(d, "try_wait on a completed phase");
    run<1>(d, "bar.sync of this warp only");
    run<2>(d, "mbarrier.arrive (observed by warp 2)");
    run<3>(d, "ld.volatile.shared");
  }
  return 0;
}
