// Microbenchmark: the decode GEMM's MMA stage in isolation -- StageAsm<16, gate|up, 1 CTA, offset,
// kKSplit> (16 tcgen05.mma M128 x N16 x K16, A in TMEM, four or two accumulate chains) issued by one
// thread with a commit per stage, completion observed by a second warp. Modes:
//   stream  -- S stages back to back (accumulator slots rotate over 4, A slots over 2, no waits)
//   serial  -- issue one stage, wait for its commit, issue the next (isolated stage latency)
// Run on 1 CTA and on 148 CTAs (every SM) to see whether the stage time is the tensor pipe's.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2504_16214_b200/csrc
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
#include "mma_stage.cuh"
using namespace w4;

constexpr int S = 64;

template <int kKSplit, bool kSerial>
__global__ void mma_stage(long long* out) {
  __shared__ __align__(1024) uint8_t smem[8192];
  __shared__ uint32_t holder;
  __shared__ __align__(8) uint64_t cbar[S];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 8192 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (warp == 0) tmem_alloc<512>(&holder);
  if (threadIdx.x == 32) {
    for (int i = 0; i < S; ++i) mbar_init(&cbar[i], 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = holder;
  long long* o = out + blockIdx.x * 2 * S;
  if (warp == 1) {
    constexpr uint32_t idesc = make_idesc_f16(128, 16, false);
    const uint64_t bdesc = make_sdesc_sw128(smem_u32(smem));
    constexpr int kAccCols = 2 * kKSplit * 16;
    for (int s = 0; s < S; ++s) {
      if (elect_one()) {
        StageAsm<16, 1, 1, true, kKSplit>::issue(tb + (s % 4) * kAccCols, tb + 256 + (s % 2) * 128, bdesc, idesc, 0u);
        umma_commit(&cbar[s]);
      }
      __syncwarp();
      long long t = clock64();
      if (lane == 0) o[s] = t;
      if (kSerial) mbar_wait(&cbar[s], 0);
    }
  } else if (warp == 2) {
    for (int s = 0; s < S; ++s) {
      mbar_wait(&cbar[s], 0);
      long long t = clock64();
      if (lane == 0) o[S + s] = t;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tb); }
}

template <int kKSplit, bool kSerial>
void run(long long* d, int grid, const char* what) {
  cudaMemset(d, 0, sizeof(long long) * 2 * S * 148);
  mma_stage<kKSplit, kSerial><<<grid, 96>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  static long long h[2 * S * 148];
  cudaMemcpy(h, d, sizeof(long long) * 2 * S * grid, cudaMemcpyDeviceToHost);
  double lat = 0, per = 0;
  int lo = S / 4, hi = 3 * S / 4;
  for (int b = 0; b < grid; ++b) {
    const long long* o = h + b * 2 * S;
    for (int s = lo; s < hi; ++s) lat += o[S + s] - o[s];
    per += double(o[S + hi] - o[S + lo]) / (hi - lo);
  }
  printf("%-34s grid %3d: issue->complete %7.1f cyc, completion period %7.1f cyc/stage%s%s\n", what, grid,
         lat / (grid * (hi - lo)), per / grid, e == cudaSuccess ? "" : " ", e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * 2 * S * 148);
  for (int r = 0; r < 2; ++r) {
    for (int g : {1, 148}) {
      run<2, false>(d, g, "stream, k-split 2 (4 chains x 4)");
      run<2, true>(d, g, "serial, k-split 2 (4 chains x 4)");
      run<1, false>(d, g, "stream, k-split 1 (2 chains x 8)");
      run<1, true>(d, g, "serial, k-split 1 (2 chains x 8)");
    }
  }
  return 0;
}
