// Microbenchmark: cycles per tcgen05.mma.cta_group::2.kind::f16 (M=256 over a CTA pair, K=16, A in
// TMEM) issued back to back by the leader CTA, for several N, against cta_group::1 M=128 (mma_rate.cu).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2504_16214_b200/csrc
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace w4;

template <int N>
__global__ void __cluster_dims__(2, 1, 1) mma_pair(int iters, long long* out) {
  __shared__ __align__(1024) uint8_t smem[16384];
  __shared__ uint32_t holder;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32;
  const uint32_t rank = cluster_ctarank();
  for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (warp == 0) tmem_alloc_pair<512>(&holder);
  if (threadIdx.x == 32) { mbar_init(&bar, 1); fence_mbar_init(); }
  fence_proxy_async_smem();
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tb = holder;
  if (warp == 1 && rank == 0) {
    constexpr uint32_t idesc = make_idesc_f16(256, N, false);
    const uint64_t bdesc = make_sdesc_sw128(smem_u32(smem));
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const uint32_t d = tb + (k % 2) * (N > 128 ? 128 : N);
        asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, 1, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                     "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                     "r"(tb + 384 + (k & 7) * 8), "l"(bdesc + (k & 3) * 2), "r"(idesc) : "memory");
      }
    }
    long long t1 = clock64();
    umma_commit_pair_warp(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    if (threadIdx.x == 32) { out[0] = t1 - t0; out[1] = t2 - t0; }
  } else if (warp == 1 && rank == 1) {
    mbar_wait(&bar, 0);  // the multicast commit arrives here too
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 0) { tc_fence_after(); tmem_dealloc_pair<512>(tb); }
}

template <int N>
void run(long long* d) {
  const int iters = 200;
  cudaMemset(d, 0, 32);
  mma_pair<N><<<2, 64>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[2];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("pair M=256 N=%3d ts: issue %.1f cyc/mma, complete %.1f cyc/mma (per-SM share = M128 x N) %s\n", N,
         (double)h[0] / (iters * 16), (double)h[1] / (iters * 16), e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  run<32>(d); run<64>(d); run<128>(d); run<256>(d);
  return 0;
}
