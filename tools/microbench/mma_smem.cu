// Microbenchmark: does TMA (cp.async.bulk) traffic into shared memory slow tcgen05.mma (A in TMEM,
// B = 128 rows x K16 from SMEM)? One CTA: warp 1 issues M128 x N x K16 MMAs back to back, warp 2
// streams bulk copies (4 x 16 KB in flight) from global into a separate smem region until the MMAs
// are done, optionally warps 3.. read smem with ld.shared.v4 (the dequant's code loads).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2504_16214_b200/csrc
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace w4;

constexpr int kTmaBytes = 4 * 16384;

template <int N, bool kTma, int kLdsWarps, bool kPairB, bool kRand = false>
__global__ void mma_smem(int iters, const uint8_t* src, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];  // [0,32K) B tile, [32K, 32K+64K) TMA landing
  __shared__ uint32_t holder;
  __shared__ __align__(8) uint64_t bar, tbar;
  __shared__ volatile int done;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // kRand: random fp16 in [-1, 1) for B and A (data-dependent tensor-core power probe)
  auto rnd = [](uint32_t i) {
    uint32_t h = i * 2654435761u;
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    h ^= h >> 15;
    return ((h & 0x03ff03ffu) | 0x38003800u) ^ (h & 0x80008000u);  // |x| in [0.5, 1), random sign
  };
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = kRand ? rnd(i) : 0x3c003c00u;
  if (warp == 0) tmem_alloc<512>(&holder);
  if (threadIdx.x == 32) { mbar_init(&bar, 1); mbar_init(&tbar, 1); done = 0; fence_mbar_init(); }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = holder;
  if (kRand && warp < 4) {  // A region cols 256..511, lane quadrant of this warp
    uint32_t r[16];
    for (int c = 0; c < 16; ++c) {
#pragma unroll
      for (int i = 0; i < 16; ++i) r[i] = rnd(threadIdx.x * 977 + c * 16 + i);
      tmem_st_x16(tb + ((warp & 3) * 32 << 16) + 256 + c * 16, r);
    }
    tc_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    constexpr uint32_t idesc = make_idesc_f16(128, N, false);
    const uint64_t bdesc = make_sdesc_sw128(smem_u32(smem));
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        // gate/up pattern: two MMAs (different A, accumulators) read the same B slice
        const uint32_t d = tb + (k & 1) * 128;
        umma_ts_f16_warp(d, tb + 256 + (k & 7) * 8, bdesc + (kPairB ? ((k >> 1) & 3) : (k & 3)) * 2, idesc, 1);
      }
    }
    long long t1 = clock64();
    umma_commit_warp(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    if (lane == 0) { out[0] = t1 - t0; out[1] = t2 - t0; done = 1; }
  } else if (warp == 2 && kTma) {
    long long bytes = 0, t0 = clock64();
    uint32_t ph = 0;
    if (lane == 0) {
      while (!done) {
        mbar_arrive_expect_tx(&tbar, kTmaBytes);
        for (int c = 0; c < 4; ++c) bulk_g2s(smem + 32768 + c * 16384, src + c * 16384, 16384, &tbar);
        mbar_wait(&tbar, ph);
        ph ^= 1;
        bytes += kTmaBytes;
      }
      out[2] = bytes;
      out[3] = clock64() - t0;
    }
  } else if (warp >= 4 && warp < 4 + kLdsWarps) {
    uint32_t acc = 0;
    const uint32_t base = smem_u32(smem + 32768) + lane * 16;
    while (!done) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        uint4 v;
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(base + c * 512 + (warp - 4) * 4096));
        acc ^= v.x ^ v.w;
      }
    }
    if (acc == 0x12345) out[4] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tb); }
}

template <int N, bool kTma, int kLdsWarps, bool kPairB = false, bool kRand = false>
void run(long long* d, const uint8_t* src) {
  const int iters = 400;
  cudaMemset(d, 0, 64);
  auto k = mma_smem<N, kTma, kLdsWarps, kPairB, kRand>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 + kTmaBytes);
  k<<<1, 128 + 32 * kLdsWarps, 32768 + kTmaBytes>>>(iters, src, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[4];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("rand=%d ", kRand);
  printf("N=%3d tma=%d lds_warps=%d sameB=%d: %.1f cyc/mma; TMA %.1f B/cyc %s\n", N, kTma, kLdsWarps, kPairB,
         (double)h[1] / (iters * 16), h[3] ? (double)h[2] / h[3] : 0.0, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  long long* d;
  uint8_t* src;
  cudaMalloc(&d, 64);
  cudaMalloc(&src, 1 << 20);
  cudaMemset(src, 0x11, 1 << 20);
  run<128, false, 0>(d, src);
  run<128, false, 0, false, true>(d, src);
  run<128, true, 4, false, true>(d, src);
  run<64, false, 0, false, true>(d, src);
  run<128, true, 0>(d, src);
  run<128, true, 4>(d, src);
  run<128, false, 4>(d, src);
  run<128, true, 0, true>(d, src);
  run<64, true, 0>(d, src);
  run<256, true, 0>(d, src);
  return 0;
}
