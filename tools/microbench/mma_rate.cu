// Microbenchmark: cycles per tcgen05.mma.cta_group::1.kind::f16 (M=128, K=16) issued back to back by
// one thread, for A in TMEM (ts) or SMEM (ss), several N, and 1 or 4 independent accumulators.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2504_16214_b200/csrc
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace w4;

template <int N, bool kTS, int kChains, int kStWarps = 0, int kSmemWarps = 0, int kCommits = 0>
__global__ void mma_rate(int iters, long long* out) {
  __shared__ __align__(1024) uint8_t smem[2 * 16384 + 1024];
  __shared__ uint32_t holder;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t cbar[4];
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < (2 * 16384) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (warp == 0) tmem_alloc<512>(&holder);
  if (threadIdx.x == 32) { mbar_init(&bar, 1); for (int i = 0; i < 4; ++i) mbar_init(&cbar[i], 1); fence_mbar_init(); }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = holder;
  if (warp == 1) {
    constexpr uint32_t idesc = make_idesc_f16(128, N, false);
    const uint64_t bdesc = make_sdesc_sw128(smem_u32(smem));
    const uint64_t adesc = make_sdesc_sw128(smem_u32(smem + 16384));
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const uint32_t d = tb + (k % kChains) * N;
        if constexpr (kTS) umma_ts_f16_warp(d, tb + 256 + (k & 7) * 8, bdesc + (k & 3) * 2, idesc, 1);
        else {
          asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, 1, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                       "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                       "l"(adesc + (k & 3) * 2), "l"(bdesc + (k & 3) * 2), "r"(idesc) : "memory");
        }
        // kCommits commits per 16 MMAs (never waited on): does a commit serialise the MMA pipe?
        if (kCommits > 0 && (k + 1) % (16 / (kCommits > 0 ? kCommits : 1)) == 0) umma_commit_warp(&cbar[k & 3]);
      }
    }
    long long t1 = clock64();
    umma_commit_warp(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    if (threadIdx.x == 32) { out[0] = t1 - t0; out[1] = t2 - t0; }
  } else if (warp >= 2 + kStWarps && warp < 2 + kStWarps + kSmemWarps) {
    // shared-memory write traffic into the B buffer region's tail (like TMA landing the next tiles)
    uint4* dst = reinterpret_cast<uint4*>(smem + 8192);
    const uint4 v = make_uint4(0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u);
    for (int it = 0; it < iters * 16; ++it) {
#pragma unroll
      for (int c = 0; c < 8; ++c) dst[((threadIdx.x & 31) + c * 32) & 511] = v;
    }
  } else if (warp >= 2 && warp < 2 + kStWarps) {
    // concurrent tcgen05.st traffic into columns 384..511 (like the dequant warps): each warp writes its
    // lane quadrant, 16 columns per instruction, 8 instructions per "stage"
    const uint32_t quad = warp & 3;
    uint32_t r[16];
    for (int i = 0; i < 16; ++i) r[i] = 0x3c003c00u + i;
    const int st_iters = iters * 4;
    long long t0 = clock64();
    for (int it = 0; it < st_iters; ++it) {
#pragma unroll
      for (int c = 0; c < 8; ++c) tmem_st_x16(tb + ((quad * 32) << 16) + 384 + c * 16, r);
      tc_wait_st();
    }
    long long t1 = clock64();
    if ((threadIdx.x & 31) == 0 && warp == 2) out[2] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tb); }
}

template <int N, bool kTS, int kChains, int kStWarps = 0, int kSmemWarps = 0, int kCommits = 0>
void run(long long* d) {
  const int iters = 200;
  cudaMemset(d, 0, 32);
  mma_rate<N, kTS, kChains, kStWarps, kSmemWarps, kCommits><<<1, 64 + 32 * (kStWarps + kSmemWarps)>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[3];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("commits/16=%d ", kCommits);
  printf("smemw=%d N=%3d %s chains=%d st_warps=%d : issue %.1f cyc/mma, complete %.1f cyc/mma; st %.1f cyc per 8xSTTM %s\n", N,
         kSmemWarps, kTS ? "ts" : "ss", kChains, kStWarps, (double)h[0] / (iters * 16), (double)h[1] / (iters * 16),
         kStWarps ? (double)h[2] / (iters * 4) : 0.0, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  run<128, true, 2>(d); run<128, true, 2, 4>(d); run<128, true, 2, 4, 4>(d); run<128, true, 2, 8, 4>(d);
  run<128, true, 2, 0, 0, 1>(d); run<128, true, 2, 0, 0, 2>(d); run<128, true, 2, 0, 0, 4>(d);
  run<16, true, 4, 0, 0, 1>(d); run<16, true, 4, 0, 0, 4>(d);
  run<64, true, 2>(d); run<64, true, 2, 4, 4>(d); run<16, true, 4, 4, 4>(d);
  return 0;
}
