// Probe: TMA tile::gather4 (4 arbitrary rows of a 2-D fp16 tensor, 64 columns each, 128B swizzle)
// into shared memory. Checks the data and the swizzle placement against the SW128 K-major layout the
// GEMM's B operand uses (row r of a 1 KB atom at r * 128 B, 16 B chunk c at c ^ (r % 8)).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2504_16214_b200/csrc tma_gather4.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include "ptx.cuh"
using namespace w4;

__global__ void g4(const __grid_constant__ CUtensorMap m, const int* rows, int n4, uint16_t* out) {
  __shared__ __align__(1024) uint8_t s[8192];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, n4 * 4 * 128);
    for (int g = 0; g < n4; ++g)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(
              smem_u32(s + g * 512)),
          "l"(&m), "r"(0), "r"(rows[4 * g]), "r"(rows[4 * g + 1]), "r"(rows[4 * g + 2]), "r"(rows[4 * g + 3]),
          "r"(smem_u32(&bar))
          : "memory");
  }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < n4 * 4 * 64; i += blockDim.x) out[i] = reinterpret_cast<uint16_t*>(s)[i];
}

int main() {
  const int R = 64, K = 256, n4 = 4;
  std::vector<uint16_t> h(R * K);
  for (int r = 0; r < R; ++r)
    for (int k = 0; k < K; ++k) h[r * K + k] = static_cast<uint16_t>(r * 256 + k);
  uint16_t *dx, *dout;
  int* drows;
  cudaMalloc(&dx, h.size() * 2);
  cudaMemcpy(dx, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  int rows[16] = {5, 2, 9, 0, 63, 7, 7, 31, 1, 2, 3, 4, 40, 41, 17, 12};
  cudaMalloc(&drows, sizeof(rows));
  cudaMemcpy(drows, rows, sizeof(rows), cudaMemcpyHostToDevice);
  cudaMalloc(&dout, n4 * 4 * 64 * 2);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  for (int boxr : {1, 4}) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)R};
    cuuint64_t strides[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)boxr};
    cuuint32_t es[2] = {1, 1};
    CUresult cr = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, dx, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    int* hrows;
    cudaMallocHost(&hrows, sizeof(rows));
    memcpy(hrows, rows, sizeof(rows));
    g4<<<1, 128>>>(m, hrows, n4, dout);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<uint16_t> o(n4 * 4 * 64);
    if (e == cudaSuccess) cudaMemcpy(o.data(), dout, o.size() * 2, cudaMemcpyDeviceToHost);
    int bad = 0, bad_noswz = 0;
    for (int i = 0; i < n4 * 4; ++i)     // smem row i holds source row rows[i]
      for (int c = 0; c < 8; ++c)        // 16 B chunk (8 halves)
        for (int j = 0; j < 8; ++j) {
          const uint16_t want = static_cast<uint16_t>(rows[i] * 256 + c * 8 + j);
          const int pc = c ^ (i % 8);  // SW128 placement
          if (o[i * 64 + pc * 8 + j] != want) ++bad;
          if (o[i * 64 + c * 8 + j] != want) ++bad_noswz;
        }
    printf("box rows %d: encode %d, kernel %s, mismatches (SW128 layout) %d, (unswizzled) %d\n", boxr, (int)cr,
           e == cudaSuccess ? "ok" : cudaGetErrorString(e), bad, bad_noswz);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
