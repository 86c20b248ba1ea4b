// tma_issue.cu — development microbenchmark: how many cycles does one warp spend issuing a bulk
// copy (cp.async.bulk, elected lane) or a 2D/3D TMA box load, back to back, and does a second
// issuing warp add throughput?  Sources are L2-resident (small buffer re-read).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2511_22880_b200/csrc tools/tma_issue.cu -o tools/tma_issue -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include "lsv_common.cuh"
using namespace lsv;

__global__ void __launch_bounds__(128, 1) issue_kernel(const uint8_t* src, int nops, int bytes, int nwarps,
                                                       unsigned long long* out, const __grid_constant__ CUtensorMap map,
                                                       int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < 4) mbar_init(&bar[threadIdx.x], 1);
  fence_mbar_init();
  __syncthreads();
  if (warp < nwarps) {
    const uint32_t fb = smem_u32(&bar[warp]);
    const uint32_t dst = smem_u32(sm) + warp * 65536;
    uint64_t t0 = clock64(), issue = 0;
    uint32_t phase = 0;
    for (int i = 0; i < nops; i += 16) {
      mbar_arrive_expect_tx_elect(fb, (uint32_t)(16 * bytes));
      const uint64_t a = clock64();
      for (int j = 0; j < 16; ++j) {
        if (mode == 0) bulk_load_elect(dst + (j % 4) * bytes, src + ((i + j) % 64) * bytes, bytes, fb);
        else tma_load_2d_elect(dst + (j % 4) * bytes, &map, fb, 0, ((i + j) % 64) * (bytes / 128));
      }
      issue += clock64() - a;
      mbar_wait(&bar[warp], phase);
      phase ^= 1;
    }
    uint64_t t1 = clock64();
    if (lane == 0) { out[(blockIdx.x * 4 + warp) * 2] = t1 - t0; out[(blockIdx.x * 4 + warp) * 2 + 1] = issue; }
  }
}

int main() {
  uint8_t* src;
  cudaMalloc(&src, 64 << 20);
  cudaMemset(src, 1, 64 << 20);
  unsigned long long* out;
  cudaMalloc(&out, 148 * 4 * 16);
  CUtensorMap map;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                           const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                           CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill)>(fn);
  cudaFuncSetAttribute(issue_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 65536);
  for (int bytes : {1024, 4096, 16384}) {
    cuuint64_t dims[2] = {64, (cuuint64_t)(64 << 20) / 128};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, (cuuint32_t)(bytes / 128)};
    cuuint32_t es[2] = {1, 1};
    enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int mode = 0; mode < 2; ++mode)
      for (int nw : {1, 2}) {
        for (int grid : {1, 148}) {
          const int nops = 1024;
          issue_kernel<<<grid, 128, 3 * 65536>>>(src, nops, bytes, nw, out, map, mode);
          cudaDeviceSynchronize();
          unsigned long long h[8];
          cudaMemcpy(h, out, 64, cudaMemcpyDeviceToHost);
          printf("%s %6d B  warps %d grid %3d: %7.1f cycles per op per warp (issue alone %6.1f), %6.1f B/cycle per SM\n",
                 mode ? "tma2d" : "bulk ", bytes, nw, grid, (double)h[0] / nops, (double)h[1] / nops,
                 (double)nops * bytes * nw / h[0]);
        }
      }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
