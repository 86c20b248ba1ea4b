// micro_layout.cu — development microbenchmark: tcgen05.mma (kind::f16, M=128, K=16) issue cost
// per instruction as a function of the operand smem layout and of whether successive MMAs read
// distinct smem (as a streaming kernel does) or the same tile again.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/micro_layout tools/micro_layout.cu
#include <cstdio>
#include "../paper_2511_22880_b200/csrc/lsv_common.cuh"
using namespace lsv;

// layout: 2 = SW128 K-major (rows of 128 B = 64 k), 6 = SW32 K-major (rows of 32 B = 16 k),
//         0 = interleaved (8x16B core matrices; [kgroup][mgroup] order), 4 = SW64
__device__ __forceinline__ uint64_t desc_for(uint32_t base, int layout, int rows, int kslice, int distinct) {
  switch (layout) {
    case 2: {  // tile [rows][128B]; k-slice kk -> +32 B inside the row; distinct tiles every 16 KB
      const uint32_t t = distinct ? (kslice >> 2) * (rows * 128) : 0;
      return smem_desc(base + t + (kslice & 3) * 32, 16, 1024, 2);
    }
    case 4: {  // tile [rows][64B]; k-slice -> +32 B
      const uint32_t t = distinct ? (kslice >> 1) * (rows * 64) : 0;
      return smem_desc(base + t + (kslice & 1) * 32, 16, 512, 4);
    }
    case 6: {  // tile [rows][32B] per k-slice: 8-row atoms of 256 B
      const uint32_t t = distinct ? kslice * (rows * 32) : 0;
      return smem_desc(base + t, 16, 256, 6);
    }
    default: {  // interleaved: [2 k core][rows/8][128 B]; LBO = k-core stride, SBO = m-group stride
      const uint32_t t = distinct ? kslice * (rows * 32) : 0;
      return smem_desc(base + t, rows * 16, 128, 0);
    }
  }
}

__global__ void __launch_bounds__(64, 1) bench(unsigned long long* out, int n_mma, int N, int layout, int distinct,
                                               int M) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* buf = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(buf + 200 * 1024);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
  for (int i = threadIdx.x; i < 200 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(buf)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
  if (threadIdx.x >= 32) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (M == 0 && threadIdx.x >= 32) {   // warp-converged issue, one elected lane (CuTe style)
    const uint32_t idesc = idesc_bf16(128, N, 0);
    const uint32_t a = smem_u32(buf), b = smem_u32(buf + 128 * 1024);
    unsigned long long t0 = clock64();
    for (int j = 0; j < n_mma; ++j) {
      const int ks = j & 15;
      const uint64_t da = desc_for(a, layout, 128, ks, distinct), db = desc_for(b, layout, N, ks & 7, distinct);
      if (elect_one()) umma_bf16(tmem, da, db, idesc, j > 0);
      __syncwarp();
    }
    if (elect_one()) umma_commit(bar);
    __syncwarp();
    mbar_wait(bar, 0);
    if (threadIdx.x == 32) out[0] = clock64() - t0;
  } else if (M == 0) {
  } else if (threadIdx.x == 32) {
    const uint32_t idesc = idesc_bf16(M, N, 0);
    const uint32_t a = smem_u32(buf), b = smem_u32(buf + 128 * 1024);
    unsigned long long t0 = clock64();
    for (int j = 0; j < n_mma; ++j) {
      const int ks = j & 15;  // 16 distinct k-slices = 4 SW128 tiles of 16 KB (A) -> 64 KB
      umma_bf16(tmem, desc_for(a, layout, M, ks, distinct), desc_for(b, layout, N, ks & 7, distinct), idesc, j > 0);
    }
    umma_commit(bar);
    mbar_wait(bar, 0);
    out[0] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x >= 32) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  const int smem = 200 * 1024 + 2048;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int n = 512;
  const char* lname[8] = {"interleaved", "?", "SW128", "?", "SW64", "?", "SW32", "?"};
  for (int M : {128, 0})
    for (int layout : {2, 6})
      for (int distinct : {0, 1})
        for (int N : {16, 64, 128}) {
          unsigned long long h = 0;
          for (int it = 0; it < 2; ++it) {
            bench<<<1, 64, smem>>>(d, n, N, layout, distinct, M);
            cudaDeviceSynchronize();
          }
          cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
          printf("M=%3d %-11s %-8s N=%3d: %6.1f cycles/MMA (%s)\n", M, lname[layout], distinct ? "distinct" : "same", N,
                 (double)h / n, cudaGetErrorString(cudaGetLastError()));
        }
  return 0;
}
