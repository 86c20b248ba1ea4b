// micro_floor.cu — development microbenchmark: tcgen05.mma (M=128, K=16) cost with no per-MMA
// issue arithmetic (fully unrolled, compile-time descriptor offsets), for A/B operands that walk
// through distinct shared memory like a streaming kernel versus re-reading one tile.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/micro_floor tools/micro_floor.cu
#include <cstdio>
#include "../paper_2511_22880_b200/csrc/lsv_common.cuh"
using namespace lsv;

template <int N, bool DISTINCT, int M>
__global__ void __launch_bounds__(64, 1) floor_k(unsigned long long* out, int iters) {
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
  if (threadIdx.x == 32) {
    const uint32_t idesc = idesc_bf16(M, N, 0);
    const uint64_t a0 = smem_desc(smem_u32(buf), 16, 1024, 2), b0 = smem_desc(smem_u32(buf + 128 * 1024), 16, 1024, 2);
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        // distinct: 4 tiles of [128 rows][128 B] (16 KB each) for A, [N rows][128 B] for B
        const uint64_t da = a0 + (DISTINCT ? ((j >> 2) * (M * 128) + (j & 3) * 32) >> 4 : 0);
        const uint64_t db = b0 + (DISTINCT ? ((j >> 2) * (N * 128) + (j & 3) * 32) >> 4 : 0);
        umma_bf16(tmem, da, db, idesc, (it | j) != 0);
      }
    }
    umma_commit(bar);
    mbar_wait(bar, 0);
    out[0] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x >= 32) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int N, bool D, int M>
void run(unsigned long long* d) {
  const int smem = 200 * 1024 + 2048, iters = 64;
  cudaFuncSetAttribute(floor_k<N, D, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long h = 0;
  for (int it = 0; it < 2; ++it) { floor_k<N, D, M><<<1, 64, smem>>>(d, iters); cudaDeviceSynchronize(); }
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("M=%3d N=%3d %-8s: %6.1f cycles/MMA (%s)\n", M, N, D ? "distinct" : "same", (double)h / (iters * 16),
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  run<16, false, 128>(d); run<16, true, 128>(d);
  run<32, true, 128>(d); run<64, false, 128>(d); run<64, true, 128>(d);
  run<128, false, 128>(d); run<128, true, 128>(d); run<256, true, 128>(d);
  run<16, true, 64>(d); run<64, true, 64>(d); run<128, true, 64>(d); run<256, true, 64>(d);
  return 0;
}
