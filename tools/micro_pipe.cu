// micro_pipe.cu — development microbenchmark: the shrink's producer -> MMA -> commit ring with no
// memory traffic, to separate the MMA cost from the barrier hand-off cost per pipeline stage.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/micro_pipe tools/micro_pipe.cu
#include <cstdio>
#include "../paper_2511_22880_b200/csrc/lsv_common.cuh"
using namespace lsv;

__global__ void __launch_bounds__(96, 1) pipe(unsigned long long* out, int stages, int mmas, int N, int slots,
                                              int mode) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* buf = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(buf + 131072);
  uint64_t* empty = full + 8;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(empty + 8);
  for (int i = threadIdx.x; i < 131072 / 16; i += blockDim.x) reinterpret_cast<uint4*>(buf)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    for (int b = 0; b < 8; ++b) { mbar_init(&full[b], 1); mbar_init(&empty[b], 1); }
    fence_mbar_init();
  }
  if (threadIdx.x >= 32 && threadIdx.x < 64) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long t0 = clock64();
  if (warp == 0 && lane == 0) {
    int slot = 0; uint32_t ph = 0;
    for (int s = 0; s < stages; ++s) {
      mbar_wait(&empty[slot], ph ^ 1);
      if (mode == 1) mbar_arrive_expect_tx(&full[slot], 0);
      else mbar_arrive(&full[slot]);
      if (++slot == slots) { slot = 0; ph ^= 1; }
    }
  } else if (warp == 1 && lane == 0) {
    const uint32_t idesc = idesc_bf16(128, N, 0);
    const uint32_t a = smem_u32(buf), b = smem_u32(buf + 65536);
    int slot = 0; uint32_t ph = 0;
    uint32_t acc = 0;
    for (int s = 0; s < stages; ++s) {
      mbar_wait(&full[slot], ph);
      tc_fence_after();
      for (int j = 0; j < mmas; ++j) {
        umma_bf16(tmem, smem_desc(a + (j & 3) * 32, 16, 1024, 2), smem_desc(b + (j & 3) * 32, 16, 1024, 2), idesc, acc);
        acc = 1;
      }
      umma_commit(&empty[slot]);
      if (++slot == slots) { slot = 0; ph ^= 1; }
    }
    // drain
    umma_commit(&full[7]);
    mbar_wait(&full[7], 0);
    out[0] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  const int smem = 131072 + 2048;
  cudaFuncSetAttribute(pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  struct C { int mmas, N, slots, mode; } cs[] = {
      {16, 16, 4, 1}, {16, 16, 4, 0}, {16, 32, 4, 1}, {16, 64, 4, 1}, {8, 128, 4, 1}, {16, 128, 4, 1},
      {4, 16, 4, 1}, {1, 16, 4, 1}, {32, 16, 4, 1}, {64, 16, 4, 1}, {16, 16, 8, 1}, {4, 128, 4, 1}, {64, 128, 4, 1}};
  const int stages = 256;
  for (auto c : cs) {
    unsigned long long h = 0;
    for (int it = 0; it < 2; ++it) {
      pipe<<<1, 96, smem>>>(d, stages, c.mmas, c.N, c.slots, c.mode);
      cudaDeviceSynchronize();
    }
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("mmas/stage %2d N=%3d slots %d mode %d: %8.1f cycles/stage  %6.1f cycles/MMA  (%s)\n", c.mmas, c.N, c.slots,
           c.mode, (double)h / stages, (double)h / stages / c.mmas, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
