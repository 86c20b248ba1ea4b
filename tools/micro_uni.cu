// micro_uni.cu — development microbenchmark: per-MMA issue cost of a shrink-like stage loop whose
// descriptor inputs come from memory (record fields), for different ways of telling the compiler
// they are warp-uniform.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/micro_uni tools/micro_uni.cu
#include <cstdio>
#include "../paper_2511_22880_b200/csrc/lsv_common.cuh"
using namespace lsv;

// tcgen05.mma issued by one elected lane, the election inside the asm (no divergent branch)
__device__ __forceinline__ void umma_elect(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ int uniform_ballot(int v) {
  return (int)__ballot_sync(0xffffffffu, (v >> (threadIdx.x & 31)) & 1);
}

template <int MODE>
__global__ void __launch_bounds__(64, 1) uni(unsigned long long* out, const int* params, int stages) {
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
  if (threadIdx.x >= 32) {
    int np8 = params[0], r = params[1], kc = params[2];
    if (MODE == 1) { np8 = __shfl_sync(~0u, np8, 0); r = __shfl_sync(~0u, r, 0); kc = __shfl_sync(~0u, kc, 0); }
    if (MODE >= 2) { np8 = uniform_ballot(np8); r = uniform_ballot(r); kc = uniform_ballot(kc); }
    const uint32_t idesc = idesc_bf16(128, max(16, round_up(r, 16)));
    const uint32_t ring = smem_u32(buf);
    unsigned long long t0 = clock64();
    uint32_t acc = 0;
    int slot = 0;
    for (int s = 0; s < stages; ++s) {
      const uint32_t xb = ring + slot * 49152;
      uint64_t adesc = smem_desc(xb, 16, 1024, 2), bdesc = smem_desc(xb + kc * np8 * 128, 16, 1024, 2);
      const uint32_t xstep = (uint32_t)(np8 * 128) >> 4, astep = (uint32_t)(r * 128) >> 4;
      for (int c = 0; c < kc; ++c) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          if (MODE == 3) {
            if (elect_one()) umma_bf16(tmem, adesc + 2 * kk, bdesc + 2 * kk, idesc, acc);
          } else {
            umma_elect(tmem, adesc + 2 * kk, bdesc + 2 * kk, idesc, acc);
          }
          acc = 1;
        }
        adesc += xstep;
        bdesc += astep;
      }
      if (++slot == 4) slot = 0;
    }
    if (elect_one()) umma_commit(bar);
    __syncwarp();
    mbar_wait(bar, 0);
    if (threadIdx.x == 32) out[0] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x >= 32) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int MODE>
void run(unsigned long long* d, int* p, const char* name) {
  const int smem = 200 * 1024 + 2048, stages = 64;
  cudaFuncSetAttribute(uni<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long h = 0;
  for (int it = 0; it < 2; ++it) { uni<MODE><<<1, 64, smem>>>(d, p, stages); cudaDeviceSynchronize(); }
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-40s %6.1f cycles/MMA (%s)\n", name, (double)h / (stages * 4 * 4), cudaGetErrorString(cudaGetLastError()));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  int* p;
  cudaMalloc(&p, 16);
  int hp[4] = {48, 16, 4, 0};
  cudaMemcpy(p, hp, 16, cudaMemcpyHostToDevice);
  run<0>(d, p, "R values, elect inside asm");
  run<1>(d, p, "shfl values, elect inside asm");
  run<2>(d, p, "ballot-uniform values, elect inside asm");
  run<3>(d, p, "ballot-uniform values, if(elect) branch");
  return 0;
}
