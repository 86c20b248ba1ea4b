// Microbenchmark (development aid): cost of single-thread tcgen05 issue-path operations on one SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/micro_issue tools/micro_issue.cu
#include <cstdio>
#include "../paper_2511_22880_b200/csrc/lsv_common.cuh"
using namespace lsv;

__global__ void __launch_bounds__(128, 1) micro(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* buf = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(buf + 65536);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 8);
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) reinterpret_cast<uint4*>(buf)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    for (int b = 0; b < 8; ++b) mbar_init(&bars[b], 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(buf), b = smem_u32(buf + 32768);
    const uint32_t idesc = idesc_bf16(128, 128, 0);
    unsigned long long t0, t1;
    // (1) clock read overhead
    t0 = clock64(); for (int i = 0; i < iters; ++i) { asm volatile("" ::: "memory"); } t1 = clock64(); out[0] = (t1 - t0);
    // (2) globaltimer read
    t0 = clock64(); unsigned long long acc = 0; for (int i = 0; i < iters; ++i) acc += globaltimer_ns(); t1 = clock64(); out[1] = (t1 - t0); out[15] = acc;
    // (3) mbarrier arrive + try_wait on the completed phase
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { mbar_arrive(&bars[0]); mbar_wait(&bars[0], i & 1); }
    t1 = clock64(); out[2] = (t1 - t0);
    // (4) issue one 128x128x16 MMA (SW128 K-major operands) per iteration, no waits
    t0 = clock64();
    for (int i = 0; i < iters; ++i) umma_bf16(tmem, smem_desc(a, 16, 1024, 2), smem_desc(b, 16, 1024, 2), idesc, i > 0);
    t1 = clock64(); out[3] = (t1 - t0);
    umma_commit(&bars[1]); mbar_wait(&bars[1], 0);
    t1 = clock64(); out[4] = (t1 - t0);  // including drain
    // (5) MMA + commit + wait each iteration (round trip latency)
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      umma_bf16(tmem, smem_desc(a, 16, 1024, 2), smem_desc(b, 16, 1024, 2), idesc, 1);
      umma_commit(&bars[2]); mbar_wait(&bars[2], i & 1);
    }
    t1 = clock64(); out[5] = (t1 - t0);
    // (6) 4 MMAs (N=128) then commit+wait (pipelined group)
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      for (int j = 0; j < 4; ++j) umma_bf16(tmem + 128 * (j & 1), smem_desc(a + 32 * j, 16, 1024, 2), smem_desc(b + 32 * j, 16, 1024, 2), idesc, 1);
      umma_commit(&bars[3]); mbar_wait(&bars[3], i & 1);
    }
    t1 = clock64(); out[6] = (t1 - t0);
    // (7) MN-major B (SW128) 128x128x16
    const uint32_t idesc_mn = idesc_bf16(128, 128, 1);
    t0 = clock64();
    for (int i = 0; i < iters; ++i) umma_bf16(tmem, smem_desc(a, 16, 1024, 2), smem_desc(b, 1024, 2048, 2), idesc_mn, 1);
    umma_commit(&bars[4]); mbar_wait(&bars[4], 0);
    t1 = clock64(); out[7] = (t1 - t0);
    // (8) no-swizzle (interleaved) operands
    t0 = clock64();
    for (int i = 0; i < iters; ++i) umma_bf16(tmem, smem_desc(a, 128, 256, 0), smem_desc(b, 128, 256, 0), idesc, 1);
    umma_commit(&bars[5]); mbar_wait(&bars[5], 0);
    t1 = clock64(); out[8] = (t1 - t0);
    // (9) commit alone
    t0 = clock64();
    for (int i = 0; i < iters; ++i) umma_commit(&bars[6]);
    t1 = clock64(); out[9] = (t1 - t0);
    mbar_wait(&bars[6], (iters - 1) & 1);
    // (10) 128x256x16 MMAs
    const uint32_t idesc256 = idesc_bf16(128, 256, 0);
    t0 = clock64();
    for (int i = 0; i < iters; ++i) umma_bf16(tmem, smem_desc(a, 16, 1024, 2), smem_desc(b, 16, 1024, 2), idesc256, 1);
    umma_commit(&bars[7]); mbar_wait(&bars[7], 0);
    t1 = clock64(); out[10] = (t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16 * sizeof(unsigned long long));
  cudaMemset(d, 0, 16 * 8);
  const int smem = 65536 + 1024 + 1024;
  cudaFuncSetAttribute(micro, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 256;
  micro<<<1, 128, smem>>>(d, iters);
  micro<<<1, 128, smem>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[16];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const char* names[] = {"empty loop", "globaltimer read", "mbar arrive+wait(done)", "MMA 128x128x16 issue",
                         "  ... incl drain", "MMA+commit+wait roundtrip", "4 MMA+commit+wait", "MMA MN-major B",
                         "MMA interleaved", "commit alone", "MMA 128x256x16"};
  printf("status %s\n", cudaGetErrorString(e));
  for (int i = 0; i < 11; ++i) printf("%-28s %8.1f cycles/iter\n", names[i], (double)h[i] / iters);
  return 0;
}
