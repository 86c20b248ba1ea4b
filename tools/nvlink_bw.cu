// NVLink peer-read bandwidth on this box (the ceiling for config 4's in-kernel peer loads).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvlink_bw tools/nvlink_bw.cu && tools/nvlink_bw
// GPU 0 reads a 2 GiB buffer resident on GPU 1: (a) cp.async.bulk into shared memory (what the
// delta kernels do), every SM streaming 32 KB chunks with 4 in flight; (b) 16-byte ld.global per
// thread; (c) copy engine (cudaMemcpyPeerAsync).  Also (d) the same bulk reads from local HBM, and
// (e) local + peer at once (two buffers, half the CTAs each) to see whether they add up.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(128) bulk_read(const uint8_t* src, size_t bytes, int chunk, unsigned long long* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[4];
  const int nbuf = 4;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nbuf; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const size_t nchunks = bytes / chunk;
  uint32_t phase[4] = {0, 0, 0, 0};
  size_t k = 0;
  for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++k) {
    const int b = k % nbuf;
    if (k >= (size_t)nbuf) {   // wait for this buffer's previous copy
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.b32 %0, 1, 0, P;\n\t}\n"
                     : "=r"(done) : "r"(smem_u32(&bar[b])), "r"(phase[b]) : "memory");
      phase[b] ^= 1;
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[b])), "r"(chunk) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(sm + b * chunk)), "l"(src + c * chunk), "r"(chunk), "r"(smem_u32(&bar[b]))
                 : "memory");
  }
  for (int b = 0; b < nbuf && (size_t)b < k; ++b) {
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.b32 %0, 1, 0, P;\n\t}\n"
                   : "=r"(done) : "r"(smem_u32(&bar[b])), "r"(phase[b]) : "memory");
  }
  if (sm[0] == 0x5a && sm[1] == 0x5b) atomicAdd(sink, 1ull);
}

__global__ void ld_read(const uint4* src, size_t n, unsigned long long* sink) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const uint4 v = __ldcg(src + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678) atomicAdd(sink, 1ull);
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) { printf("need 2 GPUs\n"); return 1; }
  const size_t bytes = 2ull << 30;
  uint8_t *remote, *local, *local2;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&remote, bytes));
  CK(cudaMemset(remote, 1, bytes));
  CK(cudaDeviceSynchronize());
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&local, bytes));
  CK(cudaMalloc(&local2, bytes));
  CK(cudaMemset(local, 1, bytes));
  unsigned long long* sink;
  CK(cudaMalloc(&sink, 8));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int chunk = 32768;
  CK(cudaFuncSetAttribute(bulk_read, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * chunk));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto fn, double nbytes) {
    fn();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) fn();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-44s %8.1f GB/s\n", name, nbytes * 5 / (ms * 1e-3) / 1e9);
  };
  for (int ctas : {sms, 2 * sms}) {
    char nm[96];
    snprintf(nm, sizeof nm, "peer  bulk 32KB x4/CTA, %d CTAs", ctas);
    timeit(nm, [&] { bulk_read<<<ctas, 128, 4 * chunk>>>(remote, bytes, chunk, sink); }, (double)bytes);
  }
  timeit("peer  ld.global.cg 16B, 148x4 x 512 thr", [&] { ld_read<<<sms * 4, 512>>>((const uint4*)remote, bytes / 16, sink); }, (double)bytes);
  timeit("peer  copy engine (cudaMemcpyPeerAsync)", [&] { cudaMemcpyPeerAsync(local2, 0, remote, 1, bytes); }, (double)bytes);
  timeit("local bulk 32KB x4/CTA", [&] { bulk_read<<<sms, 128, 4 * chunk>>>(local, bytes, chunk, sink); }, (double)bytes);
  // both at once: two streams
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  timeit("local + peer together (74 CTAs each, sum)", [&] {
    bulk_read<<<sms / 2, 128, 4 * chunk, s1>>>(local, bytes, chunk, sink);
    bulk_read<<<sms / 2, 128, 4 * chunk, s2>>>(remote, bytes, chunk, sink);
    cudaStreamSynchronize(s1);
    cudaStreamSynchronize(s2);
  }, 2.0 * bytes);
  return 0;
}
