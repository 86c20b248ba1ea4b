// tma_bw.cu — development microbenchmark: HBM read bandwidth of a persistent TMA streaming
// kernel over a row-major [rows][cols] bf16 matrix (the shrink's x access pattern), as a
// function of the box height R, the chunks per pipeline stage S and the number of stages NS;
// plus contiguous cp.async.bulk streaming for comparison.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2511_22880_b200/csrc \
//        tools/tma_bw.cu -o tools/tma_bw -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>

#include "lsv_common.cuh"
using namespace lsv;

struct Args {
  CUtensorMap map;
  const uint8_t* flat;
  int rows, cols, R, S, NS, slot_bytes, mode, bulk_bytes;
  long long total_bytes;
};

__global__ void __launch_bounds__(64, 1) tma_stream(const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* ring = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + a.NS * a.slot_bytes);
  uint64_t* empty = full + a.NS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < a.NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  const int chunks = a.cols / 64;
  const int bands = a.rows / a.R;
  if (a.mode == 0) {
    // 2D TMA: band b (R rows), stage = S consecutive 64-column chunks
    const int stages_per_band = chunks / a.S;
    if (warp == 0) {
      int slot = 0; uint32_t ph = 0;
      for (int b = blockIdx.x; b < bands; b += gridDim.x) {
        for (int st = 0; st < stages_per_band; ++st) {
          if (lane == 0) {
            mbar_wait(&empty[slot], ph ^ 1);
            mbar_arrive_expect_tx(&full[slot], (uint32_t)(a.S * a.R * 128));
          }
          __syncwarp();
          if (lane < a.S)
            tma_load_2d(ring + slot * a.slot_bytes + lane * a.R * 128, &a.map, &full[slot], (st * a.S + lane) * 64,
                        b * a.R);
          if (++slot == a.NS) { slot = 0; ph ^= 1; }
        }
      }
    } else if (lane == 0) {
      int slot = 0; uint32_t ph = 0;
      for (int b = blockIdx.x; b < bands; b += gridDim.x)
        for (int st = 0; st < stages_per_band; ++st) {
          mbar_wait(&full[slot], ph);
          mbar_arrive(&empty[slot]);
          if (++slot == a.NS) { slot = 0; ph ^= 1; }
        }
    }
  } else {
    // contiguous bulk copies of bulk_bytes, CTA-interleaved
    const long long n = a.total_bytes / a.bulk_bytes;
    if (warp == 0) {
      if (lane == 0) {
        int slot = 0; uint32_t ph = 0;
        for (long long i = blockIdx.x; i < n; i += gridDim.x) {
          mbar_wait(&empty[slot], ph ^ 1);
          mbar_arrive_expect_tx(&full[slot], (uint32_t)a.bulk_bytes);
          bulk_load(ring + slot * a.slot_bytes, a.flat + i * a.bulk_bytes, a.bulk_bytes, &full[slot]);
          if (++slot == a.NS) { slot = 0; ph ^= 1; }
        }
      }
    } else if (lane == 0) {
      int slot = 0; uint32_t ph = 0;
      for (long long i = blockIdx.x; i < n; i += gridDim.x) {
        mbar_wait(&full[slot], ph);
        mbar_arrive(&empty[slot]);
        if (++slot == a.NS) { slot = 0; ph ^= 1; }
      }
    }
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int rows = 32768, cols = 4096;
  const size_t bytes = (size_t)rows * cols * 2;
  uint8_t* x;
  cudaMalloc(&x, bytes);
  cudaMemset(x, 1, bytes);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)p;
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Cfg { int mode, R, S, NS, bulk; const char* l2; };
  std::vector<Cfg> cfgs = {
      {0, 48, 1, 8, 0, "none"}, {0, 48, 4, 4, 0, "none"}, {0, 48, 4, 8, 0, "none"}, {0, 48, 8, 4, 0, "none"},
      {0, 48, 16, 2, 0, "none"}, {0, 48, 8, 6, 0, "none"},
      {0, 128, 1, 8, 0, "none"}, {0, 128, 2, 6, 0, "none"}, {0, 128, 4, 3, 0, "none"},
      {0, 48, 4, 4, 0, "256B"}, {0, 48, 8, 4, 0, "256B"},
      {0, 16, 16, 4, 0, "none"}, {0, 8, 16, 8, 0, "none"},
      {1, 0, 0, 4, 16384, ""}, {1, 0, 0, 4, 32768, ""}, {1, 0, 0, 6, 32768, ""}, {1, 0, 0, 4, 49152, ""},
      {1, 0, 0, 8, 16384, ""}, {1, 0, 0, 12, 16384, ""}, {1, 0, 0, 3, 65536, ""},
  };
  for (const Cfg& c : cfgs) {
    Args a{};
    a.rows = rows; a.cols = cols; a.R = c.R; a.S = c.S; a.NS = c.NS; a.mode = c.mode; a.flat = x;
    a.total_bytes = (long long)bytes; a.bulk_bytes = c.bulk;
    if (c.mode == 0) {
      a.slot_bytes = c.S * c.R * 128;
      cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
      cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
      cuuint32_t box[2] = {64, (cuuint32_t)c.R};
      cuuint32_t es[2] = {1, 1};
      CUtensorMapL2promotion prom = c.l2[0] == '2' ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE;
      CUresult r = enc(&a.map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, prom, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); continue; }
    } else {
      a.slot_bytes = c.bulk;
    }
    const int smem = a.NS * a.slot_bytes + 2 * a.NS * 8 + 1024;
    if (smem > 220 * 1024) { printf("skip smem %d\n", smem); continue; }
    float best = 1e9;
    for (int it = 0; it < 6; ++it) {
      cudaEventRecord(e0);
      tma_stream<<<nsm, 64, smem>>>(a);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it > 0 && ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    if (c.mode == 0)
      printf("2D  R=%3d S=%2d NS=%2d slot=%6d KB in flight/SM=%4d l2=%s: %7.1f GB/s %s\n", c.R, c.S, c.NS, a.slot_bytes,
             a.NS * a.slot_bytes / 1024, c.l2, bytes / (best * 1e-3) / 1e9, cudaGetErrorString(err));
    else
      printf("BULK bytes=%6d NS=%2d in flight/SM=%4d KB: %7.1f GB/s %s\n", c.bulk, c.NS, a.NS * c.bulk / 1024,
             bytes / (best * 1e-3) / 1e9, cudaGetErrorString(err));
  }
  return 0;
}
