// expand_mem_bw.cu — development microbenchmark: the expand's memory traffic alone (no MMA, no
// cross-item dependencies).  Items = (48-row token tile m, 256-column h_out tile j): TMA-load the
// y tile (4 column blocks of 64, boxes of 32 + 16 rows, SWIZZLE_128B) and a contiguous B tile of
// BKB KB into a ring slot, then TMA-store the y tile back.  Reports GB/s of (B + 2 y) bytes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2511_22880_b200/csrc \
//        tools/expand_mem_bw.cu -o tools/expand_mem_bw -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <vector>
#include "lsv_common.cuh"
using namespace lsv;

struct Args {
  CUtensorMap ymap32, ymap16;
  const uint8_t* bsrc;
  int rows, cols, ntiles_m, ntiles_j, bkb, ns, slot;
  size_t bbytes_total;
  __nv_bfloat16* y;
  int stg;   // 1: write y back like the expand epilogue (thread = row, 16-byte stores) instead of TMA
};

__device__ __forceinline__ void tma_store_2d_(const void* tmap, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(tmap),
               "r"(smem_u32(src)), "r"(c0), "r"(c1) : "memory");
}

__global__ void __launch_bounds__(192, 1) kern(const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* ring = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + a.ns * a.slot);
  uint64_t* empty = full + 16;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < a.ns; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], a.stg ? 4 : 1); }
    fence_mbar_init();
  }
  __syncthreads();
  const int nitems = a.ntiles_m * a.ntiles_j;
  const uint32_t ybytes = 4 * 48 * 128, bbytes = a.bkb * 1024;
  if (warp == 0) {   // producer
    int slot = 0; uint32_t ph = 0;
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
      const int m = it / a.ntiles_j, j = it % a.ntiles_j;
      if (lane == 0) {
        mbar_wait(&empty[slot], ph ^ 1);
        mbar_arrive_expect_tx(&full[slot], ybytes + bbytes);
      }
      __syncwarp();
      uint8_t* dst = ring + slot * a.slot;
      if (lane == 0) {
        const size_t boff = ((size_t)(m * 131 + j) * bbytes) % (a.bbytes_total - bbytes);
        bulk_load(dst + ybytes, a.bsrc + boff / 1024 * 1024, bbytes, &full[slot]);
      } else if (lane <= 8) {
        const int h = (lane - 1) >> 1, part = (lane - 1) & 1;
        if (part == 0) tma_load_2d(dst + h * 48 * 128, &a.ymap32, &full[slot], j * 256 + h * 64, m * 48);
        else tma_load_2d(dst + h * 48 * 128 + 32 * 128, &a.ymap16, &full[slot], j * 256 + h * 64, m * 48 + 32);
      }
      if (++slot == a.ns) { slot = 0; ph ^= 1; }
    }
  } else if (a.stg && warp >= 2) {   // 4 warps: thread = row (48 rows), 32 x 16-byte STG per row
    const int t = (warp - 2) * 32 + lane;
    int slot = 0; uint32_t ph = 0;
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
      const int m = it / a.ntiles_j, j = it % a.ntiles_j;
      mbar_wait(&full[slot], ph);
      const uint8_t* src = ring + slot * a.slot;
      if (t < 48) {
        __nv_bfloat16* yrow = a.y + (size_t)(m * 48 + t) * a.cols + j * 256;
        for (int h = 0; h < 4; ++h)
          for (int c = 0; c < 8; ++c) {
            const uint4 w = *reinterpret_cast<const uint4*>(src + h * 48 * 128 + t * 128 + ((c ^ (t & 7)) << 4));
            *reinterpret_cast<uint4*>(yrow + h * 64 + c * 8) = w;
          }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      if (++slot == a.ns) { slot = 0; ph ^= 1; }
    }
  } else if (!a.stg && warp == 1 && lane == 0) {   // "consumer": stores the y tile back, then frees the slot
    int slot = 0; uint32_t ph = 0;
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
      const int m = it / a.ntiles_j, j = it % a.ntiles_j;
      mbar_wait(&full[slot], ph);
      uint8_t* src = ring + slot * a.slot;
      fence_proxy_async_smem();
      for (int h = 0; h < 4; ++h) {
        tma_store_2d_(&a.ymap32, src + h * 48 * 128, j * 256 + h * 64, m * 48);
        tma_store_2d_(&a.ymap16, src + h * 48 * 128 + 32 * 128, j * 256 + h * 64, m * 48 + 32);
      }
      bulk_commit_group();
      bulk_wait_group_read<0>();
      mbar_arrive(&empty[slot]);
      if (++slot == a.ns) { slot = 0; ph ^= 1; }
    }
    bulk_wait_group<0>();
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  const int rows = 4096, cols = 11008;
  const size_t ybytes = (size_t)rows * cols * 2, bt = 512ull << 20;
  uint8_t *y, *b;
  cudaMalloc(&y, ybytes); cudaMalloc(&b, bt);
  cudaMemset(y, 1, ybytes); cudaMemset(b, 2, bt);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)p;
  int nsm = 0; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int stg : {0, 1}) for (int bkb : {8, 32, 64}) for (int ns : {2, 3, 4}) {
    Args a{};
    a.stg = stg; a.y = reinterpret_cast<__nv_bfloat16*>(y);
    a.rows = rows; a.cols = cols; a.bsrc = b; a.bbytes_total = bt; a.bkb = bkb; a.ns = ns;
    a.slot = ((4 * 48 * 128 + bkb * 1024) + 1023) / 1024 * 1024;
    if (ns * a.slot + 1024 + 256 > 220 * 1024) continue;
    a.ntiles_m = rows / 48; a.ntiles_j = cols / 256;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows}, strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t b32[2] = {64, 32}, b16[2] = {64, 16}, es[2] = {1, 1};
    enc(&a.ymap32, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, y, dims, strides, b32, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&a.ymap16, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, y, dims, strides, b16, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int smem = ns * a.slot + 1024 + 256;
    float best = 1e9;
    for (int it = 0; it < 5; ++it) {
      cudaEventRecord(e0);
      kern<<<nsm, 192, smem>>>(a);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (it > 0 && ms < best) best = ms;
    }
    const double items = (double)a.ntiles_m * a.ntiles_j;
    const double bytes = items * (2.0 * 4 * 48 * 128 + bkb * 1024.0);
    printf("%s B tile %2d KB, %d slots x %3d KB: %7.1f us, %7.1f GB/s (%s)\n", stg ? "STG" : "TMA", bkb, ns, a.slot / 1024, best * 1e3,
           bytes / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
