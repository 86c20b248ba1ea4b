// tma_red_bw.cu — development microbenchmark: can the expand add its delta into y with a TMA
// bulk tensor reduce-add (performed in L2) at HBM speed?  y = [4096 x 11008] bf16 (90 MB), tiles
// of 48 rows x 256 columns (4 boxes of 48x64, SWIZZLE_128B) like the expand's items, 148 CTAs
// striding over the tiles.  Modes: 0 = TMA reduce-add from smem, 1 = TMA store from smem,
// 2 = TMA load + TMA store (the y read-modify-write the expand does today, minus the math).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tma_red_bw tools/tma_red_bw.cu -lcuda
#include <cuda.h>
#include <cstdio>
#include <vector>
#include "../paper_2511_22880_b200/csrc/lsv_common.cuh"
using namespace lsv;

constexpr int ROWS = 48, COLS = 256, TOK = 4096, HOUT = 11008;
constexpr int TILE_BYTES = ROWS * COLS * 2;   // 24 KB
#ifndef NBUF_
#define NBUF_ 4
#endif
constexpr int NBUF = NBUF_;

__device__ __forceinline__ void tma_reduce_add_2d(const void* tmap, const void* src, int c0, int c1) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(tmap),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}

__global__ void __launch_bounds__(128, 1) bw(const __grid_constant__ CUtensorMap map, int mode, int ntiles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* buf = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(buf + NBUF * TILE_BYTES);
  for (int i = threadIdx.x; i < NBUF * TILE_BYTES / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(buf)[i] = make_uint4(0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { for (int b = 0; b < NBUF; ++b) mbar_init(&bar[b], 1); fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int tiles_c = HOUT / COLS, tiles_r = TOK / ROWS;
  int k = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
    const int tr = (t / tiles_c) % tiles_r, tc = t % tiles_c;
    const int b = k % NBUF;
    uint8_t* s = buf + b * TILE_BYTES;
    if (k >= NBUF) bulk_wait_group_read<NBUF - 1>();   // this buffer's previous TMA has read smem
    if (mode == 2) {
      mbar_arrive_expect_tx(&bar[b], TILE_BYTES);
      for (int h = 0; h < 4; ++h) tma_load_2d(s + h * ROWS * 128, &map, &bar[b], tc * COLS + h * 64, tr * ROWS);
      mbar_wait(&bar[b], (k / NBUF) & 1);
    }
    for (int h = 0; h < 4; ++h) {
      if (mode == 0) tma_reduce_add_2d(&map, s + h * ROWS * 128, tc * COLS + h * 64, tr * ROWS);
      else tma_store_2d(&map, s + h * ROWS * 128, tc * COLS + h * 64, tr * ROWS);
    }
    bulk_commit_group();
  }
  bulk_wait_group<0>();
}

int main() {
  void* y;
  const size_t bytes = (size_t)TOK * HOUT * 2;
  cudaMalloc(&y, bytes);
  cudaMemset(y, 0, bytes);
  CUtensorMap map;
  cuuint64_t dims[2] = {HOUT, TOK}, strides[1] = {HOUT * 2};
  cuuint32_t box[2] = {64, ROWS}, es[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, y, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  const int smem = NBUF * TILE_BYTES + 2048;
  cudaFuncSetAttribute(bw, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int ntiles = (TOK / ROWS) * (HOUT / COLS);
  const size_t moved = (size_t)ntiles * TILE_BYTES;   // bytes of y covered (each read + written in DRAM)
  // L2 flush buffer
  void* flush; cudaMalloc(&flush, 256 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[3] = {"TMA reduce-add bf16", "TMA store", "TMA load + TMA store"};
  for (int mode = 0; mode < 3; ++mode) {
    float best = 1e9;
    for (int it = 0; it < 5; ++it) {
      cudaMemset(flush, it, 256 << 20);
      cudaEventRecord(e0);
      bw<<<148, 128, smem>>>(map, mode, ntiles);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (it > 0 && ms < best) best = ms;
    }
    const double rw = (mode == 1 ? 1.0 : 2.0) * moved;   // DRAM bytes: store = write only; reduce / RMW = read + write
    printf("%-22s %8.1f us  y %5.1f MB  DRAM-equivalent %7.1f GB/s  (%s)\n", names[mode], best * 1e3, moved / 1e6,
           rw / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
