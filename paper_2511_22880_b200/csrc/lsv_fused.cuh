// lsv_fused.cuh — the base projection GEMM with the LoRA expand fused into its TMEM tile.
//
//     y[t, :] = x[t, :] · W^T  +  (x[t, :] · A_s^T) · B_s^T        t in segment s
//
// SURVEY §8(f) item 4.  The reference prices a LoRA projection as one batch cost that includes the
// base model's GEMM (costmodel.py:104-105, (b + a·ΣL)·(1 + c·r/tp)); S-LoRA, which the paper runs on
// (PAPER.md:532, :203), folds the delta into the base output.  Here the delta never touches y in
// HBM on its own: per output tile D[128 tokens × 256 h_out] (fp32, TMEM) the kernel runs the base
// GEMM's K loop (D += x_tile · W_tile^T, both K-major SWIZZLE_128B TMA boxes), then, for every
// segment piece inside the 128-token tile, D += v_piece · B_s (v from the shrink of a tile-aligned
// plan: a 128-row image with zeros outside the piece, so the M=128 MMA adds only into the piece's
// rows; with split v, once for v_hi and once for v_lo), and the epilogue writes y once.  Bytes
// saved against base GEMM + separate expand: the expand's y read-modify-write (4 · N · h_out).
//
// Persistent, one CTA per SM, items = (member, 128-token tile, 256-wide h_out tile) dealt round
// robin; warp 0 = TMA producer, warp 1 = MMA issuer (TMEM owner), warps 4..7 = epilogue (TMEM lane
// quadrant warp % 4), two 256-column TMEM accumulators so the epilogue of item k overlaps the
// main loop of item k+1.  Stage ring: 3 × 64 KB slots; a base stage is x [128 × 64] (16 KB) + W
// [256 × 64] (32 KB); a LoRA stage is one K chunk (ck = swizzle-row elements of the v image) of the
// piece's v image (128 × S bytes, hi then lo) + the matching k-groups of its B tile (ck/8 × 4 KB).
#pragma once
#include <cuda.h>

#include "lsv_common.cuh"
#include "lsv_plan.h"

namespace lsv {

constexpr int kFusedThreads = 256;
constexpr int kFusedSlots = 3;
constexpr int kFusedSlotBytes = 64 * 1024;
constexpr int kFusedTileN = 256;
constexpr int kFusedTmemCols = 512;   // two 256-column accumulators

struct alignas(64) FusedParams {
  CUtensorMap xmap;                    // x [num_tokens][h_in], box {64 cols, 128 rows}, SWIZZLE_128B
  CUtensorMap wmap[kMaxProj];          // W_p [h_out_p][h_in] (nn.Linear weight), box {64, 256}, SW128
  const int32_t* plan;                 // tile-aligned plan (device)
  const void* const* b_ptrs[kMaxProj]; // per member: [S] device pointers to the segments' B tiles
  const uint8_t* ws;                   // workspace holding the shrink's v images
  __nv_bfloat16* y[kMaxProj];
  int64_t ldy[kMaxProj];
  int ws_vimg[kMaxProj];               // byte offset of member p's v images in ws
  int n_ntiles[kMaxProj];              // h_out_p / 256
  int item_base[kMaxProj + 1];         // items of member p: [item_base[p], item_base[p+1])
  int num_tokens, h_in, vsplit, n_mtiles;
  int off_mtiles, off_tile_mt;
};

__host__ __device__ constexpr int fused_smem_bytes() { return 1024 + kFusedSlots * kFusedSlotBytes + 1024; }

// The item's (member, tile m, tile n).  n fastest: the CTAs resident at once share x rows and
// sweep W, which together fit the 126 MB L2 for every Llama shape.
__device__ __forceinline__ void fused_item(const FusedParams& p, int item, int& pp, int& m, int& n) {
  pp = 0;
  while (item >= p.item_base[pp + 1]) ++pp;
  const int q = item - p.item_base[pp];
  m = q / p.n_ntiles[pp];
  n = q % p.n_ntiles[pp];
}

__global__ void __launch_bounds__(kFusedThreads, 1) fused_linear_kernel(const __grid_constant__ FusedParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* ring = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + kFusedSlots * kFusedSlotBytes);
  uint64_t* empty = full + kFusedSlots;
  uint64_t* tfull = empty + kFusedSlots;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kFusedSlots; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 4); }
    fence_mbar_init();
    prefetch_tmap(&p.xmap);
    for (int q = 0; q < kMaxProj; ++q)
      if (p.y[q]) prefetch_tmap(&p.wmap[q]);
  }
  if (warp == 1) tmem_alloc(tmem_slot, kFusedTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  asm volatile("griddepcontrol.wait;" ::: "memory");   // v images come from the shrink launch
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  const int n_items = p.item_base[kMaxProj];
  const int kch = p.h_in / kChunk;
  const MTile* mts = reinterpret_cast<const MTile*>(p.plan + p.off_mtiles);
  const int32_t* tile_mt = p.plan + p.off_tile_mt;

  if (warp == 0) {  // ---------------- TMA producer (lane 0)
    if (lane == 0) {
      int slot = 0;
      uint32_t phase = 0;
      auto next = [&]() { if (++slot == kFusedSlots) { slot = 0; phase ^= 1; } };
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        int pp, m, n;
        fused_item(p, item, pp, m, n);
        for (int c = 0; c < kch; ++c) {   // base GEMM: x and W boxes of K chunk c
          mbar_wait(&empty[slot], phase ^ 1);
          uint8_t* dst = ring + slot * kFusedSlotBytes;
          mbar_arrive_expect_tx(&full[slot], (kTileM + kFusedTileN) * 128);
          tma_load_2d(dst, &p.xmap, &full[slot], c * kChunk, m * kTileM);
          tma_load_2d(dst + kTileM * 128, &p.wmap[pp], &full[slot], c * kChunk, n * kFusedTileN);
          next();
        }
        const int j1 = tile_mt[m + 1];
        for (int j = tile_mt[m]; j < j1; ++j) {   // LoRA: every segment piece of this token tile
          const MTile mt = mts[j];
          const int kp = kpad(mt.rank), S = kmajor_row_bytes(kp), ck = S / 2;
          const uint8_t* vimg = p.ws + p.ws_vimg[pp] + mt.vimg_off;
          const uint8_t* btile = static_cast<const uint8_t*>(p.b_ptrs[pp][mt.seg]) + (size_t)n * kFusedTileN * kp * 2;
          const uint32_t vb = kTileM * S, bb = ck / 8 * 4096;
          for (int c = 0; c < kp / ck; ++c) {
            mbar_wait(&empty[slot], phase ^ 1);
            uint8_t* dst = ring + slot * kFusedSlotBytes;
            mbar_arrive_expect_tx(&full[slot], vb * (p.vsplit ? 2 : 1) + bb);
            bulk_load(dst, vimg + (size_t)c * vb, vb, &full[slot]);
            if (p.vsplit) bulk_load(dst + 16384, vimg + vimg_bytes(kTileM, kp) + (size_t)c * vb, vb, &full[slot]);
            bulk_load(dst + 32768, btile + (size_t)c * bb, bb, &full[slot]);
            next();
          }
        }
      }
    }
  } else if (warp == 1) {  // ---------------- MMA issuer (lane 0)
    if (lane == 0) {
      int slot = 0;
      uint32_t phase = 0;
      auto next = [&]() { if (++slot == kFusedSlots) { slot = 0; phase ^= 1; } };
      const uint32_t ring_base = smem_u32(ring);
      const uint32_t idesc_kk = idesc_bf16(kTileM, kFusedTileN, 0);   // A, B K-major
      const uint32_t idesc_kn = idesc_bf16(kTileM, kFusedTileN, 1);   // B MN-major (the B tile)
      int k = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++k) {
        int pp, m, n;
        fused_item(p, item, pp, m, n);
        const int buf = k & 1;
        mbar_wait(&tempty[buf], ((k >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + buf * kFusedTileN;
        for (int c = 0; c < kch; ++c) {
          mbar_wait(&full[slot], phase);
          tc_fence_after();
          const uint32_t sb = ring_base + slot * kFusedSlotBytes;
          const uint64_t adesc = smem_desc(sb, 16, 1024, 2);
          const uint64_t bdesc = smem_desc(sb + kTileM * 128, 16, 1024, 2);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) umma_bf16(d, adesc + 2 * kk, bdesc + 2 * kk, idesc_kk, (c | kk) ? 1u : 0u);
          umma_commit(&empty[slot]);
          next();
        }
        const int j1 = tile_mt[m + 1];
        for (int j = tile_mt[m]; j < j1; ++j) {
          const MTile mt = mts[j];
          const int kp = kpad(mt.rank), S = kmajor_row_bytes(kp), ck = S / 2;
          const uint32_t vlay = umma_layout(S);
          for (int c = 0; c < kp / ck; ++c) {
            mbar_wait(&full[slot], phase);
            tc_fence_after();
            const uint32_t sb = ring_base + slot * kFusedSlotBytes;
            for (int h = 0; h < (p.vsplit ? 2 : 1); ++h)
              for (int ks = 0; ks < ck / 16; ++ks) {   // K=16 steps inside the chunk
                const uint64_t adesc = smem_desc(sb + h * 16384 + ks * 32, 16, 8 * S, vlay);
                const uint64_t bdesc = smem_desc(sb + 32768 + ks * 2 * 4 * 1024, 1024, 4 * 1024, 2);
                umma_bf16(d, adesc, bdesc, idesc_kn, 1u);
              }
            umma_commit(&empty[slot]);
            next();
          }
        }
        umma_commit(&tfull[buf]);
      }
    }
  } else if (warp >= 4) {  // ---------------- epilogue: thread = token row of TMEM quadrant q
    const int q = warp & 3;
    int k = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++k) {
      int pp, m, n;
      fused_item(p, item, pp, m, n);
      const int buf = k & 1;
      mbar_wait(&tfull[buf], (k >> 1) & 1);
      tc_fence_after();
      const int t = m * kTileM + q * 32 + lane;
      const bool valid = t < p.num_tokens;
      __nv_bfloat16* yrow = p.y[pp] + (int64_t)(valid ? t : 0) * p.ldy[pp] + n * kFusedTileN;
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + buf * kFusedTileN;
      auto put = [&](const uint32_t* r, int cc) {
        uint32_t w[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) w[e] = pack_bf16x2(__uint_as_float(r[2 * e]), __uint_as_float(r[2 * e + 1]));
#pragma unroll
        for (int u = 0; u < 2; ++u) st_global_v8_if(yrow + cc + u * 16, &w[8 * u], valid);
      };
      uint32_t ra[32], rb[32];
      tmem_ld_32x32b_x32_nowait(taddr, ra);
#pragma unroll 1
      for (int cc = 0; cc < kFusedTileN; cc += 64) {   // chunk i+1's TMEM load overlaps chunk i's stores
        tmem_wait_ld_regs(ra);
        tmem_ld_32x32b_x32_nowait(taddr + cc + 32, rb);
        put(ra, cc);
        tmem_wait_ld_regs(rb);
        if (cc + 64 < kFusedTileN) tmem_ld_32x32b_x32_nowait(taddr + cc + 64, ra);
        put(rb, cc + 32);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) { tc_fence_after(); tmem_dealloc(tmem_base, kFusedTmemCols); }
}

}  // namespace lsv
