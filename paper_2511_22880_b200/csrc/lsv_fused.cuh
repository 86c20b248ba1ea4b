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
// main loop of item k+1.  Stage ring: 4 × 48 KB slots; a base stage is x [128 × 64] (16 KB) + W
// [256 × 64] (32 KB); a LoRA stage is one K chunk (ck = swizzle-row elements of the v image) of the
// piece's v image (128 × S bytes; the hi image's chunks, then the lo image's) + the matching
// k-groups of its B tile (ck/8 × 4 KB).
#pragma once
#include <cuda.h>

#include "lsv_common.cuh"
#include "lsv_plan.h"

namespace lsv {

constexpr int kFusedThreads = 256;
#ifndef LSV_FUSED_SLOTS
#define LSV_FUSED_SLOTS 4
#endif
constexpr int kFusedSlots = LSV_FUSED_SLOTS;
constexpr int kFusedSlotBytes = 48 * 1024;
constexpr int kFusedTileN = 256;
constexpr int kFusedTmemCols = 512;   // two 256-column accumulators
constexpr int kMaxPieces = 128;       // segment pieces in one 128-token tile, at most

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
  uint64_t* trace;                     // debug timeline (nullptr = off): [cta][item][16], slots 8..15 clock64
  int trace_items;
  int dbg;                             // debug ablations (0 in production): 1 = skip the LoRA stages,
                                       // 2 = skip their MMAs, 4 = skip their loads, 8 = K-major B idesc
};

__host__ __device__ constexpr int fused_smem_bytes() {
  return 1024 + kFusedSlots * kFusedSlotBytes + 1024 + 2 * kMaxPieces * (int)sizeof(MTile);
}

// The item's (member, tile m, tile n).  m fastest: the CTAs resident at once work on a few W
// n-tiles for every token tile, so each W tile is read from HBM once, while x (N x h_in, e.g.
// 33.5 MB at C2) stays L2-resident across the waves.  (n fastest streamed all of W once per wave:
// 2.0 GB of DRAM reads for C2's gate/up group, measured with ncu.)
__device__ __forceinline__ void fused_item(const FusedParams& p, int item, int& pp, int& m, int& n) {
  pp = 0;
  while (item >= p.item_base[pp + 1]) ++pp;
  const int q = item - p.item_base[pp];
  m = q % p.n_mtiles;
  n = q / p.n_mtiles;
}

// Base stages after which a LoRA stage is interleaved (LSV_FUSED_INTERLEAVE = 4: one per four base
// stages).  Default 0: every LoRA stage after the base loop.  Measured on C2's q/k/v group: after
// the loop 337 us, interleaved every 4th stage 353 us (the short LoRA stages then cut the ring's
// lead for the base stages that follow them in the middle of the loop).
__device__ __forceinline__ void fstamp(const FusedParams& p, int k, int slot) {
  if (p.trace != nullptr && k < p.trace_items) p.trace[((size_t)blockIdx.x * p.trace_items + k) * 16 + slot] = clock64();
}
#ifndef LSV_FUSED_INTERLEAVE
#define LSV_FUSED_INTERLEAVE 0
#endif
__device__ __forceinline__ bool fused_lora_slot(int c) {
  return LSV_FUSED_INTERLEAVE > 0 && c >= 4 && c % (LSV_FUSED_INTERLEAVE > 0 ? LSV_FUSED_INTERLEAVE : 1) == 0;
}

// LoRA units of an item, packed into stages: piece j's K chunk c (ck = S/2 k of its v image, S the
// v image's swizzle row bytes) as [v_hi chunk][v_lo chunk][B chunk] = 512·S bytes when split v fits
// (S <= 64), else one unit per half, [v chunk][B chunk] = 384·S bytes.  Consecutive units share a
// stage while they fit kFusedSlotBytes, so the low-rank pieces of a tile (S = 32 or 64) cost one
// stage together instead of one pipeline turn each.  Producer and MMA issuer walk the same cursor.
struct LoraCursor {
  int j, c, h;      // piece, chunk, half (split v with S = 128: 0 = hi, 1 = lo)
};
struct LoraUnit {
  MTile mt;
  int kp, S, ck;
  bool both;        // hi and lo in this unit
  uint32_t bytes;
};
__device__ __forceinline__ void lora_unit(const MTile* mts, const LoraCursor& cur, int vsplit, LoraUnit& u) {
  u.mt = mts[cur.j];
  u.kp = kpad(u.mt.rank);
  u.S = kmajor_row_bytes(u.kp);
  u.ck = u.S / 2;
  u.both = vsplit && u.S <= 64;
  u.bytes = (uint32_t)(u.both ? 512 : 384) * u.S;
}
__device__ __forceinline__ void lora_advance(LoraCursor& cur, const LoraUnit& u, int vsplit) {
  if (vsplit && !u.both && cur.h == 0) { cur.h = 1; return; }
  cur.h = 0;
  if (++cur.c == u.kp / u.ck) { cur.c = 0; ++cur.j; }
}
// Units of the stage starting at cur (advances cur past them); returns the stage's bytes.
__device__ __forceinline__ uint32_t lora_stage(const MTile* mts, LoraCursor& cur, int j1, int vsplit, int& nunits) {
  uint32_t used = 0;
  nunits = 0;
  while (cur.j < j1) {
    LoraUnit u;
    lora_unit(mts, cur, vsplit, u);
    if (used + u.bytes > (uint32_t)kFusedSlotBytes) break;
    used += u.bytes;
    ++nunits;
    lora_advance(cur, u, vsplit);
  }
  return used;
}

// A tile's piece records (<= 128: a tile has 128 tokens) copied to the warp's shared-memory cache.
// The loads are issued early in the item (tile bounds at base stage 0, records a few stages later)
// and stored after the base loop, so the plan's dependent global loads never stall the pipeline
// (measured: ~9K cycles per item when the MMA warp read them from L2 between LoRA stages).
struct PieceRegs {
  int tb;           // lane 0: tile_mt[m], lane 1: tile_mt[m + 1]
  int j0, j1;
  int4 r0, r1;      // lane l: record j0 + l
};
__device__ __forceinline__ void pieces_bounds(const int32_t* tile_mt, int m, int lane, PieceRegs& pr) {
  if (lane < 2) pr.tb = tile_mt[m + lane];
}
__device__ __forceinline__ void pieces_records(const MTile* mts, int lane, PieceRegs& pr) {
  pr.j0 = __shfl_sync(0xffffffffu, pr.tb, 0);
  pr.j1 = __shfl_sync(0xffffffffu, pr.tb, 1);
  if (lane < pr.j1 - pr.j0) {
    const int4* src = reinterpret_cast<const int4*>(mts + pr.j0 + lane);
    pr.r0 = src[0];
    pr.r1 = src[1];
  }
}
__device__ __forceinline__ void pieces_store(const MTile* mts, int lane, const PieceRegs& pr, MTile* cache) {
  const int n = min(pr.j1 - pr.j0, kMaxPieces);
  if (lane < n) {
    int4* dst = reinterpret_cast<int4*>(cache + lane);
    dst[0] = pr.r0;
    dst[1] = pr.r1;
  }
  for (int i = 32 + lane; i < n; i += 32) cache[i] = mts[pr.j0 + i];
  __syncwarp();
}

__global__ void __launch_bounds__(kFusedThreads, 1) fused_linear_kernel(const __grid_constant__ FusedParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* ring = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + kFusedSlots * kFusedSlotBytes);
  uint64_t* empty = full + kFusedSlots;
  uint64_t* tfull = empty + kFusedSlots;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  MTile* pcache = reinterpret_cast<MTile*>(ring + kFusedSlots * kFusedSlotBytes + 1024);   // [2][kMaxPieces]

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

  if (warp == 0) {  // ---------------- TMA producer: the warp walks the items, lane 0 issues
    MTile* cache = pcache;
    int slot = 0;
    uint32_t phase = 0;
    auto next = [&]() { if (++slot == kFusedSlots) { slot = 0; phase ^= 1; } };
    int kt = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++kt) {
      int pp, m, n;
      fused_item(p, item, pp, m, n);
      if (lane == 0) fstamp(p, kt, 8);
      PieceRegs pr;
      pieces_bounds(tile_mt, m, lane, pr);
      int np = 0;
      LoraCursor cur{0, 0, 0};
      auto lora_stage_issue = [&]() {   // one packed stage of the tile's LoRA units
        LoraCursor at = cur;
        int nu;
        const uint32_t bytes = lora_stage(cache, cur, np, p.vsplit, nu);
        if (lane == 0) {
          mbar_wait(&empty[slot], phase ^ 1);
          uint8_t* dst = ring + slot * kFusedSlotBytes;
          mbar_arrive_expect_tx(&full[slot], (p.dbg & 4) ? 0u : bytes);
          for (int i = 0; i < nu && !(p.dbg & 4); ++i) {
            LoraUnit u;
            lora_unit(cache, at, p.vsplit, u);
            const uint8_t* vimg = p.ws + p.ws_vimg[pp] + u.mt.vimg_off;
            const uint32_t vb = kTileM * u.S, bb = u.ck / 8 * 4096, lo = vimg_bytes(kTileM, u.kp);
            LSV_DCHECK(u.mt.tok_begin / kTileM == m && u.mt.tok_begin + u.mt.ntok <= p.num_tokens);
            LSV_DCHECK(bytes <= (uint32_t)kFusedSlotBytes && at.c * u.ck < u.kp);
            const uint8_t* bt = static_cast<const uint8_t*>(p.b_ptrs[pp][u.mt.seg]) + (size_t)n * kFusedTileN * u.kp * 2;
            bulk_load(dst, vimg + (at.h ? lo : 0u) + (size_t)at.c * vb, vb, &full[slot]);
            if (u.both) bulk_load(dst + vb, vimg + lo + (size_t)at.c * vb, vb, &full[slot]);
            bulk_load(dst + (u.both ? 2 : 1) * vb, bt + (size_t)at.c * bb, bb, &full[slot]);
            dst += u.bytes;
            lora_advance(at, u, p.vsplit);
          }
        }
        __syncwarp();
        next();
      };
      for (int c = 0; c < kch; ++c) {   // base GEMM: x and W boxes of K chunk c
        if (c == min(1, kch - 1)) pieces_records(mts, lane, pr);
        if (lane == 0) {
          mbar_wait(&empty[slot], phase ^ 1);
          uint8_t* dst = ring + slot * kFusedSlotBytes;
          mbar_arrive_expect_tx(&full[slot], (kTileM + kFusedTileN) * 128);
          tma_load_2d(dst, &p.xmap, &full[slot], c * kChunk, m * kTileM);
          tma_load_2d(dst + kTileM * 128, &p.wmap[pp], &full[slot], c * kChunk, n * kFusedTileN);
        }
        __syncwarp();
        next();
        if (c == min(3, kch - 1)) {
          pieces_store(mts, lane, pr, cache);
          np = (p.dbg & 1) ? 0 : min(pr.j1 - pr.j0, kMaxPieces);
        }
        if (fused_lora_slot(c) && cur.j < np) lora_stage_issue();
      }
      if (lane == 0) fstamp(p, kt, 9);
      while (cur.j < np) lora_stage_issue();   // what did not fit between the base stages
      if (lane == 0) fstamp(p, kt, 10);
    }
  } else if (warp == 1) {  // ---------------- MMA issuer: the whole converged warp runs the loop, the
    // election happens inside each MMA's asm (no per-instruction uniformization waterfall)
    int slot = 0;
    uint32_t phase = 0;
    auto next = [&]() { if (++slot == kFusedSlots) { slot = 0; phase ^= 1; } };
    const uint32_t ring_base = smem_u32(ring);
    const uint32_t idesc_kk = idesc_bf16(kTileM, kFusedTileN, 0);   // A, B K-major
    const uint32_t idesc_kn = idesc_bf16(kTileM, kFusedTileN, 1);   // B MN-major (the B tile)
    MTile* cache = pcache + kMaxPieces;
    int k = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++k) {
      int pp, m, n;
      fused_item(p, item, pp, m, n);
      PieceRegs pr;
      pieces_bounds(tile_mt, m, lane, pr);
      const int buf = k & 1;
      mbar_wait(&tempty[buf], ((k >> 1) & 1) ^ 1);
      tc_fence_after();
      if (lane == 0) fstamp(p, k, 11);
      const uint32_t d = tmem_base + buf * kFusedTileN;
      int np = 0;
      LoraCursor cur{0, 0, 0};
      auto lora_stage_mma = [&]() {   // D += v · B for the units of one packed stage
        LoraCursor at = cur;
        int nu;
        lora_stage(cache, cur, np, p.vsplit, nu);
        mbar_wait(&full[slot], phase);
        tc_fence_after();
        uint32_t sb = ring_base + slot * kFusedSlotBytes;
        for (int i = 0; i < nu; ++i) {
          LoraUnit u;
          lora_unit(cache, at, p.vsplit, u);
          const uint32_t vlay = umma_layout(u.S), vb = kTileM * u.S, boff = (u.both ? 2 : 1) * vb;
          for (int ks = 0; ks < u.ck / 16 && !(p.dbg & 2); ++ks) {   // K=16 steps inside the chunk
            const uint64_t bdesc = smem_desc(sb + boff + ks * 2 * 4 * 1024, 1024, 4 * 1024, 2);
            umma_bf16_elect(d, smem_desc(sb + ks * 32, 16, 8 * u.S, vlay), bdesc, idesc_kn, 1u);
            if (u.both) umma_bf16_elect(d, smem_desc(sb + vb + ks * 32, 16, 8 * u.S, vlay), bdesc, idesc_kn, 1u);
          }
          sb += u.bytes;
          lora_advance(at, u, p.vsplit);
        }
        umma_commit_elect(&empty[slot]);
        next();
      };
      for (int c = 0; c < kch; ++c) {
        if (c == min(1, kch - 1)) pieces_records(mts, lane, pr);
        mbar_wait(&full[slot], phase);
        tc_fence_after();
        const uint32_t sb = ring_base + slot * kFusedSlotBytes;
        const uint64_t adesc = smem_desc(sb, 16, 1024, 2);
        const uint64_t bdesc = smem_desc(sb + kTileM * 128, 16, 1024, 2);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16_elect(d, adesc + 2 * kk, bdesc + 2 * kk, idesc_kk, (c | kk) ? 1u : 0u);
        umma_commit_elect(&empty[slot]);
        next();
        if (c == min(3, kch - 1)) {
          pieces_store(mts, lane, pr, cache);
          np = (p.dbg & 1) ? 0 : min(pr.j1 - pr.j0, kMaxPieces);
        }
        if (fused_lora_slot(c) && cur.j < np) lora_stage_mma();
      }
      if (lane == 0) fstamp(p, k, 12);
      while (cur.j < np) lora_stage_mma();
      if (lane == 0) fstamp(p, k, 13);
      umma_commit_elect(&tfull[buf]);
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
      if (q == 0 && lane == 0) fstamp(p, k, 14);
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
      if (q == 0 && lane == 0) fstamp(p, k, 15);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) { tc_fence_after(); tmem_dealloc(tmem_base, kFusedTmemCols); }
}

}  // namespace lsv
