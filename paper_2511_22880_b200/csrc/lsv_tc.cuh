// lsv_tc.cuh — tcgen05 (5th-gen tensor core) tier of the mixed-rank LoRA delta.
//
// Shrink  D[128 tok × N=rank16] += x_tile[128 × 64k] · A_s^T            (TMEM accumulator)
//   x tile: TMA (cp.async.bulk.tensor, SWIZZLE_128B) of exactly ceil8(n) token rows per
//   64-column chunk, composed from 128/64/32/16/8-row boxes; A_s: one cp.async.bulk of a
//   pre-swizzled [kch chunks][rank][64] slab run.  Rows past the segment / columns past the
//   rank are garbage in, garbage out (row i of D only reads row i of x; column j only
//   row j of A) and are never stored.  k-splits are reduced deterministically by the
//   last-arriving CTA (fixed summation order) into the bf16 "v image".
// Expand  D[128 h_out × N=ntok16] = B_s^T[128 × rank16] · v^T            (swap-AB)
//   B tile and v image: one cp.async.bulk each; epilogue stages D through shared memory so
//   the y read-modify-write is 256-byte coalesced rows of 16-byte vectors.
//
// Warp roles (192 threads, one CTA per SM, persistent over a host-LPT-sorted work list
// assigned snake-wise): warp 0 = producer (one lane), warp 1 = MMA issuer (one lane) and
// TMEM owner, warps 2..5 = epilogue (warp w reads TMEM lanes 32*(w%4)..+31).
#pragma once
#include <cuda.h>

#include "lsv_common.cuh"
#include "lsv_plan.h"

namespace lsv {

constexpr int kTcThreads = 192;
constexpr int kTmemCols = 256;  // two 128-column accumulators (double buffer)
constexpr int kStgStride = 132; // floats per staged token row in the expand epilogue

struct alignas(64) ShrinkParams {
  CUtensorMap xmap[5];          // x [num_tokens][h_in], boxes {64 cols × 8<<b rows}, SWIZZLE_128B
  const int32_t* plan;
  const void* const* a_ptrs;
  uint8_t* ws;
  int n_items, off_items, off_mtiles, ws_partials, ws_vimg, ws_counters;
};

struct ExpandParams {
  const int32_t* plan;
  const void* const* b_ptrs;
  const uint8_t* ws;
  __nv_bfloat16* y;
  int64_t ldy;
  int n_items, off_items, off_mtiles, ws_vimg;
};

__device__ __forceinline__ int snake_item(int round, int cta, int grid) {
  return round * grid + ((round & 1) ? (grid - 1 - cta) : cta);
}

__host__ __device__ constexpr int shrink_smem_bytes() {
  return 1024 + kShrinkSlots * kShrinkSlotBytes + kShrinkGuardBytes + 256;
}
__host__ __device__ constexpr int expand_smem_bytes() {
  return 1024 + kExpandSlots * kExpandSlotBytes + 32 * kStgStride * 4 + 256;
}

// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kTcThreads, 1) shrink_tc_kernel(const __grid_constant__ ShrinkParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + kShrinkSlots * kShrinkSlotBytes + kShrinkGuardBytes);
  uint64_t* empty = full + kShrinkSlots;
  uint64_t* tfull = empty + kShrinkSlots;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const ShrinkItem* items = reinterpret_cast<const ShrinkItem*>(p.plan + p.off_items);
  const MTile* mtiles = reinterpret_cast<const MTile*>(p.plan + p.off_mtiles);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kShrinkSlots; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 4); }
    fence_mbar_init();
    for (int b = 0; b < 5; ++b) prefetch_tmap(&p.xmap[b]);
  }
  if (warp == 1) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int grid = gridDim.x, cta = blockIdx.x;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- producer
      int slot = 0; uint32_t phase = 0;
      for (int rnd = 0;; ++rnd) {
        const int idx = snake_item(rnd, cta, grid);
        if (idx >= p.n_items) break;
        const ShrinkItem it = items[idx];
        const MTile mt = mtiles[it.mtile];
        const int r = mt.rank, np8 = round_up(mt.ntok, 8), kch = it.split_kch >> 16;
        const uint8_t* a = static_cast<const uint8_t*>(p.a_ptrs[mt.seg]);
        for (int g = it.chunk_begin; g < it.chunk_end; g += kch) {
          const int kc = min(kch, it.chunk_end - g);
          mbar_wait(&empty[slot], phase ^ 1);
          uint8_t* dst = ring + slot * kShrinkSlotBytes;
          mbar_arrive_expect_tx(&full[slot], (uint32_t)(kc * (np8 + r) * 128));
          for (int c = 0; c < kc; ++c) {
            int row = 0;
            for (int b = 4; b >= 0; --b) {
              const int R = 8 << b;
              if (np8 - row >= R) {
                tma_load_2d(dst + (c * np8 + row) * 128, &p.xmap[b], &full[slot], (g + c) * kChunk,
                            mt.tok_begin + row);
                row += R;
              }
            }
          }
          bulk_load(dst + kc * np8 * 128, a + (size_t)g * r * 128, (uint32_t)(kc * r * 128), &full[slot]);
          if (++slot == kShrinkSlots) { slot = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      int slot = 0; uint32_t phase = 0; int ai = 0;
      for (int rnd = 0;; ++rnd) {
        const int idx = snake_item(rnd, cta, grid);
        if (idx >= p.n_items) break;
        const ShrinkItem it = items[idx];
        const MTile mt = mtiles[it.mtile];
        const int r = mt.rank, np8 = round_up(mt.ntok, 8), kch = it.split_kch >> 16;
        const int buf = ai & 1;
        mbar_wait(&tempty[buf], ((ai >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + buf * 128;
        const uint32_t idesc = idesc_bf16(128, max(16, round_up(r, 16)));
        uint32_t accumulate = 0;
        for (int g = it.chunk_begin; g < it.chunk_end; g += kch) {
          const int kc = min(kch, it.chunk_end - g);
          mbar_wait(&full[slot], phase);
          tc_fence_after();
          const uint32_t xb = smem_u32(ring + slot * kShrinkSlotBytes);
          const uint32_t ab = xb + kc * np8 * 128;
          for (int c = 0; c < kc; ++c) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t adesc = smem_desc(xb + c * np8 * 128 + kk * 32, 16, 1024, 2);
              const uint64_t bdesc = smem_desc(ab + c * r * 128 + kk * 32, 16, 1024, 2);
              umma_bf16(d, adesc, bdesc, idesc, accumulate);
              accumulate = 1;
            }
          }
          umma_commit(&empty[slot]);
          if (++slot == kShrinkSlots) { slot = 0; phase ^= 1; }
        }
        umma_commit(&tfull[buf]);
        ++ai;
      }
    }
  } else {  // ---------------------------- epilogue (warps 2..5)
    const int q = warp & 3, row = q * 32 + lane, etid = threadIdx.x - 64;
    float* partials = reinterpret_cast<float*>(p.ws + p.ws_partials);
    int* counters = reinterpret_cast<int*>(p.ws + p.ws_counters);
    int ai = 0;
    for (int rnd = 0;; ++rnd) {
      const int idx = snake_item(rnd, cta, grid);
      if (idx >= p.n_items) break;
      const ShrinkItem it = items[idx];
      const MTile mt = mtiles[it.mtile];
      const int r = mt.rank, nt = mt.ntok, kp16 = max(16, r), split = it.split_kch & 0xffff;
      const int buf = ai & 1;
      mbar_wait(&tfull[buf], (ai >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + buf * 128;
      const bool valid = row < nt;
      uint8_t* vimg = p.ws + p.ws_vimg + mt.vimg_off;
      float* part = partials + mt.part_off + (size_t)split * nt * r;
      for (int cc = 0; cc < r; cc += 16) {
        float v[16];
        tmem_ld_32x32b_x16(taddr + cc, v);
        if (valid) {
          if (mt.nsplit == 1) {
            for (int h = 0; h < 2; ++h) {
              uint4 w;
              const int k0 = cc + h * 8;
              w.x = pack_bf16x2(k0 + 0 < r ? v[h * 8 + 0] : 0.f, k0 + 1 < r ? v[h * 8 + 1] : 0.f);
              w.y = pack_bf16x2(k0 + 2 < r ? v[h * 8 + 2] : 0.f, k0 + 3 < r ? v[h * 8 + 3] : 0.f);
              w.z = pack_bf16x2(k0 + 4 < r ? v[h * 8 + 4] : 0.f, k0 + 5 < r ? v[h * 8 + 5] : 0.f);
              w.w = pack_bf16x2(k0 + 6 < r ? v[h * 8 + 6] : 0.f, k0 + 7 < r ? v[h * 8 + 7] : 0.f);
              if (k0 < kp16) *reinterpret_cast<uint4*>(vimg + vimg_off(row, k0, kp16)) = w;
            }
          } else {
            float4* dst = reinterpret_cast<float4*>(part + (size_t)row * r + cc);
            const int nvec = min(16, r - cc) / 4;
            for (int u = 0; u < nvec; ++u) dst[u] = make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
      if (mt.nsplit > 1) {
        __threadfence();
        named_bar_sync(1, 128);
        if (etid == 0) *last_flag = (atomicAdd(&counters[mt.counter], 1) == mt.nsplit - 1);
        named_bar_sync(1, 128);
        if (*last_flag) {
          __threadfence();
          const float* base = partials + mt.part_off;
          const size_t stride = (size_t)nt * r;
          // one thread per (token, 8-rank unit): fixed-order sum over splits, 16-byte store
          const int units = nt * (kp16 / 8);
          for (int u = etid; u < units; u += 128) {
            const int t = u / (kp16 / 8), k0 = (u % (kp16 / 8)) * 8;
            float s[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) s[e] = 0.f;
            if (k0 < r) {
              for (int j = 0; j < mt.nsplit; ++j) {
                const float4* src = reinterpret_cast<const float4*>(base + j * stride + (size_t)t * r + k0);
                const float4 lo = __ldcg(src), hi = __ldcg(src + 1);
                s[0] += lo.x; s[1] += lo.y; s[2] += lo.z; s[3] += lo.w;
                s[4] += hi.x; s[5] += hi.y; s[6] += hi.z; s[7] += hi.w;
              }
            }
            uint4 w;
            w.x = pack_bf16x2(s[0], s[1]); w.y = pack_bf16x2(s[2], s[3]);
            w.z = pack_bf16x2(s[4], s[5]); w.w = pack_bf16x2(s[6], s[7]);
            *reinterpret_cast<uint4*>(vimg + vimg_off(t, k0, kp16)) = w;
          }
          if (etid == 0) counters[mt.counter] = 0;  // leave the workspace clean for the next call
        }
        named_bar_sync(1, 128);
      }
      ++ai;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) { tc_fence_after(); tmem_dealloc(tmem_base, kTmemCols); }
}

// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kTcThreads, 1) expand_tc_kernel(const __grid_constant__ ExpandParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* stg = reinterpret_cast<float*>(ring + kExpandSlots * kExpandSlotBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + 32 * kStgStride);
  uint64_t* empty = full + kExpandSlots;
  uint64_t* tfull = empty + kExpandSlots;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const ExpandItem* items = reinterpret_cast<const ExpandItem*>(p.plan + p.off_items);
  const MTile* mtiles = reinterpret_cast<const MTile*>(p.plan + p.off_mtiles);

  // The K=16 MMA of a rank-8 adapter reads one 8-wide k-core past the tile (multiplied by
  // the zero k-padding of v); zero the ring once so that memory is never NaN.
  for (int i = threadIdx.x; i < kExpandSlots * kExpandSlotBytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(ring)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    for (int s = 0; s < kExpandSlots; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 4); }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int grid = gridDim.x, cta = blockIdx.x;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- producer
      int slot = 0; uint32_t phase = 0;
      for (int rnd = 0;; ++rnd) {
        const int idx = snake_item(rnd, cta, grid);
        if (idx >= p.n_items) break;
        const ExpandItem it = items[idx];
        const MTile mt = mtiles[it.mtile];
        const int r = mt.rank, kp16 = max(16, r), np16 = round_up(mt.ntok, 16);
        const uint8_t* b = static_cast<const uint8_t*>(p.b_ptrs[mt.seg]);
        const uint32_t bbytes = 128 * r * 2, vbytes = np16 * kp16 * 2;
        mbar_wait(&empty[slot], phase ^ 1);
        uint8_t* dst = ring + slot * kExpandSlotBytes;
        mbar_arrive_expect_tx(&full[slot], bbytes + vbytes);
        bulk_load(dst, b + (size_t)it.jtile * bbytes, bbytes, &full[slot]);
        bulk_load(dst + kExpandSlotBytes / 2, p.ws + p.ws_vimg + mt.vimg_off, vbytes, &full[slot]);
        if (++slot == kExpandSlots) { slot = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      int slot = 0; uint32_t phase = 0; int ai = 0;
      for (int rnd = 0;; ++rnd) {
        const int idx = snake_item(rnd, cta, grid);
        if (idx >= p.n_items) break;
        const ExpandItem it = items[idx];
        const MTile mt = mtiles[it.mtile];
        const int r = mt.rank, kp16 = max(16, r), np16 = round_up(mt.ntok, 16);
        const int buf = ai & 1;
        mbar_wait(&tempty[buf], ((ai >> 1) & 1) ^ 1);
        tc_fence_after();
        mbar_wait(&full[slot], phase);
        tc_fence_after();
        const uint32_t bb = smem_u32(ring + slot * kExpandSlotBytes);
        const uint32_t vb = bb + kExpandSlotBytes / 2;
        const uint32_t idesc = idesc_bf16(128, np16);
        const uint32_t d = tmem_base + buf * 128;
        for (int ks = 0; ks < kp16 / 16; ++ks) {
          const uint64_t adesc = smem_desc(bb + ks * 256, 128, r * 16, 0);
          const uint64_t bdesc = smem_desc(vb + ks * 256, 128, kp16 * 16, 0);
          umma_bf16(d, adesc, bdesc, idesc, ks > 0 ? 1u : 0u);
        }
        umma_commit(&empty[slot]);
        umma_commit(&tfull[buf]);
        if (++slot == kExpandSlots) { slot = 0; phase ^= 1; }
        ++ai;
      }
    }
  } else {  // ---------------------------- epilogue (warps 2..5)
    const int q = warp & 3, jrow = q * 32 + lane, etid = threadIdx.x - 64;
    int ai = 0;
    for (int rnd = 0;; ++rnd) {
      const int idx = snake_item(rnd, cta, grid);
      if (idx >= p.n_items) break;
      const ExpandItem it = items[idx];
      const MTile mt = mtiles[it.mtile];
      const int nt = mt.ntok;
      const int buf = ai & 1;
      mbar_wait(&tfull[buf], (ai >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + buf * 128;
      __nv_bfloat16* ybase = p.y + (int64_t)mt.tok_begin * p.ldy + it.jtile * 128;
      for (int c0 = 0; c0 < nt; c0 += 32) {
        float v[32];
        tmem_ld_32x32b_x16(taddr + c0, v);
        tmem_ld_32x32b_x16(taddr + c0 + 16, v + 16);
#pragma unroll
        for (int t = 0; t < 32; ++t) stg[t * kStgStride + jrow] = v[t];
        named_bar_sync(1, 128);
        const int rows = min(32, nt - c0);
        for (int task = etid; task < rows * 16; task += 128) {
          const int t = task >> 4, u = task & 15;
          uint4* gy = reinterpret_cast<uint4*>(ybase + (int64_t)(c0 + t) * p.ldy + u * 8);
          const uint4 yv = *gy;
          const float4 d0 = *reinterpret_cast<const float4*>(stg + t * kStgStride + u * 8);
          const float4 d1 = *reinterpret_cast<const float4*>(stg + t * kStgStride + u * 8 + 4);
          uint4 o;
          o.x = pack_bf16x2(bf16_lo(yv.x) + d0.x, bf16_hi(yv.x) + d0.y);
          o.y = pack_bf16x2(bf16_lo(yv.y) + d0.z, bf16_hi(yv.y) + d0.w);
          o.z = pack_bf16x2(bf16_lo(yv.z) + d1.x, bf16_hi(yv.z) + d1.y);
          o.w = pack_bf16x2(bf16_lo(yv.w) + d1.z, bf16_hi(yv.w) + d1.w);
          *gy = o;
        }
        named_bar_sync(1, 128);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
      ++ai;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) { tc_fence_after(); tmem_dealloc(tmem_base, kTmemCols); }
}

}  // namespace lsv
