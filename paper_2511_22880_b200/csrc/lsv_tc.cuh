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
//   B tile and v image: one cp.async.bulk each; the item's y rows arrive by TMA (exact row
//   count, boxes of 128..1 rows) into the same ring allocation, so the y read is prefetched as
//   deep as the ring; the epilogue adds D and writes bf16x2 words straight back to HBM.
//
// Both kernels: 192 threads, one persistent CTA per SM, each streaming its own list of fully
// decoded work records (the host planner assigns records to CTAs LPT-greedy on estimated bytes,
// so there are no device atomics and no dependent descriptor loads on the critical path).
// warp 0 = producer (one lane), warp 1 = MMA issuer (one lane) and TMEM owner, warps 2..5 =
// epilogue (warp w reads TMEM lanes 32*(w%4)..+31).  Launched with programmatic dependent
// launch: the prologue (barrier init, TMEM alloc) overlaps the previous kernel's tail.
#pragma once
#include <cuda.h>

#include "lsv_common.cuh"
#include "lsv_plan.h"

namespace lsv {

constexpr int kTcThreads = 192;
constexpr int kTmemCols = 256;  // two 128-column accumulators (double buffer)
constexpr int kItemQ = 8;       // expand: ring allocations in flight

struct alignas(64) ShrinkParams {
  CUtensorMap xmap[5];          // x [num_tokens][h_in], boxes {64 cols × 8<<b rows}, SWIZZLE_128B
  const int32_t* plan;
  const void* const* a_ptrs;
  uint8_t* ws;
  int off_recs, off_cta, ws_partials, ws_vimg, ws_counters;
  uint64_t* trace;              // debug timeline (nullptr = off): [cta][item][8] globaltimer stamps
  int trace_items;
};

struct alignas(64) ExpandParams {
  CUtensorMap ymap[8];          // y [num_tokens][h_out], boxes {128 cols × 1<<b rows}, no swizzle
  const int32_t* plan;
  const void* const* b_ptrs;
  uint8_t* ws;
  __nv_bfloat16* y;
  int64_t ldy;
  int off_recs, off_cta, ws_vimg;
  uint64_t* trace;
  int trace_items;
  int dbg;                      // debug ablations (0 in production)
};

__device__ __forceinline__ void trace_stamp(uint64_t* trace, int trace_items, int cta, int i, int k) {
  if (trace != nullptr && i < trace_items) {
    trace[((size_t)cta * trace_items + i) * 16 + k] = globaltimer_ns();
    trace[((size_t)cta * trace_items + i) * 16 + 8 + k] = clock64();
  }
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Streams one CTA's record list with a one-record lookahead (the next load is in flight while
// the current record is processed).
template <typename Rec>
struct RecStream {
  const Rec* recs;
  int k, end;
  Rec next;
  __device__ __forceinline__ RecStream(const int32_t* plan, int off_recs, int off_cta, int cta) {
    recs = reinterpret_cast<const Rec*>(plan + off_recs);
    k = plan[off_cta + cta];
    end = plan[off_cta + cta + 1];
    if (k < end) next = recs[k];
  }
  __device__ __forceinline__ bool pop(Rec& r) {
    if (k >= end) return false;
    r = next;
    if (++k < end) next = recs[k];
    return true;
  }
};

__host__ __device__ constexpr int shrink_smem_bytes() {
  return 1024 + kShrinkSlots * kShrinkSlotBytes + kShrinkGuardBytes + 1024;
}
__host__ __device__ constexpr int expand_smem_bytes() {
  return 1024 + kExpandRingBytes + kExpandGuardBytes + 1024;
}

// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kTcThreads, 1) shrink_tc_kernel(const __grid_constant__ ShrinkParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* ring = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + kShrinkSlots * kShrinkSlotBytes + kShrinkGuardBytes);
  uint64_t* empty = full + kShrinkSlots;
  uint64_t* tfull = empty + kShrinkSlots;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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
  const int cta = blockIdx.x;
  pdl_wait();                 // x, workspace and counters are written by earlier launches
  pdl_launch_dependents();

  if (warp == 0) {
    if (lane == 0) {  // ---------------- producer
      RecStream<ShrinkRec> rs(p.plan, p.off_recs, p.off_cta, cta);
      ShrinkRec inf;
      int slot = 0; uint32_t phase = 0;
      for (int k = 0; rs.pop(inf); ++k) {
        trace_stamp(p.trace, p.trace_items, cta, k, 0);
        const int r = inf.rank, np8 = round_up(inf.ntok, 8), kch = inf.kch;
        const uint8_t* a = static_cast<const uint8_t*>(p.a_ptrs[inf.seg]);
        for (int g = inf.chunk_begin; g < inf.chunk_end; g += kch) {
          const int kc = min(kch, inf.chunk_end - g);
          mbar_wait(&empty[slot], phase ^ 1);
          uint8_t* dst = ring + slot * kShrinkSlotBytes;
          mbar_arrive_expect_tx(&full[slot], (uint32_t)(kc * (np8 + r) * 128));
          for (int c = 0; c < kc; ++c) {
            int row = 0;
            for (int b = 4; b >= 0; --b) {
              const int R = 8 << b;
              if (np8 - row >= R) {
                tma_load_2d(dst + (c * np8 + row) * 128, &p.xmap[b], &full[slot], (g + c) * kChunk,
                            inf.tok_begin + row);
                row += R;
              }
            }
          }
          bulk_load(dst + kc * np8 * 128, a + (size_t)g * r * 128, (uint32_t)(kc * r * 128), &full[slot]);
          if (++slot == kShrinkSlots) { slot = 0; phase ^= 1; }
        }
        trace_stamp(p.trace, p.trace_items, cta, k, 1);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      RecStream<ShrinkRec> rs(p.plan, p.off_recs, p.off_cta, cta);
      ShrinkRec inf;
      int slot = 0; uint32_t phase = 0;
      for (int k = 0; rs.pop(inf); ++k) {
        const int r = inf.rank, np8 = round_up(inf.ntok, 8), kch = inf.kch;
        const int buf = k & 1;
        mbar_wait(&tempty[buf], ((k >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + buf * 128;
        const uint32_t idesc = idesc_bf16(128, max(16, round_up(r, 16)));
        uint32_t accumulate = 0;
        for (int g = inf.chunk_begin; g < inf.chunk_end; g += kch) {
          const int kc = min(kch, inf.chunk_end - g);
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
        trace_stamp(p.trace, p.trace_items, cta, k, 2);
      }
    }
  } else {  // ---------------------------- epilogue (warps 2..5)
    const int q = warp & 3, row = q * 32 + lane, etid = threadIdx.x - 64;
    float* partials = reinterpret_cast<float*>(p.ws + p.ws_partials);
    int* counters = reinterpret_cast<int*>(p.ws + p.ws_counters);
    RecStream<ShrinkRec> rs(p.plan, p.off_recs, p.off_cta, cta);
    ShrinkRec inf;
    for (int k = 0; rs.pop(inf); ++k) {
      const int r = inf.rank, nt = inf.ntok, kp16 = max(16, r);
      const int buf = k & 1;
      mbar_wait(&tfull[buf], (k >> 1) & 1);
      tc_fence_after();
      if (etid == 0) trace_stamp(p.trace, p.trace_items, cta, k, 3);
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + buf * 128;
      const bool valid = row < nt;
      uint8_t* vimg = p.ws + p.ws_vimg + inf.vimg_off;
      float* part = partials + inf.part_off + (size_t)inf.split * nt * r;
      for (int cc = 0; cc < r; cc += 16) {
        float v[16];
        tmem_ld_32x32b_x16(taddr + cc, v);
        if (valid) {
          if (inf.nsplit == 1) {
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
      if (etid == 0) trace_stamp(p.trace, p.trace_items, cta, k, 4);
      if (inf.nsplit > 1) {
        __threadfence();
        named_bar_sync(1, 128);
        if (etid == 0) *last_flag = (atomicAdd(&counters[inf.counter], 1) == inf.nsplit - 1);
        named_bar_sync(1, 128);
        if (*last_flag) {
          __threadfence();
          const float* base = partials + inf.part_off;
          const size_t stride = (size_t)nt * r;
          // one thread per (token, 8-rank unit), four units in flight per thread; fixed-order sum
          const int upr = kp16 / 8, units = nt * upr;
          for (int u0 = etid; u0 < units; u0 += 4 * 128) {
            float s[4][8];
#pragma unroll
            for (int g = 0; g < 4; ++g)
#pragma unroll
              for (int e = 0; e < 8; ++e) s[g][e] = 0.f;
            for (int j = 0; j < inf.nsplit; ++j) {
              float4 lo[4], hi[4];
#pragma unroll
              for (int g = 0; g < 4; ++g) {
                const int u = u0 + g * 128, t = u / upr, k0 = (u % upr) * 8;
                if (u < units && k0 < r) {
                  const float4* src = reinterpret_cast<const float4*>(base + j * stride + (size_t)t * r + k0);
                  lo[g] = __ldcg(src);
                  hi[g] = __ldcg(src + 1);
                } else {
                  lo[g] = hi[g] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
              }
#pragma unroll
              for (int g = 0; g < 4; ++g) {
                s[g][0] += lo[g].x; s[g][1] += lo[g].y; s[g][2] += lo[g].z; s[g][3] += lo[g].w;
                s[g][4] += hi[g].x; s[g][5] += hi[g].y; s[g][6] += hi[g].z; s[g][7] += hi[g].w;
              }
            }
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              const int u = u0 + g * 128, t = u / upr, k0 = (u % upr) * 8;
              if (u < units) {
                uint4 w;
                w.x = pack_bf16x2(s[g][0], s[g][1]); w.y = pack_bf16x2(s[g][2], s[g][3]);
                w.z = pack_bf16x2(s[g][4], s[g][5]); w.w = pack_bf16x2(s[g][6], s[g][7]);
                *reinterpret_cast<uint4*>(vimg + vimg_off(t, k0, kp16)) = w;
              }
            }
          }
          if (etid == 0) counters[inf.counter] = 0;  // leave the workspace clean for the next call
        }
        named_bar_sync(1, 128);
      }
      if (etid == 0) trace_stamp(p.trace, p.trace_items, cta, k, 5);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) { tc_fence_after(); tmem_dealloc(tmem_base, kTmemCols); }
}

// ------------------------------------------------------------------------------------------
// Expand: per item (m-tile, 128-wide h_out tile) the producer moves B tile + v image (bulk
// copies) and the item's y rows (TMA, exact row count) into a variable-size byte ring; the
// epilogue adds D (TMEM) to the prefetched y rows and stores bf16x2 words back to HBM.
__global__ void __launch_bounds__(kTcThreads, 1) expand_tc_kernel(const __grid_constant__ ExpandParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* ring = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint32_t* offs = reinterpret_cast<uint32_t*>(ring + kExpandRingBytes + kExpandGuardBytes);  // [kItemQ]
  uint64_t* full = reinterpret_cast<uint64_t*>(offs + 2 * kItemQ);
  uint64_t* empty = full + kItemQ;
  uint64_t* tfull = empty + kItemQ;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // The K=16 MMA of a rank-8 adapter reads one 8-wide k-core past its B tile (multiplied by the
  // zero k-padding of v): zero the ring once so that memory is never NaN.
  for (int i = threadIdx.x; i < (kExpandRingBytes + kExpandGuardBytes) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(ring)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  // Ring allocations in flight: full[s] = the item's bytes landed (the producer's arrive also
  // publishes offs[s]), empty[s] = the 4 epilogue warps are done with them.
  if (threadIdx.x == 0) {
    for (int s = 0; s < kItemQ; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 4); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 4); }
    fence_mbar_init();
    for (int b = 0; b < 8; ++b) prefetch_tmap(&p.ymap[b]);
  }
  if (warp == 1) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int cta = blockIdx.x;
  pdl_wait();                 // v images come from the shrink launch; y from earlier work
  pdl_launch_dependents();

  if (warp == 0) {
    if (lane == 0) {  // ---------------- producer: byte-ring allocation in list order
      RecStream<ExpandRec> rs(p.plan, p.off_recs, p.off_cta, cta);
      ExpandRec inf;
      uint32_t head = 0, tail = 0;
      uint32_t vbegin[kItemQ];
      int retired = 0;
      for (int k = 0; rs.pop(inf); ++k) {
        const int kp16 = max(16, inf.rank), np16 = round_up(inf.ntok, 16);
        const uint32_t bbytes = 128 * inf.rank * 2, vbytes = np16 * kp16 * 2, ybytes = inf.ntok * 256;
        const uint32_t size = round_up(bbytes, 128) + round_up(vbytes, 128) + round_up(ybytes, 128);
        if ((head % kExpandRingBytes) + size > kExpandRingBytes)
          head = (head / kExpandRingBytes + 1) * kExpandRingBytes;
        trace_stamp(p.trace, p.trace_items, cta, k, 0);
        // retire in FIFO order until an allocation slot and the ring bytes are free
        while (k - retired == kItemQ || head + size - tail > (uint32_t)kExpandRingBytes) {
          mbar_wait(&empty[retired % kItemQ], (retired / kItemQ) & 1);
          ++retired;
          tail = retired < k ? vbegin[retired % kItemQ] : head;
        }
        const int qs = k % kItemQ;
        vbegin[qs] = head;
        const uint32_t ring_off = head % kExpandRingBytes;
        offs[qs] = ring_off;
        trace_stamp(p.trace, p.trace_items, cta, k, 1);
        uint8_t* dst = ring + ring_off;
        const uint8_t* b = static_cast<const uint8_t*>(p.b_ptrs[inf.seg]);
        mbar_arrive_expect_tx(&full[qs], bbytes + vbytes + ybytes);
        bulk_load(dst, b + (size_t)inf.jtile * bbytes, bbytes, &full[qs]);
        uint8_t* vdst = dst + round_up(bbytes, 128);
        bulk_load(vdst, p.ws + p.ws_vimg + inf.vimg_off, vbytes, &full[qs]);
        uint8_t* ydst = vdst + round_up(vbytes, 128);
        int row = 0;
        for (int bb = 7; bb >= 0; --bb) {
          if (inf.ntok - row >= (1 << bb)) {
            tma_load_2d(ydst + row * 256, &p.ymap[bb], &full[qs], inf.jtile * 128, inf.tok_begin + row);
            row += 1 << bb;
          }
        }
        head += size;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      RecStream<ExpandRec> rs(p.plan, p.off_recs, p.off_cta, cta);
      ExpandRec inf;
      for (int k = 0; rs.pop(inf); ++k) {
        const int qs = k % kItemQ;
        const int r = inf.rank, kp16 = max(16, r), np16 = round_up(inf.ntok, 16);
        const int buf = k & 1;
        mbar_wait(&tempty[buf], ((k >> 1) & 1) ^ 1);
        mbar_wait(&full[qs], (k / kItemQ) & 1);
        tc_fence_after();
        const uint32_t bb = smem_u32(ring + offs[qs]);
        const uint32_t vb = bb + round_up(128 * r * 2, 128);
        const uint32_t idesc = idesc_bf16(128, np16);
        const uint32_t d = tmem_base + buf * 128;
        for (int ks = 0; ks < kp16 / 16; ++ks) {
          const uint64_t adesc = smem_desc(bb + ks * 256, 128, r * 16, 0);
          const uint64_t bdesc = smem_desc(vb + ks * 256, 128, kp16 * 16, 0);
          umma_bf16(d, adesc, bdesc, idesc, ks > 0 ? 1u : 0u);
        }
        umma_commit(&tfull[buf]);
        trace_stamp(p.trace, p.trace_items, cta, k, 2);
      }
    }
  } else {  // ---------------------------- epilogue (warps 2..5)
    const int q = warp & 3, etid = threadIdx.x - 64;
    // Lane pairs (2m, 2m+1) own columns (c, c+1), c = 32q + 2m.  For each token pair (t, t+1)
    // one shuffle gives the even lane both columns of token t and the odd lane both columns of
    // token t+1, so every y access is a 32-bit word: LDS from the TMA-prefetched tile, STG of
    // the updated pair straight to HBM (fire-and-forget).
    const bool odd = lane & 1;
    const int c = q * 32 + (lane & ~1);
    const int64_t ldw = p.ldy >> 1;  // row stride in 32-bit words
    RecStream<ExpandRec> rs(p.plan, p.off_recs, p.off_cta, cta);
    ExpandRec inf;
    for (int k = 0; rs.pop(inf); ++k) {
      const int qs = k % kItemQ;
      const int nt = inf.ntok, r = inf.rank, kp16 = max(16, r), np16 = round_up(nt, 16);
      const int buf = k & 1;
      mbar_wait(&tfull[buf], (k >> 1) & 1);
      mbar_wait(&full[qs], (k / kItemQ) & 1);  // y rows landed (TMA writes visible)
      tc_fence_after();
      if (etid == 0) trace_stamp(p.trace, p.trace_items, cta, k, 3);
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + buf * 128;
      const uint8_t* ytile = ring + offs[qs] + round_up(128 * r * 2, 128) + round_up(np16 * kp16 * 2, 128);
      const uint32_t* ysm = reinterpret_cast<const uint32_t*>(ytile) + (c >> 1);
      uint32_t* yg = reinterpret_cast<uint32_t*>(p.y + (int64_t)inf.tok_begin * p.ldy + inf.jtile * 128 + c);
      for (int c0 = 0; c0 < nt; c0 += 32) {
        if (etid == 0 && c0 == 32) trace_stamp(p.trace, p.trace_items, cta, k, 5);
        float v[32];
        if (!(p.dbg & 4)) {
          tmem_ld_32x32b_x16(taddr + c0, v);
          tmem_ld_32x32b_x16(taddr + c0 + 16, v + 16);
        } else {
#pragma unroll
          for (int t = 0; t < 32; ++t) v[t] = 0.f;
        }
        const int rows = min(32, nt - c0);
        uint32_t yw[16], out[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int tl = 2 * u + (odd ? 1 : 0);
          yw[u] = ld_shared_b32_if(ysm + (c0 + tl) * 64, tl < rows && !(p.dbg & 2));
        }
        // shuffle phase: no control flow, so the warp stays converged without reconvergence code
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const float send = odd ? v[2 * u] : v[2 * u + 1];
          const float recv = __shfl_xor_sync(0xffffffffu, send, 1);
          const float d0 = odd ? recv : v[2 * u];          // column c
          const float d1 = odd ? v[2 * u + 1] : recv;      // column c+1
          out[u] = pack_bf16x2(bf16_lo(yw[u]) + d0, bf16_hi(yw[u]) + d1);
        }
        // store phase: branch-free predicated 32-bit stores
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int tl = 2 * u + (odd ? 1 : 0);
          st_global_b32_if(yg + (int64_t)(c0 + tl) * ldw, out[u], tl < rows && !(p.dbg & 1));
        }
      }
      if (etid == 0) trace_stamp(p.trace, p.trace_items, cta, k, 6);
      tc_fence_before();
      __syncwarp();
      if (etid == 0) trace_stamp(p.trace, p.trace_items, cta, k, 7);
      if (lane == 0) {
        mbar_arrive(&tempty[buf]);
        mbar_arrive(&empty[qs]);  // this warp is done with the item's ring bytes
      }
      if (etid == 0) trace_stamp(p.trace, p.trace_items, cta, k, 4);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) { tc_fence_after(); tmem_dealloc(tmem_base, kTmemCols); }
}

}  // namespace lsv
