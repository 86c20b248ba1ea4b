// lsv_tc.cuh — tcgen05 (5th-gen tensor core) tier of the mixed-rank LoRA delta.
//
// Shrink  D[128 tok × N = members·rank] += x_tile[128 × 64k] · A_s^T     (TMEM accumulator)
//   x tile: TMA (cp.async.bulk.tensor, SWIZZLE_128B) of exactly ceil8(n) token rows per
//   64-column chunk, composed from 128/64/32/16/8-row boxes; A_s: one cp.async.bulk of a
//   pre-swizzled [kch chunks][rows][64] slab run.  Rows past the segment / columns past the
//   rank are garbage in, garbage out (row i of D only reads row i of x; column j only
//   row j of A) and are never stored.  k-split partials are summed in split order (bit-
//   reproducible) into the v images: after a grid barrier in the standalone kernel, per tile by
//   the reducer warp in the group kernel.
// Expand  D[128 tok × 256 h_out] = v_hi·B_s^T + v_lo·B_s^T + I·y          (y added on the tensor core)
//   B tile and v image pair: one cp.async.bulk each; the item's y rows: one 3D TMA box per row
//   range into an MN-major SWIZZLE_128B operand; the epilogue is LDTM -> cvt -> 32-byte stores.
//
// Kernels: shrink_tc_kernel and expand_tc_kernel (standalone entry points, TP) and
// group_tc_kernel<NG> (lsv_lora_forward: NG input groups' shrinks and expands in one launch,
// per-m-tile readiness instead of a grid barrier).  One persistent CTA per SM streams its own
// lists of fully decoded records (host LPT assignment: no device atomics on the critical path).
// Warp roles (256 threads; the group kernel adds warp 8): 0, 1, 6, 7 epilogue (warp w reads TMEM
// lanes 32*(w%4)..+31), 2 (+ 4 / 8) copy issue, 3 MMA issue and TMEM owner; in the group kernel
// 4 publishes stored records and checks expand readiness, 5 reduces split-K shares.  Every copy
// and MMA is issued by an elected lane of a converged warp.  Launched with programmatic dependent
// launch: the prologue (barrier init, TMEM alloc) overlaps the previous kernel's tail.
#pragma once
#include <cuda.h>

#include "lsv_common.cuh"
#include "lsv_plan.h"

namespace lsv {

constexpr int kTcThreads = 192;
constexpr int kMaxTp = 8;       // tensor-parallel ranks a scatter shrink writes to
constexpr int kTmemCols = 512;  // four 128-column accumulators
constexpr int kAccBufs = 4;
#ifndef LSV_EXPAND_ITEMQ
#define LSV_EXPAND_ITEMQ 6
#endif
constexpr int kItemQ = LSV_EXPAND_ITEMQ;   // expand: ring allocations in flight

struct alignas(64) ShrinkParams {
  CUtensorMap xmap[5];          // x [num_tokens][h_in], boxes {64 cols × 8<<b rows}, SWIZZLE_128B
  const int32_t* plan;
  const void* const* a_ptrs;
  uint8_t* ws;
  int off_recs, off_cta, ws_partials, ws_vimg;
  int off_mtiles, off_red, n_red, red_units, off_red_cta;   // grid-wide split-K reduction
  int* gbar;                    // grid barrier {arrive, done} in the workspace's barrier header
  int num_proj, vimg_stride;    // input group: projections shrunk together, bytes between their v images
  int acc_cols;                 // TMEM accumulator width (128 -> 4 buffers, 256 -> 2)
  int vsplit;                   // 1: v images are bf16 (hi, lo) pairs (PlanHeader::vsplit)
  int tile_aligned;             // 1: 128-row tile-aligned images, zero rows outside the piece
  int wait_prev;                // 0: the previous launch is another input group's expand, which this
                                // launch neither reads nor overwrites: start without waiting for it
  // tensor-parallel scatter (tp > 0): instead of this rank's shard images, every (token, member,
  // 8-column) unit goes to column tp_rank*rs + k of the member's full-rank image on every rank
  // (vdst[d]: rank d's image base for this layer/group, CUDA-IPC-mapped); the last CTA then bumps
  // every rank's flag.  fplan: the full-rank plan (same m-tiles) on the device.
  int tp, tp_rank, vstride_f, f_off_mtiles;
  int tp_rr;                    // 1: shard = the 8-row groups g of the full rank with g % tp == tp_rank
                                //    (balanced shards, no padding); 0: contiguous rows [tp_rank*rs, +rs)
  const int32_t* fplan;
  uint8_t* vdst[kMaxTp];
  int* flags[kMaxTp];
  int tp_row;                   // row-parallel: vdst[d] is rank d's exchange buffer; this rank's fp32
  int xslot;                    // partial v goes to slot tp_rank (xslot bytes per slot) on every rank
  uint64_t* trace;              // debug timeline (nullptr = off): [cta][item][8] globaltimer stamps
  int trace_items;
  int dbg;                      // debug ablations (0 in production)
  int num_tokens, h_in;         // bounds for the checked build (LSV_DCHECK)
  int64_t ws_bytes;
};

struct alignas(64) ExpandParams {
  // per member: y [num_tokens][h_out] as 3D {64 cols, rows, h_out/64 blocks} (strides 2 B, ldy*2 B,
  // 128 B), SWIZZLE_128B boxes {64, 8<<b rows, 4 blocks} (256-wide items) / {64, 8<<b, 2} (128-wide):
  // one copy lands a row range of every 64-column block of the item as [block][rows][64]
  CUtensorMap ymap[kMaxProj][5];
  CUtensorMap ymap2[kMaxProj][5];
  const int32_t* plan;
  const void* const* b_ptrs[kMaxProj];
  uint8_t* ws;
  __nv_bfloat16* y[kMaxProj];
  int64_t ldy[kMaxProj];
  int ws_vimg[kMaxProj];        // byte offset of each member's v images
  int tws[kMaxProj];            // each member's h_out tile width (its B slab layout: 128 or 256)
  int st32[kMaxProj];           // 1: y base and row stride are 32-byte aligned -> 32-byte (full sector) stores
  int tw_max;                   // TMEM accumulator width
  int off_recs, off_cta;
  int* wait_flag;               // TP: wait until *wait_flag == wait_target (every rank's shard written),
  int wait_target;              //     then the last CTA through re-arms it ([0] flag, [1] pass counter)
  const uint8_t* xsum;          // TP row groups: this rank's exchange buffer (wait_target fp32 partial
  int xslot, ws_vimg0;          //   slots); summed into the v images (at ws + ws_vimg0) before expanding
  int off_mtiles, n_mtiles, num_proj, vimg_stride;
  int* gbar;                    // TP row-sum grid barrier {arrive, done} (workspace barrier header)
  int vsplit;                   // 1: v images are bf16 (hi, lo) pairs: two v MMAs per K step
  uint64_t* trace;
  int trace_items;
  int dbg;                      // debug ablations (0 in production)
  int num_tokens;               // bounds for the checked build (LSV_DCHECK)
  int h_outs[kMaxProj];
  int64_t ws_bytes;
  // layer kernel, dynamic dispatch (cursor != nullptr): CTAs take items of the list in the plan's
  // off_dyn order from a global cursor instead of walking their own LPT lists
  int* cursor;
  int off_dyn, n_dyn;
};

__device__ __forceinline__ void trace_stamp(uint64_t* trace, int trace_items, int cta, int i, int k) {
  if (trace != nullptr && i < trace_items) {
#ifndef LSV_TRACE_CLOCK_ONLY   // the globaltimer read is slow enough to perturb per-item timings
    trace[((size_t)cta * trace_items + i) * 16 + k] = globaltimer_ns();
#endif
    trace[((size_t)cta * trace_items + i) * 16 + 8 + k] = clock64();
  }
}
// Clock-only trace builds: extra per-item stamps in the (unused) globaltimer slots.
__device__ __forceinline__ void trace_aux(uint64_t* trace, int trace_items, int cta, int i, int k) {
#ifdef LSV_TRACE_CLOCK_ONLY
  if (trace != nullptr && i < trace_items) trace[((size_t)cta * trace_items + i) * 16 + k] = clock64();
#endif
}
// CTA-level phase stamps land in the last item slot of the trace buffer.
__device__ __forceinline__ void phase_stamp(uint64_t* trace, int trace_items, int cta, int k) {
  if (trace != nullptr) trace_stamp(trace, trace_items, cta, trace_items - 1, k);
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Warp-cooperative stream over one CTA's record list: every lane of the warp calls pop(); a
// refill loads the next CH records (one per lane) plus each record's adapter pointer into the
// warp's shared-memory buffer, so the dependent global loads cost one latency per CH items
// instead of one per item.
template <typename Rec, int CH>
struct WarpRecBuf {
  Rec rec[CH];
  const uint8_t* ptr[CH];
};

__device__ __forceinline__ int rec_table(const ShrinkRec&) { return 0; }
__device__ __forceinline__ int rec_table(const ExpandRec& r) { return r.proj; }

template <typename Rec, int CH>
struct WarpRecStream {
  WarpRecBuf<Rec, CH>* buf;
  const Rec* recs;
  const void* const* const* tables;   // adapter pointer table of each member (nullptr: no pointers)
  int next, end, j, n;
  __device__ __forceinline__ WarpRecStream(WarpRecBuf<Rec, CH>* b, const int32_t* plan, int off_recs, int off_cta,
                                           int cta, const void* const* const* adapter_tables) {
    buf = b;
    recs = reinterpret_cast<const Rec*>(plan + off_recs);
    tables = adapter_tables;
    next = plan[off_cta + cta];
    end = plan[off_cta + cta + 1];
    j = n = 0;
  }
  // all 32 lanes must call; returns the same record on every lane
  __device__ __forceinline__ bool pop(Rec& r, const uint8_t*& ptr) {
    if (j == n) {
      if (next >= end) return false;
      __syncwarp();
      const int lane = threadIdx.x & 31;
      n = min(CH, end - next);
      if (lane < n) {
        const Rec rr = recs[next + lane];
        buf->rec[lane] = rr;
        buf->ptr[lane] = tables ? static_cast<const uint8_t*>(tables[rec_table(rr)][rr.seg]) : nullptr;
      }
      __syncwarp();
      next += n;
      j = 0;
    }
    r = buf->rec[j];
    ptr = buf->ptr[j];
    ++j;
    return true;
  }
};

constexpr int kShrinkRecCh = 16;
#ifndef LSV_EXPAND_RECCH
#define LSV_EXPAND_RECCH 32
#endif
constexpr int kExpandRecCh = LSV_EXPAND_RECCH;
using ShrinkRecBuf = WarpRecBuf<ShrinkRec, kShrinkRecCh>;
using ExpandRecBuf = WarpRecBuf<ExpandRec, kExpandRecCh>;

// Dynamic expand dispatch (layer kernel): the dispatcher warp takes the next item index from the
// group's global cursor and publishes its record here; every expand role reads the records in
// publication order.  A record with ntok == 0 ends the CTA's phase.  Slot reuse: the dispatcher
// leads the copy warp by at most kVQ items (v-ready queue), which leads the MMA by kItemQ and the
// epilogue by the TMEM buffers, plus one end record per phase: fewer than kDynQ positions.
constexpr int kDynQ = 48;
struct DynRing {
  ExpandRec rec[kDynQ];
  const uint8_t* ptr[kDynQ];
  int published;                 // records published (monotone over the launch)
};
__device__ __forceinline__ int ld_acquire_cta_shared(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta_shared(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
// An expand role's record source: its CTA's static list, or the dynamic ring (dyn != nullptr;
// q = the role's ring position, carried over phases).
struct ExpSrc {
  WarpRecStream<ExpandRec, kExpandRecCh> rs;
  DynRing* dyn;
  int* q;
  __device__ __forceinline__ ExpSrc(ExpandRecBuf* b, const int32_t* plan, int off_recs, int off_cta, int cta,
                                    const void* const* const* tables, DynRing* d, int* qpos)
      : rs(b, plan, off_recs, off_cta, cta, tables), dyn(d), q(qpos) {}
  __device__ __forceinline__ bool pop(ExpandRec& r, const uint8_t*& ptr) {
    if (dyn == nullptr) return rs.pop(r, ptr);
    const int pos = *q;
    uint64_t t0 = 0;
    for (uint32_t spin = 0; ld_acquire_cta_shared(&dyn->published) <= pos; ++spin) {
      if ((spin & 1023u) == 1023u) {   // bounded like every other wait: trap after ~4 s instead of hanging
        const uint64_t now = globaltimer_ns();
        if (t0 == 0) t0 = now;
        else if (now - t0 > 4000000000ull) __trap();
      }
    }
    r = dyn->rec[pos % kDynQ];
    ptr = dyn->ptr[pos % kDynQ];
    *q = pos + 1;
    return r.ntok != 0;
  }
};

// Full-rank image column of local shard column k (a multiple of 8): contiguous shards put it at
// tp_rank * rs + k; round-robin shards own every tp-th 8-row group, starting at group tp_rank.
__device__ __forceinline__ int tp_full_col(const ShrinkParams& p, int k, int rs) {
  return p.tp_rr ? 8 * (p.tp_rank + p.tp * (k >> 3)) + (k & 7) : p.tp_rank * rs + k;
}
// TP scatter of one 16-byte unit (8 k of member pp, token t of m-tile mtile; k local to the shard)
// into every rank's full-rank image at column tp_full_col of K = kpad(full rank).
__device__ __forceinline__ void tp_scatter(const ShrinkParams& p, int mtile, int pp, int t, int k, int rs, int np16,
                                           const uint4& w, const uint4& wlo) {
  const MTile mf = reinterpret_cast<const MTile*>(p.fplan + p.f_off_mtiles)[mtile];
  const uint32_t off = (uint32_t)pp * p.vstride_f + mf.vimg_off + vimg_off(t, tp_full_col(p, k, rs), kpad(mf.rank), np16);
  const uint32_t lo = vimg_bytes(mf.ntok, kpad(mf.rank));
  for (int d = 0; d < p.tp; ++d) {
    *reinterpret_cast<uint4*>(p.vdst[d] + off) = w;
    if (p.vsplit) *reinterpret_cast<uint4*>(p.vdst[d] + off + lo) = wlo;
  }
}
// The full image's k pad (full rank % 16 == 8) is written as zeros by the last shard's rank.
__device__ __forceinline__ void tp_scatter_pad(const ShrinkParams& p, int mtile, int pp, int t, int np16) {
  const MTile mf = reinterpret_cast<const MTile*>(p.fplan + p.f_off_mtiles)[mtile];
  const int kpf = kpad(mf.rank);
  // written by the rank holding the last real 8-row group (contiguous: the last rank)
  const int writer = p.tp_rr ? (mf.rank / 8 - 1) % p.tp : p.tp - 1;
  if (p.tp_rank != writer || kpf == mf.rank) return;
  const uint32_t off = (uint32_t)pp * p.vstride_f + mf.vimg_off + vimg_off(t, mf.rank, kpf, np16);
  const uint32_t lo = vimg_bytes(mf.ntok, kpf);
  for (int d = 0; d < p.tp; ++d) {
    *reinterpret_cast<uint4*>(p.vdst[d] + off) = make_uint4(0, 0, 0, 0);
    if (p.vsplit) *reinterpret_cast<uint4*>(p.vdst[d] + off + lo) = make_uint4(0, 0, 0, 0);
  }
}
// Row-parallel TP: 8 fp32 partial-v values (member pp, token t of m-tile mtile, k..k+7) into slot
// tp_rank of every rank's exchange buffer (per m-tile fp32 [np16][kp] at 2 * vimg_off).
__device__ __forceinline__ void tp_row_put(const ShrinkParams& p, int mtile, int pp, int t, int k, const float* v8) {
  const MTile mt = reinterpret_cast<const MTile*>(p.plan + p.off_mtiles)[mtile];
  const size_t off = (size_t)p.tp_rank * p.xslot + (size_t)pp * 2 * p.vimg_stride + 2 * (size_t)mt.vimg_off +
                     ((size_t)t * kpad(mt.rank) + k) * 4;
  const float4 lo = make_float4(v8[0], v8[1], v8[2], v8[3]), hi = make_float4(v8[4], v8[5], v8[6], v8[7]);
  for (int d = 0; d < p.tp; ++d) {
    float4* dst = reinterpret_cast<float4*>(p.vdst[d] + off);
    dst[0] = lo;
    dst[1] = hi;
  }
}
// No split tiles: the CTAs count themselves out (counter slot after the grid barrier's) and the
// last one signals every rank.
__device__ __forceinline__ void tp_signal(const ShrinkParams& p) {
  if (threadIdx.x != 0) return;
  int* bar = p.gbar;
  if (atomicAdd(&bar[1], 1) == (int)gridDim.x - 1) {
    bar[1] = 0;
    for (int d = 0; d < p.tp; ++d) red_release_sys_add(p.flags[d], 1);
  }
}

// Copy-issuing warps per pipeline: a warp spends ~130 cycles issuing each bulk / TMA copy
// (tools/tma_issue.cu), two warps issue twice as many.  The second part runs on warp 4 in the
// standalone kernels (idle otherwise) and on warp 8 in the group kernel.
#ifndef LSV_PROD_PARTS
#define LSV_PROD_PARTS 2
#endif
constexpr int kProdParts = LSV_PROD_PARTS;
constexpr int kProdWarp2 = 4;
// Shrink warp roles: as the expand's (below), layout 1 keeps the producer and the MMA issuer off
// the sub-partitions of the busy epilogue quadrants 0 and 1.
#ifndef LSV_SHRINK_LAYOUT
#define LSV_SHRINK_LAYOUT 1
#endif
#if LSV_SHRINK_LAYOUT
constexpr int kShrProdWarp = 2, kShrMmaWarp = 3, kShrinkThreads = 256;
__device__ __forceinline__ bool shrink_epi_warp(int w) { return w < 2 || w == 6 || w == 7; }
#else
constexpr int kShrProdWarp = 0, kShrMmaWarp = 1, kShrinkThreads = 192;
__device__ __forceinline__ bool shrink_epi_warp(int w) { return w >= 2; }
#endif
constexpr int kShrinkRecBufs = kShrinkThreads / 32;
__host__ __device__ constexpr int shrink_smem_bytes() {
  return 1024 + kShrinkSlots * kShrinkSlotBytes + kShrinkGuardBytes + kShrinkRecBufs * (int)sizeof(ShrinkRecBuf) + 1024;
}
#ifndef LSV_EXPAND_EPI_PIPE
#define LSV_EXPAND_EPI_PIPE 1
#endif
#ifndef LSV_EXPAND_ST32
#define LSV_EXPAND_ST32 1
#endif
// Quadrant rotation of small expand tiles.  An M=128 MMA writes A row i to TMEM lane i, so an item
// of <= 32 (<= 64) tokens whose A descriptors start 32*qb rows early lands in lane quadrant(s)
// qb.. and is stored by that quadrant's epilogue warp.  Consecutive small items then drain on
// different warps in parallel instead of queueing on the quadrant-0 warp.  0: off; 1: <= 32-token
// items alternate quadrants 0/1; 2: <= 32-token items rotate over 0..3, <= 64-token over {0, 2}.
#ifndef LSV_EXPAND_QROT
#define LSV_EXPAND_QROT 0
#endif
__device__ __forceinline__ int expand_qbase(int k, int ntok) {
#if LSV_EXPAND_QROT == 2
  return ntok <= 32 ? (k & 3) : ntok <= 64 ? ((k & 1) << 1) : 0;
#elif LSV_EXPAND_QROT == 1
  return ntok <= 32 ? (k & 1) : 0;
#else
  return 0;
#endif
}
#ifndef LSV_EXPAND_EPI_WARPS
#define LSV_EXPAND_EPI_WARPS 4
#endif
constexpr int kExpandEpiWarps = LSV_EXPAND_EPI_WARPS;   // 4: one per TMEM lane quadrant; 8: two, each half the columns
// Expand warp roles.  An epilogue warp can only read its TMEM lane quadrant (warp % 4), and
// tiles of <= 64 tokens (most of them) keep only quadrants 0 and 1 busy with LDTM + stores, which
// congest their SM sub-partition's memory-instruction queue.  Layout 1 therefore puts the
// producer and the MMA issuer (serial chains of shared-memory / mbarrier ops) on sub-partitions
// 2 and 3: warps 0, 1, 6, 7 = epilogue quadrants 0..3, 2 = producer, 3 = MMA, 4 and 5 idle.
// Layout 0: 0 = producer, 1 = MMA, 2.. = epilogue.
#ifndef LSV_EXPAND_LAYOUT
#define LSV_EXPAND_LAYOUT 1
#endif
#if LSV_EXPAND_LAYOUT
static_assert(LSV_EXPAND_EPI_WARPS == 4, "layout 1 has one epilogue warp per quadrant");
constexpr int kExpProdWarp = 2, kExpMmaWarp = 3, kExpandThreads = 256;
__device__ __forceinline__ bool expand_epi_warp(int w) { return w < 2 || w == 6 || w == 7; }
#else
constexpr int kExpProdWarp = 0, kExpMmaWarp = 1, kExpandThreads = 64 + 32 * kExpandEpiWarps;
__device__ __forceinline__ bool expand_epi_warp(int w) { return w >= 2; }
#endif
constexpr int kExpRecBufs = kExpandThreads / 32;   // one record buffer per warp (indexed by warp)
__host__ __device__ constexpr int expand_smem_bytes() {
  return 1024 + kExpandRingBytes + kExpandGuardBytes + 256 * 16 * 2 + kExpRecBufs * (int)sizeof(ExpandRecBuf) + 1024;
}

// ------------------------------------------------------------------------------------------
// One split-K reduce unit: 8 k of member pp for token t of split tile e (entry in the plan's
// reduce table).  Resolving it reads only static plan data.
struct RedUnit {
  MTile mt;
  int e, t, pp, k0;
};
__device__ __forceinline__ RedUnit red_unit(const ShrinkParams& p, int u, int e) {
  const int32_t* red = p.plan + p.off_red;
  while (e + 1 < p.n_red && red[2 * (e + 1) + 1] <= u) ++e;
  RedUnit ru;
  ru.mt = reinterpret_cast<const MTile*>(p.plan + p.off_mtiles)[red[2 * e]];
  ru.e = e;
  const int upr = kpad(ru.mt.rank) / 8, v = u - red[2 * e + 1];
  const int upt = p.num_proj * upr;   // units per token: projections x k units
  ru.t = v / upt;
  ru.pp = (v % upt) / upr;
  ru.k0 = (v % upr) * 8;
  return ru;
}
// Sum of the unit's partials over its splits, in split order (bit-reproducible).
__device__ __forceinline__ void red_sum(const ShrinkParams& p, const RedUnit& ru, float* s8) {
#pragma unroll
  for (int q8 = 0; q8 < 8; ++q8) s8[q8] = 0.f;
  if (ru.k0 >= ru.mt.rank || ru.t >= ru.mt.ntok) return;   // k pad / tile-aligned zero rows
  const float* partials = reinterpret_cast<const float*>(p.ws + p.ws_partials);
  const int G = p.num_proj * ru.mt.rank;
  const size_t stride = (size_t)ru.mt.ntok * G;
  const float* base = partials + ru.mt.part_off + (size_t)ru.t * G + ru.pp * ru.mt.rank + ru.k0;
  for (int j = 0; j < ru.mt.nsplit; ++j) {
    const float4 lo4 = __ldcg(reinterpret_cast<const float4*>(base + j * stride));
    const float4 hi4 = __ldcg(reinterpret_cast<const float4*>(base + j * stride) + 1);
    s8[0] += lo4.x; s8[1] += lo4.y; s8[2] += lo4.z; s8[3] += lo4.w;
    s8[4] += hi4.x; s8[5] += hi4.y; s8[6] += hi4.z; s8[7] += hi4.w;
  }
}
__device__ __forceinline__ void red_store(const ShrinkParams& p, const RedUnit& ru, const float* s8) {
  const int32_t* red = p.plan + p.off_red;
  const int kp = kpad(ru.mt.rank), np16 = round_up(ru.mt.ntok, 16);
  uint4 w, wlo;
  split_bf16x8(s8, w, wlo);
  if (p.tp > 0 && p.tp_row) {
    if (ru.k0 < ru.mt.rank) tp_row_put(p, red[2 * ru.e], ru.pp, ru.t, ru.k0, s8);
  } else if (p.tp > 0) {
    if (ru.k0 < ru.mt.rank) tp_scatter(p, red[2 * ru.e], ru.pp, ru.t, ru.k0, ru.mt.rank, np16, w, wlo);
    if (ru.k0 == 0) tp_scatter_pad(p, red[2 * ru.e], ru.pp, ru.t, np16);   // once per (token, member)
  } else {
    // tile-aligned: the piece's rows sit at its offset inside the 128-row tile image
    const int irow = p.tile_aligned ? ((ru.mt.tok_begin + ru.t) & (kTileM - 1)) : ru.t;
    const int rpad = p.tile_aligned ? kTileM : np16;
    uint8_t* dst = p.ws + p.ws_vimg + (size_t)ru.pp * p.vimg_stride + ru.mt.vimg_off + vimg_off(irow, ru.k0, kp, rpad);
    *reinterpret_cast<uint4*>(dst) = w;
    if (p.vsplit) *reinterpret_cast<uint4*>(dst + vimg_bytes(rpad, kp)) = wlo;
  }
}

// ---- shrink roles (shrink_tc_kernel and the group kernel) ---------------------------------
struct ShrinkSm {
  uint8_t* ring;
  ShrinkRecBuf* recbuf;   // indexed by warp
  uint64_t *full, *empty, *tfull, *tempty;
  uint32_t* offs;         // [kShrinkStages] ring offset of the stage behind each full barrier
};
// Pipeline position that carries over when one CTA runs several input groups back to back (the
// layer kernel): every barrier's parity follows from these running counts.  Each role keeps its
// own copy of the fields it uses (producer parts and MMA: the slot ring and the item count; MMA and
// epilogue: the TMEM buffers' parity bits; epilogue and signal warp: the record count).
struct PipeState {
  int s_slot = 0;
  uint32_t s_phase = 0;     // shrink slot ring position
  uint32_t s_tbits = 0;     // shrink TMEM buffers: bit b = parity of buffer b's next tfull wait
  int s_rec = 0;            // shrink records so far (recdone queue)
  int e_item = 0;           // expand items so far (ring allocations, v-ready queue)
  int e_q = 0;              // dynamic dispatch ring position (items + end records)
  uint32_t e_tbits = 0;     // expand TMEM buffers: bit b = parity of buffer b's next tfull wait
};
// Byte ring shared by every pipeline a CTA runs (the layer kernel: shrink stages and expand items
// of consecutive phases back to back).  Allocations are contiguous, 1024-byte aligned and released
// in allocation order (the MMA warp consumes them in that order, across phases), each when its
// release barrier completes the recorded phase; a phase's first copies therefore go out while the
// previous phase's last items are still landing — there is no drain between phases.  Every
// producer part keeps an identical copy of this bookkeeping.
// An allocation's barriers (shrink slot or expand queue entry) are reused only after the FIFO has
// released their previous allocation, so every FIFO wait names an unambiguous phase.
constexpr int kRingQ = 16;   // allocations in flight, both pipelines (>= kShrinkStages + kItemQ)
constexpr int kRingBars = 16;   // barrier ids: shrink slot s -> s, expand queue entry q -> kShrinkStages + q
constexpr int kRingTableWords = 2 * kRingQ + kRingBars;   // per producer part, in shared memory
// The counters stay in registers; the tables live in shared memory (local-memory tables queue
// behind the epilogue's global stores in L1 and slowed the producers by ~15%).
struct RingAlloc {
  uint32_t head = 0, tail = 0;   // bytes allocated / start of the oldest live allocation (monotone)
  int n = 0, r = 0;              // allocations made / released
  uint32_t* beg;                 // [kRingQ] start of allocation i % kRingQ
  uint32_t* bar;                 // [kRingQ] its release barrier: shared address | phase parity
  int* last;                     // [kRingBars] per barrier id: index of its latest allocation (-1: none)
  // tab: this part's kRingTableWords words; the whole warp calls this
  __device__ explicit RingAlloc(uint32_t* tab, int lane)
      : beg(tab), bar(tab + kRingQ), last(reinterpret_cast<int*>(tab + 2 * kRingQ)) {
    if (lane < kRingBars) last[lane] = -1;
    __syncwarp();
  }
};
__device__ __forceinline__ void ring_release_one(RingAlloc& ra) {
  const uint32_t b = ra.bar[ra.r % kRingQ];
  mbar_wait_addr(b & ~1u, b & 1u);
  ++ra.r;
  ra.tail = ra.r < ra.n ? ra.beg[ra.r % kRingQ] : ra.head;
}
// size bytes once they are free.  The allocation ends before ring_bytes + spill (free shared
// memory past the ring) and `extent` bytes from its start (the MMAs over-read past short tiles)
// before ring_bytes + guard (shared memory the over-read may touch: garbage there only reaches
// accumulator rows/columns nobody stores); else it starts at the next wrap.  Returns the offset.
__device__ __forceinline__ uint32_t ring_alloc(RingAlloc& ra, uint32_t size, uint32_t extent, uint32_t ring_bytes,
                                               uint32_t spill, uint32_t guard, int bar_id, uint32_t bar_addr,
                                               uint32_t parity) {
  uint32_t head = (ra.head + 1023u) & ~1023u;
  const uint32_t off = head % ring_bytes;
  if (off + size > ring_bytes + spill || off + extent > ring_bytes + guard) head = (head / ring_bytes + 1) * ring_bytes;
  ra.head = head;
  if (ra.r == ra.n) ra.tail = head;
  const int prev = ra.last[bar_id];   // the barriers' previous allocation must be released first
  while (ra.r <= prev || ra.n - ra.r == kRingQ || head + size - ra.tail > ring_bytes) ring_release_one(ra);
  ra.last[bar_id] = ra.n;
  ra.beg[ra.n % kRingQ] = head;
  ra.bar[ra.n % kRingQ] = bar_addr | parity;
  ++ra.n;
  ra.head = head + size;
  return head % ring_bytes;
}
// Producer: streams every record's stages into the byte ring (stage slot = barrier pair + offset).
__device__ __forceinline__ void shrink_producer(const ShrinkParams& p, const ShrinkSm& sm, int cta, int warp, int lane,
                                                int part, int nparts, PipeState& st, RingAlloc& ra, uint32_t ring_bytes,
                                                uint32_t spill) {
  // nparts warps run this loop with the same slot and ring bookkeeping; a stage's copies (A first,
  // then the x boxes) go round-robin to the parts, each arriving on full[slot] with its own bytes:
  // one warp spends ~130 cycles issuing each copy, so copies from two warps double the issue rate.
  uint8_t* ring = sm.ring;
  ShrinkRecBuf* recbuf = sm.recbuf;
  uint64_t* full = sm.full;
  uint64_t* empty = sm.empty;
  WarpRecStream<ShrinkRec, kShrinkRecCh> rs(&recbuf[warp], p.plan, p.off_recs, p.off_cta, cta, &p.a_ptrs);
  ShrinkRec inf;
  const uint8_t* a;
  int slot = st.s_slot; uint32_t phase = st.s_phase;
  int pstage = 0;   // debug stage stamps (LSV_DEBUG_SHRINK bit 16)
  const bool stamp = part == 0 && lane == 0;
  const uint32_t ring_base = smem_u32(ring);
  for (int k = 0; rs.pop(inf, a); ++k) {
    if (!(p.dbg & 16) && stamp) trace_stamp(p.trace, p.trace_items, cta, k, 0);
    // rows [p0*r, (p0+np)*r) of the group A tile (G = num_proj*r rows per 64-column chunk)
    const int r = inf.rank, G = p.num_proj * r, rows = inf.np * r, np8 = round_up(inf.ntok, 8), kch = inf.kch;
    const uint8_t* asub = a + (size_t)inf.p0 * r * 128;
    LSV_DCHECK(inf.ntok >= 1 && inf.ntok <= kTileM && inf.tok_begin >= 0 && inf.tok_begin + inf.ntok <= p.num_tokens);
    LSV_DCHECK(r >= 8 && r <= 256 && r % 8 == 0 && rows <= 256 && inf.p0 + inf.np <= p.num_proj);
    LSV_DCHECK(inf.chunk_begin >= 0 && inf.chunk_begin < inf.chunk_end && inf.chunk_end * kChunk <= p.h_in);
    LSV_DCHECK(kch >= 1 && kch * (np8 + rows) * 128 <= kShrinkSlotBytes && a != nullptr);
    const int m = np8 >> 3;   // x boxes per chunk: one per set bit of np8/8
    for (int g = inf.chunk_begin; g < inf.chunk_end; g += kch) {
      const int kc = min(kch, inf.chunk_end - g);
      if ((p.dbg & 16) && stamp) trace_stamp(p.trace, p.trace_items, cta, pstage, 3);
      // x chunks [kc][np8 rows], then A [kc][rows]; the M=128 MMA reads 16 KB from each x chunk and
      // N = round_up(rows, 16) A rows
      // (the standalone kernel's ring holds kShrinkSlots whole slots: fixed-size stages, no wrap waste)
      const uint32_t size = ring_bytes == kShrinkSlots * kShrinkSlotBytes ? kShrinkSlotBytes : (uint32_t)(kc * (np8 + rows) * 128);
      const uint32_t extent = max(size + (uint32_t)((round_up(rows, 16) - rows) * 128),
                                  (uint32_t)((kc - 1) * np8 * 128 + kTileM * 128));
      const uint32_t off = ring_alloc(ra, size, extent, ring_bytes, spill, kShrinkGuardBytes, slot, smem_u32(&empty[slot]), phase);
      if (part == 0) sm.offs[slot] = off;   // every lane: the elected arriving lane's own store
      if ((p.dbg & 16) && stamp) trace_stamp(p.trace, p.trace_items, cta, pstage, 4);
      const uint32_t fb = smem_u32(&full[slot]);
      // part 0 copies A; chunk c's x boxes belong to part (c + 1) % nparts
      const bool do_a = part == 0 && !(p.dbg & 2), do_x = !(p.dbg & 4);
      const int my_chunks = do_x ? (kc + nparts - 1 - (part + nparts - 1) % nparts) / nparts : 0;
      mbar_arrive_expect_tx_elect(fb, (uint32_t)((do_a ? kc * rows : 0) + my_chunks * np8) * 128);
      const uint32_t dst = ring_base + off;
      if (do_a) {
        if (rows == G) {       // whole group: the kc chunks are one contiguous run
          bulk_load_elect(dst + kc * np8 * 128, a + (size_t)g * G * 128, (uint32_t)(kc * G * 128), fb);
        } else {               // projection subset: one copy per chunk
          for (int c = 0; c < kc; ++c)
            bulk_load_elect(dst + (kc * np8 + c * rows) * 128, asub + (size_t)(g + c) * G * 128, (uint32_t)(rows * 128), fb);
        }
      }
      if (do_x) {
        for (int c = (part + nparts - 1) % nparts; c < kc; c += nparts) {
          int mm = m, row = 0;
          while (mm) {
            const int bb = 31 - __clz(mm);
            tma_load_2d_elect(dst + (c * np8 + row) * 128, &p.xmap[bb], fb, (g + c) * kChunk, inf.tok_begin + row);
            row += 8 << bb;
            mm &= ~(1 << bb);
          }
        }
      }
      if ((p.dbg & 16) && stamp) trace_stamp(p.trace, p.trace_items, cta, pstage++, 5);
      if (++slot == kShrinkStages) { slot = 0; phase ^= 1; }
    }
    if (!(p.dbg & 16) && stamp) trace_stamp(p.trace, p.trace_items, cta, k, 1);
    __syncwarp();
  }
  st.s_slot = slot;
  st.s_phase = phase;
}
// MMA issuer: the whole warp runs the loop (warp-uniform values stay in uniform registers, so each
// MMA costs a few uniform adds), one lane issues.  Returns the number of records.
__device__ __forceinline__ int shrink_mma(const ShrinkParams& p, const ShrinkSm& sm, uint32_t tmem_base, int cta, int warp,
                                          int lane, PipeState& st) {
  uint8_t* ring = sm.ring;
  ShrinkRecBuf* recbuf = sm.recbuf;
  uint64_t* full = sm.full;
  uint64_t* empty = sm.empty;
  uint64_t* tfull = sm.tfull;
  uint64_t* tempty = sm.tempty;
  // the whole warp runs the loop (warp-uniform values stay in uniform registers, so each MMA costs a
  // few uniform adds); an elected lane issues
  WarpRecStream<ShrinkRec, kShrinkRecCh> rs(&recbuf[warp], p.plan, p.off_recs, p.off_cta, cta, nullptr);
  ShrinkRec inf;
  const uint8_t* unused;
  int slot = st.s_slot; uint32_t phase = st.s_phase;
  int dbg_stage = 0;
  const uint32_t ring_base = __shfl_sync(0xffffffffu, smem_u32(ring), 0);
  const int nbuf = kTmemCols / p.acc_cols;
  int k = 0;
  for (; rs.pop(inf, unused); ++k) {
    const int rows = __shfl_sync(0xffffffffu, inf.rank * inf.np, 0);
    const int np8 = round_up(__shfl_sync(0xffffffffu, inf.ntok, 0), 8);
    const int kch = __shfl_sync(0xffffffffu, inf.kch, 0);
    const int cb = __shfl_sync(0xffffffffu, inf.chunk_begin, 0), ce = __shfl_sync(0xffffffffu, inf.chunk_end, 0);
    const int buf = k % nbuf;
    mbar_wait(&tempty[buf], ((st.s_tbits >> buf) & 1) ^ 1);
    tc_fence_after();
    const uint32_t d = tmem_base + buf * p.acc_cols;
    const uint32_t idesc = idesc_bf16(128, max(16, round_up(rows, 16)));
    const uint32_t xstep = (uint32_t)(np8 * 128) >> 4, astep = (uint32_t)(rows * 128) >> 4;  // per chunk, desc units
    uint32_t accumulate = 0;
    for (int g = cb; g < ce; g += kch) {
      const int kc = min(kch, ce - g);
      if ((p.dbg & 16) && lane == 0) trace_stamp(p.trace, p.trace_items, cta, dbg_stage, 6);
      mbar_wait(&full[slot], phase);
      tc_fence_after();
      if ((p.dbg & 16) && lane == 0) trace_stamp(p.trace, p.trace_items, cta, dbg_stage++, 7);
      const uint32_t xb = ring_base + sm.offs[slot];
      uint64_t adesc = smem_desc(xb, 16, 1024, 2);
      uint64_t bdesc = smem_desc(xb + kc * np8 * 128, 16, 1024, 2);
      for (int c = 0; c < kc; ++c) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {   // K=16 steps inside the 128-byte swizzle row: +32 B = +2
          umma_bf16_elect(d, adesc + 2 * kk, bdesc + 2 * kk, idesc, accumulate);
          accumulate = 1;
        }
        adesc += xstep;
        bdesc += astep;
      }
      umma_commit_elect(&empty[slot]);
      if (++slot == kShrinkStages) { slot = 0; phase ^= 1; }
    }
    umma_commit_elect(&tfull[buf]);
    st.s_tbits ^= 1u << buf;
    if (!(p.dbg & 16) && lane == 0) trace_stamp(p.trace, p.trace_items, cta, k, 2);
  }
  st.s_slot = slot;
  st.s_phase = phase;
  return k;
}
// Epilogue: thread = token row of quadrant q.  In the group kernel (recdone != nullptr) each warp
// arrives on recdone[k % kRecQ] once its rows of record k are stored; the signal warp publishes
// (and counts the records it has published in the int after the barriers: back-pressure).
constexpr int kRecQ = 16;   // recdone barriers, then the signal warp's progress counter
__device__ __forceinline__ void shrink_epilogue(const ShrinkParams& p, const ShrinkSm& sm, uint32_t tmem_base, int cta,
                                                int warp, int lane, uint64_t* recdone, PipeState& st) {
  ShrinkRecBuf* recbuf = sm.recbuf;
  uint64_t* tfull = sm.tfull;
  uint64_t* tempty = sm.tempty;
  const int q = warp & 3, row = q * 32 + lane;
  float* partials = reinterpret_cast<float*>(p.ws + p.ws_partials);
  WarpRecStream<ShrinkRec, kShrinkRecCh> rs(&recbuf[warp], p.plan, p.off_recs, p.off_cta, cta, nullptr);
  ShrinkRec inf;
  const uint8_t* unused;
  const int nbuf = kTmemCols / p.acc_cols;
  int k = 0;
  for (; rs.pop(inf, unused); ++k) {
    const int r = inf.rank, nt = inf.ntok, kp = kpad(r), np16 = round_up(nt, 16);
    const int G = p.num_proj * r, rows = inf.np * r;
    const int buf = k % nbuf;
    mbar_wait(&tfull[buf], (st.s_tbits >> buf) & 1);
    st.s_tbits ^= 1u << buf;
    tc_fence_after();
    if (!(p.dbg & 16) && q == 0 && lane == 0) trace_stamp(p.trace, p.trace_items, cta, k, 3);
    const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + buf * p.acc_cols;
    const bool valid = row < nt && !(p.dbg & 8);
    uint8_t* vimg = p.ws + p.ws_vimg + inf.vimg_off;          // + projection * vimg_stride
    // tile-aligned images (fused base GEMM): 128 rows, this piece at rows tok_begin % 128 + row,
    // every other row zero; each thread writes image row (tok_begin + row) % 128, zeros if !valid
    const bool ta = p.tile_aligned != 0;
    const int irow = ta ? ((inf.tok_begin + row) & (kTileM - 1)) : row, rpad = ta ? kTileM : np16;
    const bool wimg = ta ? !(p.dbg & 8) : valid;              // writes an image row (nsplit == 1)
    const uint32_t vlo = vimg_bytes(rpad, kp);                // hi image -> lo image (split v)
    LSV_DCHECK(p.tp > 0 || (int64_t)p.ws_vimg + (int64_t)(p.num_proj - 1) * p.vimg_stride + inf.vimg_off +
                                 (int64_t)vlo * (p.vsplit ? 2 : 1) <= p.ws_bytes);
    LSV_DCHECK(inf.nsplit == 1 || (int64_t)p.ws_partials + 4 * ((int64_t)inf.part_off +
                                 (int64_t)inf.nsplit * nt * G) <= p.ws_bytes);
    float* part = partials + inf.part_off + ((size_t)inf.split * nt + row) * G + inf.p0 * r;
    for (int cc = 0; cc < rows; cc += 16) {
      float v[16];
      tmem_ld_32x32b_x16(taddr + cc, v);
      if (valid || (wimg && inf.nsplit == 1)) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int j0 = cc + h * 8;          // 8 columns, all of projection p0 + j0 / r (r % 8 == 0)
          if (j0 < rows) {
            if (inf.nsplit == 1) {
              uint4 w, wlo;
              split_bf16x8(v + h * 8, w, wlo);
              if (!valid) w = wlo = make_uint4(0, 0, 0, 0);   // tile-aligned zero row
              const int pp = inf.p0 + j0 / r;
              if (p.tp > 0 && p.tp_row) tp_row_put(p, inf.mtile, pp, row, j0 % r, v + h * 8);
              else if (p.tp > 0) tp_scatter(p, inf.mtile, pp, row, j0 % r, r, np16, w, wlo);
              else {
                uint8_t* dst = vimg + (size_t)pp * p.vimg_stride + vimg_off(irow, j0 % r, kp, rpad);
                *reinterpret_cast<uint4*>(dst) = w;
                if (p.vsplit) *reinterpret_cast<uint4*>(dst + vlo) = wlo;
              }
            } else {
              float* dst = part + j0;
              if ((reinterpret_cast<uintptr_t>(dst) & 31) == 0) {   // one full sector per row
                st_global_v8_if(dst, reinterpret_cast<const uint32_t*>(v + h * 8), true);
              } else {
                reinterpret_cast<float4*>(dst)[0] = make_float4(v[h * 8 + 0], v[h * 8 + 1], v[h * 8 + 2], v[h * 8 + 3]);
                reinterpret_cast<float4*>(dst)[1] = make_float4(v[h * 8 + 4], v[h * 8 + 5], v[h * 8 + 6], v[h * 8 + 7]);
              }
            }
          }
        }
      }
    }
    if (valid && inf.nsplit == 1 && p.tp > 0) {
      if (!p.tp_row)
        for (int pp = inf.p0; pp < inf.p0 + inf.np; ++pp) tp_scatter_pad(p, inf.mtile, pp, row, np16);
    } else if (wimg && inf.nsplit == 1 && kp != r) {   // the k pad of each v image (r % 16 == 8) is zero
      for (int pp = inf.p0; pp < inf.p0 + inf.np; ++pp) {
        uint8_t* dst = vimg + (size_t)pp * p.vimg_stride + vimg_off(irow, r, kp, rpad);
        *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
        if (p.vsplit) *reinterpret_cast<uint4*>(dst + vlo) = make_uint4(0, 0, 0, 0);
      }
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&tempty[buf]);
    if (recdone != nullptr && lane == 0) {   // group kernel: stored (the signal warp is < kRecQ behind)
      const volatile int* sigc = reinterpret_cast<const volatile int*>(recdone + kRecQ);
      const int kg = st.s_rec + k;   // record index over every group this CTA has run
      while (kg >= kRecQ && *sigc <= kg - kRecQ) __nanosleep(32);
      mbar_arrive(&recdone[kg % kRecQ]);
    }
    if (!(p.dbg & 16) && q == 0 && lane == 0) trace_stamp(p.trace, p.trace_items, cta, k, 4);
    if (!(p.dbg & 16) && q == 0 && lane == 0) trace_stamp(p.trace, p.trace_items, cta, k, 5);
  }
  st.s_rec += k;
  }

__global__ void __launch_bounds__(kShrinkThreads, 1) shrink_tc_kernel(const __grid_constant__ ShrinkParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* ring = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  ShrinkRecBuf* recbuf = reinterpret_cast<ShrinkRecBuf*>(ring + kShrinkSlots * kShrinkSlotBytes + kShrinkGuardBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(recbuf + kShrinkRecBufs);
  uint64_t* empty = full + kShrinkStages;
  uint64_t* tfull = empty + kShrinkStages;
  uint64_t* tempty = tfull + kAccBufs;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + kAccBufs);
  uint32_t* offs = tmem_slot + 1;
  uint32_t* ring_tab = offs + kShrinkStages;   // [kProdParts][kRingTableWords]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) phase_stamp(p.trace, p.trace_items, blockIdx.x, 0);
  if (threadIdx.x == 0) {
  for (int s = 0; s < kShrinkStages; ++s) { mbar_init(&full[s], kProdParts); mbar_init(&empty[s], 1); }
  for (int b = 0; b < kAccBufs; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 4); }
  fence_mbar_init();
  for (int b = 0; b < 5; ++b) prefetch_tmap(&p.xmap[b]);
  }
  if (warp == kShrMmaWarp) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int cta = blockIdx.x;
  if (threadIdx.x == 0) phase_stamp(p.trace, p.trace_items, cta, 1);
  if (p.wait_prev) pdl_wait();   // x, workspace and counters are written by earlier launches
  pdl_launch_dependents();
  if (threadIdx.x == 0) phase_stamp(p.trace, p.trace_items, cta, 2);
  const ShrinkSm sm{ring, recbuf, full, empty, tfull, tempty, offs};
  if (warp == kShrProdWarp || (warp == kProdWarp2 && kProdParts == 2)) {
  PipeState st;
  RingAlloc ra(ring_tab + (warp == kShrProdWarp ? 0 : kRingTableWords), lane);
  shrink_producer(p, sm, cta, warp, lane, warp == kShrProdWarp ? 0 : 1, kProdParts, st, ra, kShrinkSlots * kShrinkSlotBytes,
                  kShrinkGuardBytes);
  } else if (warp == kShrMmaWarp) {
  PipeState st;
  shrink_mma(p, sm, tmem_base, cta, warp, lane, st);
  } else if (shrink_epi_warp(warp)) {
  PipeState st;
  shrink_epilogue(p, sm, tmem_base, cta, warp, lane, nullptr, st);
  }
  // CTA c owns split-K reduce units [c*U/G, (c+1)*U/G) of the concatenated split tiles; the host
  // recorded the table entry holding its first unit.  Each thread resolves its first two units
  // (static plan data, dependent loads) now, while other warps finish, so that after the grid
  // barrier it only loads and sums partials.
  const int u0 = (int)((int64_t)p.red_units * blockIdx.x / gridDim.x);
  const int u1 = (int)((int64_t)p.red_units * (blockIdx.x + 1) / gridDim.x);
  const int ua = u0 + threadIdx.x, ub = ua + blockDim.x;
  RedUnit ra{}, rb{};
  if (p.n_red > 0 && ua < u1) {
  ra = red_unit(p, ua, p.plan[p.off_red_cta + blockIdx.x]);
  if (ub < u1) rb = red_unit(p, ub, ra.e);
  }
  tc_fence_before();
  __threadfence();             // partials visible device-wide before the grid barrier
  if (p.tp > 0) __threadfence_system();   // scattered images visible to the peers
  __syncthreads();
  if (threadIdx.x == 0) phase_stamp(p.trace, p.trace_items, cta, 3);
  if (warp == kShrMmaWarp) { tc_fence_after(); tmem_dealloc(tmem_base, kTmemCols); }
  if (p.n_red == 0) {
  if (p.tp > 0) tp_signal(p);
  return;
  }

  // ---- grid-wide split-K reduction (all CTAs are co-resident: grid <= SMs, 1 CTA per SM) ----
  // Every (token, 8-wide k unit) of every split tile is summed over its splits in fixed split
  // order by one thread, so results are bit-identical from run to run.
  int* bar = p.gbar;
  if (threadIdx.x == 0) {
  atomicAdd(&bar[0], 1);
  int seen = 0;
  uint64_t t0 = 0;
  for (uint32_t spin = 0;; ++spin) {
    seen = ld_relaxed_gpu(&bar[0]);
    if (seen >= (int)gridDim.x) { (void)ld_acquire_gpu(&bar[0]); break; }
    __nanosleep(64);
    if ((spin & 1023u) == 1023u) {   // bounded: trap after ~4 s instead of hanging the GPU
      const uint64_t now = globaltimer_ns();
      if (t0 == 0) t0 = now;
      else if (now - t0 > 4000000000ull) __trap();
    }
  }
  }
  __syncthreads();
  if (threadIdx.x == 0) phase_stamp(p.trace, p.trace_items, cta, 4);
  if (ua < u1) {
  float sa[8], sb[8];
  red_sum(p, ra, sa);                  // both units' loads in flight before either store
  if (ub < u1) red_sum(p, rb, sb);
  red_store(p, ra, sa);
  if (ub < u1) red_store(p, rb, sb);
  int e = ub < u1 ? rb.e : ra.e;
  for (int u = ub + blockDim.x; u < u1; u += blockDim.x) {
    const RedUnit ru = red_unit(p, u, e);
    e = ru.e;
    float s8[8];
    red_sum(p, ru, s8);
    red_store(p, ru, s8);
  }
  }
  if (p.tp > 0) __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) phase_stamp(p.trace, p.trace_items, cta, 5);
  if (threadIdx.x == 0 && atomicAdd(&bar[1], 1) == (int)gridDim.x - 1) {
  bar[0] = 0;                // every CTA is past the barrier: re-arm it for the next launch
  bar[1] = 0;
  if (p.tp > 0)              // the last CTA out: every rank's copy of this group is complete
    for (int d = 0; d < p.tp; ++d) red_release_sys_add(p.flags[d], 1);
  }
}

// ------------------------------------------------------------------------------------------
// Expand: per item (m-tile of <=128 tokens, tw-wide h_out tile, tw = 256 or 128):
//     D[tok x tw] = v[tok x K=kp] . B_s[K x tw]  +  I[tok x K=tok16] . y[K=tok16 x tw]
// The first MMA group is the LoRA expand (A = v image, K-major swizzled; B = the B tile, MN-major
// SWIZZLE_128B); the second adds the current y rows on the tensor core: A = a 0/1 identity
// block, B = the y tile TMA-loaded as an MN-major SWIZZLE_128B operand.  TMEM lane = token,
// columns = h_out, so the epilogue is LDTM -> cvt.bf16x2 -> 16-byte stores of contiguous row
// pieces (~0.7 instructions per element), and the ring bytes are released as soon as the MMAs
// have read them.  The producer warp issues an item's copies from several lanes at once.
constexpr int kIdentRows = 256;  // identity block at rows [128, 144) of a zero [256 x 16] A tile

// Row-parallel TP: CTA c sums m-tiles c, c + grid, ... over the wait_target fp32 partial slots
// (rank order 0..T-1: every rank computes the same bits) into the bf16 v images; k pads are zero.
__device__ __forceinline__ void tp_row_sum(const ExpandParams& p) {
  const MTile* mts = reinterpret_cast<const MTile*>(p.plan + p.off_mtiles);
  for (int m = blockIdx.x; m < p.n_mtiles; m += gridDim.x) {
    const MTile mt = mts[m];
    const int kp = kpad(mt.rank), upr = kp / 8, np16 = round_up(mt.ntok, 16);
    const int units = mt.ntok * upr * p.num_proj;
    for (int u = threadIdx.x; u < units; u += blockDim.x) {
      const int pp = u / (mt.ntok * upr), rem = u % (mt.ntok * upr), t = rem / upr, k0 = (rem % upr) * 8;
      float s8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      if (k0 < mt.rank) {
        const size_t off = (size_t)pp * 2 * p.vimg_stride + 2 * (size_t)mt.vimg_off + ((size_t)t * kp + k0) * 4;
        for (int d = 0; d < p.wait_target; ++d) {
          const float4* src = reinterpret_cast<const float4*>(p.xsum + (size_t)d * p.xslot + off);
          const float4 lo = __ldcg(src), hi = __ldcg(src + 1);
          s8[0] += lo.x; s8[1] += lo.y; s8[2] += lo.z; s8[3] += lo.w;
          s8[4] += hi.x; s8[5] += hi.y; s8[6] += hi.z; s8[7] += hi.w;
        }
      }
      uint4 w, wlo;
      split_bf16x8(s8, w, wlo);
      uint8_t* dst = p.ws + p.ws_vimg0 + (size_t)pp * p.vimg_stride + mt.vimg_off + vimg_off(t, k0, kp, np16);
      *reinterpret_cast<uint4*>(dst) = w;
      if (p.vsplit) *reinterpret_cast<uint4*>(dst + vimg_bytes(mt.ntok, kp)) = wlo;
    }
  }
}

// y rows [tok_begin, tok_begin + np16) as nb 64-column SWIZZLE_128B blocks; each block is np16/8 =
// a sum of powers of two 8-row groups -> one TMA box per set bit.  Box `box` (one per lane):
// 64-column block h, first row `row`, box map index bb (8 << bb rows).  False: no such box.
__device__ __forceinline__ bool y_box(int np16, int nb, int box, int& h, int& row, int& bb) {
  const int m = np16 >> 3, pc = __popc(m);
  if (box < 0 || box >= nb * pc) return false;
  h = box / pc;
  const int i = box % pc;
  int mm = m;
  row = 0;
  bb = -1;
  for (int s2 = 0; s2 <= i; ++s2) {       // i-th set bit from the top
    bb = 31 - __clz(mm);
    if (s2 < i) { row += 8 << bb; mm &= ~(1 << bb); }
  }
  return true;
}

// ---- expand roles (expand_tc_kernel and the group kernel) ---------------------------------
constexpr int kVQ = 16;   // group kernel: v-ready queue between the ready checker and the producer
struct ExpandSm {
  uint8_t* ring;
  uint8_t* ident;
  ExpandRecBuf* recbuf;   // indexed by warp
  uint32_t* offs;
  uint64_t *full, *empty, *tfull, *tempty;
  DynRing* dyn;           // dynamic dispatch (layer kernel) or nullptr
};
// Producer (whole warp, converged): every lane keeps the same ring bookkeeping and computes the
// same copy operands; each copy is issued by one elected lane inside its asm (issuing the y
// boxes from different lanes made ptxas serialise them through a per-lane uniformization loop,
// ~1800 cycles per item).  B and y are issued first; in the group kernel (vfull != nullptr) the
// v copy waits until the ready checker has seen the item's m-tile complete.
__device__ __forceinline__ void expand_producer(const ExpandParams& p, const ExpandSm& sm, int cta, int warp, int lane,
                                                uint64_t* vfull, uint64_t* vempty, int part, int nparts, PipeState& st,
                                                RingAlloc& ra) {
  // nparts (1 or 2) warps run this loop with the same ring bookkeeping: part 0 copies B and v
  // (and y when alone), part 1 the y boxes; each arrives on full[] with its own bytes.
  uint8_t* ring = sm.ring;
  ExpandRecBuf* recbuf = sm.recbuf;
  uint32_t* offs = sm.offs;
  uint64_t* full = sm.full;
  uint64_t* empty = sm.empty;
  // Every lane keeps the same ring bookkeeping and computes the same copy operands; each copy
  // is issued by one elected lane inside its asm.  (Issuing the y boxes from different lanes
  // made ptxas serialise them through a per-lane uniformization loop: ~1800 cycles per item.)
  ExpSrc rs(&recbuf[warp], p.plan, p.off_recs, p.off_cta, cta, p.b_ptrs, sm.dyn, &st.e_q);
  ExpandRec inf;
  const uint8_t* b;
  const int k0 = st.e_item;
  const uint32_t ring_base = __shfl_sync(0xffffffffu, smem_u32(ring), 0);
  int k = k0;
  for (; rs.pop(inf, b); ++k) {
    const int twl = p.tws[inf.proj], tw = expand_item_tw(inf.rank, twl), nb = tw / 64;
    const int kp = kpad(inf.rank), np16 = round_up(inf.ntok, 16), S = kmajor_row_bytes(kp);
    const uint32_t vlo = vimg_bytes(inf.ntok, kp);
    const uint32_t bbytes = tw * kp * 2, vbytes = np16 * kp * 2 + (p.vsplit ? vlo : 0), ybytes = nb * np16 * 128;
    const uint32_t voff = round_up(bbytes, 1024), yoff = round_up(voff + vbytes, 1024);
    const uint32_t size = yoff + ybytes;
    const int qs = k % kItemQ;
    const uint32_t extent =
        max(size, voff + (p.vsplit ? vlo : 0u) + (uint32_t)((kp * 2 / S - 1) * np16 * S + 128 * S));
    LSV_DCHECK(extent <= (uint32_t)(kExpandRingBytes + kExpandGuardBytes) && size <= (uint32_t)kExpandRingBytes);
    LSV_DCHECK(inf.ntok >= 1 && inf.ntok <= kTileM && inf.tok_begin + inf.ntok <= p.num_tokens);
    LSV_DCHECK(inf.proj >= 0 && inf.proj < kMaxProj && (inf.jtile + 1) * tw <= p.h_outs[inf.proj]);
    LSV_DCHECK(p.wait_flag != nullptr || (int64_t)p.ws_vimg[inf.proj] + inf.vimg_off + vbytes <= p.ws_bytes);
    const bool p0 = part == 0, stamp = p0 && lane == 0, do_y = nparts == 1 || part == 1;
    if (stamp) trace_stamp(p.trace, p.trace_items, cta, k - k0, 0);
    const uint32_t ring_off = ring_alloc(ra, size, extent, kExpandRingBytes, kExpandGuardBytes, kExpandGuardBytes, kShrinkStages + qs,
                                         smem_u32(&empty[qs]), (k / kItemQ) & 1);
    if (stamp) offs[qs] = ring_off;
    const int dbg = p.dbg;
    const uint32_t fb = smem_u32(&full[qs]);
    mbar_arrive_expect_tx_elect(fb, (p0 ? ((dbg & 16) ? 0 : bbytes) + ((dbg & 32) ? 0 : vbytes) : 0u) +
                                        (do_y ? ((dbg & 8) ? 0 : ybytes) : 0u));
    if (stamp) trace_stamp(p.trace, p.trace_items, cta, k - k0, 1);
    const uint32_t dst = ring_base + ring_off;
    if (p0 && !(dbg & 16)) {
      if (tw < twl) {   // a 128-wide half of a 256-wide layout tile: 2 KB per 8-k group
        const int halves = twl / tw, jt = inf.jtile / halves, sub = inf.jtile % halves;
        const uint8_t* src = b + (size_t)jt * twl * kp * 2 + sub * nb * 1024;
        for (int kg = 0; kg < kp / 8; ++kg)
          bulk_load_elect(dst + kg * nb * 1024, src + (size_t)kg * (twl / 64) * 1024, (uint32_t)(nb * 1024), fb);
      } else {
        bulk_load_elect(dst, b + (size_t)inf.jtile * bbytes, bbytes, fb);
      }
    }
    if (stamp) trace_aux(p.trace, p.trace_items, cta, k - k0, 3);
    if (do_y && !(dbg & 8)) {
      // y rows [tok_begin, +np16): one 3D box per set bit of np16 / 8 (largest first), each
      // [nb blocks][R rows][64] at yoff + row * nb * 128
      const CUtensorMap* ym = nb == 4 ? p.ymap[inf.proj] : p.ymap2[inf.proj];
      int mm = np16 >> 3, row = 0;
      while (mm) {
        const int bbit = 31 - __clz(mm);
        tma_load_3d_elect(dst + yoff + row * nb * 128, &ym[bbit], fb, 0, inf.tok_begin + row, inf.jtile * nb);
        row += 8 << bbit;
        mm &= ~(1 << bbit);
      }
    }
    if (p0 && vfull != nullptr) {   // group kernel: the tile's v images are complete (ready checker warp)
      if (stamp) trace_aux(p.trace, p.trace_items, cta, k - k0, 5);
      mbar_wait(&vfull[k % kVQ], (k / kVQ) & 1);
      if (stamp) trace_aux(p.trace, p.trace_items, cta, k - k0, 6);
      if (lane == 0) mbar_arrive(&vempty[k % kVQ]);
    }
    if (p0 && !(dbg & 32)) bulk_load_elect(dst + voff, p.ws + p.ws_vimg[inf.proj] + inf.vimg_off, vbytes, fb);
    if (stamp) trace_aux(p.trace, p.trace_items, cta, k - k0, 4);
    __syncwarp();
  }
  st.e_item = k;
}
// MMA issuer (whole warp): the election happens inside the MMA asm, so ptxas emits no per-MMA
// uniformization loop; descriptors advance by constant steps (start address field = byte
// address >> 4, below 2^14 in shared memory).
__device__ __forceinline__ void expand_mma(const ExpandParams& p, const ExpandSm& sm, uint32_t tmem_base, int cta, int warp,
                                           int lane, PipeState& st) {
  uint8_t* ring = sm.ring;
  uint8_t* ident = sm.ident;
  ExpandRecBuf* recbuf = sm.recbuf;
  uint32_t* offs = sm.offs;
  uint64_t* full = sm.full;
  uint64_t* empty = sm.empty;
  uint64_t* tfull = sm.tfull;
  uint64_t* tempty = sm.tempty;
  const int nbuf = kTmemCols / p.tw_max;     // TMEM accumulators in flight
  // Every lane runs the loop and computes the same descriptors; the election happens inside the
  // MMA asm, so ptxas emits no per-MMA uniformization loop.  Descriptors advance by constant
  // steps (start address field = byte address >> 4, which stays below 2^14 in shared memory).
  ExpSrc rs(&recbuf[warp], p.plan, p.off_recs, p.off_cta, cta, nullptr, sm.dyn, &st.e_q);
  ExpandRec inf;
  const uint8_t* unused;
  const uint32_t ib = smem_u32(ident);
  const uint32_t ring_base = __shfl_sync(0xffffffffu, smem_u32(ring), 0);
  const int k0 = st.e_item;
  int k = k0;
  for (; rs.pop(inf, unused); ++k) {
    const int r = inf.rank;
    const int tw = expand_item_tw(r, p.tws[inf.proj]), nb = tw / 64;
    const uint32_t idesc_mn = idesc_bf16(128, tw, 1);
    const int qs = k % kItemQ;
    const int kp = kpad(r), np16 = round_up(inf.ntok, 16);
    const int S = kmajor_row_bytes(kp), ck = S / 2;
    const uint32_t vlay = umma_layout(S);
    const int buf = (k - k0) % nbuf;
    mbar_wait(&tempty[buf], ((st.e_tbits >> buf) & 1) ^ 1);
    if (lane == 0) trace_stamp(p.trace, p.trace_items, cta, k - k0, 5);
    mbar_wait(&full[qs], (k / kItemQ) & 1);
    if (lane == 0) trace_stamp(p.trace, p.trace_items, cta, k - k0, 6);
    tc_fence_after();
    const uint32_t bb = ring_base + offs[qs];
    const uint32_t voff = round_up(tw * kp * 2, 1024);
    const uint32_t vb = bb + voff;
    const uint32_t vlo = vimg_bytes(inf.ntok, kp);
    const uint32_t yb = bb + round_up(voff + np16 * kp * 2 + (p.vsplit ? vlo : 0u), 1024);
    const uint32_t d = tmem_base + buf * p.tw_max;
    const int qrow = 32 * expand_qbase(k - k0, inf.ntok);
    const int nv = (p.dbg & 128) ? 1 : kp / 16, ny = (p.dbg & 64) ? 0 : np16 / 16;
    // D = v . B (+ v_lo . B): A = v image (K-major, swizzled by kp), B = B tile (MN-major SW128).
    // K step ks: A advances 32 B inside a swizzle row, np16 rows of S bytes per ck-element chunk;
    // B advances one 2 * nb KB group of 16 k.
    const uint64_t a0 = smem_desc(vb - qrow * S, 16, 8 * S, vlay);
    const uint64_t b0 = smem_desc(bb, 1024, nb * 1024, 2);
    const uint32_t bstep = (2 * nb * 1024) >> 4, cstep = (np16 * S) >> 4;
    for (int h = 0; h < (p.vsplit ? 2 : 1); ++h) {
      uint64_t arow = a0 + (h ? (vlo >> 4) : 0u), bd = b0;
      for (int ks = 0; ks < nv; ++ks) {
        const uint32_t in_row = (uint32_t)((ks * 16) % ck) * 2 >> 4;
        umma_bf16_elect(d, arow + in_row, bd, idesc_mn, (h | ks) ? 1u : 0u);
        bd += bstep;
        if (((ks + 1) * 16) % ck == 0) arow += cstep;
      }
    }
    // D += I . y : A = identity rows shifted by 16*ks (K-major SW32), B = y (MN-major SW128)
    // y sits in boxes of R = 8 << b rows (largest first), box at yb + row0 * nb * 128 with block
    // stride R * 128; every box holds whole 16-row K steps (np16 / 8 is even)
    uint64_t ai = smem_desc(ib + (128 - qrow) * 32, 16, 256, 6);
    {
      int mm = np16 >> 3, row0 = 0, ks = 0;
      while (mm && ks < ny) {
        const int bbit = 31 - __clz(mm), R = 8 << bbit;
        uint64_t by = smem_desc(yb + row0 * nb * 128, R * 128, 1024, 2);
        for (int r = 0; r < R && ks < ny; r += 16, ++ks) {
          umma_bf16_elect(d, ai, by, idesc_mn, 1u);
          ai -= 32;      // 16 identity rows x 32 B
          by += 128;     // 16 y rows x 128 B
        }
        row0 += R;
        mm &= ~(1 << bbit);
      }
    }
    umma_commit_elect(&empty[qs]);   // ring bytes free once these MMAs have read them
    umma_commit_elect(&tfull[buf]);
    st.e_tbits ^= 1u << buf;
    if (lane == 0) trace_stamp(p.trace, p.trace_items, cta, k - k0, 2);
    __syncwarp();
  }
  st.e_item = k;
}
// Epilogue: thread = token row of quadrant q.
__device__ __forceinline__ void expand_epilogue(const ExpandParams& p, const ExpandSm& sm, uint32_t tmem_base, int cta,
                                                int warp, int lane, PipeState& st) {
  ExpandRecBuf* recbuf = sm.recbuf;
  uint64_t* tfull = sm.tfull;
  uint64_t* tempty = sm.tempty;
  const int nbuf = kTmemCols / p.tw_max;
  const int q = warp & 3;
  const int half = (warp - 2) >> 2;          // with 8 epilogue warps: which half of the columns
  ExpSrc rs(&recbuf[warp], p.plan, p.off_recs, p.off_cta, cta, nullptr, sm.dyn, &st.e_q);
  ExpandRec inf;
  const uint8_t* unused;
  for (int k = 0; rs.pop(inf, unused); ++k) {
    const int buf = k % nbuf;
    mbar_wait(&tfull[buf], (st.e_tbits >> buf) & 1);
    st.e_tbits ^= 1u << buf;
    tc_fence_after();
    if (q == 0 && lane == 0) trace_stamp(p.trace, p.trace_items, cta, k, 3);
    const int qr = q - expand_qbase(k, inf.ntok);   // this warp's quadrant within the item
    const int t = qr * 32 + lane;
    if (qr >= 0 && qr * 32 < inf.ntok) {   // warp-uniform: other quadrants have no rows
      const int tw = expand_item_tw(inf.rank, p.tws[inf.proj]);
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + buf * p.tw_max;
      const bool valid = t < inf.ntok && !(p.dbg & 1);
      __nv_bfloat16* yrow = p.y[inf.proj] + (int64_t)(inf.tok_begin + (valid ? t : 0)) * p.ldy[inf.proj] + inf.jtile * tw;
      const int c_lo = kExpandEpiWarps == 8 ? half * (tw / 2) : 0, c_hi = kExpandEpiWarps == 8 ? c_lo + tw / 2 : tw;
      // each lane writes its own token row: 32-byte stores are one full sector per row and half
      // the store wavefronts of 16-byte ones; streaming (evict-first) since y is not re-read here
      const bool st32 = LSV_EXPAND_ST32 && p.st32[inf.proj];
#if LSV_EXPAND_EPI_PIPE
      // two 32-column chunks in flight: chunk i+1's TMEM load overlaps chunk i's convert + stores
      auto put = [&](const uint32_t* r, int cc) {
        uint32_t w[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) w[e] = pack_bf16x2(__uint_as_float(r[2 * e]), __uint_as_float(r[2 * e + 1]));
        if (st32) {
#pragma unroll
          for (int u = 0; u < 2; ++u) st_global_v8_cs_if(yrow + cc + u * 16, &w[8 * u], valid);
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            st_global_v4_if(yrow + cc + u * 8, w[4 * u], w[4 * u + 1], w[4 * u + 2], w[4 * u + 3], valid);
        }
      };
      uint32_t ra[32], rb[32];
      tmem_ld_32x32b_x32_nowait(taddr + c_lo, ra);
#pragma unroll 1
      for (int cc = c_lo; cc < c_hi; cc += 64) {   // (c_hi - c_lo) is a multiple of 64
        tmem_wait_ld_regs(ra);
        tmem_ld_32x32b_x32_nowait(taddr + cc + 32, rb);
        put(ra, cc);
        tmem_wait_ld_regs(rb);
        if (cc + 64 < c_hi) tmem_ld_32x32b_x32_nowait(taddr + cc + 64, ra);
        put(rb, cc + 32);
      }
#else
#pragma unroll 1
      for (int cc = c_lo; cc < c_hi; cc += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(taddr + cc, r);
        uint32_t w[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) w[e] = pack_bf16x2(__uint_as_float(r[2 * e]), __uint_as_float(r[2 * e + 1]));
        if (st32) {
#pragma unroll
          for (int u = 0; u < 2; ++u) st_global_v8_cs_if(yrow + cc + u * 16, &w[8 * u], valid);
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            st_global_v4_if(yrow + cc + u * 8, w[4 * u], w[4 * u + 1], w[4 * u + 2], w[4 * u + 3], valid);
        }
      }
#endif
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&tempty[buf]);
    if (q == 0 && lane == 0) trace_stamp(p.trace, p.trace_items, cta, k, 4);
  }
  }

__global__ void __launch_bounds__(kExpandThreads, 1) expand_tc_kernel(const __grid_constant__ ExpandParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* ring = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ident = ring + kExpandRingBytes + kExpandGuardBytes;                    // 8 KB
  ExpandRecBuf* recbuf = reinterpret_cast<ExpandRecBuf*>(ident + kIdentRows * 16 * 2);
  uint32_t* offs = reinterpret_cast<uint32_t*>(recbuf + kExpRecBufs);     // [kItemQ]
  uint64_t* full = reinterpret_cast<uint64_t*>(offs + 2 * kItemQ);
  uint64_t* empty = full + kItemQ;
  uint64_t* tfull = empty + kItemQ;
  uint64_t* tempty = tfull + kAccBufs;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + kAccBufs);
  uint32_t* ring_tab = tmem_slot + 1;   // [kProdParts][kRingTableWords]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) phase_stamp(p.trace, p.trace_items, blockIdx.x, 0);
  // No ring zeroing is needed: B tiles are stored padded to kp rows (zeros past the rank) and
  // every other over-read (v rows past the tile's tokens) only feeds discarded D rows.
  // identity A tile, K-major SWIZZLE_32B [256 rows][16 k]: 1.0 at (128 + k, k)
  for (int i = threadIdx.x; i < kIdentRows * 16; i += blockDim.x) {
  const int t = i / 16, k = i % 16;
  reinterpret_cast<uint16_t*>(ident)[swz(t * 32 + k * 2, 32) / 2] = (t == 128 + k) ? 0x3F80u : 0u;
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
  for (int s = 0; s < kItemQ; ++s) { mbar_init(&full[s], kProdParts); mbar_init(&empty[s], 1); }
  for (int b = 0; b < kAccBufs; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], kExpandEpiWarps); }
  fence_mbar_init();
  for (int pp = 0; pp < kMaxProj; ++pp)
    if (p.y[pp])
      for (int b = 0; b < 5; ++b) { prefetch_tmap(&p.ymap[pp][b]); prefetch_tmap(&p.ymap2[pp][b]); }
  }
  if (warp == kExpMmaWarp) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int cta = blockIdx.x;
  if (threadIdx.x == 0) phase_stamp(p.trace, p.trace_items, cta, 1);
  pdl_wait();                 // v images come from the shrink launch; y from earlier work
  if (p.wait_flag != nullptr) {   // TP: the peers' shards of the v images have landed here too
  if (threadIdx.x == 0) {
    wait_flag_geq(p.wait_flag, p.wait_target);
    fence_proxy_async_global();
    if (atomicAdd(p.wait_flag + 1, 1) == (int)gridDim.x - 1) {   // last CTA through: re-arm
      p.wait_flag[1] = 0;
      p.wait_flag[0] = 0;
    }
  }
  __syncthreads();
  if (p.xsum != nullptr) {      // row group: v = sum of every rank's fp32 partial, fixed rank order
    tp_row_sum(p);
    __threadfence();
    __syncthreads();
    int* bar = p.gbar;
    if (threadIdx.x == 0) {
      atomicAdd(&bar[0], 1);
      uint64_t t0 = 0;
      for (uint32_t spin = 0; ld_relaxed_sys(&bar[0]) < (int)gridDim.x; ++spin) {
        __nanosleep(32);
        if ((spin & 1023u) == 1023u) {
          const uint64_t now = globaltimer_ns();
          if (t0 == 0) t0 = now;
          else if (now - t0 > 4000000000ull) __trap();
        }
      }
      (void)ld_acquire_sys(&bar[0]);
      fence_proxy_async_global();   // generic-proxy v writes -> the bulk copies that read them
    }
    __syncthreads();
  }
  }
  pdl_launch_dependents();
  if (threadIdx.x == 0) phase_stamp(p.trace, p.trace_items, cta, 2);

  const ExpandSm sm{ring, ident, recbuf, offs, full, empty, tfull, tempty, nullptr};
  PipeState st;
  if (warp == kExpProdWarp || (warp == kProdWarp2 && kProdParts == 2)) {
    const int part = warp == kExpProdWarp ? 0 : 1;
    RingAlloc ra(ring_tab + part * kRingTableWords, lane);
    expand_producer(p, sm, cta, warp, lane, nullptr, nullptr, part, kProdParts, st, ra);
  }
  else if (warp == kExpMmaWarp) expand_mma(p, sm, tmem_base, cta, warp, lane, st);
  else if (expand_epi_warp(warp)) expand_epilogue(p, sm, tmem_base, cta, warp, lane, st);
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) phase_stamp(p.trace, p.trace_items, cta, 3);
  if (warp == kExpMmaWarp) { tc_fence_after(); tmem_dealloc(tmem_base, kTmemCols); }
  if (p.xsum != nullptr && threadIdx.x == 0) {   // every CTA is past the sum barrier: re-arm it
  int* bar = p.gbar;
  if (atomicAdd(&bar[1], 1) == (int)gridDim.x - 1) { bar[0] = 0; bar[1] = 0; }
  }
}


// ------------------------------------------------------------------------------------------
// Group kernel: one input group's shrink and expand in one persistent launch.  Each CTA runs its
// shrink records, then its expand items; an item's v copy waits only for its own m-tile:
//   ready[mt]      = records of the tile whose v images are written (split tiles: whose share of
//                    the split-K reduction is written), target MTile::counter (= its records);
//   split_done[mt] = split records of the tile whose fp32 partials are written.
// Warp 4 publishes each stored record, then walks the CTA's expand list ahead of the producer and
// releases each item's v copy when its tile is complete; warp 5 reduces the CTA's split records
// (tokens split, split + nsplit, ... of the record's members) once every split of the tile is in.  There is no grid barrier
// and no second launch; CTAs that finish their shrink early expand the tiles already complete.
struct alignas(64) GroupParams {
  ShrinkParams s;
  ExpandParams e;
  int* ready;          // [n_mtiles], zero at launch (lsv_lora_forward zero-fills them per call)
  int* split_done;     // [n_mtiles]
  int s_grid, e_grid;  // CTAs with shrink records / expand items
  int wait_prev;       // 1: griddepcontrol.wait first (the previous launch may touch our buffers)
  uint64_t* tl;        // development timeline (nullptr = off): [cta][16] = {entry, setup done, exit, SM id,
                       // end of phase i (epilogue warp 0) at 4 + i}
};
// A layer kernel runs NG input groups back to back in every CTA (lsv_lora_forward, overlap-free
// calls): the groups' parameters travel together as kernel parameters (4 groups: ~26 KB).
template <int NG>
struct alignas(64) LayerParams {
  GroupParams g[NG];
  int ngroups;
  int lookahead;       // phase order: group g's expand runs after the shrinks of groups <= g + lookahead
  int dyn;             // 1: expand items by dynamic dispatch (every group's e.cursor set)
};
union RecBufU {
  ShrinkRecBuf s;
  ExpandRecBuf e;
};
__host__ __device__ constexpr int group_smem_bytes() {
  return 1024 + kExpandRingBytes + kExpandGuardBytes + kIdentRows * 16 * 2 + 9 * (int)sizeof(RecBufU) + 2 * kItemQ * 4 +
         8 * (2 * kShrinkStages + 2 * kAccBufs + 2 * kItemQ + 2 * kAccBufs + 2 * kVQ + kRecQ) + 32 +
         2 * kRingTableWords * 4 + (int)sizeof(DynRing) + 16 + 1024;
}
static_assert(kShrinkGuardBytes <= kExpandGuardBytes + kIdentRows * 16 * 2 + 9 * (int)sizeof(RecBufU),
              "a shrink stage's MMA over-read past the ring end stays inside the group kernel's shared memory");
static_assert(kShrinkStages <= kItemQ, "the shrink stage offsets live in the second half of offs[]");
static_assert(8 * (2 * kShrinkStages + 2 * kAccBufs) + 4 + 4 * kShrinkStages + 2 * 4 * kRingTableWords <= 1024 &&
                  4 * 2 * kItemQ + 8 * (2 * kItemQ + 2 * kAccBufs) + 4 + 2 * 4 * kRingTableWords <= 1024,
              "the standalone kernels' barriers, offsets and ring tables fit their last 1 KB of shared memory");
static_assert(kShrinkStages + kItemQ <= kRingQ && kShrinkStages + kItemQ <= kRingBars,
              "ring allocations in flight across a phase boundary: at most one per barrier pair");

// Warp 5: this CTA's share of the split-K reduction of its split records.
__device__ __forceinline__ void group_reducer(const ShrinkParams& p, ShrinkRecBuf* rb, int cta, int lane, int* ready,
                                              const int* split_done) {
  WarpRecStream<ShrinkRec, kShrinkRecCh> rs(rb, p.plan, p.off_recs, p.off_cta, cta, nullptr);
  ShrinkRec inf;
  const uint8_t* unused;
  const MTile* mts = reinterpret_cast<const MTile*>(p.plan + p.off_mtiles);
  while (rs.pop(inf, unused)) {
    if (inf.nsplit == 1) continue;
    if (lane == 0) wait_geq_gpu(&split_done[inf.mtile], inf.counter);   // every split record of the tile
    __syncwarp();
    RedUnit ru;
    ru.mt = mts[inf.mtile];
    ru.e = 0;
    const int upr = kpad(inf.rank) / 8, per_tok = inf.np * upr;
    const int ntk = (inf.ntok - inf.split + inf.nsplit - 1) / inf.nsplit;   // tokens split, split + nsplit, ...
    for (int u = lane; u < ntk * per_tok; u += 32) {
      ru.t = inf.split + (u / per_tok) * inf.nsplit;
      ru.pp = inf.p0 + (u % per_tok) / upr;
      ru.k0 = (u % upr) * 8;
      float s8[8];
      red_sum(p, ru, s8);
      red_store(p, ru, s8);
    }
    __syncwarp();
    if (lane == 0) {
      fence_proxy_async_global();
      red_release_gpu_add(&ready[inf.mtile], 1);
    }
  }
}
// Warp 4, shrink phase: publishes each of the CTA's records once its four epilogue warps have
// stored it (recdone): ready[mt] for a whole tile's images, split_done[mt] for split partials.
// It never waits on other CTAs, so every record's signal goes out whatever the reducers wait on.
// The release is cumulative over the epilogue warps' stores it acquired through the mbarrier.
__device__ __forceinline__ void group_signaler(const ShrinkParams& p, ShrinkRecBuf* rb, int cta, int lane, int* ready,
                                               int* split_done, uint64_t* recdone, int& rec_base) {
  WarpRecStream<ShrinkRec, kShrinkRecCh> rs(rb, p.plan, p.off_recs, p.off_cta, cta, nullptr);
  ShrinkRec inf;
  const uint8_t* unused;
  int k = rec_base;   // record index over every group this CTA has run (recdone queue)
  for (; rs.pop(inf, unused); ++k) {
    mbar_wait(&recdone[k % kRecQ], (k / kRecQ) & 1);
    if (lane == 0) {
      fence_proxy_async_global();   // the expand reads the images with bulk copies (async proxy)
      red_release_gpu_add(inf.nsplit > 1 ? &split_done[inf.mtile] : &ready[inf.mtile], 1);
      *reinterpret_cast<volatile int*>(recdone + kRecQ) = k + 1;
    }
    __syncwarp();
  }
  rec_base = k;
}
// Warp 4, expand phase: walks the expand list ahead of the producer; releases item k's v copy (vfull) once its
// m-tile is complete.  The acquire + proxy fence make the images (generic-proxy stores of other
// CTAs) visible to the producer's bulk copy.
__device__ __forceinline__ void group_ready_checker(const ExpandParams& p, ExpandRecBuf* rb, int cta, int lane,
                                                    const int* ready, uint64_t* vfull, uint64_t* vempty, int& item_base) {
  WarpRecStream<ExpandRec, kExpandRecCh> rs(rb, p.plan, p.off_recs, p.off_cta, cta, nullptr);
  ExpandRec inf;
  const uint8_t* unused;
  const MTile* mts = reinterpret_cast<const MTile*>(p.plan + p.off_mtiles);
  int last = -1;
  int k = item_base;   // item index over every group this CTA has run (v-ready queue)
  for (; rs.pop(inf, unused); ++k) {
    mbar_wait(&vempty[k % kVQ], ((k / kVQ) & 1) ^ 1);
    if (inf.mtile != last) {
      if (lane == 0) {
        wait_geq_gpu(&ready[inf.mtile], mts[inf.mtile].counter);
        fence_proxy_async_global();
      }
      last = inf.mtile;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&vfull[k % kVQ]);
  }
  item_base = k;
}
// Warp 4, expand phase with dynamic dispatch: takes the group's items in batches of kDynBatch
// (one atomicAdd on the cursor; the lanes load the records and adapter pointers in parallel),
// publishes them to the CTA's expand roles, then releases each item's v copy once its m-tile is
// complete.  A batch is taken only when the copy warp has taken item k - kDynLead, so every CTA
// holds about the same few items when the list runs out (the phase ends together on every SM).
// The end record goes out when the list is exhausted.
#ifndef LSV_DYN_BATCH
#define LSV_DYN_BATCH 4
#endif
#ifndef LSV_DYN_LEAD
#define LSV_DYN_LEAD 4
#endif
constexpr int kDynBatch = LSV_DYN_BATCH;
constexpr int kDynLead = LSV_DYN_LEAD;
static_assert(kDynBatch - 1 + kDynLead < kVQ && kDynLead + kDynBatch + kVQ + kItemQ + 4 + 4 < kDynQ,
              "dynamic dispatch lead within the v-ready queue and the record ring");
__device__ __forceinline__ void group_dispatcher(const ExpandParams& p, DynRing* dr, int lane, const int* ready,
                                                 uint64_t* vfull, uint64_t* vempty, int& item_base, int& q_base) {
  const MTile* mts = reinterpret_cast<const MTile*>(p.plan + p.off_mtiles);
  const ExpandRec* recs = reinterpret_cast<const ExpandRec*>(p.plan + p.off_recs);
  const int32_t* order = p.plan + p.off_dyn;
  int k = item_base, q = q_base;
  for (bool done = false; !done;) {
    const int j = k - kDynLead;   // the copy warp took item j: bounded lead (and v-queue slots free)
    if (j >= 0) mbar_wait(&vempty[j % kVQ], (j / kVQ) & 1);
    int base = 0;
    if (lane == 0) base = atomicAdd(p.cursor, kDynBatch);
    base = __shfl_sync(0xffffffffu, base, 0);
    const int nvalid = max(0, min(kDynBatch, p.n_dyn - base));
    done = nvalid < kDynBatch;
    const int npub = nvalid + (done ? 1 : 0);   // + the end record
    if (lane < npub) {
      ExpandRec r{};
      const uint8_t* ptr = nullptr;
      if (lane < nvalid) {
        r = recs[order[base + lane]];
        ptr = static_cast<const uint8_t*>(p.b_ptrs[r.proj][r.seg]);
      }
      dr->rec[(q + lane) % kDynQ] = r;
      dr->ptr[(q + lane) % kDynQ] = ptr;
    }
    __syncwarp();
    if (lane == 0) st_release_cta_shared(&dr->published, q + npub);
    if (lane < nvalid) {   // each lane releases its item's v copy when the m-tile is complete (any order)
      const int mt = dr->rec[(q + lane) % kDynQ].mtile;
      wait_geq_gpu(&ready[mt], mts[mt].counter);
      fence_proxy_async_global();
      mbar_arrive(&vfull[(k + lane) % kVQ]);
    }
    __syncwarp();
    k += nvalid;
    q += npub;
  }
  item_base = k;
  q_base = q;
}

constexpr int kGroupThreads = 288;   // the standalone layout + warp 8 (second copy-issuing part)
template <int NG>
__global__ void __launch_bounds__(kGroupThreads, 1) group_tc_kernel(const __grid_constant__ LayerParams<NG> lp) {
  static_assert(kShrinkThreads == kExpandThreads && kShrProdWarp == kExpProdWarp && kShrMmaWarp == kExpMmaWarp,
                "the group kernel runs both pipelines with one warp layout");
  const GroupParams& gp = lp.g[0];   // launch-wide fields (timeline, wait) and the first group's maps
  const ShrinkParams& sp = gp.s;
  const ExpandParams& ep = gp.e;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* ring = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // shrink slots / expand ring
  uint8_t* ident = ring + kExpandRingBytes + kExpandGuardBytes;                     // 8 KB
  RecBufU* recbuf = reinterpret_cast<RecBufU*>(ident + kIdentRows * 16 * 2);       // one per warp, both phases
  uint32_t* offs = reinterpret_cast<uint32_t*>(recbuf + kGroupThreads / 32);
  uint64_t* s_full = reinterpret_cast<uint64_t*>(offs + 2 * kItemQ);
  uint64_t* s_empty = s_full + kShrinkStages;
  uint64_t* s_tfull = s_empty + kShrinkStages;
  uint64_t* s_tempty = s_tfull + kAccBufs;
  uint64_t* e_full = s_tempty + kAccBufs;
  uint64_t* e_empty = e_full + kItemQ;
  uint64_t* e_tfull = e_empty + kItemQ;
  uint64_t* e_tempty = e_tfull + kAccBufs;
  uint64_t* vfull = e_tempty + kAccBufs;
  uint64_t* vempty = vfull + kVQ;
  uint64_t* recdone = vempty + kVQ;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(recdone + kRecQ) + 1;   // [0]: published-record count
  uint32_t* ring_tab = tmem_slot + 1;                                          // [kProdParts][kRingTableWords]
  DynRing* dyn = reinterpret_cast<DynRing*>(
      (reinterpret_cast<uintptr_t>(ring_tab + kProdParts * kRingTableWords) + 15) & ~uintptr_t(15));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cta = blockIdx.x;
  if (gp.tl != nullptr && threadIdx.x == 0) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    gp.tl[cta * 16 + 0] = globaltimer_ns();
    gp.tl[cta * 16 + 3] = smid;
  }
  for (int i = threadIdx.x; i < kIdentRows * 16; i += blockDim.x) {   // identity A tile (expand y add)
    const int t = i / 16, k = i % 16;
    reinterpret_cast<uint16_t*>(ident)[swz(t * 32 + k * 2, 32) / 2] = (t == 128 + k) ? 0x3F80u : 0u;
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    for (int s = 0; s < kShrinkStages; ++s) { mbar_init(&s_full[s], kProdParts); mbar_init(&s_empty[s], 1); }
    for (int b = 0; b < kAccBufs; ++b) { mbar_init(&s_tfull[b], 1); mbar_init(&s_tempty[b], 4); }
    for (int s = 0; s < kItemQ; ++s) { mbar_init(&e_full[s], kProdParts); mbar_init(&e_empty[s], 1); }
    for (int b = 0; b < kAccBufs; ++b) { mbar_init(&e_tfull[b], 1); mbar_init(&e_tempty[b], kExpandEpiWarps); }
    for (int q = 0; q < kVQ; ++q) { mbar_init(&vfull[q], 1); mbar_init(&vempty[q], 1); }
    for (int q = 0; q < kRecQ; ++q) mbar_init(&recdone[q], 4);
    *reinterpret_cast<volatile int*>(recdone + kRecQ) = 0;
    dyn->published = 0;
    fence_mbar_init();
    for (int b = 0; b < 5; ++b) prefetch_tmap(&sp.xmap[b]);
    for (int pp = 0; pp < kMaxProj; ++pp)
      if (ep.y[pp])
        for (int b = 0; b < 5; ++b) { prefetch_tmap(&ep.ymap[pp][b]); prefetch_tmap(&ep.ymap2[pp][b]); }
  }
  if (warp == kExpMmaWarp) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) phase_stamp(sp.trace, sp.trace_items, cta, 0);
  if (gp.tl != nullptr && threadIdx.x == 0) gp.tl[cta * 16 + 1] = globaltimer_ns();
  if (gp.wait_prev) pdl_wait();
  pdl_launch_dependents();
  const ShrinkSm ssm{ring, &recbuf[0].s, s_full, s_empty, s_tfull, s_tempty, offs + kItemQ};
  const bool dyn_on = NG > 1 && lp.dyn;
  const ExpandSm esm{ring, ident, &recbuf[0].e, offs, e_full, e_empty, e_tfull, e_tempty, dyn_on ? dyn : nullptr};
  // dynamic dispatch: every CTA of the launch runs every expand phase (it takes items until the
  // group's list is exhausted)
  auto runs_expand = [&](const GroupParams& G) { return dyn_on || cta < G.e_grid; };
  // the role functions index recbuf by warp: give each a pointer whose [warp] is this warp's union slot
  ShrinkSm ssw = ssm;
  ssw.recbuf = reinterpret_cast<ShrinkRecBuf*>(&recbuf[warp]) - warp;
  ExpandSm esw = esm;
  esw.recbuf = reinterpret_cast<ExpandRecBuf*>(&recbuf[warp]) - warp;
  const int ng = NG == 1 ? 1 : lp.ngroups;
  // Each role runs the layer's 2*ng phases in the same order, its pipeline position carried over
  // (PipeState).  Default order (lookahead 3): every shrink, then every expand — a group's m-tiles
  // (split-K reductions included) on other CTAs have the later shrinks' time to complete before
  // its expand asks for them, which absorbs the start skew of back-to-back layer launches
  // (lookahead 1, S0 S1 E0 S2 E1 S3 E2 E3, measured 9.1 vs 8.73 ms per C2 step).  Shrink stages and expand items share one byte ring
  // (RingAlloc): the copy warps start a phase's loads behind the previous phase's last items; the
  // MMA warp drains a phase's accumulators before the next phase writes TMEM.  No CTA-wide barrier.
  const int nph = 2 * ng;
  // lookahead d: S0 .. Sd, then E0 S(d+1) E1 S(d+2) ..., then the remaining expands
  // (d = 1: S0 S1 E0 S2 E1 S3 E2 E3; d = 3: S0 S1 S2 S3 E0 E1 E2 E3)
  const int npre = min(ng, (NG == 1 ? 1 : max(lp.lookahead, 1)) + 1), m = ng - npre;
  auto phase_of = [&](int i, int& g) -> bool {   // true: expand phase of group g
    if (i < npre) { g = i; return false; }
    const int j = i - npre;
    if (j < 2 * m) {
      g = j / 2 + (j % 2 ? npre : 0);
      return j % 2 == 0;
    }
    g = m + (j - 2 * m);
    return true;
  };
  if (warp == kExpProdWarp || (warp == 8 && kProdParts == 2)) {
    const int part = warp == 8 ? 1 : 0;
    PipeState st;
    RingAlloc ra(ring_tab + part * kRingTableWords, lane);
    for (int i = 0; i < nph; ++i) {
      int g;
      const bool ex = phase_of(i, g);
      const GroupParams& G = lp.g[g];
      if (!ex) {
        if (g > 0 && part == 0 && lane == 0) {   // this group's tensor maps
          for (int b = 0; b < 5; ++b) prefetch_tmap(&G.s.xmap[b]);
          for (int pp = 0; pp < kMaxProj; ++pp)
            if (G.e.y[pp])
              for (int b = 0; b < 5; ++b) { prefetch_tmap(&G.e.ymap[pp][b]); prefetch_tmap(&G.e.ymap2[pp][b]); }
        }
        if (cta < G.s_grid) shrink_producer(G.s, ssw, cta, warp, lane, part, kProdParts, st, ra, kExpandRingBytes,
                                            kExpandGuardBytes);
        if (lane == 0 && part == 0) phase_stamp(G.s.trace, G.s.trace_items, cta, 2);   // shrink stages issued
      } else if (runs_expand(G)) {
        expand_producer(G.e, esw, cta, warp, lane, vfull, vempty, part, kProdParts, st, ra);
      }
    }
  } else if (warp == kExpMmaWarp) {
    PipeState st;
    for (int i = 0; i < nph; ++i) {
      int g;
      const bool ex = phase_of(i, g);
      const GroupParams& G = lp.g[g];
      if (!ex && cta < G.s_grid) {
        shrink_mma(G.s, ssw, tmem_base, cta, warp, lane, st);
        for (int b = 0; b < kAccBufs; ++b) mbar_wait(&s_tempty[b], ((st.s_tbits >> b) & 1) ^ 1);   // accumulators drained
        tc_fence_after();
      } else if (ex && runs_expand(G)) {
        expand_mma(G.e, esw, tmem_base, cta, warp, lane, st);
        if (i + 1 < nph) {
          for (int b = 0; b < kAccBufs; ++b) mbar_wait(&e_tempty[b], ((st.e_tbits >> b) & 1) ^ 1);
          tc_fence_after();
        }
      }
    }
  } else if (expand_epi_warp(warp)) {
    PipeState st;
    for (int i = 0; i < nph; ++i) {
      int g;
      const bool ex = phase_of(i, g);
      const GroupParams& G = lp.g[g];
      if (!ex && cta < G.s_grid) shrink_epilogue(G.s, ssw, tmem_base, cta, warp, lane, recdone, st);
      if (ex && runs_expand(G)) expand_epilogue(G.e, esw, tmem_base, cta, warp, lane, st);
      if (warp == 0 && lane == 0) phase_stamp(G.s.trace, G.s.trace_items, cta, ex ? 4 : 1);   // phase stored
      if (gp.tl != nullptr && warp == 0 && lane == 0 && i < 12) gp.tl[cta * 16 + 4 + i] = globaltimer_ns();
    }
  } else if (warp == 4) {
    int rec_base = 0, item_base = 0, q_base = 0;
    for (int i = 0; i < nph; ++i) {
      int g;
      const bool ex = phase_of(i, g);
      const GroupParams& G = lp.g[g];
      if (!ex && cta < G.s_grid) group_signaler(G.s, &recbuf[warp].s, cta, lane, G.ready, G.split_done, recdone, rec_base);
      if (ex && dyn_on) group_dispatcher(G.e, dyn, lane, G.ready, vfull, vempty, item_base, q_base);
      else if (ex && cta < G.e_grid) group_ready_checker(G.e, &recbuf[warp].e, cta, lane, G.ready, vfull, vempty, item_base);
    }
  } else if (warp == 5) {
    for (int i = 0; i < nph; ++i) {
      int g;
      if (phase_of(i, g)) continue;
      const GroupParams& G = lp.g[g];
      if (cta < G.s_grid) group_reducer(G.s, &recbuf[warp].s, cta, lane, G.ready, G.split_done);
      if (lane == 0) phase_stamp(G.s.trace, G.s.trace_items, cta, 3);   // split-K shares reduced
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kExpMmaWarp) { tc_fence_after(); tmem_dealloc(tmem_base, kTmemCols); }
  if (gp.tl != nullptr && threadIdx.x == 0) gp.tl[cta * 16 + 2] = globaltimer_ns();
}

}  // namespace lsv
