// lsv_plan.h — the int32 plan blob shared by the host planner (lsv_plan.cpp) and the kernels.
//
// One plan covers one co-batched token batch (the reference's prefill batch,
// simengine.py:96-152 schedule_server) for one projection shape (h_in, h_out).  It is
// built on the host from the segment indexer's output and copied to HBM once; every
// layer/projection of that shape reuses it.
#pragma once
#include <stdint.h>

namespace lsv {

constexpr int32_t kPlanMagic = 0x5056534c;  // "LSVP"
constexpr int32_t kPlanVersion = 3;
constexpr int kMaxProj = 4;    // projections per input group (q/k/v = 3)

enum Tier : int32_t { kTierNone = 0, kTierSimt = 1, kTierTc = 2 };

struct PlanHeader {            // 64 int32
  int32_t magic, version;
  int32_t num_segments, num_tokens, h_in, h_out;
  int32_t n_simt_items;        // SIMT tier work items: <= kSimtMaxTok tokens of one segment
  int32_t n_mtiles;            // tcgen05 tier 128-token tiles
  int32_t n_shrink_items;      // tcgen05 shrink work items (mtile, k-range)
  int32_t n_expand_items;      // tcgen05 expand work items (mtile, 128-wide h_out tile)
  int32_t shrink_grid, expand_grid;
  // int32 offsets of the arrays inside the blob
  int32_t off_seg_indptr, off_seg_rank, off_seg_tier;
  int32_t off_simt_items, off_mtiles;
  int32_t off_shrink_recs, off_shrink_cta;   // records grouped per CTA + [grid+1] CTA offsets
  int32_t off_expand_recs, off_expand_cta;
  int32_t total_ints;
  // workspace layout, byte offsets (workspace < 2 GiB)
  int32_t ws_counters, ws_partials, ws_vimg, ws_simt_v, ws_bytes;
  int32_t n_counters;
  int32_t simt_segments;
  int32_t off_red, n_red, red_units;   // split-K reduction table: [n_red] {mtile, unit prefix}
  int32_t off_red_cta;                 // [shrink_grid + 1] first reduction entry of each CTA's unit range
  // input groups: num_proj projections share x (q/k/v, gate/up) and are shrunk together from a
  // group A tile [chunk][num_proj*rank rows][64]; each has its own h_out, expand list and v images
  int32_t num_proj;
  int32_t vimg_stride;                 // bytes between the v-image regions of consecutive projections
  int32_t simt_stride;                 // floats between the SIMT v regions of consecutive projections
  int32_t acc_cols;                    // shrink TMEM accumulator width (128 or 256 columns)
  int32_t h_outs[kMaxProj];
  int32_t off_expand_recs_p[kMaxProj], off_expand_cta_p[kMaxProj];
  int32_t expand_grid_p[kMaxProj], n_expand_items_p[kMaxProj];
  int32_t off_expand_recs_all, off_expand_cta_all, expand_grid_all, n_expand_all;  // every member, one LPT list
  int32_t vsplit;                      // 1: each tcgen05 v image is a bf16 (hi, lo) pair, v = hi + lo to ~2^-16
  // tile-aligned plans (LSV_PLAN_TILE_ALIGNED, for the fused base-GEMM kernel): m-tiles are the
  // pieces of segments inside each 128-token tile of the batch; a piece's v image has 128 rows (the
  // tile's) with the piece at rows [tok_begin % 128, +ntok) and zeros elsewhere
  int32_t tile_aligned;
  // [n] int32: the group kernel's expand list (all members when num_proj > 1, else member 0's) in
  // global readiness order, for the layer kernel's dynamic expand dispatch (0: none)
  int32_t off_dyn;
};
static_assert(sizeof(PlanHeader) == 64 * 4, "plan header size");

struct SimtItem {              // 4 int32
  int32_t seg, tok_begin;
  int32_t nt_rank;             // ntok | rank << 16: the kernels need both before their first weight load
  int32_t v_off;               // float index of this item's fp32 v [ntok][rank]
};
#ifndef LSV_SIMT_SHR_ROWS
#define LSV_SIMT_SHR_ROWS 16
#endif
constexpr int kSimtShrRows = LSV_SIMT_SHR_ROWS;   // group-A rows per SIMT shrink block (8 or 16)
__host__ __device__ inline int simt_nt(const SimtItem& it) { return it.nt_rank & 0xffff; }
__host__ __device__ inline int simt_rank(const SimtItem& it) { return it.nt_rank >> 16; }
// Tile-aligned plans append [n_gemm_tiles + 1] first-piece indices after the split-K tables
// (off_tile_mt = total_ints - n_gemm_tiles - 1; n_gemm_tiles = ceil(num_tokens / 128)).
// The SIMT tail of a plan, after the items: the shrink's row-block prefix [n + 1] over the items
// (8-row blocks of each item's group A), then one int per row block: item << 8 | row block.

struct MTile {                 // 8 int32
  int32_t seg, tok_begin, ntok, rank;
  int32_t nsplit;              // shrink k-splits reduced by the last-arriving CTA
  int32_t part_off;            // float index of partials [nsplit][ntok][rank] (if nsplit > 1)
  int32_t vimg_off;            // byte offset of the bf16 v image (16-byte aligned)
  int32_t counter;             // index of this tile's split-arrival counter
};

// Fully decoded work records: the host assigns them to CTAs (LPT greedy on estimated bytes)
// and stores each CTA's list contiguously, so the kernels need no atomics and no dependent
// descriptor loads on their critical path.
struct ShrinkRec {             // 16 int32
  int32_t seg, tok_begin, ntok, rank;
  int32_t chunk_begin, chunk_end, kch, split;   // k-range in 64-element chunks of h_in
  int32_t nsplit, part_off, vimg_off, counter;
  int32_t mtile, p0, np, pad;                   // projections [p0, p0+np) of the group: N = np*rank
};

struct ExpandRec {             // 8 int32
  int32_t seg, tok_begin, ntok, rank;
  int32_t jtile, vimg_off, mtile, proj;         // member proj's h_out columns [jtile*tw, jtile*tw+tw)
};

// Workspace barrier header.  Every workspace starts with kBarHeaderBytes of grid-barrier words that
// are zero at rest (zero-filled once; every kernel re-arms what it used before it exits).  A plan's
// own scratch (split-K partials, v images, SIMT v) starts after it, so reusing one workspace for
// plans of different layouts (a new batch every step) never lands a barrier on stale scratch.
// Pair 0 serves the standalone entry points; lsv_lora_forward gives (layer l, group g) pair
// 1 + l * num_groups + g.
constexpr int kBarHeaderBytes = 64 * 1024;
constexpr int kMaxBarPairs = kBarHeaderBytes / 8;

// Pipeline geometry (bytes of shared memory).
#ifndef LSV_SHRINK_SLOT_KB
#define LSV_SHRINK_SLOT_KB 64
#define LSV_SHRINK_SLOTS 3
#endif
#ifndef LSV_SHRINK_MAX_KCH
#define LSV_SHRINK_MAX_KCH 16
#endif
constexpr int kShrinkMaxKch = LSV_SHRINK_MAX_KCH;   // 64-column chunks per pipeline stage, at most
constexpr int kShrinkSlotBytes = LSV_SHRINK_SLOT_KB * 1024;
constexpr int kShrinkSlots = LSV_SHRINK_SLOTS;     // the standalone shrink kernel's ring: whole slots
#ifndef LSV_SHRINK_STAGES
#define LSV_SHRINK_STAGES LSV_SHRINK_SLOTS
#endif
constexpr int kShrinkStages = LSV_SHRINK_STAGES;   // stage barrier pairs (stages in flight), both kernels
constexpr int kShrinkGuardBytes = 16 * 1024;   // the M=128 MMA over-reads past short token tiles
#ifndef LSV_EXPAND_RING_KB
#define LSV_EXPAND_RING_KB 200
#endif
constexpr int kExpandRingBytes = LSV_EXPAND_RING_KB * 1024;   // variable-size items, allocated in issue order
constexpr int kExpandGuardBytes = 2 * 1024;    // rank-8 K=16 MMA reads one k-core past its tile
constexpr int kExpandInflight = 8;
// SIMT shrink k-splits: h_in's 64-column chunks are split into ~48-chunk ranges, one block each.
// With one launch stream, 16-chunk splits measured best (4.24-4.41 ms decode step; the few rank-row
// blocks of a decode batch need the split to spread over the SMs).  With lsv_lora_forward's groups on
// concurrent streams the other groups fill the SMs instead, and fewer splits win (decode step 3.04 ms
// at 48 vs 3.06 at 64, 3.20 at 32, 3.42 at 16, 3.61 at 128; tools/gpu_ab_lib.sh --config decode); the
// serialised step pays for it (6.6 vs 5.4 ms).  Each split writes its own fp32 partial v; the SIMT
// expand sums the splits in split order (deterministic).
#ifndef LSV_SIMT_SPLIT_CHUNKS
#define LSV_SIMT_SPLIT_CHUNKS 48
#endif
__host__ __device__ constexpr int simt_ksplit(int h_in) {
  return h_in / 64 / LSV_SIMT_SPLIT_CHUNKS < 1 ? 1 : h_in / 64 / LSV_SIMT_SPLIT_CHUNKS;
}

}  // namespace lsv
