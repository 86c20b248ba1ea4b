// lsv_api.cu — liblsv C ABI: planner, adapter packing, apply / shrink / expand, peers.
// See include/lsv.h for the reference interfaces each entry point replaces.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <queue>
#include <unordered_map>
#include <vector>

#include "../../include/lsv.h"
#include "lsv_common.cuh"
#include "lsv_fused.cuh"
#include "lsv_plan.h"
#include "lsv_simt.cuh"
#include "lsv_tc.cuh"

using namespace lsv;

namespace {

thread_local char g_err[512] = "";
// Development hooks, not part of any compute path's state: a per-thread trace buffer
// (lsv_debug_set_trace: launches issued from the calling thread stamp it) and ablation bits read
// once from the environment (0 in production).
thread_local uint64_t* g_trace = nullptr;
thread_local int g_trace_items = 0;   // < 0: group-kernel timeline mode, -(launches) records
thread_local int g_tl_launch = 0;
const int g_debug_shrink = [] { const char* e = std::getenv("LSV_DEBUG_SHRINK"); return e ? std::atoi(e) : 0; }();
const int g_debug_expand = [] { const char* e = std::getenv("LSV_DEBUG_EXPAND"); return e ? std::atoi(e) : 0; }();
// LSV_SIMT_WAIT=1: SIMT shrinks always wait for the previous launch (A/B timing of the overlap)
const bool g_simt_wait = [] { const char* e = std::getenv("LSV_SIMT_WAIT"); return e && std::atoi(e) != 0; }();
// LSV_GROUP_KERNEL=0: lsv_lora_forward runs each group as a shrink launch + an expand launch
// instead of one group kernel (A/B timing)
const bool g_group_kernel = [] { const char* e = std::getenv("LSV_GROUP_KERNEL"); return !e || std::atoi(e) != 0; }();
// LSV_FWD_STREAMS=0: an overlap-free forward that cannot use layer kernels (SIMT-tier groups: decode)
// issues every group on the caller's stream instead of one stream per group index
const bool g_fwd_streams = [] { const char* e = std::getenv("LSV_FWD_STREAMS"); return !e || std::atoi(e) != 0; }();
// LSV_LAYER_KERNEL=0: one group kernel per (layer, group) instead of one layer kernel per layer
const bool g_layer_kernel = [] { const char* e = std::getenv("LSV_LAYER_KERNEL"); return !e || std::atoi(e) != 0; }();
// LSV_READY_ORDER=0: keep each CTA's expand items in LPT order instead of estimated m-tile
// readiness order (A/B timing)
// layer kernel phase order (lsv_tc.cuh group_tc_kernel): group g's expand after the shrinks of groups <= g + d
const int g_phase_lookahead = [] { const char* e = std::getenv("LSV_PHASE_LOOKAHEAD"); return e ? std::atoi(e) : 3; }();
// layer kernel: expand items by dynamic dispatch from a per-group global cursor (lsv_tc.cuh group_dispatcher)
// in calls of several layers (C2 8.43-8.57 ms vs 8.91-9.05 with each CTA's static LPT list, same box:
// the static lists let the CTAs drift apart over a step's back-to-back layer launches, up to ~100 µs
// by layer 8); a one-layer call keeps the static lists (no drift to absorb; 134 vs 142 µs for mlp_in)
const bool g_dyn_expand = [] { const char* e = std::getenv("LSV_DYN_EXPAND"); return !e || std::atoi(e) != 0; }();
const int g_dyn_order = [] { const char* e = std::getenv("LSV_DYN_ORDER"); return e ? std::atoi(e) : 1; }();
const bool g_ready_order = [] { const char* e = std::getenv("LSV_READY_ORDER"); return !e || std::atoi(e) != 0; }();
const int g_debug_fused = [] { const char* e = std::getenv("LSV_DEBUG_FUSED"); return e ? std::atoi(e) : 0; }();

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

#define LSV_CUDA_CHECK(expr)                                                        \
  do {                                                                              \
    cudaError_t e__ = (expr);                                                       \
    if (e__ != cudaSuccess)                                                         \
      return fail(LSV_ECUDA, "%s failed: %s", #expr, cudaGetErrorString(e__));       \
  } while (0)

// ---- planner knobs ------------------------------------------------------------------------
// AUTO tier rule: a segment of n tokens and rank r goes to the SIMT tier iff n <= simt_max_tok(r),
// else to tcgen05.  From the (n, r) sweep in profiles/r2_tier_sweep.txt (tools/tier_sweep.py:
// batches of S equal segments, gate 4096->11008 and down 11008->4096, both tiers forced, CUDA-event
// time; ncu dram% / tensor-pipe% beside it): the threshold is the largest n at which the SIMT
// tier's summed gate + down time is lower.  The SIMT expand re-reads each B tile per 2-token pass,
// so its cost grows with n; the tcgen05 tier's per-item cost is flat in n up to a 128-row tile, so
// its advantage comes earlier the higher the rank.  Rank 256 runs on 64-token tiles with 128-wide
// expand items (mtile_rows, expand_item_tw), which moves its crossover back up by one step.
//     r:        8   16   32   64   128   256
//     SIMT n <= 4    4    2    1    0     1
int simt_max_tok(int rank) {
  if (rank <= 16) return 4;
  if (rank <= 32) return 2;
  if (rank <= 64) return 1;
  if (rank <= 128) return 0;
  return 1;
}
bool auto_simt(int n, int rank) { return n <= simt_max_tok(rank); }
// Batch level: a decode-shaped batch (no segment longer than kSimtMaxTok tokens) runs entirely on
// the SIMT tier.  The sweep's thresholds compare batches of one (n, r) class; in a decode batch
// the few segments they would move to tcgen05 bring that tier's launches (shrink + expand per
// input group) for little work: C2's decode step (128 requests x 1 token, 100 adapters) measured
// 7.32 ms per-segment vs 5.79 ms all-SIMT (profiles/r2_tier_sweep.txt, batch-level note).
bool decode_shaped(int32_t S, const int32_t* indptr) {
  for (int s = 0; s < S; ++s)
    if (indptr[s + 1] - indptr[s] > kSimtMaxTok) return false;
  return true;
}
constexpr int64_t kMinItemBytes = 64 * 1024;  // smallest shrink k-split worth a pipeline fill
#ifndef LSV_SHRINK_WAVES
#define LSV_SHRINK_WAVES 2
#endif
constexpr int kShrinkWaves = LSV_SHRINK_WAVES;  // target shrink items per SM (balance vs split cost): with the layer kernel's S(g+1)-before-E(g) order 2 measured best (8.67 / 8.95 ms vs 8.76 / 8.94 at 4, 8.93 at 8; 1 within noise)
// LPT cost of an item = its bytes + a fixed per-item cost (pipeline fill, barrier round trips,
// epilogue), in byte-equivalents
#ifndef LSV_EXPAND_ITEM_FIXED_KB
#define LSV_EXPAND_ITEM_FIXED_KB 8
#endif
// Fixed costs per shrink record / stage: with the layer kernel's byte ring (no pipeline refill per
// phase) small ones balance the CTAs best (C2 8.38-8.48 ms at 16 / 8 KB vs 8.61-8.75 at the
// standalone-kernel-era 64 / 96 KB; 0-16 KB all within noise of each other)
#ifndef LSV_SHRINK_REC_FIXED_KB
#define LSV_SHRINK_REC_FIXED_KB 16
#endif
constexpr int64_t kExpandItemFixed = (int64_t)LSV_EXPAND_ITEM_FIXED_KB * 1024;
constexpr int64_t kShrinkRecFixed = (int64_t)LSV_SHRINK_REC_FIXED_KB * 1024;
#ifndef LSV_SHRINK_STAGE_FIXED_KB
#define LSV_SHRINK_STAGE_FIXED_KB 8
#endif
constexpr int64_t kShrinkStageFixed = (int64_t)LSV_SHRINK_STAGE_FIXED_KB * 1024;
// Remote segments (adapter owned by an NVLink peer, LSV_SEG_REMOTE): their A/B bytes weigh
// kRemoteWeight local bytes in the LPT cost (HBM ~6.5 TB/s against ~0.9 TB/s of NVLink ingress per
// GPU), so the peer reads spread evenly over the CTAs; each CTA's list then alternates remote and
// local records, keeping NVLink and HBM busy together instead of one after the other.
const int kRemoteWeight = [] { const char* e = std::getenv("LSV_REMOTE_WEIGHT"); return e ? std::atoi(e) : 7; }();

// Per-device side streams for lsv_lora_forward's group-parallel mode (created once, never freed):
// the groups of an overlap-free call are independent, so group g's launches go to stream g % 4
// (forked from and joined back into the caller's stream with events; graph capture records the
// fork/join as parallel branches).
#ifndef LSV_FWD_NSTREAMS
#define LSV_FWD_NSTREAMS 4
#endif
constexpr int kFwdStreams = LSV_FWD_NSTREAMS;
struct FwdStreams {
  cudaStream_t s[kFwdStreams - 1] = {};
  cudaEvent_t fork = nullptr, join[kFwdStreams - 1] = {};
  bool ok = false;
};
FwdStreams* fwd_streams() {
  static FwdStreams per_dev[16];
  static std::mutex mu;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  FwdStreams& f = per_dev[dev];
  if (!f.ok) {
    bool good = cudaEventCreateWithFlags(&f.fork, cudaEventDisableTiming) == cudaSuccess;
    for (int i = 0; i < kFwdStreams - 1 && good; ++i)
      good = cudaStreamCreateWithFlags(&f.s[i], cudaStreamNonBlocking) == cudaSuccess &&
             cudaEventCreateWithFlags(&f.join[i], cudaEventDisableTiming) == cudaSuccess;
    if (!good) { cudaGetLastError(); return nullptr; }
    f.ok = true;
  }
  return &f;
}
int num_sms_cached() {
  static int sms = -1;
  static std::once_flag once;
  std::call_once(once, [] {
    int n = 0;
    if (cudaGetDeviceCount(&n) == cudaSuccess && n > 0) {
      int dev = 0, v = 0;
      cudaGetDevice(&dev);
      if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0) sms = v;
    }
    cudaGetLastError();
    if (sms <= 0) sms = kNumSmsDefault;
  });
  return sms;
}

struct PlanBuilder {
  PlanHeader h{};
  std::vector<int32_t> indptr, rank, tier;
  std::vector<SimtItem> simt;
  std::vector<MTile> mtiles;
  std::vector<ShrinkRec> shrink;     // grouped per CTA
  std::vector<int32_t> shrink_cta;   // [grid+1]
  std::vector<ExpandRec> expand[kMaxProj];
  std::vector<int32_t> expand_cta[kMaxProj];
  std::vector<ExpandRec> expand_all;   // every member's items, one LPT assignment
  std::vector<int32_t> expand_all_cta;
  std::vector<int32_t> red;          // {mtile, first unit} per split tile
  int32_t red_units = 0;
  std::vector<int32_t> red_cta;
  std::vector<int32_t> tile_mt;      // tile-aligned plans: [n_gemm_tiles + 1] first piece per tile
  std::vector<int32_t> dyn;          // dynamic expand dispatch order (PlanHeader::off_dyn)
};

// LPT greedy: items (already sorted by non-increasing cost) go to the least-loaded CTA; each
// CTA's list keeps that order.  Returns records regrouped per CTA and the [grid+1] offsets.
// Least-loaded CTA with the lowest index among equals, via a tournament tree over the CTA loads:
// the root holds the winner, an update replays one leaf-to-root path (log2(grid) compares).
struct LoadTree {
  int n = 1;
  std::vector<int64_t> load;
  std::vector<int32_t> win;   // [2n): win[1] is the overall least-loaded CTA
  explicit LoadTree(int grid) {
    while (n < grid) n <<= 1;
    load.assign(n, INT64_MAX);
    for (int c = 0; c < grid; ++c) load[c] = 0;
    win.assign(2 * n, 0);
    for (int i = 0; i < n; ++i) win[n + i] = i;
    for (int i = n - 1; i >= 1; --i) win[i] = better(win[2 * i], win[2 * i + 1]);
  }
  int better(int a, int b) const { return (load[b] < load[a] || (load[b] == load[a] && b < a)) ? b : a; }
  int top() const { return win[1]; }
  void add(int c, int64_t v) {
    load[c] += v;
    for (int i = (n + c) >> 1; i >= 1; i >>= 1) win[i] = better(win[2 * i], win[2 * i + 1]);
  }
};

// LPT greedy: items (already sorted by non-increasing cost) go to the least-loaded CTA; each
// CTA's list keeps that order.  Returns records regrouped per CTA and the [grid+1] offsets.
// finish (optional): each record's estimated completion, its CTA's load once it is done.
template <typename Rec>
void lpt_assign(const std::vector<std::pair<int64_t, Rec>>& costed, int grid, std::vector<Rec>& out,
                std::vector<int32_t>& cta_off, const std::vector<uint8_t>* remote = nullptr,
                std::vector<int64_t>* finish = nullptr) {
  std::vector<int32_t> owner(costed.size());
  std::vector<int64_t> done(costed.size());
  LoadTree tree(grid);
  for (size_t i = 0; i < costed.size(); ++i) {
    const int c = tree.top();
    owner[i] = c;
    tree.add(c, costed[i].first);
    done[i] = tree.load[c];
  }
  cta_off.assign(grid + 1, 0);
  for (int32_t o : owner) ++cta_off[o + 1];
  for (int c = 0; c < grid; ++c) cta_off[c + 1] += cta_off[c];
  out.resize(costed.size());
  if (finish) finish->resize(costed.size());
  std::vector<int32_t> fill(cta_off.begin(), cta_off.end() - 1);
  for (size_t i = 0; i < costed.size(); ++i) {   // keeps LPT order per CTA
    if (finish) (*finish)[fill[owner[i]]] = done[i];
    out[fill[owner[i]]++] = costed[i].second;
  }
  if (remote == nullptr) return;
  // per CTA: remote and local records alternate (each kind in LPT order), remote first
  std::vector<Rec> rem, loc;
  for (int c = 0; c < grid; ++c) {
    rem.clear();
    loc.clear();
    for (int i = cta_off[c]; i < cta_off[c + 1]; ++i) ((*remote)[out[i].seg] ? rem : loc).push_back(out[i]);
    size_t a = 0, b = 0;
    for (int i = cta_off[c]; i < cta_off[c + 1]; ++i)
      out[i] = (a < rem.size() && (b >= loc.size() || a <= b)) ? rem[a++] : loc[b++];
  }
}

int validate_segments(int32_t S, const int32_t* indptr, const int32_t* rank, int32_t h_in, int32_t P,
                      const int32_t* h_outs) {
  if (S < 0) return fail(LSV_EINVAL, "num_segments must be >= 0, got %d", S);
  if (S > 0 && (!indptr || !rank)) return fail(LSV_EINVAL, "seg_indptr/seg_rank must be non-null");
  if (h_in <= 0 || h_in % 128) return fail(LSV_EINVAL, "h_in must be a positive multiple of 128, got %d", h_in);
  if (P < 1 || P > kMaxProj) return fail(LSV_EINVAL, "num_proj must be in [1, %d], got %d", kMaxProj, P);
  if (!h_outs) return fail(LSV_EINVAL, "h_outs must be non-null");
  for (int p = 0; p < P; ++p)
    if (h_outs[p] <= 0 || h_outs[p] % 128)
      return fail(LSV_EINVAL, "h_out must be a positive multiple of 128, got %d", h_outs[p]);
  if (S > 0 && indptr[0] != 0) return fail(LSV_EINVAL, "seg_indptr[0] must be 0, got %d", indptr[0]);
  for (int s = 0; s < S; ++s) {
    if (indptr[s + 1] < indptr[s])
      return fail(LSV_EINVAL, "seg_indptr must be non-decreasing (segment %d: %d < %d)", s, indptr[s + 1], indptr[s]);
    if (rank[s] < 8 || rank[s] > 256 || rank[s] % 8)
      return fail(LSV_EINVAL, "segment %d: rank must be a multiple of 8 in [8, 256], got %d", s, rank[s]);
  }
  return LSV_OK;
}

// Projections [p0, p0+np) of one record: the widest prefix whose rows (np*rank) fit one
// M=128 tcgen05 MMA (N <= 256).
int subset_np(int P, int p0, int r) { return std::max(1, std::min(P - p0, 256 / r)); }

int build_plan(PlanBuilder& pb, int32_t S, const int32_t* indptr, const int32_t* rank, int32_t h_in, int32_t P,
               const int32_t* h_outs, int32_t policy, const int32_t* seg_flags = nullptr) {
  if (int rc = validate_segments(S, indptr, rank, h_in, P, h_outs)) return rc;
  if (policy & ~(0xff | LSV_PLAN_V_BF16 | LSV_PLAN_TILE_ALIGNED | (0xff << 16)))
    return fail(LSV_EINVAL, "unknown plan flags 0x%x", policy);
  const int sm_budget = (policy >> 16) & 0xff;   // LSV_PLAN_SMS(n): grids of at most n CTAs (0: all SMs)
  const int vsplit = (policy & LSV_PLAN_V_BF16) ? 0 : 1;
  const bool tile_aligned = (policy & LSV_PLAN_TILE_ALIGNED) != 0;
  policy &= 0xff;
  if (policy != LSV_TIER_AUTO && policy != LSV_TIER_SIMT && policy != LSV_TIER_TC)
    return fail(LSV_EINVAL, "unknown tier policy %d", policy);
  if (tile_aligned && policy == LSV_TIER_SIMT)
    return fail(LSV_EINVAL, "tile-aligned plans (LSV_PLAN_TILE_ALIGNED) are tensor-core tier only");
  if (tile_aligned) policy = LSV_TIER_TC;   // every segment's v feeds the fused GEMM's M=128 tiles
  const int N = S > 0 ? indptr[S] : 0;
  pb.indptr.assign(indptr, indptr + S + 1);
  if (S == 0) pb.indptr.assign(1, 0);
  pb.rank.assign(rank, rank + S);
  pb.tier.assign(S, kTierNone);
  std::vector<uint8_t> remote(S, 0);
  bool any_remote = false;
  for (int s = 0; s < S && seg_flags; ++s) {
    remote[s] = (seg_flags[s] & LSV_SEG_REMOTE) ? 1 : 0;
    any_remote |= remote[s] != 0;
  }
  const std::vector<uint8_t>* rem = any_remote ? &remote : nullptr;
  // LSV_SEG_NOSHRINK: the segment's m-tiles stay in the plan (indices match a full-rank plan of the
  // same batch) but this plan shrinks nothing for it (a TP rank holding no rows of its adapter)
  std::vector<uint8_t> noshrink(S, 0);
  for (int s = 0; s < S && seg_flags; ++s) noshrink[s] = (seg_flags[s] & LSV_SEG_NOSHRINK) ? 1 : 0;
  const int nsm = sm_budget > 0 ? std::min(sm_budget, num_sms_cached()) : num_sms_cached();

  // tier per segment
  const bool all_simt = policy == LSV_TIER_AUTO && decode_shaped(S, indptr);
  int64_t v_off = 0;
  for (int s = 0; s < S; ++s) {
    const int n = indptr[s + 1] - indptr[s];
    if (n == 0 || (seg_flags && (seg_flags[s] & LSV_SEG_SKIP))) continue;   // no work (range kept)
    bool simt;
    if (policy == LSV_TIER_SIMT) simt = true;
    else if (policy == LSV_TIER_TC) simt = false;
    else simt = all_simt || auto_simt(n, rank[s]);
    pb.tier[s] = simt ? kTierSimt : kTierTc;
    if (simt) {
      for (int tb = 0; tb < n; tb += kSimtMaxTok) {
        const int nt = std::min(kSimtMaxTok, n - tb);
        pb.simt.push_back(SimtItem{s, indptr[s] + tb, nt | rank[s] << 16, (int32_t)v_off});
        v_off += (int64_t)nt * rank[s];
      }
    } else if (tile_aligned) {   // pieces of the segment inside each 128-token tile of the batch
      for (int t = indptr[s]; t < indptr[s + 1];) {
        const int e = std::min(indptr[s + 1], (t / kTileM + 1) * kTileM);
        MTile mt{};
        mt.seg = s; mt.tok_begin = t; mt.ntok = e - t; mt.rank = rank[s];
        pb.mtiles.push_back(mt);
        t = e;
      }
    } else {
      const int tm = mtile_rows(rank[s]);
      for (int tb = 0; tb < n; tb += tm) {
        MTile mt{};
        mt.seg = s; mt.tok_begin = indptr[s] + tb; mt.ntok = std::min(tm, n - tb); mt.rank = rank[s];
        pb.mtiles.push_back(mt);
      }
    }
  }
  // shrink: every m-tile is cut into projection subsets (N = np*rank <= 256) and k-splits that
  // balance bytes across ~kShrinkWaves waves of the SMs
  const int chunks = h_in / kChunk;
  int64_t total = 0;
  int acc_cols = 128;
  for (const MTile& mt : pb.mtiles) {
    const int np8 = round_up(mt.ntok, 8);
    for (int p0 = 0; p0 < P; p0 += subset_np(P, p0, mt.rank)) {
      const int rows = subset_np(P, p0, mt.rank) * mt.rank;
      total += (int64_t)(np8 + rows) * 128 * chunks;
      if (round_up(rows, 16) > 128) acc_cols = 256;
    }
  }
  const int64_t target = std::max<int64_t>(kMinItemBytes, total / std::max(1, kShrinkWaves * nsm));
  int64_t part_off = 0, vimg_off = 0;
  int counter = 0;
  std::vector<std::pair<int64_t, ShrinkRec>> shrink_costed;
  for (size_t i = 0; i < pb.mtiles.size(); ++i) {
    MTile& mt = pb.mtiles[i];
    const int r = mt.rank, G = P * r, np8 = round_up(mt.ntok, 8);
    const int64_t mt_bytes = (int64_t)(np8 + G) * 128 * chunks;
    int nsplit = (int)std::min<int64_t>(chunks, std::max<int64_t>(1, (mt_bytes + target - 1) / target));
    int cps = (chunks + nsplit - 1) / nsplit;          // chunks per split, whole 4-chunk stages
    if (nsplit > 1) cps = std::min(chunks, round_up(cps, kShrinkMaxKch));
    nsplit = (chunks + cps - 1) / cps;
    if (noshrink[mt.seg]) nsplit = 1;
    mt.nsplit = nsplit;
    mt.part_off = (int32_t)part_off;
    if (nsplit > 1) part_off += (int64_t)nsplit * mt.ntok * G;
    mt.vimg_off = (int32_t)vimg_off;  // 1024-aligned: the v image's swizzle atoms are address-based
    // split v: hi image, lo image; tile-aligned images span the whole 128-row tile
    vimg_off += (int64_t)vimg_bytes(tile_aligned ? kTileM : mt.ntok, kpad(r)) * (vsplit ? 2 : 1);
    int nsub = 0;
    for (int p0 = 0; p0 < P; p0 += subset_np(P, p0, r)) ++nsub;
    mt.counter = noshrink[mt.seg] ? 0 : nsplit * nsub;   // shrink records of the tile (group kernel's ready target)
    ++counter;
    if (noshrink[mt.seg]) continue;
    if (nsplit > 1) {  // reduction units: (token, projection, 8 padded-k) of this tile, reduced grid-wide
      pb.red.push_back((int32_t)i);
      pb.red.push_back(pb.red_units);
      pb.red_units += (tile_aligned ? kTileM : mt.ntok) * P * (kpad(r) / 8);   // tile-aligned: zero rows too
    }
    for (int p0 = 0; p0 < P; p0 += subset_np(P, p0, r)) {
      const int np = subset_np(P, p0, r), rows = np * r;
      const int64_t row_bytes = (int64_t)(np8 + rows) * 128;
      const int kch = (int)std::max<int64_t>(1, std::min<int64_t>(kShrinkMaxKch, kShrinkSlotBytes / row_bytes));
      for (int sp = 0; sp < nsplit; ++sp) {
        ShrinkRec rc{};
        rc.seg = mt.seg; rc.tok_begin = mt.tok_begin; rc.ntok = mt.ntok; rc.rank = r;
        rc.chunk_begin = sp * cps;
        rc.chunk_end = std::min(chunks, (sp + 1) * cps);
        rc.kch = kch; rc.split = sp;
        rc.nsplit = nsplit; rc.part_off = mt.part_off; rc.vimg_off = mt.vimg_off; rc.counter = mt.counter;
        rc.mtile = (int32_t)i; rc.p0 = p0; rc.np = np;
        // bytes moved + a fixed cost per pipeline stage and per record (epilogue, split partials).
        // The standalone shrink (round-2 start, tools/shrink_balance.py) paid a near fixed share of
        // the load latency per stage; the layer kernel streams stages back to back across phases,
        // and bytes predict a CTA's time (tools/timeline_step.py per-CTA phase ends vs its plan).
        const int nstage = (rc.chunk_end - rc.chunk_begin + kch - 1) / kch;
        const int64_t cost = row_bytes * (rc.chunk_end - rc.chunk_begin) + kShrinkRecFixed +
                             kShrinkStageFixed * nstage + (nsplit > 1 ? (int64_t)mt.ntok * rows * 8 : 0) +
                             (remote[mt.seg] ? (int64_t)(kRemoteWeight - 1) * rows * 128 * (rc.chunk_end - rc.chunk_begin) : 0);
        shrink_costed.push_back({cost, rc});
      }
    }
  }
  std::stable_sort(shrink_costed.begin(), shrink_costed.end(),
                   [](const auto& a, const auto& b) { return a.first > b.first; });
  const int shrink_grid = (int)std::min<size_t>(shrink_costed.size(), (size_t)nsm);
  std::vector<int64_t> shrink_finish;
  lpt_assign(shrink_costed, std::max(shrink_grid, 1), pb.shrink, pb.shrink_cta, rem, &shrink_finish);
  // estimated time each m-tile's v images are complete (its last shrink record; split tiles also
  // wait for their reduction): the group kernel's CTAs take their expand items in this order
  std::vector<int64_t> tile_ready(pb.mtiles.size(), 0);
  for (size_t i = 0; i < pb.shrink.size(); ++i) {
    const ShrinkRec& rc = pb.shrink[i];
    tile_ready[rc.mtile] = std::max(tile_ready[rc.mtile], shrink_finish[i] + (rc.nsplit > 1 ? kShrinkRecFixed : 0));
  }
  auto ready_order = [&](std::vector<ExpandRec>& recs, const std::vector<int32_t>& off) {
    for (size_t c = 0; c + 1 < off.size(); ++c)
      std::stable_sort(recs.begin() + off[c], recs.begin() + off[c + 1], [&](const ExpandRec& a, const ExpandRec& b) {
        return tile_ready[a.mtile] < tile_ready[b.mtile];
      });
  };

  // expand: per projection, items = (m-tile, tw-wide h_out tile); plus all members in one list.
  // An item's cost depends only on (m-tile, member), so the (m-tile, member) classes are sorted
  // (stable, a few hundred) and their h_out tiles emitted in that order: the LPT input order of a
  // stable sort of the items, without sorting the items.
  struct ItemClass { int64_t cost; int32_t mt, p; };
  auto emit = [&](const std::vector<ItemClass>& cls, std::vector<std::pair<int64_t, ExpandRec>>& out) {
    for (const ItemClass& c : cls) {
      const MTile& mt = pb.mtiles[c.mt];
      const int tw = expand_item_tw(mt.rank, b_tile_width(h_outs[c.p]));
      for (int jt = 0; jt < h_outs[c.p] / tw; ++jt) {
        ExpandRec r{};
        r.seg = mt.seg; r.tok_begin = mt.tok_begin; r.ntok = mt.ntok; r.rank = mt.rank;
        r.jtile = jt; r.vimg_off = mt.vimg_off; r.mtile = c.mt; r.proj = c.p;
        out.push_back({c.cost, r});
      }
    }
  };
  auto by_cost = [](const ItemClass& a, const ItemClass& b) { return a.cost > b.cost; };
  int expand_grid[kMaxProj] = {0, 0, 0, 0};
  std::vector<ItemClass> all_cls;
  for (int p = 0; p < P; ++p) {
    std::vector<ItemClass> cls;
    size_t n_items = 0;
    for (size_t i = 0; i < pb.mtiles.size(); ++i) {
      const MTile& mt = pb.mtiles[i];
      const int tw = expand_item_tw(mt.rank, b_tile_width(h_outs[p]));
      const int64_t bbytes = (int64_t)tw * kpad(mt.rank) * 2;
      cls.push_back({bbytes * (remote[mt.seg] ? kRemoteWeight : 1) + (int64_t)mt.ntok * tw * 4 + kExpandItemFixed,
                     (int32_t)i, p});
      n_items += h_outs[p] / tw;
    }
    all_cls.insert(all_cls.end(), cls.begin(), cls.end());
    std::stable_sort(cls.begin(), cls.end(), by_cost);
    std::vector<std::pair<int64_t, ExpandRec>> expand_costed;
    expand_costed.reserve(n_items);
    emit(cls, expand_costed);
    expand_grid[p] = (int)std::min<size_t>(expand_costed.size(), (size_t)nsm);
    lpt_assign(expand_costed, std::max(expand_grid[p], 1), pb.expand[p], pb.expand_cta[p], rem);
    if (g_ready_order && !rem) ready_order(pb.expand[p], pb.expand_cta[p]);
  }
  std::stable_sort(all_cls.begin(), all_cls.end(), by_cost);
  std::vector<std::pair<int64_t, ExpandRec>> all_costed;
  emit(all_cls, all_costed);
  const int expand_grid_all = (int)std::min<size_t>(all_costed.size(), (size_t)nsm);
  lpt_assign(all_costed, std::max(expand_grid_all, 1), pb.expand_all, pb.expand_all_cta, rem);
  if (g_ready_order && !rem) ready_order(pb.expand_all, pb.expand_all_cta);
  {   // dynamic dispatch order over the group kernel's list: estimated tile readiness, then larger first
    const std::vector<ExpandRec>& gl = P > 1 ? pb.expand_all : pb.expand[0];
    std::vector<int64_t> key(gl.size());
    for (size_t i = 0; i < gl.size(); ++i) {
      const ExpandRec& r = gl[i];
      const int tw = expand_item_tw(r.rank, b_tile_width(h_outs[r.proj]));
      key[i] = (int64_t)tw * kpad(r.rank) * 2 + (int64_t)r.ntok * tw * 4;
    }
    pb.dyn.resize(gl.size());
    for (size_t i = 0; i < gl.size(); ++i) pb.dyn[i] = (int32_t)i;
    int64_t max_ready = 1;
    for (int64_t t : tile_ready) max_ready = std::max(max_ready, t);
    const int nb = g_dyn_order == 1 ? 8 : 1;   // 1: readiness in 8 buckets, h_out tiles interleaved inside each
    std::stable_sort(pb.dyn.begin(), pb.dyn.end(), [&](int32_t a, int32_t b) {
      const ExpandRec &x = gl[a], &y = gl[b];
      if (g_dyn_order == 2) {   // h_out-tile major: consecutive items from different m-tiles
        if (x.jtile != y.jtile) return x.jtile < y.jtile;
      } else if (g_dyn_order == 1) {
        const int64_t ba = tile_ready[x.mtile] * nb / (max_ready + 1), bb = tile_ready[y.mtile] * nb / (max_ready + 1);
        if (ba != bb) return ba < bb;
        if (x.jtile != y.jtile) return x.jtile < y.jtile;
      }
      const int64_t ra = tile_ready[x.mtile], rb = tile_ready[y.mtile];
      return ra != rb ? ra < rb : key[a] > key[b];
    });
    if (rem) {   // peer-owned items (NVLink) and local ones (HBM) merged by their estimated time on
                 // each link, so both stay busy to the end of the list (~8x HBM / NVLink bandwidth)
      std::vector<int32_t> loc, rmt;
      for (int32_t i : pb.dyn) (remote[gl[i].seg] ? rmt : loc).push_back(i);
      pb.dyn.clear();
      int64_t tl = 0, tr = 0;
      size_t il = 0, ir = 0;
      while (il < loc.size() || ir < rmt.size()) {
        if (ir < rmt.size() && (il == loc.size() || tr <= tl)) {
          const ExpandRec& r = gl[rmt[ir]];
          tr += (int64_t)expand_item_tw(r.rank, b_tile_width(h_outs[r.proj])) * kpad(r.rank) * 2 * 8;
          pb.dyn.push_back(rmt[ir++]);
        } else {
          tl += key[loc[il]];
          pb.dyn.push_back(loc[il++]);
        }
      }
    }
  }

  // header + workspace layout
  PlanHeader& h = pb.h;
  h.magic = kPlanMagic; h.version = kPlanVersion;
  h.num_segments = S; h.num_tokens = N; h.h_in = h_in; h.h_out = h_outs[0];
  h.num_proj = P;
  h.acc_cols = acc_cols;
  h.vsplit = vsplit;
  h.n_simt_items = (int32_t)pb.simt.size();
  h.n_mtiles = (int32_t)pb.mtiles.size();
  h.n_shrink_items = (int32_t)pb.shrink.size();
  h.shrink_grid = shrink_grid;
  int32_t off = sizeof(PlanHeader) / 4;
  h.off_seg_indptr = off; off += S + 1;
  h.off_seg_rank = off; off += S;
  h.off_seg_tier = off; off += S;
  off = round_up(off, 4);
  h.off_simt_items = off; off += 4 * h.n_simt_items;
  // SIMT tail (lsv_plan.h): row-block prefix [n + 1], row-block map [n_rb]
  if (h.n_simt_items > 0) {
    int n_rb = 0;
    for (const SimtItem& it : pb.simt) n_rb += (P * simt_rank(it) + kSimtShrRows - 1) / kSimtShrRows;
    off += h.n_simt_items + 1 + n_rb;
  }
  off = round_up(off, 4);
  h.off_mtiles = off; off += 8 * h.n_mtiles;
  h.off_shrink_recs = off; off += 16 * h.n_shrink_items;
  h.off_shrink_cta = off; off += (int32_t)pb.shrink_cta.size();
  for (int p = 0; p < P; ++p) {
    off = round_up(off, 4);
    h.h_outs[p] = h_outs[p];
    h.n_expand_items_p[p] = (int32_t)pb.expand[p].size();
    h.expand_grid_p[p] = expand_grid[p];
    h.off_expand_recs_p[p] = off; off += 8 * h.n_expand_items_p[p];
    h.off_expand_cta_p[p] = off; off += (int32_t)pb.expand_cta[p].size();
  }
  off = round_up(off, 4);
  h.n_expand_all = (int32_t)pb.expand_all.size();
  h.expand_grid_all = expand_grid_all;
  h.off_expand_recs_all = off; off += 8 * h.n_expand_all;
  h.off_expand_cta_all = off; off += (int32_t)pb.expand_all_cta.size();
  h.n_expand_items = h.n_expand_items_p[0];
  h.expand_grid = h.expand_grid_p[0];
  h.off_expand_recs = h.off_expand_recs_p[0];
  h.off_expand_cta = h.off_expand_cta_p[0];
  h.off_red = off; off += (int32_t)pb.red.size();
  h.n_red = (int32_t)pb.red.size() / 2;
  h.red_units = pb.red_units;
  // split-K reduction: CTA c reduces units [c*U/G, (c+1)*U/G); record the entry holding its first
  std::vector<int32_t> red_cta(shrink_grid + 1, 0);
  for (int c = 0; c <= shrink_grid; ++c) {
    const int64_t u0 = shrink_grid > 0 ? (int64_t)pb.red_units * c / shrink_grid : 0;
    int e = 0;
    while (e + 1 < h.n_red && pb.red[2 * (e + 1) + 1] <= u0) ++e;
    red_cta[c] = e;
  }
  h.off_red_cta = off; off += (int32_t)red_cta.size();
  pb.red_cta = red_cta;
  h.off_dyn = off; off += (int32_t)pb.dyn.size();
  h.tile_aligned = tile_aligned ? 1 : 0;
  if (tile_aligned) {   // [n_gemm_tiles + 1] first piece of every 128-token tile (pieces are in token order)
    const int nt = (N + kTileM - 1) / kTileM;
    pb.tile_mt.assign(nt + 1, 0);
    size_t i = 0;
    for (int t = 0; t <= nt; ++t) {
      while (i < pb.mtiles.size() && pb.mtiles[i].tok_begin < t * kTileM) ++i;
      pb.tile_mt[t] = (int32_t)i;
    }
    off += nt + 1;
  }
  h.total_ints = off;
  int64_t ws = 0;
  h.ws_counters = 0; ws += kBarHeaderBytes;   // barrier header (lsv_plan.h): pair 0 for standalone calls
  h.ws_partials = (int32_t)ws; ws += (part_off * 4 + 255) / 256 * 256;
  const int64_t vstride = (vimg_off + 1023) / 1024 * 1024;
  h.ws_vimg = (int32_t)ws; ws += vstride * P;
  h.simt_stride = (int32_t)((v_off + 63) / 64 * 64);
  h.ws_simt_v = (int32_t)ws; ws += (int64_t)h.simt_stride * 4 * P * simt_ksplit(h_in);
  if (ws > INT32_MAX) return fail(LSV_EUNSUPPORTED, "workspace of %lld bytes exceeds 2 GiB", (long long)ws);
  h.vimg_stride = (int32_t)vstride;
  h.ws_bytes = (int32_t)ws;
  h.n_counters = 0;
  (void)counter;
  int simt_segs = 0;
  for (int s = 0; s < S; ++s) simt_segs += pb.tier[s] == kTierSimt;
  h.simt_segments = simt_segs;
  return LSV_OK;
}

const PlanHeader* check_plan(const void* plan_host) {
  const PlanHeader* h = static_cast<const PlanHeader*>(plan_host);
  if (!h || h->magic != kPlanMagic || h->version != kPlanVersion) return nullptr;
  return h;
}

// ---- driver entry point for TMA descriptors (no link-time libcuda dependency) -------------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
    cudaGetLastError();
  });
  return fn;
}

// Tensor maps are pure functions of (pointer, row stride, rows, cols); encoding costs ~1 µs of
// host time, so they are cached (a model step reuses the same activation buffers every layer).
struct MapKey {
  uintptr_t ptr; int64_t ld; int32_t rows, cols, kind;
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && ld == o.ld && rows == o.rows && cols == o.cols && kind == o.kind;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    size_t h = std::hash<uintptr_t>()(k.ptr);
    h ^= std::hash<int64_t>()(k.ld * 1315423911LL + k.rows) + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2);
    h ^= std::hash<int64_t>()((int64_t)k.cols * 31 + k.kind) + (h << 6) + (h >> 2);
    return h;
  }
};
std::mutex g_map_mu;
std::unordered_map<MapKey, std::vector<CUtensorMap>, MapKeyHash> g_map_cache;

// kind 0: x maps (5 boxes of 64 cols x 8<<b rows, SWIZZLE_128B)
// kind 1: expand y maps, 3D {64 cols, rows, cols/64 blocks} (strides ld*2, 128 B): 10 boxes
//         {64, 8<<b rows, 4 blocks} (b = 0..4) then {64, 8<<b, 2 blocks}, SWIZZLE_128B
// kind 2: base-weight maps (1 box of 64 cols x 256 rows, SWIZZLE_128B)
int get_maps(CUtensorMap* out, int kind, const void* ptr, int64_t ld, int32_t rows, int32_t cols) {
  const MapKey key{reinterpret_cast<uintptr_t>(ptr), ld, rows, cols, kind};
  const int nmaps = kind == 0 ? 5 : kind == 1 ? 10 : 1;
  {
    std::lock_guard<std::mutex> lk(g_map_mu);
    auto it = g_map_cache.find(key);
    if (it != g_map_cache.end()) {
      std::memcpy(out, it->second.data(), sizeof(CUtensorMap) * nmaps);
      return LSV_OK;
    }
  }
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return fail(LSV_ECUDA, "cuTensorMapEncodeTiled entry point unavailable");
  std::vector<CUtensorMap> maps(nmaps);
  for (int b = 0; b < nmaps && kind == 1; ++b) {
    if (cols % 64) return fail(LSV_EINVAL, "y width %d is not a multiple of 64", cols);
    const cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(cols / 64)};
    const cuuint64_t strides[2] = {(cuuint64_t)ld * 2, 128};
    const cuuint32_t box[3] = {64, (cuuint32_t)(8 << (b % 5)), b < 5 ? 4u : 2u};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(&maps[b], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(LSV_ECUDA, "cuTensorMapEncodeTiled failed (%d) for a 3D y map, box %d", (int)r, b);
  }
  for (int b = 0; b < nmaps && kind != 1; ++b) {
    const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
    const cuuint32_t box[2] = {(cuuint32_t)kChunk, kind == 0 ? (cuuint32_t)(8 << b) : (cuuint32_t)kFusedTileN};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&maps[b], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
      return fail(LSV_ECUDA, "cuTensorMapEncodeTiled failed (%d) kind %d box %d", (int)r, kind, b);
  }
  std::memcpy(out, maps.data(), sizeof(CUtensorMap) * nmaps);
  std::lock_guard<std::mutex> lk(g_map_mu);
  if (g_map_cache.size() > 8192) g_map_cache.clear();
  g_map_cache.emplace(key, std::move(maps));
  return LSV_OK;
}

int ensure_smem_attrs() {
  static int rc = -1;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaError_t e1 = cudaFuncSetAttribute(shrink_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          shrink_smem_bytes());
    cudaError_t e2 = cudaFuncSetAttribute(expand_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          expand_smem_bytes());
    cudaError_t e3 = cudaFuncSetAttribute(fused_linear_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          fused_smem_bytes());
    cudaError_t e4 = cudaFuncSetAttribute(group_tc_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          group_smem_bytes());
    if (e4 == cudaSuccess)
      e4 = cudaFuncSetAttribute(group_tc_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, group_smem_bytes());
    if (e2 == cudaSuccess) e2 = e3;
    if (e2 == cudaSuccess) e2 = e4;
    rc = (e1 == cudaSuccess && e2 == cudaSuccess) ? LSV_OK : LSV_ECUDA;
    if (rc) fail(LSV_ECUDA, "cudaFuncSetAttribute(smem) failed: %s / %s", cudaGetErrorString(e1), cudaGetErrorString(e2));
  });
  return rc;
}

// Programmatic dependent launch: the kernel may start while the previous kernel in the stream
// drains; it calls griddepcontrol.wait before touching anything that kernel wrote.
template <typename Params>
cudaError_t launch_pdl(void (*kernel)(Params), int grid, int smem, cudaStream_t st, const Params& p, bool pdl = true,
                       int threads = kTcThreads) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;     // without it the launch waits for all earlier work in the stream
  return cudaLaunchKernelEx(&cfg, kernel, p);
}

// The same for any kernel signature and grid shape (the SIMT kernels).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_any(void (*kernel)(KArgs...), dim3 grid, int threads, cudaStream_t st, bool pdl, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

int check_common(const PlanHeader* h, size_t workspace_bytes, const void* plan_dev, const void* ws) {
  if (!h) return fail(LSV_EINVAL, "plan_host is not a liblsv plan");
  if (!plan_dev) return fail(LSV_EINVAL, "plan_dev is null");
  if (workspace_bytes < (size_t)h->ws_bytes)
    return fail(LSV_EWORKSPACE, "workspace of %zu bytes is smaller than the planned %d", workspace_bytes, h->ws_bytes);
  if (h->ws_bytes > 0 && !ws) return fail(LSV_EINVAL, "workspace is null");
  return LSV_OK;
}

// wait_prev = 0: the previous launch neither writes what this shrink reads nor reads what it
// writes (lsv_lora_forward's per-(layer, group) workspace slices), so it need not wait for it;
// pdl = false: a plain launch, ordered after all earlier work in the stream.
struct TpScatter {
  int tp = 0, tp_rank = 0, row = 0, rr = 0;
  const PlanHeader* fh = nullptr;
  const int32_t* fplan = nullptr;
  void* const* vdst = nullptr;
  int32_t* const* flags = nullptr;
};

int fill_shrink_params(ShrinkParams& p, const PlanHeader* h, const void* x, int64_t ldx, int32_t num_tokens,
                       const void* const* a_ptrs, const int32_t* plan, uint8_t* ws, int* gbar);
int fill_expand_params(ExpandParams& p, const PlanHeader* h, int p0, int np, void* const* ys, const int64_t* ldys,
                       int32_t num_tokens, const void* const* const* b_ptrs, const int32_t* plan, uint8_t* ws,
                       const uint8_t* vimg_base);

int run_shrink(const PlanHeader* h, const void* x, int64_t ldx, int32_t num_tokens, const void* const* a_ptrs,
               const int32_t* plan, uint8_t* ws, cudaStream_t st, int wait_prev = 1, bool pdl = true,
               const TpScatter* tps = nullptr, bool simt_pdl = false, int* gbar = nullptr) {
  if (h->n_simt_items > 0) {
    // one block per (8-row block of an item's group A, k-split): exactly the blocks with rows
    const int32_t* hp = reinterpret_cast<const int32_t*>(h);
    const int n_rb = hp[h->off_simt_items + 4 * h->n_simt_items + h->n_simt_items];
    LSV_CUDA_CHECK(launch_pdl_any(simt_shrink_kernel, dim3(n_rb, 1, simt_ksplit(h->h_in)), 256, st, simt_pdl,
                                  static_cast<const __nv_bfloat16*>(x), ldx, (int)h->h_in, plan,
                                  (int)h->off_simt_items, (int)h->n_simt_items, a_ptrs,
                                  reinterpret_cast<float*>(ws + h->ws_simt_v), (int)h->num_proj, (int)h->simt_stride,
                                  (wait_prev || !simt_pdl || g_simt_wait) ? 1 : 0));
  }
  if (h->n_shrink_items > 0) {
    if (int rc = ensure_smem_attrs()) return rc;
    ShrinkParams p{};
    if (int rc = fill_shrink_params(p, h, x, ldx, num_tokens, a_ptrs, plan, ws, gbar)) return rc;
    p.wait_prev = (wait_prev || h->n_simt_items > 0) ? 1 : 0;   // a SIMT launch in between is not PDL
    if (tps != nullptr) {
      p.tp = tps->tp; p.tp_rank = tps->tp_rank; p.tp_rr = tps->rr;
      p.tp_row = tps->row; p.xslot = 2 * h->vimg_stride * h->num_proj;
      p.fplan = tps->fplan; p.f_off_mtiles = tps->fh->off_mtiles; p.vstride_f = tps->fh->vimg_stride;
      for (int d = 0; d < tps->tp; ++d) {
        p.vdst[d] = static_cast<uint8_t*>(tps->vdst[d]);
        p.flags[d] = tps->flags[d];
      }
    }
    LSV_CUDA_CHECK(launch_pdl(shrink_tc_kernel, h->shrink_grid, shrink_smem_bytes(), st, p, pdl, kShrinkThreads));
  }
  return LSV_OK;
}

int fill_shrink_params(ShrinkParams& p, const PlanHeader* h, const void* x, int64_t ldx, int32_t num_tokens,
                       const void* const* a_ptrs, const int32_t* plan, uint8_t* ws, int* gbar) {
  {
    if (int rc = get_maps(p.xmap, 0, x, ldx, num_tokens, h->h_in)) return rc;
    p.plan = plan; p.a_ptrs = a_ptrs; p.ws = ws;
    p.off_recs = h->off_shrink_recs; p.off_cta = h->off_shrink_cta;
    p.ws_partials = h->ws_partials; p.ws_vimg = h->ws_vimg;
    p.gbar = gbar ? gbar : reinterpret_cast<int*>(ws);
    p.off_mtiles = h->off_mtiles; p.off_red = h->off_red; p.n_red = h->n_red; p.red_units = h->red_units;
    p.off_red_cta = h->off_red_cta;
    p.num_proj = h->num_proj; p.vimg_stride = h->vimg_stride; p.acc_cols = h->acc_cols;
    p.vsplit = h->vsplit;
    p.tile_aligned = h->tile_aligned;
    p.dbg = g_debug_shrink;
    p.trace = g_trace_items > 0 ? g_trace : nullptr; p.trace_items = std::max(0, g_trace_items);
    p.num_tokens = num_tokens; p.h_in = h->h_in; p.ws_bytes = h->ws_bytes;
  }
  return LSV_OK;
}

// Expand of members [p0, p0 + np) of a plan: np == num_proj uses the combined list (one launch
// for every member), np == 1 member p0's own list.
int run_expand(const PlanHeader* h, int p0, int np, void* const* ys, const int64_t* ldys, int32_t num_tokens,
               const void* const* const* b_ptrs, const int32_t* plan, uint8_t* ws, cudaStream_t st,
               const uint8_t* vimg_base = nullptr, int32_t* wait_flag = nullptr, int32_t wait_target = 0,
               const uint8_t* xsum = nullptr, bool simt_pdl = false) {
  if (h->tile_aligned)
    return fail(LSV_EINVAL, "a tile-aligned plan (LSV_PLAN_TILE_ALIGNED) feeds lsv_lora_fused_linear, not the expand");
  if (h->n_simt_items > 0) {   // every member in one launch per token class (grid.z = member)
    SimtExpandArgs a{};
    int max_tiles = 0;
    for (int i = 0; i < np; ++i) {
      const int pp = p0 + i;
      a.y[i] = static_cast<__nv_bfloat16*>(ys[i]);
      a.ldy[i] = ldys[i];
      a.h_out[i] = h->h_outs[pp];
      a.b_ptrs[i] = b_ptrs[i];
      a.v[i] = reinterpret_cast<const float*>(ws + h->ws_simt_v) + (size_t)pp * h->simt_stride;
      max_tiles = std::max(max_tiles, (h->h_outs[pp] + kSimtExpCols - 1) / kSimtExpCols);
    }
    a.plan = plan; a.off_items = h->off_simt_items;
    a.ksplit = simt_ksplit(h->h_in); a.split_stride = (int64_t)h->num_proj * h->simt_stride;
    // one launch: the small accumulator; larger items (rare in decode) in token-pair passes
    LSV_CUDA_CHECK(launch_pdl_any(simt_expand_kernel<kSimtSmallTok>, dim3(h->n_simt_items, max_tiles, np), kSimtExpThreads, st,
                                  simt_pdl, a));
  }
  const bool all = np == h->num_proj && np > 1;
  const int n_items = all ? h->n_expand_all : h->n_expand_items_p[p0];
  if (n_items == 0) return LSV_OK;
  if (int rc = ensure_smem_attrs()) return rc;
  ExpandParams p{};
  if (int rc = fill_expand_params(p, h, p0, np, ys, ldys, num_tokens, b_ptrs, plan, ws, vimg_base)) return rc;
  p.wait_flag = wait_flag; p.wait_target = wait_target;
  if (xsum != nullptr) {
    p.xsum = xsum; p.xslot = 2 * h->vimg_stride * h->num_proj; p.ws_vimg0 = h->ws_vimg;
    p.off_mtiles = h->off_mtiles; p.n_mtiles = h->n_mtiles; p.num_proj = h->num_proj;
    p.vimg_stride = h->vimg_stride;
    p.gbar = reinterpret_cast<int*>(ws);
  }
  LSV_CUDA_CHECK(launch_pdl(expand_tc_kernel, all ? h->expand_grid_all : h->expand_grid_p[p0], expand_smem_bytes(),
                            st, p, true, kExpandThreads));
  LSV_CUDA_CHECK(cudaGetLastError());
  return LSV_OK;
}

// Expand parameters of members [p0, p0 + np) (np == num_proj > 1: the combined list).
int fill_expand_params(ExpandParams& p, const PlanHeader* h, int p0, int np, void* const* ys, const int64_t* ldys,
                       int32_t num_tokens, const void* const* const* b_ptrs, const int32_t* plan, uint8_t* ws,
                       const uint8_t* vimg_base) {
  const bool all = np == h->num_proj && np > 1;
  int tw_max = 0;
  for (int pp = 0; pp < h->num_proj; ++pp) {
    const int i = all ? pp : (pp == p0 ? 0 : -1);
    if (i < 0) continue;
    CUtensorMap ym[10];
    if (int rc = get_maps(ym, 1, ys[i], ldys[i], num_tokens, h->h_outs[pp])) return rc;
    std::memcpy(p.ymap[pp], ym, sizeof(CUtensorMap) * 5);
    std::memcpy(p.ymap2[pp], ym + 5, sizeof(CUtensorMap) * 5);
    p.y[pp] = static_cast<__nv_bfloat16*>(ys[i]);
    p.ldy[pp] = ldys[i];
    p.b_ptrs[pp] = b_ptrs[i];
    p.tws[pp] = b_tile_width(h->h_outs[pp]);
    p.st32[pp] = (reinterpret_cast<uintptr_t>(ys[i]) & 31) == 0 && ldys[i] % 16 == 0;
    p.ws_vimg[pp] = (vimg_base ? 0 : h->ws_vimg) + pp * h->vimg_stride;
    tw_max = std::max(tw_max, p.tws[pp]);
  }
  p.plan = plan; p.ws = vimg_base ? const_cast<uint8_t*>(vimg_base) : ws;
  p.vsplit = h->vsplit;
  p.off_recs = all ? h->off_expand_recs_all : h->off_expand_recs_p[p0];
  p.off_cta = all ? h->off_expand_cta_all : h->off_expand_cta_p[p0];
  p.off_mtiles = h->off_mtiles;
  p.tw_max = tw_max;
  p.dbg = g_debug_expand;
  p.trace = g_trace_items > 0 ? g_trace : nullptr; p.trace_items = std::max(0, g_trace_items);
  p.num_tokens = num_tokens; p.ws_bytes = vimg_base ? INT64_MAX : h->ws_bytes;
  for (int pp = 0; pp < h->num_proj; ++pp) p.h_outs[pp] = h->h_outs[pp];
  return LSV_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// One input group's shrink + expand as one group kernel (tensor-core plans without SIMT items):
// ready / split_done are the group's [n_mtiles] counters, zero at launch.
bool group_kernel_eligible(const PlanHeader* h) {
  return g_group_kernel && h->n_simt_items == 0 && !h->tile_aligned && h->n_shrink_items > 0 &&
         (h->num_proj > 1 ? h->n_expand_all : h->n_expand_items_p[0]) > 0;
}
// One group's parameters (its plan, x, A table, ys, B tables, workspace slice and counters).
struct GroupArgs {
  const PlanHeader* h;
  const void* x;
  int64_t ldx;
  const void* const* a_ptrs;
  void* const* ys;
  const int64_t* ldys;
  const void* const* const* b_ptrs;   // [num_proj] member tables
  const int32_t* plan;
  uint8_t* ws;
  int* gbar;
  int* ready;
};
int fill_group_params(GroupParams& gp, const GroupArgs& a, int32_t num_tokens, int wait_prev) {
  const PlanHeader* h = a.h;
  if (int rc = fill_shrink_params(gp.s, h, a.x, a.ldx, num_tokens, a.a_ptrs, a.plan, a.ws, a.gbar)) return rc;
  if (int rc = fill_expand_params(gp.e, h, 0, h->num_proj, a.ys, a.ldys, num_tokens, a.b_ptrs, a.plan, a.ws, nullptr))
    return rc;
  gp.ready = a.ready;
  gp.split_done = a.ready + h->n_mtiles;
  gp.s_grid = h->shrink_grid;
  gp.e_grid = h->num_proj > 1 ? h->expand_grid_all : h->expand_grid_p[0];
  gp.wait_prev = wait_prev;
  return LSV_OK;
}
// Development traces: timeline mode gives each launch its own [cta][16] record; item traces put the
// expand's stamps in a second buffer half.
void group_trace(GroupParams& gp) {
  if (g_trace != nullptr && g_trace_items < 0) {
    gp.s.trace = gp.e.trace = nullptr;
    gp.s.trace_items = gp.e.trace_items = 0;
    gp.tl = g_trace + (size_t)(g_tl_launch++ % -g_trace_items) * num_sms_cached() * 16;
  } else if (gp.e.trace != nullptr) {
    gp.e.trace += (size_t)num_sms_cached() * gp.e.trace_items * 16;
  }
}
int run_group(const GroupArgs& a, int32_t num_tokens, int wait_prev, bool pdl, cudaStream_t st) {
  if (int rc = ensure_smem_attrs()) return rc;
  LayerParams<1> lp{};
  if (int rc = fill_group_params(lp.g[0], a, num_tokens, wait_prev)) return rc;
  lp.ngroups = 1;
  group_trace(lp.g[0]);
  LSV_CUDA_CHECK(launch_pdl(group_tc_kernel<1>, std::max(lp.g[0].s_grid, lp.g[0].e_grid), group_smem_bytes(), st, lp,
                            pdl, kGroupThreads));
  LSV_CUDA_CHECK(cudaGetLastError());
  return LSV_OK;
}
// A layer kernel: n (<= kLayerGroups) overlap-free groups back to back in one launch.
constexpr int kLayerGroups = 4;
// dyn: expand items by dynamic dispatch (calls of several layers: back-to-back layer launches)
int run_layer(const GroupArgs* a, int n, int32_t num_tokens, int wait_prev, bool pdl, bool dyn, cudaStream_t st) {
  if (int rc = ensure_smem_attrs()) return rc;
  LayerParams<kLayerGroups> lp{};
  int grid = 0;
  for (int i = 0; i < n; ++i) {
    if (int rc = fill_group_params(lp.g[i], a[i], num_tokens, wait_prev)) return rc;
    grid = std::max(grid, std::max(lp.g[i].s_grid, lp.g[i].e_grid));
  }
  lp.ngroups = n;
  lp.lookahead = g_phase_lookahead;
  lp.dyn = dyn ? 1 : 0;
  for (int i = 0; i < n && dyn; ++i) {   // cursor: the int after the group's 2 * n_mtiles counters
    const PlanHeader* h = a[i].h;
    lp.g[i].e.cursor = lp.g[i].ready + 2 * h->n_mtiles;
    lp.g[i].e.off_dyn = h->off_dyn;
    lp.g[i].e.n_dyn = h->num_proj > 1 ? h->n_expand_all : h->n_expand_items_p[0];
  }
  group_trace(lp.g[0]);
  for (int i = 1; i < n; ++i) lp.g[i].s.trace = lp.g[i].e.trace = nullptr;
  LSV_CUDA_CHECK(launch_pdl(group_tc_kernel<kLayerGroups>, grid, group_smem_bytes(), st, lp, pdl, kGroupThreads));
  LSV_CUDA_CHECK(cudaGetLastError());
  return LSV_OK;
}
// lsv_lora_forward's group-kernel counters: 2 * n_mtiles ints per (layer, group) + the dynamic
// dispatch cursor, after the slices
size_t forward_counter_bytes(int L, int G, const PlanHeader* const* hs) {
  size_t n = 0;
  for (int g = 0; g < G; ++g) n += 2 * (size_t)hs[g]->n_mtiles + 1;
  return (n * 4 * (size_t)L + 255) / 256 * 256;
}



// lsv_lora_forward slice of one (layer, group): the plan's scratch without its barrier header
size_t forward_slice_bytes(const PlanHeader* h) {
  return ((size_t)h->ws_bytes - kBarHeaderBytes + 255) / 256 * 256;
}

// lsv_lora_forward's cross-launch overlap is safe when every y range is disjoint from every other
// y range and from every x range of the call (x ranges may overlap each other: read-only).
bool forward_ranges_disjoint(int L, int G, const PlanHeader* const* hs, int nproj, const void* const* xs,
                             const int64_t* ldxs, void* const* ys, const int64_t* ldys, int32_t num_tokens) {
  if (num_tokens <= 0) return true;
  struct Rng { uintptr_t lo, hi; bool is_y; };
  std::vector<Rng> r;
  r.reserve((size_t)L * (G + nproj));
  for (int l = 0; l < L; ++l) {
    int p0 = 0;
    for (int g = 0; g < G; ++g) {
      const PlanHeader* h = hs[g];
      const uintptr_t x = reinterpret_cast<uintptr_t>(xs[(size_t)l * G + g]);
      if (x) r.push_back({x, x + (uintptr_t)(((int64_t)(num_tokens - 1) * ldxs[(size_t)l * G + g] + h->h_in) * 2), false});
      for (int i = 0; i < h->num_proj; ++i) {
        const size_t k = (size_t)l * nproj + p0 + i;
        const uintptr_t y = reinterpret_cast<uintptr_t>(ys[k]);
        if (y) r.push_back({y, y + (uintptr_t)(((int64_t)(num_tokens - 1) * ldys[k] + h->h_outs[i]) * 2), true});
      }
      p0 += h->num_proj;
    }
  }
  std::sort(r.begin(), r.end(), [](const Rng& a, const Rng& b) { return a.lo < b.lo; });
  // sweep: an overlap involving a y range is a hazard; track the furthest-reaching x and y so far
  uintptr_t x_end = 0, y_end = 0;
  for (const Rng& q : r) {
    if (q.lo < y_end) return false;                 // overlaps an earlier y
    if (q.is_y && q.lo < x_end) return false;        // a y overlapping an earlier x
    if (q.is_y) y_end = std::max(y_end, q.hi);
    else x_end = std::max(x_end, q.hi);
  }
  return true;
}

}  // namespace

extern "C" {

int lsv_version(void) { return LSV_ABI_VERSION; }
const char* lsv_last_error(void) { return g_err; }
int lsv_num_sms(void) { return num_sms_cached(); }
int lsv_build_info(void) { return LSV_DEVICE_CHECKS ? LSV_BUILD_DEVICE_CHECKS : 0; }

size_t lsv_adapter_a_bytes(int32_t rank, int32_t h_in) {
  return (rank > 0 && h_in > 0) ? (size_t)rank * h_in * 2 : 0;
}
size_t lsv_adapter_b_bytes(int32_t rank, int32_t h_out) {
  return (rank > 0 && h_out > 0) ? (size_t)kpad(rank) * h_out * 2 : 0;  // rows padded to 16
}

static int pack_common(const void* lora_a, const void* lora_b, int32_t rank, int32_t h_in, int32_t h_out,
                       void* a_tiled, void* b_tiled, lsv_stream_t stream, int unpack, int32_t nproj = 1,
                       int32_t proj = 0) {
  if (rank < 8 || rank > 256 || rank % 8) return fail(LSV_EINVAL, "rank must be a multiple of 8 in [8, 256], got %d", rank);
  if (nproj < 1 || nproj > kMaxProj || proj < 0 || proj >= nproj)
    return fail(LSV_EINVAL, "projection %d of a group of %d (max %d)", proj, nproj, kMaxProj);
  const bool do_a = lora_a || a_tiled, do_b = lora_b || b_tiled;   // either half may be skipped
  if ((do_a && (h_in <= 0 || h_in % 128)) || (do_b && (h_out <= 0 || h_out % 128)))
    return fail(LSV_EINVAL, "h_in/h_out must be positive multiples of 128 (got %d, %d)", h_in, h_out);
  if ((do_a && !(lora_a && a_tiled)) || (do_b && !(lora_b && b_tiled)) || !(do_a || do_b))
    return fail(LSV_EINVAL, "null buffer");
  if ((do_a && (!aligned16(lora_a) || !aligned16(a_tiled))) || (do_b && (!aligned16(lora_b) || !aligned16(b_tiled))))
    return fail(LSV_EINVAL, "buffers must be 16-byte aligned");
  const int64_t units = ((do_a ? (int64_t)rank * h_in : 0) + (do_b ? (int64_t)h_out * kpad(rank) : 0)) / 8;
  const int blocks = (int)std::min<int64_t>(4096, (units + 255) / 256);
  pack_adapter_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint8_t*>(lora_a), static_cast<const uint8_t*>(lora_b), rank, do_a ? h_in : 0,
      do_b ? h_out : 0, static_cast<uint8_t*>(a_tiled), static_cast<uint8_t*>(b_tiled), unpack, nproj * rank,
      proj * rank);
  LSV_CUDA_CHECK(cudaGetLastError());
  return LSV_OK;
}

int lsv_pack_adapter(const void* lora_a, const void* lora_b, int32_t rank, int32_t h_in, int32_t h_out,
                     void* a_tiled, void* b_tiled, lsv_stream_t stream) {
  return pack_common(lora_a, lora_b, rank, h_in, h_out, a_tiled, b_tiled, stream, 0);
}

int lsv_unpack_adapter(const void* a_tiled, const void* b_tiled, int32_t rank, int32_t h_in, int32_t h_out,
                       void* lora_a, void* lora_b, lsv_stream_t stream) {
  return pack_common(lora_a, lora_b, rank, h_in, h_out, const_cast<void*>(a_tiled), const_cast<void*>(b_tiled),
                     stream, 1);
}

size_t lsv_adapter_a_group_bytes(int32_t num_proj, int32_t rank, int32_t h_in) {
  return (num_proj > 0 && rank > 0 && h_in > 0) ? (size_t)num_proj * rank * h_in * 2 : 0;
}

int lsv_pack_adapter_group(const void* lora_a, int32_t num_proj, int32_t proj, int32_t rank, int32_t h_in,
                           void* a_group_tiled, lsv_stream_t stream) {
  return pack_common(lora_a, nullptr, rank, h_in, 0, a_group_tiled, nullptr, stream, 0, num_proj, proj);
}

int lsv_unpack_adapter_group(const void* a_group_tiled, int32_t num_proj, int32_t proj, int32_t rank, int32_t h_in,
                             void* lora_a, lsv_stream_t stream) {
  return pack_common(lora_a, nullptr, rank, h_in, 0, const_cast<void*>(a_group_tiled), nullptr, stream, 1, num_proj,
                     proj);
}

static int plan_write(const PlanBuilder& pb, void* plan_host, size_t plan_bytes) {
  const PlanHeader& h = pb.h;
  if (!plan_host) return fail(LSV_EINVAL, "plan_host is null");
  if (plan_bytes < (size_t)h.total_ints * 4)
    return fail(LSV_EINVAL, "plan buffer of %zu bytes is smaller than %d", plan_bytes, h.total_ints * 4);
  int32_t* out = static_cast<int32_t*>(plan_host);
  std::memset(out, 0, (size_t)h.total_ints * 4);
  std::memcpy(out, &h, sizeof(h));
  std::copy(pb.indptr.begin(), pb.indptr.end(), out + h.off_seg_indptr);
  std::copy(pb.rank.begin(), pb.rank.end(), out + h.off_seg_rank);
  std::copy(pb.tier.begin(), pb.tier.end(), out + h.off_seg_tier);
  std::memcpy(out + h.off_simt_items, pb.simt.data(), pb.simt.size() * sizeof(SimtItem));
  if (h.n_simt_items > 0) {   // SIMT tail: row-block prefix over the items, then the row-block map
    const int n = h.n_simt_items;
    int32_t* pre = out + h.off_simt_items + 4 * n;
    int32_t* rbmap = pre + n + 1;
    pre[0] = 0;
    for (int i = 0; i < n; ++i) {
      const int nrb = (h.num_proj * simt_rank(pb.simt[i]) + kSimtShrRows - 1) / kSimtShrRows;
      for (int rb = 0; rb < nrb; ++rb) rbmap[pre[i] + rb] = i << 8 | rb;
      pre[i + 1] = pre[i] + nrb;
    }
  }
  std::memcpy(out + h.off_mtiles, pb.mtiles.data(), pb.mtiles.size() * sizeof(MTile));
  std::memcpy(out + h.off_shrink_recs, pb.shrink.data(), pb.shrink.size() * sizeof(ShrinkRec));
  std::copy(pb.shrink_cta.begin(), pb.shrink_cta.end(), out + h.off_shrink_cta);
  for (int p = 0; p < h.num_proj; ++p) {
    std::memcpy(out + h.off_expand_recs_p[p], pb.expand[p].data(), pb.expand[p].size() * sizeof(ExpandRec));
    std::copy(pb.expand_cta[p].begin(), pb.expand_cta[p].end(), out + h.off_expand_cta_p[p]);
  }
  std::memcpy(out + h.off_expand_recs_all, pb.expand_all.data(), pb.expand_all.size() * sizeof(ExpandRec));
  std::copy(pb.expand_all_cta.begin(), pb.expand_all_cta.end(), out + h.off_expand_cta_all);
  std::copy(pb.red.begin(), pb.red.end(), out + h.off_red);
  std::copy(pb.red_cta.begin(), pb.red_cta.end(), out + h.off_red_cta);
  std::copy(pb.dyn.begin(), pb.dyn.end(), out + h.off_dyn);
  if (h.tile_aligned) std::copy(pb.tile_mt.begin(), pb.tile_mt.end(), out + h.total_ints - (int32_t)pb.tile_mt.size());
  return LSV_OK;
}

// The usual call pattern is lsv_plan_size_group then lsv_plan_build_group with the same inputs:
// the last plan built on this thread is kept so the second call does not plan again.
struct PlanKey {
  std::vector<int32_t> v;
  PlanKey() = default;
  PlanKey(int32_t S, const int32_t* indptr, const int32_t* rank, int32_t h_in, int32_t P, const int32_t* h_outs,
          int32_t policy, const int32_t* flags) {
    v = {S, h_in, P, policy, num_sms_cached(), flags ? 1 : 0};
    if (h_outs) v.insert(v.end(), h_outs, h_outs + std::max(0, std::min(P, kMaxProj)));
    if (S > 0 && indptr && rank) {
      v.insert(v.end(), indptr, indptr + S + 1);
      v.insert(v.end(), rank, rank + S);
      if (flags) v.insert(v.end(), flags, flags + S);
    }
  }
};
thread_local PlanKey g_last_key;
thread_local std::unique_ptr<PlanBuilder> g_last_plan;

int plan_cached(int32_t S, const int32_t* indptr, const int32_t* rank, int32_t h_in, int32_t P, const int32_t* h_outs,
                int32_t policy, const PlanBuilder** out, const int32_t* flags = nullptr) {
  PlanKey key(S, indptr, rank, h_in, P, h_outs, policy, flags);
  if (g_last_plan && key.v == g_last_key.v) {
    *out = g_last_plan.get();
    return LSV_OK;
  }
  auto pb = std::make_unique<PlanBuilder>();
  if (int rc = build_plan(*pb, S, indptr, rank, h_in, P, h_outs, policy, flags)) return rc;
  g_last_key = std::move(key);
  g_last_plan = std::move(pb);
  *out = g_last_plan.get();
  return LSV_OK;
}

int lsv_plan_size_group(int32_t num_segments, const int32_t* seg_indptr, const int32_t* seg_rank, int32_t h_in,
                        int32_t num_proj, const int32_t* h_outs, int32_t tier_policy, size_t* plan_bytes,
                        size_t* workspace_bytes) {
  const PlanBuilder* pb = nullptr;
  if (int rc = plan_cached(num_segments, seg_indptr, seg_rank, h_in, num_proj, h_outs, tier_policy, &pb)) return rc;
  if (plan_bytes) *plan_bytes = (size_t)pb->h.total_ints * 4;
  if (workspace_bytes) *workspace_bytes = (size_t)pb->h.ws_bytes;
  return LSV_OK;
}

int lsv_plan_build_group(int32_t num_segments, const int32_t* seg_indptr, const int32_t* seg_rank, int32_t h_in,
                         int32_t num_proj, const int32_t* h_outs, int32_t tier_policy, void* plan_host,
                         size_t plan_bytes) {
  const PlanBuilder* pb = nullptr;
  if (int rc = plan_cached(num_segments, seg_indptr, seg_rank, h_in, num_proj, h_outs, tier_policy, &pb)) return rc;
  return plan_write(*pb, plan_host, plan_bytes);
}

int lsv_plan_size_group_ex(int32_t num_segments, const int32_t* seg_indptr, const int32_t* seg_rank,
                           const int32_t* seg_flags, int32_t h_in, int32_t num_proj, const int32_t* h_outs,
                           int32_t tier_policy, size_t* plan_bytes, size_t* workspace_bytes) {
  const PlanBuilder* pb = nullptr;
  if (int rc = plan_cached(num_segments, seg_indptr, seg_rank, h_in, num_proj, h_outs, tier_policy, &pb, seg_flags))
    return rc;
  if (plan_bytes) *plan_bytes = (size_t)pb->h.total_ints * 4;
  if (workspace_bytes) *workspace_bytes = (size_t)pb->h.ws_bytes;
  return LSV_OK;
}

int lsv_plan_build_group_ex(int32_t num_segments, const int32_t* seg_indptr, const int32_t* seg_rank,
                            const int32_t* seg_flags, int32_t h_in, int32_t num_proj, const int32_t* h_outs,
                            int32_t tier_policy, void* plan_host, size_t plan_bytes) {
  const PlanBuilder* pb = nullptr;
  if (int rc = plan_cached(num_segments, seg_indptr, seg_rank, h_in, num_proj, h_outs, tier_policy, &pb, seg_flags))
    return rc;
  return plan_write(*pb, plan_host, plan_bytes);
}

int lsv_plan_size(int32_t num_segments, const int32_t* seg_indptr, const int32_t* seg_rank, int32_t h_in,
                  int32_t h_out, int32_t tier_policy, size_t* plan_bytes, size_t* workspace_bytes) {
  return lsv_plan_size_group(num_segments, seg_indptr, seg_rank, h_in, 1, &h_out, tier_policy, plan_bytes,
                             workspace_bytes);
}

int lsv_plan_build(int32_t num_segments, const int32_t* seg_indptr, const int32_t* seg_rank, int32_t h_in,
                   int32_t h_out, int32_t tier_policy, void* plan_host, size_t plan_bytes) {
  return lsv_plan_build_group(num_segments, seg_indptr, seg_rank, h_in, 1, &h_out, tier_policy, plan_host,
                              plan_bytes);
}

int lsv_plan_summary(const void* plan_host, int32_t* out8) {
  const PlanHeader* h = check_plan(plan_host);
  if (!h || !out8) return fail(LSV_EINVAL, "not a liblsv plan");
  const int32_t v[8] = {h->num_segments, h->num_tokens, h->h_in, h->h_out,
                        h->simt_segments, h->n_mtiles, h->n_shrink_items, h->n_expand_items};
  std::memcpy(out8, v, sizeof(v));
  return LSV_OK;
}

int lsv_lora_shrink(const void* x, int64_t ldx, int32_t num_tokens, int32_t h_in, const void* const* a_ptrs,
                    const void* plan_dev, const void* plan_host, void* workspace, size_t workspace_bytes,
                    lsv_stream_t stream) {
  const PlanHeader* h = check_plan(plan_host);
  if (int rc = check_common(h, workspace_bytes, plan_dev, workspace)) return rc;
  if (h->h_in != h_in) return fail(LSV_EINVAL, "h_in %d does not match the plan's %d", h_in, h->h_in);
  if (num_tokens < h->num_tokens)
    return fail(LSV_EINVAL, "num_tokens %d is smaller than the plan's %d", num_tokens, h->num_tokens);
  if (h->num_tokens == 0) return LSV_OK;
  if (!x || !a_ptrs) return fail(LSV_EINVAL, "x / a_ptrs must be non-null");
  if (!aligned16(x) || ldx % 8 || ldx < h_in) return fail(LSV_EINVAL, "x must be 16-byte aligned with ldx %% 8 == 0, ldx >= h_in");
  return run_shrink(h, x, ldx, num_tokens, a_ptrs, static_cast<const int32_t*>(plan_dev),
                    static_cast<uint8_t*>(workspace), static_cast<cudaStream_t>(stream));
}

int lsv_lora_expand_proj(void* y, int64_t ldy, int32_t num_tokens, int32_t h_out, int32_t proj,
                         const void* const* b_ptrs, const void* plan_dev, const void* plan_host, void* workspace,
                         size_t workspace_bytes, lsv_stream_t stream) {
  const PlanHeader* h = check_plan(plan_host);
  if (int rc = check_common(h, workspace_bytes, plan_dev, workspace)) return rc;
  if (proj < 0 || proj >= h->num_proj) return fail(LSV_EINVAL, "projection %d of a plan for %d", proj, h->num_proj);
  if (h->h_outs[proj] != h_out)
    return fail(LSV_EINVAL, "h_out %d does not match the plan's %d", h_out, h->h_outs[proj]);
  if (num_tokens < h->num_tokens)
    return fail(LSV_EINVAL, "num_tokens %d is smaller than the plan's %d", num_tokens, h->num_tokens);
  if (h->num_tokens == 0) return LSV_OK;
  if (!y || !b_ptrs) return fail(LSV_EINVAL, "y / b_ptrs must be non-null");
  if (!aligned16(y) || ldy % 8 || ldy < h_out) return fail(LSV_EINVAL, "y must be 16-byte aligned with ldy %% 8 == 0, ldy >= h_out");
  void* ys[1] = {y};
  const int64_t ldys[1] = {ldy};
  const void* const* bt[1] = {b_ptrs};
  return run_expand(h, proj, 1, ys, ldys, num_tokens, bt, static_cast<const int32_t*>(plan_dev),
                    static_cast<uint8_t*>(workspace), static_cast<cudaStream_t>(stream));
}

namespace {
int expand_group_checked(void* const* ys, const int64_t* ldys, int32_t num_tokens, const void* const* const* b_ptrs,
                         const void* plan_dev, const void* plan_host, void* workspace, size_t workspace_bytes,
                         cudaStream_t stream, bool simt_pdl) {
  const PlanHeader* h = check_plan(plan_host);
  if (int rc = check_common(h, workspace_bytes, plan_dev, workspace)) return rc;
  if (!ys || !ldys || !b_ptrs) return fail(LSV_EINVAL, "ys / ldys / b_ptrs must be non-null host arrays");
  if (num_tokens < h->num_tokens)
    return fail(LSV_EINVAL, "num_tokens %d is smaller than the plan's %d", num_tokens, h->num_tokens);
  if (h->num_tokens == 0) return LSV_OK;
  for (int pp = 0; pp < h->num_proj; ++pp) {
    if (!ys[pp] || !b_ptrs[pp]) return fail(LSV_EINVAL, "member %d: y / b_ptrs must be non-null", pp);
    if (!aligned16(ys[pp]) || ldys[pp] % 8 || ldys[pp] < h->h_outs[pp])
      return fail(LSV_EINVAL, "member %d: y must be 16-byte aligned with ldy %% 8 == 0, ldy >= h_out", pp);
  }
  return run_expand(h, 0, h->num_proj, ys, ldys, num_tokens, b_ptrs, static_cast<const int32_t*>(plan_dev),
                    static_cast<uint8_t*>(workspace), stream, nullptr, nullptr, 0, nullptr, simt_pdl);
}
}  // namespace

int lsv_lora_expand_group(void* const* ys, const int64_t* ldys, int32_t num_tokens, const void* const* const* b_ptrs,
                          const void* plan_dev, const void* plan_host, void* workspace, size_t workspace_bytes,
                          lsv_stream_t stream) {
  return expand_group_checked(ys, ldys, num_tokens, b_ptrs, plan_dev, plan_host, workspace, workspace_bytes,
                              static_cast<cudaStream_t>(stream), false);
}

int lsv_lora_expand(void* y, int64_t ldy, int32_t num_tokens, int32_t h_out, const void* const* b_ptrs,
                    const void* plan_dev, const void* plan_host, void* workspace, size_t workspace_bytes,
                    lsv_stream_t stream) {
  return lsv_lora_expand_proj(y, ldy, num_tokens, h_out, 0, b_ptrs, plan_dev, plan_host, workspace, workspace_bytes,
                              stream);
}

int lsv_lora_forward(int32_t num_layers, int32_t num_groups, const void* const* plans_dev, const void* const* plans_host,
                     const void* const* xs, const int64_t* ldxs, void* const* ys, const int64_t* ldys,
                     const void* a_ptrs, const void* b_ptrs, int32_t num_tokens, void* workspace,
                     size_t workspace_bytes, lsv_stream_t stream) {
  return lsv_lora_forward_ex(num_layers, num_groups, plans_dev, plans_host, xs, ldxs, ys, ldys, a_ptrs, b_ptrs,
                             num_tokens, workspace, workspace_bytes, 0, stream);
}

int lsv_lora_forward_ex(int32_t num_layers, int32_t num_groups, const void* const* plans_dev,
                        const void* const* plans_host, const void* const* xs, const int64_t* ldxs, void* const* ys,
                        const int64_t* ldys, const void* a_ptrs, const void* b_ptrs, int32_t num_tokens,
                        void* workspace, size_t workspace_bytes, int32_t flags, lsv_stream_t stream) {
  if (flags & ~LSV_FWD_SERIAL) return fail(LSV_EINVAL, "lsv_lora_forward_ex: unknown flags 0x%x", flags);
  if (num_layers < 0 || num_groups < 1 || num_groups > 64)
    return fail(LSV_EINVAL, "num_layers %d / num_groups %d out of range", num_layers, num_groups);
  if (!plans_dev || !plans_host || !xs || !ldxs || !ys || !ldys || !a_ptrs || !b_ptrs)
    return fail(LSV_EINVAL, "lsv_lora_forward: null argument");
  // every (layer, group) gets its own workspace slice: nothing a shrink writes is read by any
  // other launch of this call but its own group's expand, so a shrink need not wait for the
  // expand before it (it fills the SMs that expand's tail frees).  The first launch of the call
  // is a plain one: it waits for everything earlier in the stream, including a previous call.
  const PlanHeader* hs[64];
  size_t ws_off[65];
  int nproj = 0, S = -1;
  ws_off[0] = 0;
  for (int g = 0; g < num_groups; ++g) {
    hs[g] = check_plan(plans_host[g]);
    if (!hs[g]) return fail(LSV_EINVAL, "plans_host[%d] is not a liblsv plan", g);
    if (!plans_dev[g]) return fail(LSV_EINVAL, "plans_dev[%d] is null", g);
    if (S >= 0 && hs[g]->num_segments != S) return fail(LSV_EINVAL, "group plans index different batches");
    S = hs[g]->num_segments;
    nproj += hs[g]->num_proj;
    ws_off[g + 1] = ws_off[g] + forward_slice_bytes(hs[g]);
  }
  if (1 + (int64_t)num_layers * num_groups > kMaxBarPairs)
    return fail(LSV_EUNSUPPORTED, "%d layers x %d groups exceed the workspace barrier header", num_layers, num_groups);
  const size_t per_layer = ws_off[num_groups];
  const size_t need = kBarHeaderBytes + per_layer * (size_t)num_layers + forward_counter_bytes(num_layers, num_groups, hs);
  // A shrink may skip waiting for the previous launch only if nothing it reads is written by an
  // earlier expand of this call and no two expands write overlapping y: otherwise (e.g. y buffers
  // reused across layers) every launch waits for its predecessor.
  const bool overlap_free = !(flags & LSV_FWD_SERIAL) && forward_ranges_disjoint(num_layers, num_groups, hs, nproj, xs, ldxs, ys, ldys, num_tokens);
  if (workspace_bytes < need)
    return fail(LSV_EWORKSPACE, "workspace of %zu bytes is smaller than the %zu the forward needs "
                "(lsv_lora_forward_workspace)", workspace_bytes, need);
  if (!workspace) return fail(LSV_EINVAL, "workspace is null");
  const void* const* at = static_cast<const void* const*>(a_ptrs);
  const void* const* bt = static_cast<const void* const*>(b_ptrs);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // workspace: [barrier header: pair 1 + l*G + g per (layer, group)][per layer: one slice per group].
  // A slice holds its plan's scratch without the plan's own barrier header: the kernels get a base
  // kBarHeaderBytes before the slice (plan offsets start there) and their barrier pair explicitly.
  uint8_t* const wsb = static_cast<uint8_t*>(workspace);
  // group-kernel counters (after the slices): zero-filled by this call, ordered after everything
  // earlier in the stream (a memset is never overlapped by a programmatic launch)
  int* const counters = reinterpret_cast<int*>(wsb + kBarHeaderBytes + per_layer * (size_t)num_layers);
  bool any_group = false;
  for (int g = 0; g < num_groups; ++g) any_group |= group_kernel_eligible(hs[g]) && hs[g]->num_tokens > 0;
  if (any_group && num_layers > 0)
    LSV_CUDA_CHECK(cudaMemsetAsync(counters, 0, forward_counter_bytes(num_layers, num_groups, hs), st));
  size_t cnt_off = 0;
  // layer kernels: an overlap-free call whose groups all run as group kernels issues one launch per
  // layer (every group of the layer back to back in each CTA)
  bool layer_kernel = g_layer_kernel && overlap_free && num_groups <= kLayerGroups;
  for (int g = 0; g < num_groups; ++g) layer_kernel &= hs[g]->num_tokens > 0 && group_kernel_eligible(hs[g]);
  // otherwise an overlap-free call whose groups are all SIMT tier (decode batches) spreads its
  // groups over kFwdStreams streams ((layer, group) round robin): independent groups then run
  // concurrently, which the small SIMT launches need to fill the GPU.  Never with tensor-core work:
  // its kernels (the group kernel's readiness waits, the standalone shrink's grid barrier) need
  // every CTA of the grid co-resident, which two concurrent 148-CTA grids could not guarantee.
  bool all_simt = true;
  for (int g = 0; g < num_groups; ++g) all_simt &= hs[g]->n_mtiles == 0;
  FwdStreams* const fs = (overlap_free && !layer_kernel && all_simt && g_fwd_streams && num_groups > 1 &&
                          num_layers > 0) ? fwd_streams() : nullptr;
  if (fs != nullptr) {
    LSV_CUDA_CHECK(cudaEventRecord(fs->fork, st));
    for (int i = 0; i < kFwdStreams - 1; ++i) LSV_CUDA_CHECK(cudaStreamWaitEvent(fs->s[i], fs->fork, 0));
  }
  const cudaStream_t st_main = st;
  for (int l = 0; l < num_layers; ++l) {
    int p0 = 0;
    uint8_t* wsl = wsb + per_layer * (size_t)l;   // + kBarHeaderBytes + ws_off[g] = slice (l, g)
    GroupArgs la[kLayerGroups];
    const void* const* lbt[kLayerGroups][kMaxProj];
    for (int g = 0; g < num_groups; ++g) {
      const PlanHeader* h = hs[g];
      int* gbar = reinterpret_cast<int*>(wsb) + 2 * (1 + l * num_groups + g);
      const int np = h->num_proj;
      const int64_t ldx = ldxs[l * num_groups + g];
      const void* x = xs[l * num_groups + g];
      // the first launch on each stream of this call is a plain one (waits for the fork / earlier work)
      const int si = (l * num_groups + g) % kFwdStreams;   // (layer, group) round robin over the streams
      const bool first = fs != nullptr ? l * num_groups + g < kFwdStreams : (l == 0 && g == 0);
      const cudaStream_t st = (fs != nullptr && si != 0) ? fs->s[si - 1] : st_main;
      int* const ready = counters + cnt_off;
      cnt_off += 2 * (size_t)h->n_mtiles + 1;
      if (h->num_tokens > 0 && group_kernel_eligible(h)) {
        if (!x || !aligned16(x) || ldx % 8 || ldx < h->h_in || num_tokens < h->num_tokens)
          return fail(LSV_EINVAL, "layer %d group %d: bad x", l, g);
        void* const* yg = ys + (size_t)l * nproj + p0;
        const int64_t* ldg = ldys + (size_t)l * nproj + p0;
        for (int i = 0; i < np; ++i)
          if (!yg[i] || !aligned16(yg[i]) || ldg[i] % 8 || ldg[i] < h->h_outs[i])
            return fail(LSV_EINVAL, "layer %d group %d member %d: bad y", l, g, i);
        const void* const** btab = lbt[layer_kernel ? g : 0];
        for (int i = 0; i < np; ++i) btab[i] = bt + ((size_t)l * nproj + p0 + i) * S;
        const GroupArgs ga{h, x, ldx, at + ((size_t)l * num_groups + g) * S, yg, ldg, btab,
                           static_cast<const int32_t*>(plans_dev[g]), wsl + ws_off[g], gbar, ready};
        p0 += np;
        if (layer_kernel) {
          la[g] = ga;
          continue;
        }
        // an overlap-free call's group kernels touch disjoint buffers: none waits for its predecessor
        if (int rc = run_group(ga, num_tokens, (first || !overlap_free) ? 1 : 0, !first, st)) return rc;
        continue;
      }
      if (h->num_tokens > 0) {
        if (!x || !aligned16(x) || ldx % 8 || ldx < h->h_in || num_tokens < h->num_tokens)
          return fail(LSV_EINVAL, "layer %d group %d: bad x", l, g);
        // every launch after the first may start during its predecessor's tail (PDL): inside
        // this call no kernel writes an adapter slab, so the SIMT kernels stream their first
        // weights before griddepcontrol.wait
        if (int rc = run_shrink(h, x, ldx, num_tokens, at + ((size_t)l * num_groups + g) * S,
                                static_cast<const int32_t*>(plans_dev[g]), wsl + ws_off[g], st,
                                (first || !overlap_free) ? 1 : 0, !first,
                                nullptr, !first, gbar))
          return rc;
      }
      const void* const* btab[kMaxProj];
      for (int i = 0; i < np; ++i) btab[i] = bt + ((size_t)l * nproj + p0 + i) * S;
      if (int rc = expand_group_checked(ys + (size_t)l * nproj + p0, ldys + (size_t)l * nproj + p0, num_tokens,
                                        btab, plans_dev[g], plans_host[g], wsl + ws_off[g],
                                        ws_off[g + 1] - ws_off[g] + kBarHeaderBytes, st, true))
        return rc;
      p0 += np;
    }
    if (layer_kernel)
      if (int rc = run_layer(la, num_groups, num_tokens, l == 0 ? 1 : 0, l > 0, g_dyn_expand && num_layers > 1, st_main)) return rc;
  }
  if (fs != nullptr)
    for (int i = 0; i < kFwdStreams - 1; ++i) {
      LSV_CUDA_CHECK(cudaEventRecord(fs->join[i], fs->s[i]));
      LSV_CUDA_CHECK(cudaStreamWaitEvent(st_main, fs->join[i], 0));
    }
  return LSV_OK;
}

int lsv_lora_shrink_tp_scatter(const void* x, int64_t ldx, int32_t num_tokens, int32_t h_in, const void* const* a_ptrs,
                               const void* plan_dev, const void* plan_host, void* workspace, size_t workspace_bytes,
                               int32_t tp, int32_t tp_rank, void* const* vfull_dst, const void* full_plan_dev,
                               const void* full_plan_host, int32_t* const* flags, lsv_stream_t stream) {
  const PlanHeader* h = check_plan(plan_host);
  const PlanHeader* fh = check_plan(full_plan_host);
  if (int rc = check_common(h, workspace_bytes, plan_dev, workspace)) return rc;
  if (!fh || !full_plan_dev) return fail(LSV_EINVAL, "full_plan is not a liblsv plan");
  const int rr = (tp & LSV_TP_ROUND_ROBIN) ? 1 : 0;   // shard = 8-row groups g with g % tp == tp_rank
  tp &= 0xff;
  if (tp < 1 || tp > kMaxTp || tp_rank < 0 || tp_rank >= tp || !vfull_dst || !flags)
    return fail(LSV_EINVAL, "lsv_lora_shrink_tp_scatter: bad tp / rank / destinations");
  if (fh->n_mtiles != h->n_mtiles || fh->num_proj != h->num_proj || fh->num_tokens != h->num_tokens)
    return fail(LSV_EINVAL, "shard and full plans index different tiles");
  if (fh->vsplit != h->vsplit) return fail(LSV_EINVAL, "shard and full plans differ in v precision (LSV_PLAN_V_BF16)");
  if (h->n_simt_items != 0 || fh->n_simt_items != 0)
    return fail(LSV_EUNSUPPORTED, "TP scatter needs every segment on the tensor-core tier (plan with LSV_TIER_TC)");
  if (h->h_in != h_in) return fail(LSV_EINVAL, "h_in %d does not match the plan's %d", h_in, h->h_in);
  if (h->num_tokens == 0) return LSV_OK;
  if (!x || !a_ptrs || !aligned16(x) || ldx % 8 || ldx < h_in) return fail(LSV_EINVAL, "bad x / a_ptrs");
  for (int d = 0; d < tp; ++d)
    if (!vfull_dst[d] || !flags[d]) return fail(LSV_EINVAL, "rank %d: null destination or flag", d);
  if (h->tile_aligned || fh->tile_aligned) return fail(LSV_EUNSUPPORTED, "TP scatter with a tile-aligned plan");
  TpScatter tps;
  tps.tp = tp; tps.tp_rank = tp_rank; tps.rr = rr; tps.fh = fh; tps.fplan = static_cast<const int32_t*>(full_plan_dev);
  tps.vdst = vfull_dst; tps.flags = flags;
  return run_shrink(h, x, ldx, num_tokens, a_ptrs, static_cast<const int32_t*>(plan_dev),
                    static_cast<uint8_t*>(workspace), static_cast<cudaStream_t>(stream), 1, true, &tps);
}

int lsv_lora_expand_group_tp(void* const* ys, const int64_t* ldys, int32_t num_tokens, const void* const* const* b_ptrs,
                             const void* plan_dev, const void* plan_host, const void* vimg_base, int32_t* flag,
                             int32_t expect, lsv_stream_t stream) {
  const PlanHeader* h = check_plan(plan_host);
  if (!h || !plan_dev) return fail(LSV_EINVAL, "not a liblsv plan");
  if (!ys || !ldys || !b_ptrs || !vimg_base || !flag) return fail(LSV_EINVAL, "lsv_lora_expand_group_tp: null argument");
  if (num_tokens < h->num_tokens) return fail(LSV_EINVAL, "num_tokens %d is smaller than the plan's %d", num_tokens, h->num_tokens);
  if (h->n_simt_items != 0) return fail(LSV_EUNSUPPORTED, "TP expand needs every segment on the tensor-core tier");
  if (h->num_tokens == 0) return LSV_OK;
  return run_expand(h, 0, h->num_proj, ys, ldys, num_tokens, b_ptrs, static_cast<const int32_t*>(plan_dev), nullptr,
                    static_cast<cudaStream_t>(stream), static_cast<const uint8_t*>(vimg_base), flag, expect);
}

int lsv_lora_shrink_tp_partials(const void* x, int64_t ldx, int32_t num_tokens, int32_t h_in, const void* const* a_ptrs,
                                const void* plan_dev, const void* plan_host, void* workspace, size_t workspace_bytes,
                                int32_t tp, int32_t tp_rank, void* const* xdst, int32_t* const* flags,
                                lsv_stream_t stream) {
  const PlanHeader* h = check_plan(plan_host);
  if (int rc = check_common(h, workspace_bytes, plan_dev, workspace)) return rc;
  if (tp < 1 || tp > kMaxTp || tp_rank < 0 || tp_rank >= tp || !xdst || !flags)
    return fail(LSV_EINVAL, "lsv_lora_shrink_tp_partials: bad tp / rank / destinations");
  if (h->n_simt_items != 0)
    return fail(LSV_EUNSUPPORTED, "TP partial exchange needs every segment on the tensor-core tier (LSV_TIER_TC)");
  if (h->h_in != h_in) return fail(LSV_EINVAL, "h_in %d does not match the plan's %d", h_in, h->h_in);
  if (h->num_tokens == 0) return LSV_OK;
  if (!x || !a_ptrs || !aligned16(x) || ldx % 8 || ldx < h_in) return fail(LSV_EINVAL, "bad x / a_ptrs");
  for (int d = 0; d < tp; ++d)
    if (!xdst[d] || !flags[d]) return fail(LSV_EINVAL, "rank %d: null destination or flag", d);
  if (h->tile_aligned) return fail(LSV_EUNSUPPORTED, "TP partial exchange with a tile-aligned plan");
  TpScatter tps;
  tps.tp = tp; tps.tp_rank = tp_rank; tps.row = 1; tps.fh = h; tps.fplan = static_cast<const int32_t*>(plan_dev);
  tps.vdst = xdst; tps.flags = flags;
  return run_shrink(h, x, ldx, num_tokens, a_ptrs, static_cast<const int32_t*>(plan_dev),
                    static_cast<uint8_t*>(workspace), static_cast<cudaStream_t>(stream), 1, true, &tps);
}

int lsv_lora_expand_group_tp_sum(void* const* ys, const int64_t* ldys, int32_t num_tokens,
                                 const void* const* const* b_ptrs, const void* plan_dev, const void* plan_host,
                                 void* workspace, size_t workspace_bytes, const void* xsum, int32_t tp, int32_t* flag,
                                 lsv_stream_t stream) {
  const PlanHeader* h = check_plan(plan_host);
  if (int rc = check_common(h, workspace_bytes, plan_dev, workspace)) return rc;
  if (!ys || !ldys || !b_ptrs || !xsum || !flag || tp < 1 || tp > kMaxTp)
    return fail(LSV_EINVAL, "lsv_lora_expand_group_tp_sum: bad arguments");
  if (num_tokens < h->num_tokens) return fail(LSV_EINVAL, "num_tokens %d is smaller than the plan's %d", num_tokens, h->num_tokens);
  if (h->n_simt_items != 0) return fail(LSV_EUNSUPPORTED, "TP expand needs every segment on the tensor-core tier");
  if (h->num_tokens == 0) return LSV_OK;
  return run_expand(h, 0, h->num_proj, ys, ldys, num_tokens, b_ptrs, static_cast<const int32_t*>(plan_dev),
                    static_cast<uint8_t*>(workspace), static_cast<cudaStream_t>(stream), nullptr, flag, tp,
                    static_cast<const uint8_t*>(xsum));
}

size_t lsv_lora_forward_workspace(int32_t num_layers, int32_t num_groups, const void* const* plans_host) {
  if (num_layers < 0 || num_groups < 1 || !plans_host) return 0;
  size_t per_layer = 0;
  for (int g = 0; g < num_groups; ++g) {
    const PlanHeader* h = check_plan(plans_host[g]);
    if (!h) return 0;
    per_layer += forward_slice_bytes(h);
  }
  // at least as large as any single plan's workspace, so the standalone entry points can share it
  const PlanHeader* hs[64];
  if (num_groups > 64) return 0;
  for (int g = 0; g < num_groups; ++g) hs[g] = check_plan(plans_host[g]);
  size_t need = kBarHeaderBytes + per_layer * (size_t)num_layers + forward_counter_bytes(num_layers, num_groups, hs);
  for (int g = 0; g < num_groups; ++g) need = std::max(need, (size_t)check_plan(plans_host[g])->ws_bytes);
  return need;
}

int lsv_lora_apply(const void* x, int64_t ldx, void* y, int64_t ldy, int32_t dtype, int32_t num_tokens, int32_t h_in,
                   int32_t h_out, const void* const* a_ptrs, const void* const* b_ptrs, const void* plan_dev,
                   const void* plan_host, void* workspace, size_t workspace_bytes, lsv_stream_t stream) {
  if (dtype != LSV_DTYPE_BF16) return fail(LSV_EUNSUPPORTED, "only LSV_DTYPE_BF16 is supported, got %d", dtype);
  if (int rc = lsv_lora_shrink(x, ldx, num_tokens, h_in, a_ptrs, plan_dev, plan_host, workspace, workspace_bytes,
                               stream))
    return rc;
  return lsv_lora_expand(y, ldy, num_tokens, h_out, b_ptrs, plan_dev, plan_host, workspace, workspace_bytes, stream);
}

int lsv_lora_fused_linear(const void* x, int64_t ldx, int32_t num_tokens, int32_t h_in, const void* const* a_ptrs,
                          const void* const* w, const int64_t* ldw, void* const* ys, const int64_t* ldys,
                          const void* const* const* b_ptrs, const void* plan_dev, const void* plan_host, void* workspace,
                          size_t workspace_bytes, lsv_stream_t stream) {
  const PlanHeader* h = check_plan(plan_host);
  if (int rc = check_common(h, workspace_bytes, plan_dev, workspace)) return rc;
  if (!h->tile_aligned) return fail(LSV_EINVAL, "lsv_lora_fused_linear needs a plan built with LSV_PLAN_TILE_ALIGNED");
  if (h->h_in != h_in) return fail(LSV_EINVAL, "h_in %d does not match the plan's %d", h_in, h->h_in);
  if (num_tokens < h->num_tokens)
    return fail(LSV_EINVAL, "num_tokens %d is smaller than the plan's %d", num_tokens, h->num_tokens);
  if (!x || !aligned16(x) || ldx % 8 || ldx < h_in) return fail(LSV_EINVAL, "x must be 16-byte aligned with ldx %% 8 == 0, ldx >= h_in");
  if (!w || !ldw || !ys || !ldys || !b_ptrs) return fail(LSV_EINVAL, "w / ldw / ys / ldys / b_ptrs must be non-null host arrays");
  const int P = h->num_proj;
  for (int pp = 0; pp < P; ++pp) {
    if (h->h_outs[pp] % kFusedTileN)
      return fail(LSV_EUNSUPPORTED, "member %d: h_out %d is not a multiple of %d", pp, h->h_outs[pp], kFusedTileN);
    if (!w[pp] || !aligned16(w[pp]) || ldw[pp] % 8 || ldw[pp] < h_in)
      return fail(LSV_EINVAL, "member %d: W must be [h_out][h_in] bf16, 16-byte aligned, ldw %% 8 == 0", pp);
    if (!ys[pp] || (reinterpret_cast<uintptr_t>(ys[pp]) & 31) || ldys[pp] % 16 || ldys[pp] < h->h_outs[pp])
      return fail(LSV_EINVAL, "member %d: y must be 32-byte aligned with ldy %% 16 == 0, ldy >= h_out", pp);
    if (!b_ptrs[pp]) return fail(LSV_EINVAL, "member %d: b_ptrs is null", pp);
  }
  if (num_tokens == 0) return LSV_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  // the shrink of the tile-aligned plan (skipped when a_ptrs is NULL: v images already in ws)
  if (a_ptrs && h->num_tokens > 0)
    if (int rc = run_shrink(h, x, ldx, num_tokens, a_ptrs, static_cast<const int32_t*>(plan_dev), ws, st)) return rc;
  if (int rc = ensure_smem_attrs()) return rc;
  FusedParams p{};
  CUtensorMap xm[5];
  if (int rc = get_maps(xm, 0, x, ldx, num_tokens, h_in)) return rc;
  p.xmap = xm[4];   // 64 cols x 128 rows
  int items = 0;
  const int mt = (num_tokens + kTileM - 1) / kTileM;
  for (int pp = 0; pp < P; ++pp) {
    if (int rc = get_maps(&p.wmap[pp], 2, w[pp], ldw[pp], h->h_outs[pp], h_in)) return rc;
    p.b_ptrs[pp] = b_ptrs[pp];
    p.y[pp] = static_cast<__nv_bfloat16*>(ys[pp]);
    p.ldy[pp] = ldys[pp];
    p.ws_vimg[pp] = h->ws_vimg + pp * h->vimg_stride;
    p.n_ntiles[pp] = h->h_outs[pp] / kFusedTileN;
    p.item_base[pp] = items;
    items += mt * p.n_ntiles[pp];
  }
  for (int pp = P; pp <= kMaxProj; ++pp) p.item_base[pp] = items;
  // tokens past the plan's batch (num_tokens > plan tokens) get the base GEMM only: tiles past the
  // plan's last tile see no pieces (their tile_mt range is empty)
  if (mt > (h->num_tokens + kTileM - 1) / kTileM)
    return fail(LSV_EINVAL, "num_tokens %d spans more 128-token tiles than the plan's %d tokens", num_tokens,
                h->num_tokens);
  p.plan = static_cast<const int32_t*>(plan_dev);
  p.ws = ws;
  p.num_tokens = num_tokens; p.h_in = h_in; p.vsplit = h->vsplit; p.n_mtiles = mt;
  p.off_mtiles = h->off_mtiles;
  p.off_tile_mt = h->total_ints - ((h->num_tokens + kTileM - 1) / kTileM + 1);
  p.dbg = g_debug_fused;
  p.trace = g_trace; p.trace_items = g_trace_items;
  LSV_CUDA_CHECK(launch_pdl(fused_linear_kernel, std::min(items, num_sms_cached()), fused_smem_bytes(), st, p, true,
                            kFusedThreads));
  return LSV_OK;
}

// Debug only (not part of include/lsv.h): route per-item globaltimer stamps of the tcgen05
// kernels into `buf` ([148][items][8] uint64); nullptr turns tracing off.
int lsv_debug_set_trace(void* buf, int32_t items_per_cta) {
  g_trace = static_cast<uint64_t*>(buf);
  g_trace_items = buf ? items_per_cta : 0;
  g_tl_launch = 0;
  return LSV_OK;
}

int lsv_slab_alloc(size_t bytes, int32_t device, void** dev_ptr_out) {
  if (!dev_ptr_out || bytes == 0) return fail(LSV_EINVAL, "lsv_slab_alloc: bad arguments");
  int cur = 0;
  LSV_CUDA_CHECK(cudaGetDevice(&cur));
  LSV_CUDA_CHECK(cudaSetDevice(device));
  const cudaError_t e = cudaMalloc(dev_ptr_out, bytes);
  cudaSetDevice(cur);
  if (e != cudaSuccess) return fail(LSV_ECUDA, "cudaMalloc(%zu) on device %d: %s", bytes, device, cudaGetErrorString(e));
  return LSV_OK;
}

int lsv_slab_free(void* dev_ptr) {
  if (!dev_ptr) return LSV_OK;
  LSV_CUDA_CHECK(cudaFree(dev_ptr));
  return LSV_OK;
}

int lsv_plan_vimg_region(const void* plan_host, size_t* offset, size_t* bytes) {
  const PlanHeader* h = check_plan(plan_host);
  if (!h || !offset || !bytes) return fail(LSV_EINVAL, "not a liblsv plan");
  *offset = (size_t)h->ws_vimg;           // every member's v images, contiguous (member p at p * vimg_stride)
  *bytes = (size_t)h->vimg_stride * h->num_proj;
  return LSV_OK;
}

int lsv_vimg_assemble(const void* gathered, size_t region_bytes, int32_t tp, const void* shard_plan_dev,
                      const void* shard_plan_host, const void* full_plan_dev, const void* full_plan_host,
                      void* full_workspace, lsv_stream_t stream) {
  const PlanHeader* hs = check_plan(shard_plan_host);
  const PlanHeader* hf = check_plan(full_plan_host);
  if (!hs || !hf || !shard_plan_dev || !full_plan_dev) return fail(LSV_EINVAL, "not a liblsv plan");
  if (hs->n_mtiles != hf->n_mtiles || hs->num_tokens != hf->num_tokens)
    return fail(LSV_EINVAL, "shard and full plans index different tiles (%d vs %d)", hs->n_mtiles, hf->n_mtiles);
  if (tp < 1 || !gathered || !full_workspace) return fail(LSV_EINVAL, "bad arguments");
  if (hs->num_proj != hf->num_proj) return fail(LSV_EINVAL, "shard and full plans have different members");
  if (hs->vsplit != hf->vsplit) return fail(LSV_EINVAL, "shard and full plans differ in v precision (LSV_PLAN_V_BF16)");
  if (hs->n_simt_items != 0 || hf->n_simt_items != 0)
    return fail(LSV_EUNSUPPORTED, "TP assembly needs every segment on the tensor-core tier (plan with LSV_TIER_TC)");
  if (hf->n_mtiles == 0) return LSV_OK;
  const int32_t* sp = static_cast<const int32_t*>(shard_plan_dev);
  const int32_t* fp = static_cast<const int32_t*>(full_plan_dev);
  for (int pp = 0; pp < hf->num_proj; ++pp) {   // member pp: its shard images and its full-rank images
    vimg_assemble_kernel<<<hf->n_mtiles, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint8_t*>(gathered) + (size_t)pp * hs->vimg_stride, region_bytes, tp, sp, hs->off_mtiles, 0,
        fp, hf->off_mtiles, static_cast<uint8_t*>(full_workspace), hf->ws_vimg + pp * hf->vimg_stride, hf->vsplit);
    LSV_CUDA_CHECK(cudaGetLastError());
  }
  return LSV_OK;
}

int lsv_copy_blocks(int32_t n, const void* const* src, void* const* dst, const size_t* bytes, lsv_stream_t stream) {
  if (n < 0 || (n > 0 && (!src || !dst || !bytes))) return fail(LSV_EINVAL, "lsv_copy_blocks: bad arguments");
  for (int i = 0; i < n; ++i) {
    if (bytes[i] == 0) continue;
    if (!src[i] || !dst[i]) return fail(LSV_EINVAL, "lsv_copy_blocks: null block %d", i);
    LSV_CUDA_CHECK(cudaMemcpyAsync(dst[i], src[i], bytes[i], cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream)));
  }
  return LSV_OK;
}

int lsv_ipc_get_handle(void* dev_ptr, void* handle64_out) {
  if (!dev_ptr || !handle64_out) return fail(LSV_EINVAL, "null pointer");
  cudaIpcMemHandle_t h;
  LSV_CUDA_CHECK(cudaIpcGetMemHandle(&h, dev_ptr));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(handle64_out, &h, sizeof(h));
  return LSV_OK;
}

int lsv_ipc_open_handle(const void* handle64, int32_t device, void** dev_ptr_out) {
  if (!handle64 || !dev_ptr_out) return fail(LSV_EINVAL, "null pointer");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  int cur = 0;
  LSV_CUDA_CHECK(cudaGetDevice(&cur));
  LSV_CUDA_CHECK(cudaSetDevice(device));
  const cudaError_t e = cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess);
  cudaSetDevice(cur);
  if (e != cudaSuccess) return fail(LSV_ECUDA, "cudaIpcOpenMemHandle on device %d: %s", device, cudaGetErrorString(e));
  return LSV_OK;
}

int lsv_ipc_close_handle(void* dev_ptr) {
  if (!dev_ptr) return fail(LSV_EINVAL, "null pointer");
  LSV_CUDA_CHECK(cudaIpcCloseMemHandle(dev_ptr));
  return LSV_OK;
}

int lsv_enable_peer(int32_t dev, int32_t peer) {
  if (dev == peer) return LSV_OK;
  int can = 0;
  LSV_CUDA_CHECK(cudaDeviceCanAccessPeer(&can, dev, peer));
  if (!can) return fail(LSV_EUNSUPPORTED, "device %d cannot access peer %d", dev, peer);
  int cur = 0;
  LSV_CUDA_CHECK(cudaGetDevice(&cur));
  LSV_CUDA_CHECK(cudaSetDevice(dev));
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) { cudaGetLastError(); e = cudaSuccess; }
  cudaSetDevice(cur);
  if (e != cudaSuccess) return fail(LSV_ECUDA, "cudaDeviceEnablePeerAccess(%d -> %d): %s", dev, peer, cudaGetErrorString(e));
  return LSV_OK;
}

}  // extern "C"
