/*
 * lsv.h — C ABI of liblsv, the B200 (sm_100a) mixed-rank LoRA delta path.
 *
 * What it replaces.  The reference (LoRAServe simulator, /root/reference/pkg/src/lorasim)
 * has no tensor arithmetic: "apply this co-batched prefill's LoRA deltas" exists only as
 * the cost callback
 *     costmodel.prefill_time(prompt_lengths, ranks, params, resident_max_rank)
 *         /root/reference/pkg/src/lorasim/costmodel.py:83-105
 *     costmodel.decode_iter_time(context_lengths, ranks, params)      costmodel.py:108-123
 *     costmodel.fetch_latency(size_bytes, "remote_rdma", params)      costmodel.py:129-143
 * called by schedule_server (simengine.py:139,146) on the batch it formed FIFO under the
 * token budget (simengine.py:96-152).  The entry points below are what that callback's
 * batch actually needs done on a GPU: for every segment s (the tokens of one adapter,
 * contiguous after a stable sort by adapter slot)
 *
 *     y[t, :] += (x[t, :] · A_s^T) · B_s^T            t in [seg_indptr[s], seg_indptr[s+1])
 *
 * with A_s = lora_A [rank_s, h_in] and B_s = lora_B [h_out, rank_s] (PEFT layout), bf16
 * operands, fp32 accumulation, bf16 y updated in place.  Each segment pays for its own
 * rank (the B200 path deliberately does NOT reproduce costmodel.py:104's "whole batch pays
 * the max rank").  A_s/B_s pointers may be local HBM or NVLink peer addresses: the
 * reference's remote fetch (pool.py:101-132 plan_fetch → fetch_remote, priced by
 * fetch_latency(..., "remote_rdma")) becomes a peer load inside the kernel.
 *
 * Conventions (mirroring the reference's error behaviour, costmodel.py:95-103, pool.py:75-80):
 *   - every call returns LSV_OK (0) or an error code; lsv_last_error() returns a
 *     thread-local message for the last nonzero return;
 *   - LSV_EINVAL / LSV_EWORKSPACE map to Python ValueError, LSV_ECUDA / LSV_EUNSUPPORTED
 *     to RuntimeError in the shim (paper_2511_22880_b200/native.py);
 *   - all device work is asynchronous on the caller's stream; the library never
 *     allocates device memory in lsv_lora_apply.  Its host-side mutable state is limited to
 *     caches whose contents are pure functions of their keys: cached device attributes and
 *     driver entry points, a process-wide tensor-map cache keyed by (pointer, row stride,
 *     rows, cols, box kind) under a mutex, and a per-thread cache of the last plan built
 *     (keyed by every planner input, so lsv_plan_size_* followed by lsv_plan_build_* with the
 *     same inputs plans once).  None of them changes a result.
 */
#ifndef LSV_H_
#define LSV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LSV_ABI_VERSION 3

#define LSV_OK 0
#define LSV_EINVAL 1
#define LSV_ECUDA 2
#define LSV_EUNSUPPORTED 3
#define LSV_EWORKSPACE 4

#define LSV_DTYPE_BF16 0

/* Tier policy for lsv_plan_build: AUTO chooses per segment (SIMT warp-shuffle tier for
 * short segments, tcgen05 tier otherwise); the forced policies exist for tests/benchmarks. */
#define LSV_TIER_AUTO 0
#define LSV_TIER_SIMT 1
#define LSV_TIER_TC 2
/* Plan flag, OR-ed into tier_policy: the tensor-core tier's intermediate v = x·A^T is kept as a
 * single bf16 image instead of the default bf16 (hi, lo) pair.  The pair (v_hi = bf16(v), v_lo =
 * bf16(v - v_hi)) carries v to ~16 significant bits through the expand's two bf16 MMAs, so the
 * delta matches the fp32-v SGMV result up to the final bf16 rounding of y; the single image rounds
 * v to bf16 (8 bits) first, costing less workspace and expand ring bytes. */
#define LSV_PLAN_V_BF16 0x100
/* Plan flag: tile-aligned v images for lsv_lora_fused_linear (the base projection GEMM with the
 * LoRA expand accumulated in its TMEM tile).  Every segment is split at the batch's 128-token tile
 * boundaries and each piece's v image spans its whole tile (zero rows outside the piece), so an
 * M=128 MMA adds v·B into exactly the piece's rows.  Tensor-core tier only. */
#define LSV_PLAN_TILE_ALIGNED 0x200
/* Plan flag: launch at most n CTAs (1..255) per kernel instead of one per SM, so two plans can run
 * side by side on disjoint SM sets (LSV_SEG_SKIP partitions a batch between them). */
#define LSV_PLAN_SMS(n) (((n) & 0xff) << 16)

typedef void* lsv_stream_t; /* a cudaStream_t */

/* ABI version (LSV_ABI_VERSION). */
int lsv_version(void);

/* Message for the last nonzero return on this thread ("" if none). */
const char* lsv_last_error(void);

/* ---- adapter slab format -------------------------------------------------------------
 * Replaces the reference's "adapter is GPU-resident in a slot" notion
 * (pool.py:88-99 touch_gpu / is_gpu_resident; gpu_slots config.py:29): an adapter in a GPU
 * slot is a pair of tiled buffers in HBM, packed once at load time so the kernels can
 * move them with single bulk copies. */
size_t lsv_adapter_a_bytes(int32_t rank, int32_t h_in);
size_t lsv_adapter_b_bytes(int32_t rank, int32_t h_out);

/* Slab memory: one cudaMalloc on `device` (its base is what lsv_ipc_get_handle exports). */
int lsv_slab_alloc(size_t bytes, int32_t device, void** dev_ptr_out);
int lsv_slab_free(void* dev_ptr);

/* Pack PEFT-layout device tensors lora_A [rank][h_in] and lora_B [h_out][rank] (bf16,
 * row-major, contiguous) into the tiled slab buffers a_tiled / b_tiled (device).
 * rank must be a multiple of 8 in [8, 256]; h_in, h_out multiples of 128.  Passing null for
 * both pointers of one half packs only the other (tensor-parallel shards keep A and B at
 * different ranks). */
int lsv_pack_adapter(const void* lora_a, const void* lora_b, int32_t rank, int32_t h_in,
                     int32_t h_out, void* a_tiled, void* b_tiled, lsv_stream_t stream);

/* Inverse of lsv_pack_adapter (used by tests and by peer copy-on-first-use checks). */
int lsv_unpack_adapter(const void* a_tiled, const void* b_tiled, int32_t rank, int32_t h_in,
                       int32_t h_out, void* lora_a, void* lora_b, lsv_stream_t stream);

/* Input groups.  Projections that read the same activation (q/k/v of attention, gate/up of the
 * MLP; all with the same h_in and, for one adapter, the same rank) keep their A matrices in one
 * group tile of num_proj*rank rows per 64-column chunk, so one shrink reads x once for all of them
 * (lsv_plan_build_group).  Member `proj` occupies rows [proj*rank, (proj+1)*rank).  B stays per
 * projection (lsv_pack_adapter with lora_a = a_tiled = NULL).  num_proj = 1 is exactly the
 * lsv_pack_adapter A layout. */
size_t lsv_adapter_a_group_bytes(int32_t num_proj, int32_t rank, int32_t h_in);
int lsv_pack_adapter_group(const void* lora_a, int32_t num_proj, int32_t proj, int32_t rank,
                           int32_t h_in, void* a_group_tiled, lsv_stream_t stream);
int lsv_unpack_adapter_group(const void* a_group_tiled, int32_t num_proj, int32_t proj, int32_t rank,
                             int32_t h_in, void* lora_a, lsv_stream_t stream);

/* ---- plan ------------------------------------------------------------------------------
 * Host-side work planning for one (batch, projection shape).  seg_indptr [S+1] and
 * seg_rank [S] are HOST arrays (the segment indexer's output); seg_indptr[0] must be 0,
 * non-decreasing, seg_rank[s] in {8,16,...,256}.  The plan is a self-describing int32
 * blob: segment table, per-segment tier, the LPT-ordered shrink and expand work lists
 * and the workspace layout.  Copy it to the device once and reuse it for every layer
 * and projection of the same shape. */
int lsv_plan_size(int32_t num_segments, const int32_t* seg_indptr, const int32_t* seg_rank,
                  int32_t h_in, int32_t h_out, int32_t tier_policy, size_t* plan_bytes,
                  size_t* workspace_bytes);

int lsv_plan_build(int32_t num_segments, const int32_t* seg_indptr, const int32_t* seg_rank,
                   int32_t h_in, int32_t h_out, int32_t tier_policy, void* plan_host,
                   size_t plan_bytes);

/* Plan for an input group: num_proj projections with output widths h_outs[0..num_proj) that share
 * x.  lsv_lora_shrink with this plan (a_ptrs = the segments' group A tiles) writes the v images of
 * every member; lsv_lora_expand_proj(proj) then applies member proj.  lsv_plan_build is the
 * num_proj = 1 case. */
int lsv_plan_size_group(int32_t num_segments, const int32_t* seg_indptr, const int32_t* seg_rank,
                        int32_t h_in, int32_t num_proj, const int32_t* h_outs, int32_t tier_policy,
                        size_t* plan_bytes, size_t* workspace_bytes);
int lsv_plan_build_group(int32_t num_segments, const int32_t* seg_indptr, const int32_t* seg_rank,
                         int32_t h_in, int32_t num_proj, const int32_t* h_outs, int32_t tier_policy,
                         void* plan_host, size_t plan_bytes);

/* Group plan with per-segment flags (HOST array [S], or NULL = lsv_plan_*_group).  LSV_SEG_REMOTE:
 * the segment's adapter lives in an NVLink peer's slab (the reference's fetch_remote,
 * pool.py:101-132); the planner weighs its A/B bytes by the HBM/NVLink bandwidth ratio and
 * interleaves remote and local work in every CTA's list so peer reads overlap local HBM traffic. */
#define LSV_SEG_REMOTE 1
/* LSV_SEG_SKIP: the segment keeps its token range but gets no work in this plan (two plans over one
 * batch: e.g. local segments on most SMs and peer-owned ones on a few, run on two streams). */
#define LSV_SEG_SKIP 2
/* LSV_SEG_NOSHRINK: the segment keeps its m-tiles (so the plan's tile list matches a full-rank plan of
 * the same batch) but gets no shrink work: a tensor-parallel rank that holds none of the adapter's
 * rows under balanced sharding (LSV_TP_ROUND_ROBIN).  Pass any valid rank for it. */
#define LSV_SEG_NOSHRINK 4
int lsv_plan_size_group_ex(int32_t num_segments, const int32_t* seg_indptr, const int32_t* seg_rank,
                           const int32_t* seg_flags, int32_t h_in, int32_t num_proj, const int32_t* h_outs,
                           int32_t tier_policy, size_t* plan_bytes, size_t* workspace_bytes);
int lsv_plan_build_group_ex(int32_t num_segments, const int32_t* seg_indptr, const int32_t* seg_rank,
                            const int32_t* seg_flags, int32_t h_in, int32_t num_proj, const int32_t* h_outs,
                            int32_t tier_policy, void* plan_host, size_t plan_bytes);

/* Fill out[0..7] from a host plan: {num_segments, num_tokens, h_in, h_out,
 * n_simt_segments, n_tc_mtiles, n_shrink_items, n_expand_items}. */
int lsv_plan_summary(const void* plan_host, int32_t* out8);

/* ---- apply -----------------------------------------------------------------------------
 * y[t,:] += (x[t,:]·A_s^T)·B_s^T for every segment of the plan.
 *   x  : [num_tokens][h_in] bf16, row stride ldx elements (device, 16-byte aligned rows)
 *   y  : [num_tokens][h_out] bf16, row stride ldy elements (device), updated in place
 *   a_ptrs, b_ptrs : device arrays [num_segments] of device pointers to the segment's
 *        tiled A/B (lsv_pack_adapter format); local or NVLink-peer addresses
 *   plan_dev / plan_host : the same plan blob, on device and on host
 *   workspace : device scratch of at least the planned workspace_bytes, zero-filled once
 *        at allocation (the kernels leave their counters zeroed again on exit). */
int lsv_lora_apply(const void* x, int64_t ldx, void* y, int64_t ldy, int32_t dtype,
                   int32_t num_tokens, int32_t h_in, int32_t h_out, const void* const* a_ptrs,
                   const void* const* b_ptrs, const void* plan_dev, const void* plan_host,
                   void* workspace, size_t workspace_bytes, lsv_stream_t stream);

/* Shrink only: writes the per-segment bf16 intermediate v (x·A^T) into the workspace
 * v-image area.  Together with lsv_lora_expand this splits lsv_lora_apply around an
 * exchange (tensor-parallel all-gather of v). */
int lsv_lora_shrink(const void* x, int64_t ldx, int32_t num_tokens, int32_t h_in,
                    const void* const* a_ptrs, const void* plan_dev, const void* plan_host,
                    void* workspace, size_t workspace_bytes, lsv_stream_t stream);

int lsv_lora_expand(void* y, int64_t ldy, int32_t num_tokens, int32_t h_out,
                    const void* const* b_ptrs, const void* plan_dev, const void* plan_host,
                    void* workspace, size_t workspace_bytes, lsv_stream_t stream);

/* Expand of every member of a group plan in one launch (one LPT work list over all members'
 * items): ys / ldys / b_ptrs are HOST arrays of num_proj entries (member i's y, its row stride and
 * its device table of per-segment B pointers). */
int lsv_lora_expand_group(void* const* ys, const int64_t* ldys, int32_t num_tokens,
                          const void* const* const* b_ptrs, const void* plan_dev, const void* plan_host,
                          void* workspace, size_t workspace_bytes, lsv_stream_t stream);

/* A whole model step for one batch: for every layer l and input group g, the group's fused shrink
 * and its expand.  plans_* [num_groups] (group plans of the same batch), xs/ldxs
 * [num_layers*num_groups], ys/ldys [num_layers*num_projections] (host arrays of device pointers /
 * row strides; projections numbered group by group), a_ptrs [num_layers*num_groups][S] and b_ptrs
 * [num_layers*num_projections][S] device tables.  Equivalent to the per-group calls (bit-identical
 * results), with no per-launch host round trips.  The workspace holds one slice per (layer, group)
 * plus per-m-tile counters (lsv_lora_forward_workspace bytes, zero-filled once; the call zero-fills
 * the counters itself, ordered on `stream`).  How the work is launched:
 *   - an overlap-free call (below) whose groups are all tensor-core tier: one launch per layer
 *     (every group's shrink and expand in one persistent kernel, <= 4 groups); with more than one
 *     layer its CTAs take expand items from a per-(layer, group) cursor in the counter area
 *     (dynamic dispatch; the result bits do not depend on which CTA computes an item);
 *   - otherwise each tensor-core group is one launch (shrink + expand); SIMT-tier groups are a
 *     shrink and an expand launch;
 *   - an overlap-free call without layer launches issues group g of layer l on one of 4 streams
 *     ((l * num_groups + g) % 4, forked from and joined back into `stream` with events), so
 *     independent groups (decode batches) run concurrently.  Work queued on `stream` after the call
 *     is ordered after all of it; a graph capture of `stream` records the fork/join.
 * Tensor-core launches (group / layer kernels, the standalone shrink's split-K grid barrier) wait
 * on other CTAs of their own grid, so their grid (at most one CTA per SM) must become co-resident:
 * kernels of other streams may delay them but must not wait on them.  Two lsv calls on different
 * streams of one GPU therefore need disjoint SM budgets (LSV_PLAN_SMS in the plans), as
 * SplitStep does. */
int lsv_lora_forward(int32_t num_layers, int32_t num_groups, const void* const* plans_dev,
                     const void* const* plans_host, const void* const* xs, const int64_t* ldxs,
                     void* const* ys, const int64_t* ldys, const void* a_ptrs, const void* b_ptrs,
                     int32_t num_tokens, void* workspace, size_t workspace_bytes, lsv_stream_t stream);

/* lsv_lora_forward with flags.  By default the call is overlap-free: groups run concurrently or
 * reordered (a group's shrink before the previous group's expand), which is valid only when every
 * y range of the call is disjoint from every other y range and from every x range; the library
 * checks this and falls back to full serialisation otherwise.  LSV_FWD_SERIAL forces every group
 * to wait for its predecessor (what a model whose next input depends on the previous output gets). */
#define LSV_FWD_SERIAL 1
int lsv_lora_forward_ex(int32_t num_layers, int32_t num_groups, const void* const* plans_dev,
                        const void* const* plans_host, const void* const* xs, const int64_t* ldxs,
                        void* const* ys, const int64_t* ldys, const void* a_ptrs, const void* b_ptrs,
                        int32_t num_tokens, void* workspace, size_t workspace_bytes, int32_t flags,
                        lsv_stream_t stream);

/* Workspace bytes lsv_lora_forward needs for these group plans (0 on bad input). */
size_t lsv_lora_forward_workspace(int32_t num_layers, int32_t num_groups, const void* const* plans_host);

/* Expand of member `proj` of a group plan (lsv_lora_expand is proj = 0). */
int lsv_lora_expand_proj(void* y, int64_t ldy, int32_t num_tokens, int32_t h_out, int32_t proj,
                         const void* const* b_ptrs, const void* plan_dev, const void* plan_host,
                         void* workspace, size_t workspace_bytes, lsv_stream_t stream);

/* ---- base projection GEMM with the LoRA delta fused -------------------
 * One LoRA linear layer for an input group, y_p = x · W_p^T + delta_p for every member p, with the
 * delta accumulated into the base GEMM's TMEM tile (no y read-modify-write): the prices
 * costmodel.prefill_time (costmodel.py:104-105) puts on "base GEMM + adapter" as one batch cost.
 *   x      : [num_tokens][h_in] bf16 (device), row stride ldx
 *   a_ptrs : device table [S] of the segments' group A tiles; runs the shrink of the plan first.
 *            NULL: the v images are already in the workspace (a previous lsv_lora_shrink).
 *   w, ldw : HOST arrays [num_proj]: base weight W_p [h_out_p][h_in] bf16 (nn.Linear layout, device)
 *   ys     : HOST array [num_proj] of outputs [num_tokens][h_out_p] bf16, written (not accumulated);
 *            32-byte aligned rows (ldy % 16 == 0)
 *   b_ptrs : HOST array [num_proj] of device tables [S] of B tile pointers
 * The plan must be built with LSV_PLAN_TILE_ALIGNED; every h_out must be a multiple of 256. */
int lsv_lora_fused_linear(const void* x, int64_t ldx, int32_t num_tokens, int32_t h_in, const void* const* a_ptrs,
                          const void* const* w, const int64_t* ldw, void* const* ys, const int64_t* ldys,
                          const void* const* const* b_ptrs, const void* plan_dev, const void* plan_host,
                          void* workspace, size_t workspace_bytes, lsv_stream_t stream);

/* ---- tensor parallelism -------------------------------------------------------------------
 * Column-parallel projections shard each adapter's rank over the TP group: rank t's shrink
 * (plan built with the shard ranks) writes v images of K = rank/tp; after an NCCL all-gather of
 * those workspace images into `gathered` ([tp][shard_region_bytes]), this rebuilds the full-rank
 * v images the expand (plan built with the full ranks) reads.  Both plans must index the same
 * segments.  region_bytes = the shard plan's workspace v-image region size
 * (lsv_plan_vimg_region). */
int lsv_vimg_assemble(const void* gathered, size_t region_bytes, int32_t tp, const void* shard_plan_dev,
                      const void* shard_plan_host, const void* full_plan_dev, const void* full_plan_host,
                      void* full_workspace, lsv_stream_t stream);

/* Fused compute + collective for column-parallel groups (the NCCL all-gather + assembly in one
 * kernel, over NVLink): the shrink of this rank's rank-shard plan writes every (token, member,
 * 8-column) unit of its v straight into column tp_rank*rs + k of the member's full-rank image on
 * every rank (vfull_dst[d]: rank d's image base for this layer/group, device addresses mapped with
 * lsv_ipc_open_handle; member p at p * full vimg_stride, m-tile at the full plan's offsets), then
 * its last CTA adds 1 to flags[d] on every rank (system-scope release).  full_plan: the full-rank
 * plan (same segments and members).  Tensor-core tier only (LSV_TIER_TC plans). */
/* OR-ed into lsv_lora_shrink_tp_scatter's tp: balanced shards.  Rank t holds the 8-row groups g of
 * each adapter's A with g % tp == t (possibly none: LSV_SEG_NOSHRINK), instead of a contiguous
 * 1/tp of the rank padded to a multiple of 8·tp; its local column k lands at full column
 * 8·(t + tp·(k/8)) + k%8.  The expand's B keeps the true rank. */
#define LSV_TP_ROUND_ROBIN 0x100
int lsv_lora_shrink_tp_scatter(const void* x, int64_t ldx, int32_t num_tokens, int32_t h_in,
                               const void* const* a_ptrs, const void* plan_dev, const void* plan_host,
                               void* workspace, size_t workspace_bytes, int32_t tp, int32_t tp_rank,
                               void* const* vfull_dst, const void* full_plan_dev,
                               const void* full_plan_host, int32_t* const* flags, lsv_stream_t stream);

/* The matching expand: waits until flag[0] == expect (every rank's shard has landed in vimg_base),
 * re-arms flag[0..1] for the next use, and expands every member from vimg_base (member p's images
 * at p * vimg_stride of plan). */
int lsv_lora_expand_group_tp(void* const* ys, const int64_t* ldys, int32_t num_tokens,
                             const void* const* const* b_ptrs, const void* plan_dev,
                             const void* plan_host, const void* vimg_base, int32_t* flag,
                             int32_t expect, lsv_stream_t stream);

/* Fused compute + all-reduce for row-parallel groups (o, down): the shrink of this rank's h_in
 * slice writes its fp32 partial v into slot tp_rank of every rank's exchange buffer (xdst[d]:
 * rank d's buffer for this layer/group, tp slots of 2 * vimg_stride * num_proj bytes; member p's
 * m-tile at 2 * (p * vimg_stride + vimg_off) as fp32 [rows16][kpad]) over NVLink, then signals
 * flags[d] like lsv_lora_shrink_tp_scatter. */
int lsv_lora_shrink_tp_partials(const void* x, int64_t ldx, int32_t num_tokens, int32_t h_in,
                                const void* const* a_ptrs, const void* plan_dev, const void* plan_host,
                                void* workspace, size_t workspace_bytes, int32_t tp, int32_t tp_rank,
                                void* const* xdst, int32_t* const* flags, lsv_stream_t stream);

/* The matching expand: waits for flag[0] == tp, sums the tp partial slots of xsum in rank order
 * (identical bits on every rank) into the workspace's bf16 v images, then expands every member. */
int lsv_lora_expand_group_tp_sum(void* const* ys, const int64_t* ldys, int32_t num_tokens,
                                 const void* const* const* b_ptrs, const void* plan_dev,
                                 const void* plan_host, void* workspace, size_t workspace_bytes,
                                 const void* xsum, int32_t tp, int32_t* flag, lsv_stream_t stream);

/* Byte offset and size of a plan's v-image region inside its workspace (what TP exchanges): every
 * member's images, member p at p * (size / num_proj).  lsv_vimg_assemble handles group plans
 * member by member (both plans must have the same members). */
int lsv_plan_vimg_region(const void* plan_host, size_t* offset, size_t* bytes);

/* ---- NVLink peers ----------------------------------------------------------------------
 * Replaces the reference's GPUDirect-RDMA remote fetch (pool.py:101-132, costmodel.py:139-140)
 * for single-process multi-GPU use: enable direct peer loads from `peer`'s HBM on `dev`.
 * Returns LSV_EUNSUPPORTED if the pair cannot access each other. */
int lsv_enable_peer(int32_t dev, int32_t peer);

/* Cross-process form of the same: export a device allocation (a cudaMalloc base pointer) as a
 * 64-byte CUDA IPC handle; open a peer process's handle in `device`'s context (mapping the
 * peer GPU's HBM into this GPU's address space for direct NVLink loads); close it again. */
int lsv_ipc_get_handle(void* dev_ptr, void* handle64_out);
int lsv_ipc_open_handle(const void* handle64, int32_t device, void** dev_ptr_out);
int lsv_ipc_close_handle(void* dev_ptr);

/* Fetch: n device-to-device block copies (src[i] -> dst[i], bytes[i]; host arrays of device
 * addresses) on `stream`, executed by the copy engines (NVLink for peer addresses), leaving the
 * SMs to the kernels.  The B200 form of the reference's fetch_remote (pool.py:101-132): stage a
 * peer-owned adapter's next-layer tiles in local HBM while the current layer computes. */
int lsv_copy_blocks(int32_t n, const void* const* src, void* const* dst, const size_t* bytes,
                    lsv_stream_t stream);

/* Build flags of this library: LSV_BUILD_DEVICE_CHECKS if compiled with device-side bounds checks
 * (liblsv_checked.so, the test-only build whose kernels trap on out-of-range records). */
#define LSV_BUILD_DEVICE_CHECKS 1
int lsv_build_info(void);

/* Number of SMs the planner assumes (queried from device 0 once; 148 on B200). */
int lsv_num_sms(void);

/* Development hook (tools/trace_*.py): kernels launched afterwards from the calling thread write
 * per-CTA / per-item clock stamps into buf ([grid][items_per_cta][16] uint64, device memory);
 * buf = NULL turns it off.  Not needed for any computation. */
int lsv_debug_set_trace(void* buf, int32_t items_per_cta);

#ifdef __cplusplus
}
#endif

#endif /* LSV_H_ */
