// lsv_common.cuh — sm_100a PTX wrappers and the HBM tile layouts shared by all liblsv kernels.
//
// Layouts (all bf16, fixed at adapter-load time by lsv_pack_adapter):
//
//  A tiled  (lora_A [rank][h_in]; operand B of the tcgen05 shrink, K-major, SWIZZLE_128B)
//      [h_in/64 chunks][rank rows][64 elems]; each (chunk, 8-row) block is one 1024-byte
//      swizzle atom: 16-byte unit u of row k lives at unit u ^ (k & 7).  Any run of
//      consecutive chunks is contiguous, so one stage of the shrink is one bulk copy.
//
//  B tiled  (lora_B [h_out][rank]; operand B of the tcgen05 expand, MN-major SWIZZLE_128B)
//      per tw-wide h_out tile (tw = 256, or 128 when h_out is not a multiple of 256):
//      [kp/8 k-groups][tw/64 x 64 h_out][8 k][64 h_out] with kp = rank padded to 16 (zero rows);
//      a tile is tw*kp*2 contiguous bytes, one bulk copy.
//
//  v image  (x·A^T of one 128-token tile, operand A of the expand, K-major, SWIZZLE_32/64/128B
//      by padded rank kp = round_up(max(rank,16),16)); k past the rank is zero so a rank-8
//      adapter feeds a K=16 MMA.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

namespace lsv {

constexpr int kNumSmsDefault = 148;
constexpr int kChunk = 64;          // elements per 128-byte swizzle row
constexpr int kTileM = 128;         // tokens per tcgen05 m-tile
constexpr int kSimtMaxTok = 8;      // tokens per SIMT item
#ifndef LSV_SIMT_SMALL_TOK
#define LSV_SIMT_SMALL_TOK 2
#endif
constexpr int kSimtSmallTok = LSV_SIMT_SMALL_TOK;    // SIMT items up to this many tokens use the small expand accumulator

__host__ __device__ __forceinline__ int round_up(int x, int m) { return (x + m - 1) / m * m; }

// Device-side bounds checks (the checked build, LSV_DEVICE_CHECKS=1: liblsv_checked.so, run by
// tools/gpu_checked.sh over the GPU test suite).  compute-sanitizer is not available on the GPU
// pool, so every kernel asserts its own invariants instead: plan records inside the batch, ring
// allocations inside shared memory, workspace writes inside the planned workspace.  A failed check
// prints the condition and traps (the launch fails loudly).  No-ops in the production build.
#ifndef LSV_DEVICE_CHECKS
#define LSV_DEVICE_CHECKS 0
#endif
#if LSV_DEVICE_CHECKS
#define LSV_DCHECK(cond)                                                                              \
  do {                                                                                                \
    if (!(cond)) {                                                                                    \
      printf("lsv device check failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                                      \
      __trap();                                                                                       \
    }                                                                                                 \
  } while (0)
#else
#define LSV_DCHECK(cond) do { } while (0)
#endif

// ---- layout address functions (byte offsets) -------------------------------------------
// Hardware swizzle of a byte offset inside a region aligned to the pattern period
// (SWIZZLE_32B/64B/128B = rows of 32/64/128 bytes): 16-byte unit bits [4..6] ^= bits [7..9].
__host__ __device__ __forceinline__ uint32_t swz(uint32_t off, int row_bytes) {
  const uint32_t mask = row_bytes == 128 ? 0x70u : row_bytes == 64 ? 0x30u : row_bytes == 32 ? 0x10u : 0u;
  return off ^ ((off >> 3) & mask);
}
// K padded for the 16-wide MMA K step (rank 8 -> 16, 24 -> 32, ...)
__host__ __device__ __forceinline__ int kpad(int rank) { return round_up(rank < 16 ? 16 : rank, 16); }
// v-image / K-major operand row width: the widest swizzle whose element run divides kp
__host__ __device__ __forceinline__ int kmajor_row_bytes(int kp) { return kp % 64 == 0 ? 128 : kp % 32 == 0 ? 64 : 32; }
__host__ __device__ __forceinline__ uint32_t umma_layout(int row_bytes) {
  return row_bytes == 128 ? 2u : row_bytes == 64 ? 4u : 6u;  // SWIZZLE_128B / 64B / 32B
}

// A tiled (shrink B operand, K-major SW128): [h_in/64][rank][64]
// Group form: the A tiles of an input group's projections (same h_in, same rank) interleaved per
// chunk, [h_in/64][grows = nproj*rank rows][64]; member p's rows start at p*rank (a multiple of 8,
// so every member keeps the swizzle phase it has alone).  nproj = 1 is the single-adapter layout.
__host__ __device__ __forceinline__ size_t a_tiled_off_g(int row, int i, int grows) {
  const int c = i >> 6, e = i & 63;
  return (size_t)c * grows * 128 + (size_t)row * 128 + ((((e >> 3) ^ (row & 7)) << 4) | ((e & 7) << 1));
}
__host__ __device__ __forceinline__ size_t a_tiled_off(int k, int i, int rank) { return a_tiled_off_g(k, i, rank); }
// B tiled (expand B operand, MN-major SW128): per tw-wide h_out tile (tw = b_tile_width(h_out))
// [kp/8 k-groups][tw/64 blocks of 64 h_out][8 k rows][64 h_out], 1024-byte swizzle atoms;
// kp = kpad(rank) rows, the rows past the rank are zero so a K=16 MMA step never reads stale data.
__host__ __device__ __forceinline__ int b_tile_width(int h_out) { return h_out % 256 == 0 ? 256 : 128; }
__host__ __device__ __forceinline__ size_t b_tiled_off(int j, int k, int rank, int tw) {
  const int jt = j / tw, jj = j % tw;
  const uint32_t in_atom = (uint32_t)((k & 7) * 128 + (jj & 63) * 2);
  return (size_t)jt * kpad(rank) * tw * 2 + (size_t)(k >> 3) * (tw / 64) * 1024 + (jj >> 6) * 1024 +
         swz(in_atom, 128);
}
// v image (expand A operand, K-major, swizzle by kmajor_row_bytes(kp)): rows = tokens (rows_pad =
// ntok rounded to 16), K = kp; K split in chunks of row_bytes/2 elements laid out chunk-major.
__host__ __device__ __forceinline__ uint32_t vimg_off(int t, int k, int kp, int rows_pad) {
  const int S = kmajor_row_bytes(kp), ck = S / 2;
  const uint32_t off = (uint32_t)((k / ck) * rows_pad * S + t * S + (k % ck) * 2);
  return swz(off, S);
}

// Bytes of one bf16 v image of an m-tile (rows padded to 16, K = kp), 1024-aligned.  With split v
// (PlanHeader::vsplit) the m-tile's region holds the hi image, then the lo image at +vimg_bytes.
__host__ __device__ __forceinline__ uint32_t vimg_bytes(int ntok, int kp) {
  return (uint32_t)round_up(round_up(ntok, 16) * kp * 2, 1024);
}
// Expand item tile width: ranks above 128 use 128-wide h_out tiles (a 256-wide layout tile's half)
// so that the item's B, v and y bytes fit the expand ring.
__host__ __device__ __forceinline__ int expand_item_tw(int rank, int layout_tw) {
  return rank > 128 ? 128 : layout_tw;
}
// m-tile height of a segment of this rank: 64 tokens above rank 128 (bounds an item's v image), else 128.
__host__ __device__ __forceinline__ int mtile_rows(int rank) { return rank > 128 ? 64 : 128; }

// ---- small device helpers ----------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}
// 8 fp32 values -> bf16 hi unit and the bf16 residual unit (v - hi rounded): hi + lo carries v to
// ~16 significant bits, so the expand's two MMAs (v_hi·B + v_lo·B, fp32 accumulate) see v at
// near-fp32 precision.
__device__ __forceinline__ void split_bf16x8(const float* v, uint4& hi, uint4& lo) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    h[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);
    l[i] = pack_bf16x2(v[2 * i] - __uint_as_float(h[i] << 16), v[2 * i + 1] - __uint_as_float(h[i] & 0xffff0000u));
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}
__device__ __forceinline__ uint32_t elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}\n"
      : "=r"(pred));
  return pred;
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Branch-free predicated stores (keeps warp-synchronous loops free of reconvergence code).
__device__ __forceinline__ void st_global_b32_if(void* ptr, uint32_t v, bool pred) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t@p st.global.b32 [%0], %1;\n\t}\n" ::"l"(ptr), "r"(v),
               "r"((uint32_t)pred)
               : "memory");
}
__device__ __forceinline__ uint32_t ld_shared_b32_if(const void* ptr, bool pred) {
  uint32_t v = 0;
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t@p ld.shared.b32 %0, [%1];\n\t}\n"
               : "+r"(v)
               : "r"(smem_u32(ptr)), "r"((uint32_t)pred));
  return v;
}

// ---- mbarrier ------------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Bounded wait: traps after ~4 s instead of hanging the GPU forever on a pipeline bug.
__device__ __forceinline__ void mbar_wait_addr(uint32_t addr, uint32_t parity) {
  uint32_t done = 0;
  uint64_t t0 = 0;
  for (uint32_t spin = 0;; ++spin) {
    asm volatile(
        "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.b32 %0, 1, 0, P;\n\t}\n"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
    if (done) return;
    if ((spin & 1023u) == 1023u) {   // the watchdog clock read is slow: never on the fast path
      const uint64_t now = globaltimer_ns();
      if (t0 == 0) t0 = now;
      else if (now - t0 > 4000000000ull) __trap();
    }
  }
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) { mbar_wait_addr(smem_u32(bar), parity); }

// ---- cross-GPU signalling (NVLink peers, CUDA-IPC-mapped memory) -------------------------
__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_sys_add(int* p, int v) {
  asm volatile("red.release.sys.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_gpu_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_relaxed_gpu(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// Bounded wait on a device-scope counter written by other CTAs of the same grid (traps after ~4 s).
// Spins with relaxed loads and acquires once at the end: an ld.acquire.gpu compiles to a load plus
// an invalidation of the SM's whole L1 (CCTL.IVALL); a fence.acq_rel.gpu to a full MEMBAR.GPU.
__device__ __forceinline__ void wait_geq_gpu(const int* flag, int target) {
  uint64_t t0 = 0;
  for (uint32_t spin = 0; ld_relaxed_gpu(flag) < target; ++spin) {
    __nanosleep(20);
    if ((spin & 1023u) == 1023u) {
      uint64_t now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (t0 == 0) t0 = now;
      else if (now - t0 > 4000000000ull) __trap();
    }
  }
  (void)ld_acquire_gpu(flag);   // one acquire (load + L1 invalidate) once the count is reached
}
// Bounded cross-GPU wait: traps after ~4 s instead of hanging the GPU on a missing signal.
__device__ __forceinline__ int ld_relaxed_sys(const int* p) {
  int v;
  asm volatile("ld.relaxed.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void wait_flag_geq(const int* flag, int target) {
  uint64_t t0 = 0;
  for (uint32_t spin = 0; ld_relaxed_sys(flag) < target; ++spin) {   // relaxed spin, one acquire fence
    __nanosleep(32);
    if ((spin & 1023u) == 1023u) {
      uint64_t now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (t0 == 0) t0 = now;
      else if (now - t0 > 4000000000ull) __trap();
    }
  }
  (void)ld_acquire_sys(flag);
}

// ---- async copies (TMA / bulk) -------------------------------------------------------------
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const void* tmap, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(tmap),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit_group() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_group_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_group() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// Evict-first L2 policy for operands read exactly once (adapter B tiles, the y rows the expand
// adds to), so they do not displace lines that later kernels of the step re-read.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_load_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const void* tmap, uint64_t* bar, int c0, int c1, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(
          smem_u32(dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(pol)
      : "memory");
}
// Whole-warp forms: every lane of a converged warp executes them with identical operands and one
// elected lane issues, so ptxas emits no per-lane waterfall loop around the copy instructions.
__device__ __forceinline__ void bulk_load_elect(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n\t}\n" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_elect(uint32_t dst, const void* tmap, uint32_t bar, int c0, int c1) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n\t}\n" ::"r"(dst),
      "l"(tmap), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
// 3D box {c0: 64 columns, c1: rows, c2: 64-column blocks} (see the expand's y maps)
__device__ __forceinline__ void tma_load_3d_elect(uint32_t dst, const void* tmap, uint32_t bar, int c0, int c1, int c2) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n\t}\n" ::"r"(dst),
      "l"(tmap), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx_elect(uint32_t bar, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;\n\t}\n" ::"r"(bar), "r"(bytes)
      : "memory");
}
// Bulk prefetch of [src, src + bytes) into L2 (bytes a multiple of 16): no shared memory, no barrier.
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---- tcgen05 -------------------------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// Shared-memory matrix descriptor (tcgen05 "version 1" format, see cute/arch/mma_sm100_desc.hpp).
// layout: 0 = no swizzle (interleaved core matrices), 2 = SWIZZLE_128B.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes,
                                              uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3fff);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3fff) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3fff) << 32;
  d |= (uint64_t)1 << 46;  // version = 1 (Blackwell)
  d |= (uint64_t)layout << 61;
  return d;
}
// Instruction descriptor: kind::f16, A=B=bf16, D=f32; A K-major; B K-major (b_mn_major=0) or
// MN-major (b_mn_major=1, bit 16).
__host__ __device__ __forceinline__ uint32_t idesc_bf16(int M, int N, int b_mn_major = 0) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(b_mn_major & 1) << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Whole-warp form: every lane of a converged warp executes it and the election happens inside the
// asm, so the compiler sees no divergent branch around the MMA and does not wrap it in a
// per-instruction uniformization loop (measured: ~45 vs ~100+ cycles per M=128 K=16 MMA).
__device__ __forceinline__ void umma_bf16_elect(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld_32x32b_x16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// 32 lanes x 32 columns: thread i gets TMEM lane (base + i), 32 consecutive fp32 columns.
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// The same load without the wait: pair with tmem_wait_ld_regs() before reading r.
__device__ __forceinline__ void tmem_ld_32x32b_x32_nowait(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}
// Wait for every outstanding tcgen05.ld, then re-define r so no use of it is scheduled above the wait.
__device__ __forceinline__ void tmem_wait_ld_regs(uint32_t* r) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  asm volatile(""
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]));
  asm volatile(""
               : "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]), "+r"(r[22]), "+r"(r[23]),
                 "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31]));
}
// The same with the streaming (evict-first) cache hint: for outputs nothing re-reads soon, so
// they do not displace L2 lines other traffic still needs.
__device__ __forceinline__ void st_global_v8_cs_if(void* ptr, const uint32_t* w, bool pred) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %9, 0;\n\t@p st.global.cs.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n\t}\n" ::"l"(ptr),
               "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"((int)pred)
               : "memory");
}
// 32-byte store (sm_100 STG.256); ptr must be 32-byte aligned
__device__ __forceinline__ void st_global_v8_if(void* ptr, const uint32_t* w, bool pred) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %9, 0;\n\t@p st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n\t}\n" ::"l"(ptr),
               "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"((int)pred)
               : "memory");
}
__device__ __forceinline__ void st_global_v4_if(void* ptr, uint32_t a, uint32_t b, uint32_t c, uint32_t d, bool pred) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %5, 0;\n\t@p st.global.v4.b32 [%0], {%1, %2, %3, %4};\n\t}\n" ::"l"(ptr),
               "r"(a), "r"(b), "r"(c), "r"(d), "r"((uint32_t)pred)
               : "memory");
}

}  // namespace lsv
