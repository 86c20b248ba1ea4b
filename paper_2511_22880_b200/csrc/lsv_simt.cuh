// lsv_simt.cuh — CUDA-core (warp-shuffle) tier and the adapter pack/unpack kernels.
//
// The SIMT tier serves segments too short to fill a 128-row tcgen05 tile: decode steps
// (one token per request, the reference's decode_iter_time regime, costmodel.py:108-123)
// and tiny prefill segments.  Shrink: one warp per rank row, lanes stride h_in with 16-byte
// loads of x and of the tiled A row, warp-shuffle reduction.  Expand: one thread per eight
// h_out columns (a 16-byte unit of the B tile), 16-byte read-modify-write of y.
#pragma once
#include "lsv_common.cuh"
#include "lsv_plan.h"

namespace lsv {

__device__ __forceinline__ float dot8_bf16(const uint4& a, const uint4& b) {
  float s = bf16_lo(a.x) * bf16_lo(b.x);
  s = fmaf(bf16_hi(a.x), bf16_hi(b.x), s);
  s = fmaf(bf16_lo(a.y), bf16_lo(b.y), s);
  s = fmaf(bf16_hi(a.y), bf16_hi(b.y), s);
  s = fmaf(bf16_lo(a.z), bf16_lo(b.z), s);
  s = fmaf(bf16_hi(a.z), bf16_hi(b.z), s);
  s = fmaf(bf16_lo(a.w), bf16_lo(b.w), s);
  s = fmaf(bf16_hi(a.w), bf16_hi(b.w), s);
  return s;
}

// Shrink: grid = (row blocks, 1, simt_ksplit(h_in)), block = 256: one block per (item, 8 rows of
// the item's group A, G = nproj * rank rows, one range of h_in's 64-column chunks); the plan's
// row-block map gives blockIdx.x's (item, row block) in one load.  The 8
// warps split the range's chunks (warp w takes chunks w, w + 8, ...); lane = (row of 8, quarter of
// a chunk), so a warp reads each chunk's 8 rows as 1 KB contiguous, four chunks in flight.
// Quarters reduce by shuffle, warps through shared memory in a fixed order (deterministic).  The
// split's partial v (fp32) lands in its own copy of the row's projection region.
constexpr int kSimtUnroll = 4;
#ifndef LSV_SIMT_SHR_UNROLL
#define LSV_SIMT_SHR_UNROLL (LSV_SIMT_SHR_ROWS == 8 ? 4 : 2)
#endif
constexpr int kShrRH = kSimtShrRows / 8;          // 8-row halves per block; a lane owns row rl of each
constexpr int kShrU = LSV_SIMT_SHR_UNROLL;        // chunks in flight per warp
// Resident blocks per SM the compiler must allow (register cap): 4 shrink blocks (64 registers) and
// 8 expand blocks (64 registers) instead of the 3 and 6 that 77-79 registers allow; with the decode
// batch's groups on concurrent streams the occupancy wins over the few spills (decode step 3.0 vs
// 3.6 ms for the unconstrained build, whose 91-register shrink fits 2 blocks).
#ifndef LSV_SIMT_SHR_MINB
#define LSV_SIMT_SHR_MINB 4
#endif
#ifndef LSV_SIMT_EXP_MINB
#define LSV_SIMT_EXP_MINB 8
#endif
__global__ void __launch_bounds__(256, LSV_SIMT_SHR_MINB) simt_shrink_kernel(const __nv_bfloat16* __restrict__ x, int64_t ldx,
                                                          int h_in, const int32_t* __restrict__ plan,
                                                          int off_items, int n_items,
                                                          const void* const* __restrict__ a_ptrs,
                                                          float* __restrict__ simt_v, int nproj, int simt_stride,
                                                          int wait_prev) {
  __shared__ float red[8][kSimtShrRows][kSimtMaxTok];   // [warp][row][token]
  const int m = plan[off_items + 5 * n_items + 1 + blockIdx.x];   // row-block map: item << 8 | row block
  const SimtItem it = reinterpret_cast<const SimtItem*>(plan + off_items)[m >> 8];
  const int rb = m & 255;
  const int r = simt_rank(it), G = nproj * r;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  LSV_DCHECK(simt_nt(it) >= 1 && simt_nt(it) <= kSimtMaxTok && r >= 8 && r <= 256 && rb * kSimtShrRows < G);
  LSV_DCHECK(it.v_off + simt_nt(it) * r <= simt_stride);
  const int rl = lane >> 2, k = rb * kSimtShrRows + rl, q4 = lane & 3;
  const uint8_t* arow = static_cast<const uint8_t*>(a_ptrs[it.seg]) + (size_t)k * 128;
  // row k + 8h has the same swizzle phase as row k
  const uint32_t u0 = (uint32_t)((2 * q4) ^ (k & 7)) << 4, u1 = (uint32_t)((2 * q4 + 1) ^ (k & 7)) << 4;
  bool half_ok[kShrRH];
#pragma unroll
  for (int h = 0; h < kShrRH; ++h) half_ok[h] = rb * kSimtShrRows + 8 * h < G;   // block-uniform
  const size_t cstride = (size_t)G * 128;            // bytes between consecutive chunks of a row
  const int nchunks = h_in / 64, nt = simt_nt(it), ks_n = gridDim.z;
  const int cps = (nchunks + ks_n - 1) / ks_n, cbeg = blockIdx.z * cps;
  const int chunks = min(nchunks, cbeg + cps);   // this split: chunks [cbeg, chunks)
  float acc[kShrRH][kSimtMaxTok];
#pragma unroll
  for (int h = 0; h < kShrRH; ++h)
#pragma unroll
    for (int t = 0; t < kSimtMaxTok; ++t) acc[h][t] = 0.f;
  uint4 a0[kShrU][kShrRH], a1[kShrU][kShrRH];
  auto load = [&](int c0) {
#pragma unroll
    for (int u = 0; u < kShrU; ++u) {
      const int c = c0 + 8 * u;
#pragma unroll
      for (int h = 0; h < kShrRH; ++h) {
        if (c < chunks && half_ok[h]) {
          const uint8_t* ap = arow + (size_t)c * cstride + h * 8 * 128;
          a0[u][h] = __ldg(reinterpret_cast<const uint4*>(ap + u0));
          a1[u][h] = __ldg(reinterpret_cast<const uint4*>(ap + u1));
        }
      }
    }
  };
  load(cbeg + warp);
  // PDL (lsv_lora_forward): the first A loads above may overlap the previous kernel's tail; x and
  // the v partials are touched only after it has completed.  A no-op for a normal launch.
  // wait_prev = 0: the previous launch is another input group's expand, which neither writes this
  // group's x nor reads its workspace slice (lsv_lora_forward's overlap rule): no wait at all.
  if (wait_prev) asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  for (int c0 = cbeg + warp; c0 < chunks; c0 += 8 * kShrU) {
    if (c0 != cbeg + warp) load(c0);
#pragma unroll
    for (int u = 0; u < kShrU; ++u) {
      const int c = c0 + 8 * u;
      if (c < chunks) {
        const int col = c * 64 + q4 * 16;
#pragma unroll
        for (int t = 0; t < kSimtMaxTok; ++t) {
          if (t < nt) {
            const uint4* xp = reinterpret_cast<const uint4*>(x + (int64_t)(it.tok_begin + t) * ldx + col);
            const uint4 x0 = __ldg(xp), x1 = __ldg(xp + 1);   // one x load feeds every row half
#pragma unroll
            for (int h = 0; h < kShrRH; ++h)
              if (half_ok[h]) acc[h][t] += dot8_bf16(a0[u][h], x0) + dot8_bf16(a1[u][h], x1);
          }
        }
      }
    }
  }
#pragma unroll
  for (int h = 0; h < kShrRH; ++h)
#pragma unroll
    for (int t = 0; t < kSimtMaxTok; ++t) {
      acc[h][t] += __shfl_xor_sync(0xffffffffu, acc[h][t], 1);
      acc[h][t] += __shfl_xor_sync(0xffffffffu, acc[h][t], 2);
    }
  if (q4 == 0) {
#pragma unroll
    for (int h = 0; h < kShrRH; ++h)
#pragma unroll
      for (int t = 0; t < kSimtMaxTok; ++t) red[warp][8 * h + rl][t] = acc[h][t];
  }
  __syncthreads();
  if (threadIdx.x < kSimtShrRows * kSimtMaxTok) {
    const int row = threadIdx.x / kSimtMaxTok, t = threadIdx.x % kSimtMaxTok, kk = rb * kSimtShrRows + row;
    if (t < nt && kk < G) {
      float sum = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) sum += red[w][row][t];
      simt_v[((size_t)blockIdx.z * nproj + kk / r) * simt_stride + it.v_off + t * r + kk % r] = sum;
    }
  }
}

// Expand: grid = (items, ceil(max h_out / 256), members), block = 128 (warp w: 64 columns of the
// 256); one launch per input group.
// Lane = (k row of 4, 16-byte unit of 8 columns): a warp reads four 128-byte B atom rows per
// load.  The item's v (<= 8 tokens x rank fp32) is staged in shared memory once, summing the
// shrink's k-split partials in split order, and the B loads are double-buffered (round i+1's
// kSimtExpUnroll loads are in flight while round i is multiplied), so a high-rank item costs about
// rank/32 memory latencies instead of rank/16.  [tokens][8 columns] accumulate in registers over
// k; the four k lanes reduce by shuffle and y is updated with row-contiguous 16-byte
// read-modify-writes.
#ifndef LSV_SIMT_EXP_UNROLL
#define LSV_SIMT_EXP_UNROLL 4
#endif
constexpr int kSimtExpUnroll = LSV_SIMT_EXP_UNROLL;
struct SimtExpandArgs {          // every member of an input group (grid.z = member)
  __nv_bfloat16* y[kMaxProj];
  int64_t ldy[kMaxProj];
  int h_out[kMaxProj];
  const void* const* b_ptrs[kMaxProj];
  const float* v[kMaxProj];      // member's k-split-0 v region
  const int32_t* plan;
  int off_items, ksplit;
  int64_t split_stride;          // floats between k-split copies of the v regions
};
#ifndef LSV_SIMT_EXP_COLS
#define LSV_SIMT_EXP_COLS 256
#endif
constexpr int kSimtExpCols = LSV_SIMT_EXP_COLS;            // h_out columns per block (64 per warp)
constexpr int kSimtExpThreads = kSimtExpCols / 64 * 32;
template <int NT>                // accumulator rows: tokens per pass over the item's B tile
__global__ void __launch_bounds__(kSimtExpThreads, LSV_SIMT_EXP_MINB) simt_expand_kernel(const __grid_constant__ SimtExpandArgs a) {
  __shared__ float vs[kSimtMaxTok * 256];
  const int m = blockIdx.z, h_out = a.h_out[m];
  if ((int)blockIdx.y * kSimtExpCols >= h_out) return;    // block-uniform: past this member's columns
  const SimtItem it = reinterpret_cast<const SimtItem*>(a.plan + a.off_items)[blockIdx.x];
  const int r = simt_rank(it);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.y * kSimtExpCols + warp * 64 + (lane & 7) * 8;   // this lane's 8 columns
  const bool active = blockIdx.y * kSimtExpCols + warp * 64 < h_out;      // warp-uniform (h_out % 64 == 0)
  const int ks = lane >> 3, nt = simt_nt(it);
  __nv_bfloat16* const y = a.y[m];
  const int64_t ldy = a.ldy[m];
  const uint8_t* b = static_cast<const uint8_t*>(a.b_ptrs[m][it.seg]);
  const int tw = b_tile_width(h_out);
  constexpr int U = kSimtExpUnroll;
  uint4 cur[U], nxt[U];
  auto load = [&](uint4* dst, int k0) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + u * 4 + ks;
      if (active && k < r) dst[u] = __ldg(reinterpret_cast<const uint4*>(b + b_tiled_off(j, k, r, tw)));
    }
  };
  load(cur, 0);                                  // in flight while v is staged
  // PDL (lsv_lora_forward): the B loads above may overlap the previous kernel's tail; v and y
  // are read only after it has completed.  A no-op for a normally launched grid.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const float* vp = a.v[m] + it.v_off;
  for (int i = threadIdx.x; i < nt * r; i += blockDim.x) {
    float sum = 0.f;
    for (int z = 0; z < a.ksplit; ++z) sum += __ldcg(vp + z * a.split_stride + i);
    vs[i] = sum;
  }
  __syncthreads();
  if (!active) return;
  // NT tokens per pass; items with more tokens (rare in decode) re-read their B tile from L1/L2
  for (int tb = 0; tb < nt; tb += NT) {
    if (tb > 0) load(cur, 0);
    float acc[NT][8];
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[t][e] = 0.f;
    for (int k0 = 0; k0 < r; k0 += 4 * U) {
      if (k0 + 4 * U < r) load(nxt, k0 + 4 * U);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = k0 + u * 4 + ks;
        if (k < r) {
          const float w[8] = {bf16_lo(cur[u].x), bf16_hi(cur[u].x), bf16_lo(cur[u].y), bf16_hi(cur[u].y),
                              bf16_lo(cur[u].z), bf16_hi(cur[u].z), bf16_lo(cur[u].w), bf16_hi(cur[u].w)};
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            if (tb + t < nt) {
              const float vv = vs[(tb + t) * r + k];
#pragma unroll
              for (int e = 0; e < 8; ++e) acc[t][e] = fmaf(vv, w[e], acc[t][e]);
            }
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) cur[u] = nxt[u];
    }
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        acc[t][e] += __shfl_xor_sync(0xffffffffu, acc[t][e], 8);
        acc[t][e] += __shfl_xor_sync(0xffffffffu, acc[t][e], 16);
      }
    if (ks == 0) {
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        if (tb + t < nt) {
          uint4* py = reinterpret_cast<uint4*>(y + (int64_t)(it.tok_begin + tb + t) * ldy + j);
          const uint4 yv = *py;
          uint4 o;
          o.x = pack_bf16x2(bf16_lo(yv.x) + acc[t][0], bf16_hi(yv.x) + acc[t][1]);
          o.y = pack_bf16x2(bf16_lo(yv.y) + acc[t][2], bf16_hi(yv.y) + acc[t][3]);
          o.z = pack_bf16x2(bf16_lo(yv.z) + acc[t][4], bf16_hi(yv.z) + acc[t][5]);
          o.w = pack_bf16x2(bf16_lo(yv.w) + acc[t][6], bf16_hi(yv.w) + acc[t][7]);
          *py = o;
        }
      }
    }
  }
}

// ---- tensor-parallel v assembly -------------------------------------------------------------
// grid = n_mtiles; one thread per (token, 8-wide k unit) of the full-rank image.  Shard t of a
// tile's rank holds k in [t*rs, (t+1)*rs); rs is a multiple of 8 so a unit never straddles shards.
__global__ void __launch_bounds__(256) vimg_assemble_kernel(const uint8_t* __restrict__ gathered, size_t region,
                                                            int tp, const int32_t* __restrict__ splan,
                                                            int s_off_mtiles, int s_ws_vimg,
                                                            const int32_t* __restrict__ fplan, int f_off_mtiles,
                                                            uint8_t* __restrict__ fws, int f_ws_vimg, int vsplit) {
  const MTile ms = reinterpret_cast<const MTile*>(splan + s_off_mtiles)[blockIdx.x];
  const MTile mf = reinterpret_cast<const MTile*>(fplan + f_off_mtiles)[blockIdx.x];
  const int rs = ms.rank, kps = kpad(rs), kpf = kpad(mf.rank), np16 = round_up(mf.ntok, 16);
  const int upr = kpf / 8, units = mf.ntok * upr;
  // split v: each image is a (hi, lo) pair; the lo half sits vimg_bytes after the hi half
  for (int u = threadIdx.x; u < units * (vsplit ? 2 : 1); u += blockDim.x) {
    const int half = u / units, uu = u % units;
    const int t = uu / upr, k0 = (uu % upr) * 8;
    uint4 w = make_uint4(0, 0, 0, 0);
    if (k0 < tp * rs) {
      const int sh = k0 / rs, kk = k0 % rs;
      const uint8_t* src = gathered + (size_t)sh * region + (ms.vimg_off) + vimg_off(t, kk, kps, np16) +
                           (half ? vimg_bytes(ms.ntok, kps) : 0u);
      w = *reinterpret_cast<const uint4*>(src);
    }
    *reinterpret_cast<uint4*>(fws + f_ws_vimg + mf.vimg_off + vimg_off(t, k0, kpf, np16) +
                              (half ? vimg_bytes(mf.ntok, kpf) : 0u)) = w;
  }
}

// ---- adapter slab packing ---------------------------------------------------------------
// lora_a [rank][h_in] -> A tiled; lora_b [h_out][rank] -> B tiled.  One thread per 16 bytes of
// the tiled buffers.
__global__ void pack_adapter_kernel(const uint8_t* __restrict__ lora_a, const uint8_t* __restrict__ lora_b,
                                    int rank, int h_in, int h_out, uint8_t* __restrict__ a_t,
                                    uint8_t* __restrict__ b_t, int unpack, int grows, int row0) {
  // A goes to rows [row0, row0 + rank) of a group tile of grows rows per chunk (a_tiled_off_g)
  const int kp = kpad(rank);
  const int64_t na = (int64_t)rank * h_in / 8, nb = (int64_t)h_out * kp / 8;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < na + nb;
       u += (int64_t)gridDim.x * blockDim.x) {
    if (u < na) {
      const int k = (int)(u / (h_in / 8)), i = (int)(u % (h_in / 8)) * 8;
      uint4* plain = reinterpret_cast<uint4*>(const_cast<uint8_t*>(lora_a) + ((int64_t)k * h_in + i) * 2);
      uint4* tiled = reinterpret_cast<uint4*>(a_t + a_tiled_off_g(row0 + k, i, grows));
      if (unpack) *plain = *tiled; else *tiled = *plain;
    } else {
      // one 16-byte unit of B tiled = lora_b[j .. j+7][k] (a strided column gather of lora_B);
      // k in [rank, kp) is the zero padding
      const int64_t w = u - na;
      const int k = (int)(w % kp), j = (int)(w / kp) * 8;
      uint16_t* plain = reinterpret_cast<uint16_t*>(const_cast<uint8_t*>(lora_b)) + (int64_t)j * rank + k;
      uint16_t* tiled = reinterpret_cast<uint16_t*>(b_t + b_tiled_off(j, k, rank, b_tile_width(h_out)));
      if (unpack) {
        if (k < rank)
          for (int e = 0; e < 8; ++e) plain[(int64_t)e * rank] = tiled[e];
      } else {
        alignas(16) uint16_t v[8];
        for (int e = 0; e < 8; ++e) v[e] = k < rank ? plain[(int64_t)e * rank] : (uint16_t)0;
        *reinterpret_cast<uint4*>(tiled) = *reinterpret_cast<const uint4*>(v);
      }
    }
  }
}

}  // namespace lsv
