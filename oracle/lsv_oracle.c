/*
 * lsv_oracle.c — CPU fp32 restatement of the mixed-rank LoRA delta.  TEST INFRASTRUCTURE ONLY:
 * imported by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg as the checker or the timed CPU baseline; never by the product path.
 *
 * PARITY UNPINNED BY THE REFERENCE: the reference (LoRAServe simulator) contains no LoRA
 * arithmetic (SPEC.md:8 puts kernels out of scope; costmodel.py:83-105 only prices the batch).
 * This restates the math the paper attributes to Punica SGMV / S-LoRA MBGMV
 * (PAPER.md:135, :203):  for each segment s of the adapter-sorted batch,
 *     v[t, k] = sum_i x[t, i] * lora_A_s[k, i]            (shrink, fp32 accumulate)
 *     delta[t, j] = sum_k v[t, k] * lora_B_s[j, k]        (expand, fp32 accumulate)
 * on bf16 inputs widened exactly to fp32.  Segment semantics follow the reference batch:
 * one entry per request with (prompt length, rank) (costmodel.py:83-105), formed FIFO under
 * the token budget (simengine.py:96-152); segments are that batch stably sorted by adapter.
 * The restatement is pinned against a float64 numpy computation in tests/test_oracle.py.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

static inline float bf16_to_f32(uint16_t h) {
  union { uint32_t u; float f; } v;
  v.u = (uint32_t)h << 16;
  return v.f;
}

static inline uint16_t f32_to_bf16_rne(float f) {
  union { uint32_t u; float f; } v;
  v.f = f;
  if ((v.u & 0x7f800000u) == 0x7f800000u && (v.u & 0x007fffffu)) return (uint16_t)((v.u >> 16) | 0x40);
  const uint32_t rounding = 0x7fffu + ((v.u >> 16) & 1u);
  return (uint16_t)((v.u + rounding) >> 16);
}

int lsv_oracle_threads(void) {
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

typedef struct {
  const uint16_t* x;
  int64_t ldx;
  int32_t h_in, h_out, num_segments;
  const int32_t *seg_indptr, *seg_rank;
  float* const* af; /* per segment, fp32 lora_A [rank][h_in] */
  float* const* bf; /* per segment, fp32 lora_B [h_out][rank] */
  float* delta;
  int32_t t_first, t_last; /* token range [t_first, t_last) covered by segments */
  int32_t nthreads, tid;
} job_t;

static void one_token(const job_t* J, int t, int s, float* xf) {
  const int r = J->seg_rank[s];
  float v[256];
  for (int i = 0; i < J->h_in; ++i) xf[i] = bf16_to_f32(J->x[(int64_t)t * J->ldx + i]);
  for (int k = 0; k < r; ++k) { /* shrink */
    const float* ak = J->af[s] + (int64_t)k * J->h_in;
    float acc = 0.f;
#pragma omp simd reduction(+ : acc)
    for (int i = 0; i < J->h_in; ++i) acc += xf[i] * ak[i];
    v[k] = acc;
  }
  float* dt = J->delta + (int64_t)t * J->h_out;
  for (int j = 0; j < J->h_out; ++j) { /* expand */
    const float* bj = J->bf[s] + (int64_t)j * r;
    float acc = 0.f;
#pragma omp simd reduction(+ : acc)
    for (int k = 0; k < r; ++k) acc += v[k] * bj[k];
    dt[j] = acc;
  }
}

static void* worker(void* arg) {
  const job_t* J = (const job_t*)arg;
  float* xf = (float*)malloc((size_t)J->h_in * sizeof(float));
  int s = 0;
  for (int t = J->t_first + J->tid; t < J->t_last; t += J->nthreads) {
    while (s < J->num_segments && J->seg_indptr[s + 1] <= t) ++s;
    if (s >= J->num_segments) break;
    if (t < J->seg_indptr[s]) continue;
    one_token(J, t, s, xf);
  }
  free(xf);
  return NULL;
}

/* delta[t][j] (fp32, [num_tokens][h_out], overwritten for tokens inside segments, untouched
 * elsewhere).  a[s] -> lora_A [rank][h_in] bf16, b[s] -> lora_B [h_out][rank] bf16.
 * threads <= 0 uses every online CPU. */
int lsv_oracle_delta(const uint16_t* x, int64_t ldx, int32_t h_in, int32_t h_out, int32_t num_segments,
                     const int32_t* seg_indptr, const int32_t* seg_rank, const uint16_t* const* a,
                     const uint16_t* const* b, float* delta, int32_t threads) {
  if (num_segments < 0 || h_in <= 0 || h_out <= 0) return 1;
  if (num_segments == 0) return 0;
  for (int s = 0; s < num_segments; ++s)
    if (seg_rank[s] < 1 || seg_rank[s] > 256 || seg_indptr[s + 1] < seg_indptr[s]) return 1;
  float** af = (float**)calloc((size_t)num_segments, sizeof(float*));
  float** bf = (float**)calloc((size_t)num_segments, sizeof(float*));
  int rc = 0;
  for (int s = 0; s < num_segments && !rc; ++s) {
    const int r = seg_rank[s];
    if (seg_indptr[s + 1] == seg_indptr[s]) continue;
    af[s] = (float*)malloc((size_t)r * h_in * sizeof(float));
    bf[s] = (float*)malloc((size_t)h_out * r * sizeof(float));
    if (!af[s] || !bf[s]) { rc = 2; break; }
    for (int64_t e = 0; e < (int64_t)r * h_in; ++e) af[s][e] = bf16_to_f32(a[s][e]);
    for (int64_t e = 0; e < (int64_t)h_out * r; ++e) bf[s][e] = bf16_to_f32(b[s][e]);
  }
  if (!rc) {
    int nt = threads > 0 ? threads : lsv_oracle_threads();
    if (nt > 256) nt = 256;
    pthread_t th[256];
    job_t jobs[256];
    for (int i = 0; i < nt; ++i) {
      jobs[i] = (job_t){x, ldx, h_in, h_out, num_segments, seg_indptr, seg_rank, af, bf, delta,
                        seg_indptr[0], seg_indptr[num_segments], nt, i};
    }
    int started = 0;
    for (int i = 1; i < nt; ++i)
      if (pthread_create(&th[i], NULL, worker, &jobs[i]) == 0) started = i; else break;
    worker(&jobs[0]);
    for (int i = 1; i <= started; ++i) pthread_join(th[i], NULL);
    if (started != nt - 1) rc = 3;
  }
  for (int s = 0; s < num_segments; ++s) { free(af[s]); free(bf[s]); }
  free(af);
  free(bf);
  return rc;
}

/* y[t][j] = bf16(y[t][j] + delta[t][j]) for tokens inside segments (the in-place update the
 * GPU path performs), so a y-level comparison includes the final rounding. */
void lsv_oracle_apply_bf16(uint16_t* y, int64_t ldy, const float* delta, int32_t h_out, int32_t t_begin,
                           int32_t t_end) {
  for (int t = t_begin; t < t_end; ++t)
    for (int j = 0; j < h_out; ++j) {
      const int64_t o = (int64_t)t * ldy + j;
      y[o] = f32_to_bf16_rne(bf16_to_f32(y[o]) + delta[(int64_t)t * h_out + j]);
    }
}
