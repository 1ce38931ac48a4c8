/*
 * TEST INFRASTRUCTURE ONLY - the CPU oracle for the SHM allreduce/broadcast.
 *
 * Nothing in the product path (paper_2511_09143_b200/) links or calls this
 * file.  It is used by tests/ (as the checker), by __graft_entry__.smoke()
 * (as the checker) and by bench.py's cpu_baseline / --impl reference legs
 * (as the timed CPU path).
 *
 * What it restates.  The reference holds NO arithmetic for this path: its
 * allreduce lives in NCCL 2.21.5 plus an unpublished MIG patch (reference
 * PAPER.md:353-354, 386-388, 830) and the simulator models it as
 * a constant (reference pkg/src/migsim/simcore.py:46-51, 91-100).  The
 * contract restated here is the north_star's (BASELINE.json):
 *
 *   out[i] = ((((x_0[i] + x_1[i]) + x_2[i]) + ...) + x_{n-1}[i])   in fp32,
 *
 * ranks in ascending order = the order of AllocationDecision.instances
 * produced by fm_select's round-robin (reference scheduler.py:117-136), with
 * four scale conventions:
 *   FMX_OP_SUM           no scaling
 *   FMX_OP_SUM_POSTSCALE (sum) * factor, one fp32 multiply
 *   FMX_OP_PREDIV_SUM    each x_q / factor (IEEE division) before the sum
 *   FMX_OP_PREMUL_SUM    each x_q * factor before the sum.  DDP's mean is
 *                        this op with factor = fl32(1/world): the default
 *                        hook's bucket.div_(world) (torch/distributed/
 *                        algorithms/ddp_comm_hooks/default_hooks.py:26) runs
 *                        ATen's div_true_kernel_cuda, which for a CPU-scalar
 *                        divisor multiplies by the fp32 reciprocal
 *                        (aten/src/ATen/native/cuda/BinaryDivTrueKernel.cu);
 *                        pinned on the B200 by tests/test_ddp_arith_gpu.py
 * bf16: inputs widened exactly to fp32, summed in the same order, rounded
 * once to bf16 (round-to-nearest-even).  For PREDIV / PREMUL the scaled
 * contribution is itself rounded to bf16 first (a bf16 bucket scaled in
 * place).
 * Broadcast is an exact bit copy.
 *
 * Parity status: UNPINNED against the reference (no reference arithmetic
 * exists).  Pinned instead against (a) a numpy restatement
 * (oracle/oracle.py) and (b) torch's bf16 RNE conversion, see
 * tests/golden/make_golden_data.py.
 *
 * Built by oracle/Makefile:  -O2 -fno-fast-math -ffp-contract=off so the C
 * compiler neither reassociates nor contracts.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { ORC_F32 = 0, ORC_BF16 = 1 };
enum { ORC_SUM = 0, ORC_SUM_POSTSCALE = 1, ORC_PREDIV_SUM = 2, ORC_PREMUL_SUM = 3 };

static inline float bf16_to_f32(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static inline uint16_t f32_to_bf16_rne(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu)) /* NaN: keep quiet NaN */
    return (uint16_t)((u >> 16) | 0x0040u);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

uint16_t oracle_f32_to_bf16(float f) { return f32_to_bf16_rne(f); }

static inline float contrib_f32(const void* x, int dtype, size_t i, int op, float factor) {
  if (dtype == ORC_F32) {
    float v = ((const float*)x)[i];
    return op == ORC_PREDIV_SUM ? v / factor : op == ORC_PREMUL_SUM ? v * factor : v;
  }
  float v = bf16_to_f32(((const uint16_t*)x)[i]);
  if (op == ORC_PREDIV_SUM) v = bf16_to_f32(f32_to_bf16_rne(v / factor));
  if (op == ORC_PREMUL_SUM) v = bf16_to_f32(f32_to_bf16_rne(v * factor));
  return v;
}

/* Reduce elements [lo, hi) of n contributions into out (same dtype). */
static void reduce_range(int n, const void* const* xs, void* out, int dtype, int op,
                         float factor, size_t lo, size_t hi) {
  for (size_t i = lo; i < hi; ++i) {
    float acc = contrib_f32(xs[0], dtype, i, op, factor);
    for (int q = 1; q < n; ++q) acc = acc + contrib_f32(xs[q], dtype, i, op, factor);
    if (op == ORC_SUM_POSTSCALE) acc = acc * factor;
    if (dtype == ORC_F32) ((float*)out)[i] = acc;
    else ((uint16_t*)out)[i] = f32_to_bf16_rne(acc);
  }
}

/* Single-threaded rank-order allreduce: the checker. */
void oracle_allreduce(int n, const void* const* xs, void* out, size_t count, int dtype,
                      int op, float factor) {
  reduce_range(n, xs, out, dtype, op, factor, 0, count);
}

/* ------------------------------------------------------------------------
 * CPU SHM allreduce (the "reference CPU path" timed beside the GPU).
 *
 * Same data movement as the GPU design: every rank stages its
 * non-owned chunks into a shared staging area, each owner reduces its chunk in
 * rank order (its own contribution read from its own buffer), writes the
 * result to the shared result area, and every rank gathers the other owners'
 * results.  Ranks are buffers in one address space; the work of each phase is
 * split over `nthreads` host threads.  Results are bit-identical to
 * oracle_allreduce.
 */
typedef struct {
  int n, dtype, op, phase, tid, nthreads;
  float factor;
  size_t count, chunk, esz;
  void** bufs;     /* n rank buffers, in place */
  char* staging;   /* [owner][contributor][chunk] */
  char* results;   /* [owner][chunk] */
} shm_job;

static size_t chunk_len(const shm_job* j, int owner) {
  size_t lo = (size_t)owner * j->chunk;
  if (lo >= j->count) return 0;
  size_t hi = lo + j->chunk;
  return (hi > j->count ? j->count : hi) - lo;
}

static void split(size_t total, int tid, int nt, size_t* lo, size_t* hi) {
  size_t per = (total + nt - 1) / nt;
  *lo = per * tid < total ? per * tid : total;
  *hi = *lo + per < total ? *lo + per : total;
}

static void* shm_worker(void* arg) {
  shm_job* j = (shm_job*)arg;
  size_t esz = j->esz;
  if (j->phase == 0) { /* stage: rank r copies chunk o (o != r) into staging[o][r] */
    for (int r = 0; r < j->n; ++r)
      for (int o = 0; o < j->n; ++o) {
        if (o == r) continue;
        size_t len = chunk_len(j, o), lo, hi;
        split(len, j->tid, j->nthreads, &lo, &hi);
        if (hi > lo)
          memcpy(j->staging + ((size_t)o * j->n + r) * j->chunk * esz + lo * esz,
                 (char*)j->bufs[r] + ((size_t)o * j->chunk + lo) * esz, (hi - lo) * esz);
      }
  } else if (j->phase == 1) { /* reduce: owner o sums its chunk in rank order */
    const void* xs[1024];
    for (int o = 0; o < j->n; ++o) {
      size_t len = chunk_len(j, o), lo, hi;
      split(len, j->tid, j->nthreads, &lo, &hi);
      if (hi <= lo) continue;
      for (int q = 0; q < j->n; ++q)
        xs[q] = q == o ? (const void*)((char*)j->bufs[o] + (size_t)o * j->chunk * esz)
                       : (const void*)(j->staging + ((size_t)o * j->n + q) * j->chunk * esz);
      char* res = j->results + (size_t)o * j->chunk * esz;
      reduce_range(j->n, xs, res, j->dtype, j->op, j->factor, lo, hi);
      memcpy((char*)j->bufs[o] + ((size_t)o * j->chunk + lo) * esz, res + lo * esz,
             (hi - lo) * esz);
    }
  } else { /* gather: rank r copies result chunk o (o != r) */
    for (int r = 0; r < j->n; ++r)
      for (int o = 0; o < j->n; ++o) {
        if (o == r) continue;
        size_t len = chunk_len(j, o), lo, hi;
        split(len, j->tid, j->nthreads, &lo, &hi);
        if (hi > lo)
          memcpy((char*)j->bufs[r] + ((size_t)o * j->chunk + lo) * esz,
                 j->results + (size_t)o * j->chunk * esz + lo * esz, (hi - lo) * esz);
      }
  }
  return NULL;
}

/* scratch must hold (n*n + n) * chunk * esz bytes, chunk = ceil(count/n). */
size_t oracle_shm_scratch_bytes(int n, size_t count, int dtype) {
  size_t chunk = (count + n - 1) / n;
  return ((size_t)n * n + n) * chunk * (dtype == ORC_F32 ? 4 : 2);
}

int oracle_shm_allreduce(int n, void** bufs, size_t count, int dtype, int op, float factor,
                         int nthreads, void* scratch) {
  if (n < 1 || n > 1024 || nthreads < 1 || nthreads > 256) return -1;
  shm_job base;
  memset(&base, 0, sizeof base);
  base.n = n; base.dtype = dtype; base.op = op; base.factor = factor;
  base.count = count; base.chunk = (count + n - 1) / n; base.esz = dtype == ORC_F32 ? 4 : 2;
  base.bufs = bufs; base.nthreads = nthreads;
  base.staging = (char*)scratch;
  base.results = base.staging + (size_t)n * n * base.chunk * base.esz;
  pthread_t th[256];
  shm_job jobs[256];
  for (int phase = 0; phase < 3; ++phase) {
    for (int t = 0; t < nthreads; ++t) {
      jobs[t] = base; jobs[t].phase = phase; jobs[t].tid = t;
      if (t) pthread_create(&th[t], NULL, shm_worker, &jobs[t]);
    }
    shm_worker(&jobs[0]);
    for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
  }
  return 0;
}

/* ------------------------------------------------------------------------
 * In-place host reduction (a bound, not an SHM path): every rank's buffer in
 * one address space, each of `nthreads` threads takes an element range,
 * sums it across the n buffers in rank order and writes the result back into
 * all n buffers - read n*S + write n*S, no staging copies.  It is what a
 * single host process could at best do with host-resident gradients, and is
 * reported next to the GPU e2e figure (the GPU/CPU ratio must not
 * be read as "GPU beats the host" without it).  Bit-identical results. */
typedef struct {
  int n, dtype, op;
  float factor;
  void** bufs;
  size_t lo, hi;
} inplace_job;

static void* inplace_worker(void* arg) {
  inplace_job* j = (inplace_job*)arg;
  const size_t esz = j->dtype == ORC_F32 ? 4 : 2;
  enum { B = 4096 };
  union { float f[B]; uint16_t h[B]; } tmp;
  for (size_t lo = j->lo; lo < j->hi; lo += B) {
    const size_t len = j->hi - lo < B ? j->hi - lo : B;
    const void* xs[1024];
    for (int q = 0; q < j->n; ++q) xs[q] = (const char*)j->bufs[q] + lo * esz;
    reduce_range(j->n, xs, &tmp, j->dtype, j->op, j->factor, 0, len);
    for (int q = 0; q < j->n; ++q) memcpy((char*)j->bufs[q] + lo * esz, &tmp, len * esz);
  }
  return NULL;
}

int oracle_inplace_allreduce(int n, void** bufs, size_t count, int dtype, int op, float factor,
                             int nthreads) {
  if (n < 1 || n > 1024 || nthreads < 1 || nthreads > 256) return -1;
  pthread_t th[256];
  inplace_job jobs[256];
  for (int t = 0; t < nthreads; ++t) {
    inplace_job j = {n, dtype, op, factor, bufs, 0, 0};
    split(count, t, nthreads, &j.lo, &j.hi);
    jobs[t] = j;
    if (t) pthread_create(&th[t], NULL, inplace_worker, &jobs[t]);
  }
  inplace_worker(&jobs[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
  return 0;
}
