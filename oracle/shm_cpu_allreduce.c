/*
 * TEST / BASELINE INFRASTRUCTURE ONLY - the CPU reference path of the SHM
 * allreduce as BASELINE.md §3 specifies it: ONE PROCESS PER RANK, each pinned
 * to its own host core, joined by a real POSIX shared-memory segment
 * (/dev/shm), running the same reduce-scatter / all-gather algorithm and the
 * same fixed ascending-rank fp32 sum as the GPU path (oracle/flexshm_oracle.c
 * states the arithmetic; results are bit-identical to oracle_allreduce).
 * Nothing in paper_2511_09143_b200/ runs or links this program; bench.py
 * times it as the CPU baseline and the `--impl reference` arm, and
 * tests/test_oracle.py checks its results against the checker.
 *
 *   shm_cpu_allreduce <n> <count> <dtype 0=f32,1=bf16> <op> <factor> <iters>
 *                     <warmup> <cores csv> <in path|-> <out path|->
 *
 * in path: n x count elements (rank-major) every rank copies into its
 * private buffer before the timed loop ("-": deterministic synthetic data);
 * out path: every rank's buffer after the LAST iteration.  Prints one JSON
 * line: the step time (max over ranks of the timed loop / iters), the cores
 * used and whether ranks outnumber them.
 *
 * Per iteration, rank r (owner of chunk r, chunk = ceil(count/n)):
 *   1. stage: copy its pieces of the other owners' chunks into
 *      staging[o][r] of the segment, then raise STAGED[r] = it;
 *   2. reduce: wait STAGED[q] >= it for all q, sum chunk r in rank order
 *      (its own piece from its private buffer), write results[r] and its
 *      buffer, raise REDUCED[r] = it;
 *   3. gather: wait REDUCED[q] >= it, copy results[q] into its buffer.
 * Slot reuse: stage(it+1) follows gather(it) in program order, which waited
 * for every owner's reduce(it) (the staging slots' last reader); reduce(it+1)
 * of owner o waits STAGED[q] >= it+1, raised after q's gather(it) (the
 * results slot's last reader).  Waits spin with sched_yield, so the program
 * also runs (slowly) when ranks outnumber cores.
 *
 * Built by oracle/Makefile with -O2 -fno-fast-math -ffp-contract=off.
 */
#define _GNU_SOURCE
#include <errno.h>
#include <fcntl.h>
#include <sched.h>
#include <stdatomic.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <sys/wait.h>
#include <time.h>
#include <unistd.h>

enum { F32 = 0, BF16 = 1 };
enum { OP_SUM = 0, OP_SUM_POSTSCALE = 1, OP_PREDIV_SUM = 2, OP_PREMUL_SUM = 3 };
#define MAXR 256

static inline float bf16_to_f32(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static inline uint16_t f32_to_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu)) return (uint16_t)((u >> 16) | 0x40u);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

static inline float contrib(const void* x, int dtype, size_t i, int op, float f) {
  float v = dtype == F32 ? ((const float*)x)[i] : bf16_to_f32(((const uint16_t*)x)[i]);
  if (op == OP_PREDIV_SUM) v = v / f;
  else if (op == OP_PREMUL_SUM) v = v * f;
  else return v;
  return dtype == F32 ? v : bf16_to_f32(f32_to_bf16(v));
}

typedef struct {
  _Alignas(64) atomic_uint staged;
  _Alignas(64) atomic_uint reduced;
  _Alignas(64) atomic_int ready;
  double t0, t1;
} rank_line;

typedef struct {
  _Alignas(64) atomic_int arrived;
  _Alignas(64) atomic_int go;
  rank_line r[MAXR];
} header;

static double now(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + ts.tv_nsec * 1e-9;
}

static void wait_geq(atomic_uint* p, unsigned v) {
  unsigned spins = 0;
  while ((int)(atomic_load_explicit(p, memory_order_acquire) - v) < 0)
    if (++spins > 64) sched_yield();
}

static int run_rank(int me, int n, size_t count, int dtype, int op, float factor, int iters,
                    int warmup, int core, header* h, char* staging, char* results, const char* in,
                    char* out) {
  if (core >= 0) {
    cpu_set_t set;
    CPU_ZERO(&set);
    CPU_SET(core, &set);
    sched_setaffinity(0, sizeof set, &set);
  }
  const size_t esz = dtype == F32 ? 4 : 2;
  const size_t chunk = (count + n - 1) / n;
  /* private rank buffer, first-touched on this rank's core */
  char* buf = mmap(NULL, count * esz + 64, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (buf == MAP_FAILED) return 2;
  if (in)
    memcpy(buf, in + (size_t)me * count * esz, count * esz);
  else
    for (size_t i = 0; i < count; ++i) {
      float v = (float)((int)((i * 2654435761u + (size_t)me * 40503u) % 2001u) - 1000) * 1e-6f;
      if (dtype == F32) ((float*)buf)[i] = v;
      else ((uint16_t*)buf)[i] = f32_to_bf16(v);
    }
  const void* xs[MAXR];
  atomic_fetch_add(&h->arrived, 1);
  while (atomic_load(&h->go) == 0) sched_yield();
  for (int it = 1; it <= warmup + iters; ++it) {
    if (it == warmup + 1) { /* every rank starts the timed loop together */
      atomic_store(&h->r[me].ready, it);
      for (int q = 0; q < n; ++q)
        while (atomic_load(&h->r[q].ready) < it) sched_yield();
      h->r[me].t0 = now();
    }
    /* 1. stage */
    for (int o = 0; o < n; ++o) {
      if (o == me) continue;
      const size_t lo = (size_t)o * chunk;
      if (lo >= count) continue;
      const size_t len = (lo + chunk > count ? count : lo + chunk) - lo;
      memcpy(staging + (((size_t)o * n + me) * chunk) * esz, buf + lo * esz, len * esz);
    }
    atomic_store_explicit(&h->r[me].staged, (unsigned)it, memory_order_release);
    /* 2. reduce my chunk in ascending rank order */
    const size_t lo = (size_t)me * chunk;
    const size_t len = lo >= count ? 0 : (lo + chunk > count ? count : lo + chunk) - lo;
    for (int q = 0; q < n; ++q)
      if (q != me) wait_geq(&h->r[q].staged, (unsigned)it);
    for (int q = 0; q < n; ++q)
      xs[q] = q == me ? (const void*)(buf + lo * esz)
                      : (const void*)(staging + (((size_t)me * n + q) * chunk) * esz);
    char* res = results + (size_t)me * chunk * esz;
    for (size_t i = 0; i < len; ++i) {
      float acc = contrib(xs[0], dtype, i, op, factor);
      for (int q = 1; q < n; ++q) acc = acc + contrib(xs[q], dtype, i, op, factor);
      if (op == OP_SUM_POSTSCALE) acc = acc * factor;
      if (dtype == F32) ((float*)res)[i] = acc;
      else ((uint16_t*)res)[i] = f32_to_bf16(acc);
    }
    if (len) memcpy(buf + lo * esz, res, len * esz);
    atomic_store_explicit(&h->r[me].reduced, (unsigned)it, memory_order_release);
    /* 3. gather */
    for (int q = 0; q < n; ++q) {
      if (q == me) continue;
      const size_t qlo = (size_t)q * chunk;
      if (qlo >= count) continue;
      const size_t qlen = (qlo + chunk > count ? count : qlo + chunk) - qlo;
      wait_geq(&h->r[q].reduced, (unsigned)it);
      memcpy(buf + qlo * esz, results + qlo * esz, qlen * esz);
    }
  }
  h->r[me].t1 = now();
  if (out) memcpy(out + (size_t)me * count * esz, buf, count * esz);
  return 0;
}

static void* map_file(const char* path, size_t bytes, int write) {
  int fd = open(path, write ? (O_RDWR | O_CREAT) : O_RDONLY, 0600);
  if (fd < 0) return NULL;
  if (write && ftruncate(fd, (off_t)bytes) != 0) {
    close(fd);
    return NULL;
  }
  void* p = mmap(NULL, bytes, write ? PROT_READ | PROT_WRITE : PROT_READ, MAP_SHARED, fd, 0);
  close(fd);
  return p == MAP_FAILED ? NULL : p;
}

int main(int argc, char** argv) {
  if (argc != 11) {
    fprintf(stderr, "usage: %s n count dtype op factor iters warmup cores in out\n", argv[0]);
    return 1;
  }
  const int n = atoi(argv[1]);
  const size_t count = strtoull(argv[2], NULL, 10);
  const int dtype = atoi(argv[3]), op = atoi(argv[4]);
  const float factor = strtof(argv[5], NULL);
  const int iters = atoi(argv[6]), warmup = atoi(argv[7]);
  if (n < 1 || n > MAXR || count == 0 || iters < 1 || warmup < 0) return 1;
  int cores[MAXR], ncores = 0;
  for (char* tok = strtok(argv[8], ","); tok && ncores < MAXR; tok = strtok(NULL, ","))
    cores[ncores++] = atoi(tok);
  const size_t esz = dtype == F32 ? 4 : 2;
  const char* in = NULL;
  char* out = NULL;
  if (strcmp(argv[9], "-")) in = map_file(argv[9], (size_t)n * count * esz, 0);
  if (strcmp(argv[10], "-")) out = map_file(argv[10], (size_t)n * count * esz, 1);
  if ((strcmp(argv[9], "-") && !in) || (strcmp(argv[10], "-") && !out)) {
    fprintf(stderr, "cannot map %s / %s: %s\n", argv[9], argv[10], strerror(errno));
    return 1;
  }
  /* the segment: header, staging [owner][contributor][chunk], results [owner][chunk] */
  const size_t chunk = (count + n - 1) / n;
  const size_t hdr = (sizeof(header) + 4095) / 4096 * 4096;
  const size_t stg = (size_t)n * n * chunk * esz, resb = (size_t)n * chunk * esz;
  const size_t total = hdr + stg + resb;
  char name[64];
  snprintf(name, sizeof name, "/fmx-cpuref-%d", (int)getpid());
  int fd = shm_open(name, O_CREAT | O_EXCL | O_RDWR, 0600);
  if (fd < 0 || ftruncate(fd, (off_t)total) != 0) return 3;
  char* seg = mmap(NULL, total, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  shm_unlink(name); /* children inherit the mapping */
  if (seg == MAP_FAILED) return 3;
  header* h = (header*)seg;
  memset(h, 0, sizeof *h);
  pid_t pids[MAXR];
  for (int r = 0; r < n; ++r) {
    pids[r] = fork();
    if (pids[r] == 0)
      _exit(run_rank(r, n, count, dtype, op, factor, iters, warmup,
                     ncores ? cores[r % ncores] : -1, h, seg + hdr, seg + hdr + stg, in, out));
  }
  while (atomic_load(&h->arrived) < n) usleep(100);
  atomic_store(&h->go, 1);
  int bad = 0;
  for (int r = 0; r < n; ++r) {
    int st = 0;
    waitpid(pids[r], &st, 0);
    if (!WIFEXITED(st) || WEXITSTATUS(st) != 0) bad = 1;
  }
  if (bad) return 4;
  double t0 = h->r[0].t0, t1 = h->r[0].t1;
  for (int r = 1; r < n; ++r) {
    if (h->r[r].t0 < t0) t0 = h->r[r].t0;
    if (h->r[r].t1 > t1) t1 = h->r[r].t1;
  }
  printf("{\"ms_per_step\": %.6f, \"iters\": %d, \"ranks\": %d, \"cores\": %d, "
         "\"oversubscribed\": %s, \"processes\": %d}\n",
         (t1 - t0) / iters * 1e3, iters, n, ncores ? (ncores < n ? ncores : n) : 0,
         ncores && ncores < n ? "true" : "false", n);
  if (out) munmap(out, (size_t)n * count * esz);
  return 0;
}
