/*
 * trend_oracle.c -- CPU restatement of the reference's trend/fitness hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (libebic.so, the C++
 * drop-in shim, the Python mirror) links, loads or calls this file.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use it, and
 * only as the checker / the timed CPU baseline ("kind": "port").
 *
 * Parity is PINNED: tests/test_oracle.py checks every function here against
 * (a) the hand vectors of proj/tests/test_trend.cpp:60-89, (b) the golden
 * fixtures in tests/golden/ produced by the unmodified reference sources
 * (tests/golden/make_golden.py over oracle/_ref/libbicseek_ref.so), and
 * (c) live random cases against oracle/_ref when it is built.
 *
 * Restated from /root/reference/proj/src/trend.cpp (not copied):
 *   follows_forward   trend.cpp:17-26
 *   follows_reversed  trend.cpp:28-37
 *   row_supports      trend.cpp:41-46
 *   supporting_rows   trend.cpp:48-54
 *   evaluate_population trend.cpp:56-72  (WorkerPool chunking -> pthreads here;
 *                     counts are integers so the split never changes results)
 *   fitness           trend.cpp:74-79
 *
 * Arithmetic contract: the comparison is `cur > prev - approx*|prev|` in IEEE
 * double with TWO separately rounded operations (the reference trend.o has no
 * FMA: andpd; mulsd; subsd; comisd).  This file must therefore be compiled
 * with -ffp-contract=off and without -ffast-math (see oracle/Makefile).
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <pthread.h>
#include <unistd.h>

/* Matrix view: row-major doubles, element (r, c) at m[r * n_cols + c]
 * (matrix.hpp:26,29). */

static inline int step_ok(double cur, double prev, double approx) {
  /* trend.cpp:22 / :33 -- volatile-free: -ffp-contract=off keeps mul, sub
   * separately rounded. */
  double slack = approx * fabs(prev);
  double thr = prev - slack;
  return cur > thr;
}

/* trend.cpp:17-26 */
static int follows_forward(const double* row, const uint32_t* seq, uint32_t len,
                           double approx) {
  double prev = row[seq[0]];
  for (uint32_t k = 1; k < len; ++k) {
    double cur = row[seq[k]];
    if (!step_ok(cur, prev, approx)) return 0;
    prev = cur;
  }
  return 1;
}

/* trend.cpp:28-37: walk the sequence from its last element back to the first;
 * each step has its own "prev" for the slack. */
static int follows_reversed(const double* row, const uint32_t* seq, uint32_t len,
                            double approx) {
  double prev = row[seq[len - 1]];
  for (uint32_t k = len - 1; k-- > 0;) {
    double cur = row[seq[k]];
    if (!step_ok(cur, prev, approx)) return 0;
    prev = cur;
  }
  return 1;
}

/* trend.cpp:41-46 */
int oracle_row_supports(const double* m, uint64_t n_cols, uint64_t row, const uint32_t* seq,
                        uint32_t len, double approx, int negative_trends) {
  const double* r = m + row * n_cols;
  if (len == 0) return 0;
  if (follows_forward(r, seq, len, approx)) return 1;
  return negative_trends && follows_reversed(r, seq, len, approx);
}

/* trend.cpp:48-54: ascending row list.  Returns the number of supporting rows;
 * writes at most `cap` of them. */
uint64_t oracle_supporting_rows(const double* m, uint64_t n_rows, uint64_t n_cols,
                                const uint32_t* seq, uint32_t len, double approx,
                                int negative_trends, uint32_t* rows_out, uint64_t cap) {
  uint64_t n = 0;
  for (uint64_t r = 0; r < n_rows; ++r) {
    if (oracle_row_supports(m, n_cols, r, seq, len, approx, negative_trends)) {
      if (n < cap) rows_out[n] = (uint32_t)r;
      ++n;
    }
  }
  return n;
}

/* Work sharing for the population loop: chunks of candidates handed out through
 * an atomic counter, like the reference WorkerPool (worker_pool.cpp:20-48,
 * chunk = n/(threads*8)).  Counts are integers, so the split never changes
 * the result. */
typedef struct {
  const void* m;
  int is_f32;
  uint64_t n_rows, n_cols;
  const uint32_t* cols;
  const uint32_t* offsets;
  uint64_t n_cand;
  double approx;
  int neg;
  uint32_t* counts;
  uint64_t chunk;
  uint64_t next; /* atomic */
} job_t;

static uint32_t count_f64(const job_t* j, uint64_t i) {
  const double* m = (const double*)j->m;
  const uint32_t* seq = j->cols + j->offsets[i];
  uint32_t len = j->offsets[i + 1] - j->offsets[i];
  uint32_t n = 0;
  for (uint64_t r = 0; r < j->n_rows; ++r)
    n += (uint32_t)oracle_row_supports(m, j->n_cols, r, seq, len, j->approx, j->neg);
  return n;
}

/* Same predicate over a float32 row-major matrix (values widened to double
 * before the comparison -- exactly what the reference computes on the
 * f32-quantised matrix).  Used for the CPU baseline on the bench workload. */
static uint32_t count_f32(const job_t* j, uint64_t i) {
  const float* m = (const float*)j->m;
  const uint32_t* seq = j->cols + j->offsets[i];
  uint32_t len = j->offsets[i + 1] - j->offsets[i];
  uint32_t n = 0;
  if (len == 0) return 0;
  for (uint64_t r = 0; r < j->n_rows; ++r) {
    const float* row = m + r * j->n_cols;
    int ok = 1;
    double prev = (double)row[seq[0]];
    for (uint32_t k = 1; k < len && ok; ++k) {
      double cur = (double)row[seq[k]];
      ok = step_ok(cur, prev, j->approx);
      prev = cur;
    }
    if (!ok && j->neg) {
      ok = 1;
      prev = (double)row[seq[len - 1]];
      for (uint32_t k = len - 1; k-- > 0 && ok;) {
        double cur = (double)row[seq[k]];
        ok = step_ok(cur, prev, j->approx);
        prev = cur;
      }
    }
    n += (uint32_t)ok;
  }
  return n;
}

static void* drain(void* arg) {
  job_t* j = (job_t*)arg;
  for (;;) {
    uint64_t b = __atomic_fetch_add(&j->next, j->chunk, __ATOMIC_RELAXED);
    if (b >= j->n_cand) break;
    uint64_t e = b + j->chunk < j->n_cand ? b + j->chunk : j->n_cand;
    for (uint64_t i = b; i < e; ++i) j->counts[i] = j->is_f32 ? count_f32(j, i) : count_f64(j, i);
  }
  return NULL;
}

int oracle_threads(void) {
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

static void run_job(job_t* j, int threads) {
  int nt = threads > 0 ? threads : oracle_threads();
  if (nt > 256) nt = 256;
  j->chunk = j->n_cand / ((uint64_t)nt * 8);
  if (j->chunk == 0) j->chunk = 1;
  j->next = 0;
  pthread_t tid[256];
  int started = 0;
  for (int t = 1; t < nt; ++t)
    if (pthread_create(&tid[started], NULL, drain, j) == 0) ++started;
  drain(j); /* the caller participates, like worker_pool.cpp:36 */
  for (int t = 0; t < started; ++t) pthread_join(tid[t], NULL);
}

/* trend.cpp:56-72.  Population in CSR form: candidate i owns
 * cols[offsets[i] .. offsets[i+1]).  threads <= 0 -> all online CPUs;
 * 1 -> sequential (the reference's null-pool branch, trend.cpp:67-68). */
void oracle_evaluate_population(const double* m, uint64_t n_rows, uint64_t n_cols,
                                const uint32_t* cols, const uint32_t* offsets, uint64_t n_cand,
                                double approx, int negative_trends, uint32_t* counts,
                                int threads) {
  job_t j = {m, 0, n_rows, n_cols, cols, offsets, n_cand, approx, negative_trends, counts, 1, 0};
  run_job(&j, threads);
}

void oracle_evaluate_population_f32(const float* m, uint64_t n_rows, uint64_t n_cols,
                                    const uint32_t* cols, const uint32_t* offsets,
                                    uint64_t n_cand, double approx, int negative_trends,
                                    uint32_t* counts, int threads) {
  job_t j = {m, 1, n_rows, n_cols, cols, offsets, n_cand, approx, negative_trends, counts, 1, 0};
  run_job(&j, threads);
}

/* trend.cpp:74-79: 0 below the floor, else count * 2^min(len, cap) (ldexp is
 * exact). */
double oracle_fitness(uint64_t support_count, uint64_t num_cols, uint64_t min_rows,
                      uint64_t col_cap) {
  if (support_count < min_rows) return 0.0;
  int bonus = (int)(num_cols < col_cap ? num_cols : col_cap);
  return ldexp((double)support_count, bonus);
}

