/*
 * kmeans_oracle.c — CPU restatement of the reference Lloyd hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs as the CHECKER or the CPU
 * baseline; never linked into or called by the product path
 * (paper_1402_3788_b200/).
 *
 * Restates, in plain C with the same fp64 rounding sequence (compiled with
 * -ffp-contract=off: no FMA, like the reference's numba kernels without
 * fastmath, _kernels.py:5-9), these reference functions
 * (/root/reference/pkg/src/kmeans_regimes/):
 *   ko_assign_block        _kernels.assign_block           _kernels.py:22-45
 *   ko_cluster_sums_block  _kernels.cluster_sums_block     _kernels.py:97-113
 *   ko_self_distances      _kernels.self_distances_block   _kernels.py:116-126
 *   ko_squared_distance    _kernels.squared_distance       _kernels.py:173-180
 *   ko_wcss                model.wcss / _kernels.wcss_block model.py:206-217, _kernels.py:129-141
 *   ko_update              engine.update_step + _finish_update + model.fold_blocks
 *                          engine.py:281-294, 249-278; model.py:151-173
 *   ko_update_parallel     partition.update_parallel (block spans per worker,
 *                          placement-only assembly, one fold) partition.py:172-188,237-261
 *   ko_assign_parallel     partition.assign_parallel (plan_chunks spans) partition.py:84-100,215-234
 *   ko_converged           engine.converged                engine.py:297-310
 *   ko_iterate             engine.iterate                  engine.py:320-343
 * Pinned against vectors produced by the reference itself
 * (oracle/make_golden.py → tests/golden/*.npz, tests/test_oracle_golden.py).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EXPORT __attribute__((visibility("default")))

/* _kernels.py:22-45 — strict '<' keeps the lowest index on ties. */
EXPORT void ko_assign_block(const double* coords, int64_t m, const double* centers, int64_t k, int64_t* labels,
                            int64_t start, int64_t stop) {
  for (int64_t i = start; i < stop; ++i) {
    const double* x = coords + i * m;
    int64_t best = 0;
    double best_d2 = 0.0;
    for (int64_t f = 0; f < m; ++f) {
      double d = x[f] - centers[f];
      best_d2 += d * d;
    }
    for (int64_t c = 1; c < k; ++c) {
      double d2 = 0.0;
      const double* cc = centers + c * m;
      for (int64_t f = 0; f < m; ++f) {
        double d = x[f] - cc[f];
        d2 += d * d;
      }
      if (d2 < best_d2) {
        best_d2 = d2;
        best = c;
      }
    }
    labels[i] = best;
  }
}

/* _kernels.py:97-113 */
EXPORT int64_t ko_cluster_sums_block(const double* coords, int64_t m, const int64_t* labels, int64_t k,
                                     int64_t start, int64_t stop, double* sums, int64_t* counts) {
  for (int64_t i = start; i < stop; ++i) {
    int64_t c = labels[i];
    if (c < 0 || c >= k) return i;
    counts[c] += 1;
    for (int64_t f = 0; f < m; ++f) sums[c * m + f] += coords[i * m + f];
  }
  return -1;
}

/* _kernels.py:116-126 */
EXPORT void ko_self_distances(const double* coords, int64_t m, const double* centers, const int64_t* labels,
                              int64_t start, int64_t stop, double* out) {
  for (int64_t i = start; i < stop; ++i) {
    const double* cc = centers + labels[i] * m;
    double d2 = 0.0;
    for (int64_t f = 0; f < m; ++f) {
      double d = coords[i * m + f] - cc[f];
      d2 += d * d;
    }
    out[i] = d2;
  }
}

/* _kernels.py:173-180 */
EXPORT double ko_squared_distance(const double* a, const double* b, int64_t m) {
  double acc = 0.0;
  for (int64_t f = 0; f < m; ++f) {
    double d = a[f] - b[f];
    acc += d * d;
  }
  return acc;
}

/* model.wcss (model.py:206-217): per-block sequential sums, blocks added in order. */
EXPORT double ko_wcss(const double* coords, int64_t n, int64_t m, const double* centers, const int64_t* labels,
                      int64_t block) {
  double total = 0.0;
  for (int64_t s = 0; s < n; s += block) {
    int64_t e = s + block < n ? s + block : n;
    double acc = 0.0;
    for (int64_t i = s; i < e; ++i) {
      const double* cc = centers + labels[i] * m;
      double d2 = 0.0;
      for (int64_t f = 0; f < m; ++f) {
        double d = coords[i * m + f] - cc[f];
        d2 += d * d;
      }
      acc += d2;
    }
    total += acc;
  }
  return total;
}

/* engine.converged (engine.py:297-310) */
EXPORT int ko_converged(const double* prev, const double* next, int64_t k, int64_t m, double tol) {
  double worst = 0.0;
  for (int64_t c = 0; c < k; ++c) {
    double v = sqrt(ko_squared_distance(prev + c * m, next + c * m, m));
    if (v > worst) worst = v; /* python max(worst, v) */
  }
  return worst <= tol;
}

/* ---------------------------------------------------------------------------
 * threads: the reference's ThreadPoolExecutor fan-out (partition.py:114-119,278)
 * ------------------------------------------------------------------------- */
typedef void (*task_fn)(void* arg);
typedef struct {
  task_fn fn;
  void* arg;
} task_t;

static void* task_trampoline(void* p) {
  task_t* t = (task_t*)p;
  t->fn(t->arg);
  return NULL;
}

static void run_tasks(task_fn fn, void* args, size_t arg_size, int n) {
  if (n <= 1) {
    for (int i = 0; i < n; ++i) fn((char*)args + (size_t)i * arg_size);
    return;
  }
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n);
  task_t* ts = (task_t*)malloc(sizeof(task_t) * (size_t)n);
  for (int i = 0; i < n; ++i) {
    ts[i].fn = fn;
    ts[i].arg = (char*)args + (size_t)i * arg_size;
    pthread_create(&th[i], NULL, task_trampoline, &ts[i]);
  }
  for (int i = 0; i < n; ++i) pthread_join(th[i], NULL);
  free(th);
  free(ts);
}

/* partition.plan_chunks (partition.py:84-100): first n % w spans get +1. */
static void plan_chunk(int64_t n, int w, int i, int64_t* s, int64_t* e) {
  int64_t base = n / w, extra = n % w;
  int64_t start = (int64_t)i * base + (i < extra ? i : extra);
  *s = start;
  *e = start + base + (i < extra ? 1 : 0);
}

typedef struct {
  const double* coords;
  int64_t m;
  const double* centers;
  int64_t k;
  int64_t* labels;
  int64_t s, e;
} assign_task;

static void assign_run(void* p) {
  assign_task* t = (assign_task*)p;
  ko_assign_block(t->coords, t->m, t->centers, t->k, t->labels, t->s, t->e);
}

/* partition.assign_parallel (partition.py:215-234) + counts = bincount. */
EXPORT void ko_assign_parallel(const double* coords, int64_t n, int64_t m, const double* centers, int64_t k,
                               int64_t* labels, int64_t* counts, int n_workers) {
  int w = n_workers < 1 ? 1 : n_workers;
  if (w > n) w = (int)n;
  assign_task* ts = (assign_task*)malloc(sizeof(assign_task) * (size_t)w);
  for (int i = 0; i < w; ++i) {
    ts[i].coords = coords; ts[i].m = m; ts[i].centers = centers; ts[i].k = k; ts[i].labels = labels;
    plan_chunk(n, w, i, &ts[i].s, &ts[i].e);
  }
  run_tasks(assign_run, ts, sizeof(assign_task), w);
  free(ts);
  if (counts) {
    memset(counts, 0, sizeof(int64_t) * (size_t)k);
    for (int64_t i = 0; i < n; ++i) counts[labels[i]] += 1;
  }
}

typedef struct {
  const double* coords;
  int64_t n, m, k, block;
  const int64_t* labels;
  double* sums;      /* (n_blocks, k, m) */
  int64_t* counts;   /* (n_blocks, k) */
  int64_t b0, b1;    /* block span [b0, b1) */
  int64_t bad;
} sums_task;

static void sums_run(void* p) {
  sums_task* t = (sums_task*)p;
  t->bad = -1;
  for (int64_t b = t->b0; b < t->b1; ++b) {
    int64_t s = b * t->block, e = s + t->block < t->n ? s + t->block : t->n;
    int64_t bad = ko_cluster_sums_block(t->coords, t->m, t->labels, t->k, s, e, t->sums + b * t->k * t->m,
                                        t->counts + b * t->k);
    if (bad >= 0) { t->bad = bad; return; }
  }
}

/* engine.update_step / partition.update_parallel + _finish_update.
 * labels is modified in place by the empty-cluster repair.  Returns -1 on
 * success or the first sample index with an out-of-range label. */
EXPORT int64_t ko_update_parallel(const double* coords, int64_t n, int64_t m, int64_t* labels, int64_t k,
                                  int64_t block, double* centers_out, int64_t* counts_out, int n_workers) {
  const int64_t n_blocks = (n + block - 1) / block;
  double* sums = (double*)calloc((size_t)(n_blocks * k * m), sizeof(double));
  int64_t* bcounts = (int64_t*)calloc((size_t)(n_blocks * k), sizeof(int64_t));
  /* _block_spans = np.array_split(arange(n_blocks), w): first n_blocks % w spans +1 */
  int w = n_workers < 1 ? 1 : n_workers;
  sums_task* ts = (sums_task*)malloc(sizeof(sums_task) * (size_t)w);
  for (int i = 0; i < w; ++i) {
    int64_t s, e;
    plan_chunk(n_blocks, w, i, &s, &e);
    if (n_blocks < w) { /* array_split with more parts than items: same rule, empties at the end */
      s = i < n_blocks ? i : n_blocks;
      e = i < n_blocks ? i + 1 : n_blocks;
    }
    ts[i] = (sums_task){coords, n, m, k, block, labels, sums, bcounts, s, e, -1};
  }
  run_tasks(sums_run, ts, sizeof(sums_task), w);
  int64_t bad = -1;
  for (int i = 0; i < w; ++i)
    if (ts[i].bad >= 0 && (bad < 0 || ts[i].bad < bad)) bad = ts[i].bad;
  free(ts);
  if (bad >= 0) {
    free(sums);
    free(bcounts);
    return bad;
  }
  /* fold_blocks: out = 0; for b: out += partials[b] (model.py:163-173) */
  double* fold = (double*)calloc((size_t)(k * m), sizeof(double));
  for (int64_t b = 0; b < n_blocks; ++b)
    for (int64_t i = 0; i < k * m; ++i) fold[i] += sums[b * k * m + i];
  for (int64_t c = 0; c < k; ++c) {
    int64_t cnt = 0;
    for (int64_t b = 0; b < n_blocks; ++b) cnt += bcounts[b * k + c];
    counts_out[c] = cnt;
  }
  for (int64_t c = 0; c < k; ++c) {
    if (counts_out[c] > 0) {
      for (int64_t f = 0; f < m; ++f) centers_out[c * m + f] = fold[c * m + f] / (double)counts_out[c];
    } else {
      for (int64_t f = 0; f < m; ++f) centers_out[c * m + f] = 0.0;
    }
  }
  /* repair (engine.py:265-276) */
  int any_empty = 0;
  for (int64_t c = 0; c < k; ++c) any_empty |= counts_out[c] == 0;
  if (any_empty) {
    double* d2 = (double*)malloc(sizeof(double) * (size_t)n);
    ko_self_distances(coords, m, centers_out, labels, 0, n, d2);
    /* empties = np.flatnonzero(~occupied), computed BEFORE the loop */
    int64_t* empties = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
    int64_t ne = 0;
    for (int64_t c = 0; c < k; ++c)
      if (counts_out[c] == 0) empties[ne++] = c;
    for (int64_t q = 0; q < ne; ++q) {
      int64_t c = empties[q];
      int64_t s = 0;
      for (int64_t i = 1; i < n; ++i)
        if (d2[i] > d2[s]) s = i; /* np.argmax: first maximum */
      int64_t donor = labels[s];
      labels[s] = c;
      counts_out[donor] -= 1;
      counts_out[c] += 1;
      for (int64_t f = 0; f < m; ++f) centers_out[c * m + f] = coords[s * m + f];
      d2[s] = 0.0;
    }
    free(empties);
    free(d2);
  }
  free(fold);
  free(sums);
  free(bcounts);
  return -1;
}

EXPORT int64_t ko_update(const double* coords, int64_t n, int64_t m, int64_t* labels, int64_t k, int64_t block,
                         double* centers_out, int64_t* counts_out) {
  return ko_update_parallel(coords, n, m, labels, k, block, centers_out, counts_out, 1);
}

/* engine.iterate (engine.py:320-343) with assign/update closures over
 * n_workers threads (n_workers = 1 is run_single's closures).
 * Returns iterations; *converged_out set; centers/counts/labels written. */
EXPORT int64_t ko_iterate(const double* coords, int64_t n, int64_t m, const double* c0, int64_t k,
                          int64_t max_iters, double tol, int64_t block, int n_workers, double* centers_out,
                          int64_t* counts_out, int64_t* labels_out, int* converged_out) {
  double* model = (double*)malloc(sizeof(double) * (size_t)(k * m));
  double* next = (double*)malloc(sizeof(double) * (size_t)(k * m));
  int64_t* counts = (int64_t*)calloc((size_t)k, sizeof(int64_t));
  int64_t* next_counts = (int64_t*)calloc((size_t)k, sizeof(int64_t));
  memcpy(model, c0, sizeof(double) * (size_t)(k * m));
  ko_assign_parallel(coords, n, m, model, k, labels_out, counts, n_workers);
  int64_t iterations = 0;
  int done = 0;
  for (int64_t it = 0; it < max_iters; ++it) {
    ko_update_parallel(coords, n, m, labels_out, k, block, next, next_counts, n_workers);
    iterations += 1;
    int conv = ko_converged(model, next, k, m, tol);
    memcpy(model, next, sizeof(double) * (size_t)(k * m));
    memcpy(counts, next_counts, sizeof(int64_t) * (size_t)k);
    if (conv) {
      done = 1;
      break;
    }
    ko_assign_parallel(coords, n, m, model, k, labels_out, counts, n_workers);
  }
  memcpy(centers_out, model, sizeof(double) * (size_t)(k * m));
  memcpy(counts_out, counts, sizeof(int64_t) * (size_t)k);
  *converged_out = done;
  free(model);
  free(next);
  free(counts);
  free(next_counts);
  return iterations;
}
