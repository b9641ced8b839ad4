/*
 * bf_join.c — CPU brute-force range join: TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * An exact C restatement of the reference's `brute_force_join`
 * (/root/reference/pkg/src/tickjoin/oracle.py:17-28): a query's result set is
 * every object with xa <= x <= xb and ya <= y <= yb (closed rectangle, binary64
 * compares), listed ascending by id.  It is the checker the full-size GPU parity
 * tests use where the NumPy port (oracle/quad_oracle.py) would take minutes per
 * tick; only tests/ and bench.py's CPU legs may load it.
 *
 * Acceleration without changing the semantics: objects are bucketed into a
 * G_x x G_y grid by the monotone map c(v) = clamp(trunc(fl(fl(v - lo) * inv)),
 * 0, G - 1).  Because c is non-decreasing in v, every object with
 * xa <= x <= xb lies in a column c(xa) .. c(xb) (likewise rows), so scanning
 * those cells and applying the exact closed test visits every result; the grid
 * only prunes.  Within a grid row the cells c(xa) .. c(xb) are one contiguous
 * object range (row-major counting sort).
 *
 * Outputs per query: the result count and a 64-bit order-independent digest
 * sum(mix64(id)) mod 2^64 (splitmix64 finaliser), and, for selected queries,
 * the full sorted id lists.  Multithreaded with pthreads (dynamic chunks).
 *
 * Build: gcc -O3 -shared -fPIC -pthread oracle/bf_join.c -o oracle/_lib/libbfjoin.so
 * (done by __graft_entry__.build() and by oracle/bf_join.py on first use).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int64_t n;
  double x0, y0, invx, invy;
  int32_t gx, gy;
  int64_t* start; /* gx * gy + 1 */
  double* xs;     /* objects in cell order */
  double* ys;
  int64_t* ids;
} bf_grid;

uint64_t bf_mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xbf58476d1ce4e5b9ULL;
  z ^= z >> 27;
  z *= 0x94d049bb133111ebULL;
  z ^= z >> 31;
  return z;
}

static inline int32_t cell_of(double v, double lo, double inv, int32_t g) {
  double t = (v - lo) * inv; /* two rounded binary64 ops: non-decreasing in v */
  if (!(t > 0.0)) return 0;
  if (t >= (double)(g - 1)) return g - 1;
  return (int32_t)t;
}

/* cell: desired cell edge (e.g. the query side); gmax: cap on cells per axis */
void* bf_build(int64_t n, const double* xs, const double* ys, const int64_t* ids, double cell, int32_t gmax) {
  bf_grid* g = (bf_grid*)calloc(1, sizeof(bf_grid));
  if (!g) return NULL;
  g->n = n;
  double xa = 0, ya = 0, xb = 0, yb = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (i == 0 || xs[i] < xa) xa = xs[i];
    if (i == 0 || xs[i] > xb) xb = xs[i];
    if (i == 0 || ys[i] < ya) ya = ys[i];
    if (i == 0 || ys[i] > yb) yb = ys[i];
  }
  if (gmax < 1) gmax = 1;
  if (!(cell > 0.0)) cell = 1.0;
  double w = xb - xa, h = yb - ya;
  int64_t gx = w > 0 ? (int64_t)(w / cell) + 1 : 1;
  int64_t gy = h > 0 ? (int64_t)(h / cell) + 1 : 1;
  if (gx > gmax) gx = gmax;
  if (gy > gmax) gy = gmax;
  g->gx = (int32_t)gx;
  g->gy = (int32_t)gy;
  g->x0 = xa;
  g->y0 = ya;
  g->invx = w > 0 ? (double)gx / w : 0.0;
  g->invy = h > 0 ? (double)gy / h : 0.0;
  const int64_t nc = gx * gy;
  g->start = (int64_t*)calloc((size_t)nc + 1, sizeof(int64_t));
  g->xs = (double*)malloc((size_t)(n ? n : 1) * sizeof(double));
  g->ys = (double*)malloc((size_t)(n ? n : 1) * sizeof(double));
  g->ids = (int64_t*)malloc((size_t)(n ? n : 1) * sizeof(int64_t));
  int32_t* key = (int32_t*)malloc((size_t)(n ? n : 1) * sizeof(int32_t));
  if (!g->start || !g->xs || !g->ys || !g->ids || !key) {
    free(key);
    free(g->start), free(g->xs), free(g->ys), free(g->ids), free(g);
    return NULL;
  }
  for (int64_t i = 0; i < n; ++i) {
    const int64_t c = (int64_t)cell_of(ys[i], ya, g->invy, g->gy) * gx + cell_of(xs[i], xa, g->invx, g->gx);
    key[i] = (int32_t)c;
    g->start[c + 1]++;
  }
  for (int64_t c = 0; c < nc; ++c) g->start[c + 1] += g->start[c];
  int64_t* cur = (int64_t*)malloc((size_t)nc * sizeof(int64_t));
  memcpy(cur, g->start, (size_t)nc * sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) {
    const int64_t p = cur[key[i]]++;
    g->xs[p] = xs[i];
    g->ys[p] = ys[i];
    g->ids[p] = ids[i];
  }
  free(cur);
  free(key);
  return g;
}

void bf_free(void* p) {
  bf_grid* g = (bf_grid*)p;
  if (!g) return;
  free(g->start), free(g->xs), free(g->ys), free(g->ids), free(g);
}

typedef struct {
  const bf_grid* g;
  const int64_t* rows; /* NULL: query k is row k */
  int64_t m;
  const double *qxa, *qya, *qxb, *qyb;
  int64_t* counts;
  uint64_t* digests;
  const int64_t* offsets; /* lists mode: where query k's sorted list goes */
  int64_t* out_ids;
  int64_t next;
  int64_t bad;
} bf_job;

static int cmp_i64(const void* a, const void* b) {
  const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

static void one_query(const bf_grid* g, double a, double b, double c, double d, int64_t* cnt, uint64_t* dig,
                      int64_t* out) {
  int64_t k = 0;
  uint64_t s = 0;
  if (g->n > 0 && a <= c && b <= d) {
    const int32_t cx0 = cell_of(a, g->x0, g->invx, g->gx), cx1 = cell_of(c, g->x0, g->invx, g->gx);
    const int32_t cy0 = cell_of(b, g->y0, g->invy, g->gy), cy1 = cell_of(d, g->y0, g->invy, g->gy);
    for (int32_t cy = cy0; cy <= cy1; ++cy) {
      const int64_t row = (int64_t)cy * g->gx;
      const int64_t lo = g->start[row + cx0], hi = g->start[row + cx1 + 1];
      for (int64_t i = lo; i < hi; ++i) {
        const double x = g->xs[i], y = g->ys[i];
        if (x >= a && x <= c && y >= b && y <= d) { /* oracle.py:26, closed rectangle */
          if (out) out[k] = g->ids[i];
          s += bf_mix64((uint64_t)g->ids[i]);
          ++k;
        }
      }
    }
  }
  if (out && k > 1) qsort(out, (size_t)k, sizeof(int64_t), cmp_i64);
  *cnt = k;
  *dig = s;
}

static void* worker(void* arg) {
  bf_job* j = (bf_job*)arg;
  const int64_t chunk = 2048;
  for (;;) {
    const int64_t k0 = __atomic_fetch_add(&j->next, chunk, __ATOMIC_RELAXED);
    if (k0 >= j->m) break;
    const int64_t k1 = k0 + chunk < j->m ? k0 + chunk : j->m;
    for (int64_t k = k0; k < k1; ++k) {
      const int64_t q = j->rows ? j->rows[k] : k;
      int64_t cnt;
      uint64_t dig;
      int64_t* out = j->out_ids ? j->out_ids + j->offsets[k] : NULL;
      one_query(j->g, j->qxa[q], j->qya[q], j->qxb[q], j->qyb[q], &cnt, &dig, out);
      if (j->out_ids && cnt != j->offsets[k + 1] - j->offsets[k]) __atomic_store_n(&j->bad, 1, __ATOMIC_RELAXED);
      if (j->counts) j->counts[k] = cnt;
      if (j->digests) j->digests[k] = dig;
    }
  }
  return NULL;
}

static int run(bf_job* j, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  int started = 0;
  for (int t = 1; t < nthreads; ++t)
    if (pthread_create(&th[started], NULL, worker, j) == 0) ++started;
  worker(j);
  for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
  return j->bad ? -1 : 0;
}

/* per-query result count and digest for queries rows[0..m) (rows NULL: 0..m) */
int bf_count(void* p, int64_t m, const int64_t* rows, const double* qxa, const double* qya, const double* qxb,
             const double* qyb, int64_t* counts, uint64_t* digests, int nthreads) {
  bf_job j = {(const bf_grid*)p, rows, m, qxa, qya, qxb, qyb, counts, digests, NULL, NULL, 0, 0};
  return run(&j, nthreads);
}

/* sorted id lists of queries rows[0..m) into out_ids at offsets (m + 1, from bf_count's counts) */
int bf_lists(void* p, int64_t m, const int64_t* rows, const double* qxa, const double* qya, const double* qxb,
             const double* qyb, const int64_t* offsets, int64_t* out_ids, int nthreads) {
  bf_job j = {(const bf_grid*)p, rows, m, qxa, qya, qxb, qyb, NULL, NULL, offsets, out_ids, 0, 0};
  return run(&j, nthreads);
}

/* per-segment digest sum(mix64(id)) of a CSR (the same function as above) */
void bf_csr_digests(int64_t m, const int64_t* offsets, const int64_t* ids, uint64_t* digests) {
  for (int64_t q = 0; q < m; ++q) {
    uint64_t s = 0;
    for (int64_t i = offsets[q]; i < offsets[q + 1]; ++i) s += bf_mix64((uint64_t)ids[i]);
    digests[q] = s;
  }
}
