/*
 * CPU oracle for the CAPT hot path -- TEST INFRASTRUCTURE ONLY (see
 * capt_oracle.h).  Restates /root/reference/pkg/src/captree/{tree,query,
 * morton,oracle}.py in C; each function cites the lines it follows.
 * Build: oracle/Makefile (gcc -O2 -fopenmp -ffp-contract=off).
 */
#define _GNU_SOURCE /* qsort_r */
#include "capt_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define KMAX 8

/* ------------------------------------------------------------------ */
/* numpy-order helpers                                                 */
/* ------------------------------------------------------------------ */

/* np.maximum: NaN-propagating max (numpy/_core/src/umath loops) */
static inline double np_maximum(double a, double b) {
  if (a != a) return a;
  if (b != b) return b;
  return a >= b ? a : b;
}

/* (res*res).sum(axis=-1) with res = max(lo - p, 0, p - hi): geom.py:130-134,
 * query.py:202-208.  Summation order ((r0^2 + r1^2) + r2^2). */
static inline double dist_sq_point_box(int k, const double* p, const double* lo,
                                       const double* hi) {
  double s = 0.0;
  for (int d = 0; d < k; ++d) {
    double r = np_maximum(lo[d] - p[d], 0.0);
    r = np_maximum(r, p[d] - hi[d]);
    double sq = r * r;
    s = (d == 0) ? sq : s + sq;
  }
  return s;
}

/* ------------------------------------------------------------------ */
/* construct -- tree.py:139-241                                        */
/* ------------------------------------------------------------------ */

struct oracle_tree {
  int k;
  int64_t n;       /* leaves */
  int64_t total;   /* stored points */
  float* tests;    /* n-1 */
  float* lo;       /* n*k */
  float* hi;       /* n*k */
  int64_t* offsets;/* n+1 */
  float* values;   /* total*k */
};

typedef struct {
  int k;
  int64_t n;
  const double* work; /* n*k, +inf padding rows */
  const uint8_t* finite;
  double r_min_sq, r_max_sq;
  int shortcut;
  float* tests;
  int32_t** sets;   /* per leaf: index list, rep first (-1 = infinity row) */
  int32_t* set_len;
  double* leaf_lo;  /* n*k */
  double* leaf_hi;
  int64_t ties;
} build_ctx;

typedef struct {
  const build_ctx* c;
  int axis;
} sort_arg;

/* (coordinate, original index) order; qsort_r keeps it reentrant so the
 * subtrees can be built by parallel OpenMP tasks */
static int cmp_coord_idx(const void* a, const void* b, void* arg) {
  int32_t i = *(const int32_t*)a, j = *(const int32_t*)b;
  const build_ctx* c = ((const sort_arg*)arg)->c;
  const int ax = ((const sort_arg*)arg)->axis;
  double x = c->work[(int64_t)i * c->k + ax];
  double y = c->work[(int64_t)j * c->k + ax];
  if (x < y) return -1;
  if (x > y) return 1;
  return (i > j) - (i < j);
}

/* emit_leaf -- tree.py:164-188 */
static void emit_leaf(build_ctx* c, int64_t leaf, int32_t rep, const double* lo,
                      const double* hi, const int32_t* z, int64_t nz) {
  int k = c->k;
  int32_t* set;
  int64_t m;
  if (!c->finite[rep]) {
    m = 1 + nz;
    set = (int32_t*)malloc(sizeof(int32_t) * m);
    set[0] = -1;
    memcpy(set + 1, z, sizeof(int32_t) * nz);
  } else {
    const double* p = c->work + (int64_t)rep * k;
    double s = 0.0;
    for (int d = 0; d < k; ++d) {
      double a = fabs(p[d] - lo[d]), b = fabs(p[d] - hi[d]);
      double corner = np_maximum(a, b);
      double sq = corner * corner;
      s = (d == 0) ? sq : s + sq;
    }
    if (c->shortcut && s <= c->r_min_sq) {
      m = 1;
      set = (int32_t*)malloc(sizeof(int32_t));
      set[0] = rep;
    } else {
      m = 1 + nz;
      set = (int32_t*)malloc(sizeof(int32_t) * m);
      set[0] = rep;
      memcpy(set + 1, z, sizeof(int32_t) * nz);
    }
  }
  c->sets[leaf] = set;
  c->set_len[leaf] = (int32_t)m;
  for (int d = 0; d < k; ++d) {
    double mn = INFINITY, mx = -INFINITY;
    for (int64_t i = 0; i < m; ++i) {
      double v = set[i] < 0 ? INFINITY : c->work[(int64_t)set[i] * k + d];
      if (v < mn) mn = v;
      if (v > mx) mx = v;
    }
    c->leaf_lo[leaf * k + d] = mn;
    c->leaf_hi[leaf * k + d] = mx;
  }
}

/* afforded(cand, lo, hi) -- tree.py:209-213: keep dist^2(p, cell) <= r_max^2 */
static int64_t afforded(build_ctx* c, const int32_t* a, int64_t na,
                        const int32_t* b, int64_t nb, const double* lo,
                        const double* hi, int32_t* out) {
  int64_t m = 0;
  for (int64_t i = 0; i < na + nb; ++i) {
    int32_t idx = i < na ? a[i] : b[i - na];
    if (dist_sq_point_box(c->k, c->work + (int64_t)idx * c->k, lo, hi) <=
        c->r_max_sq)
      out[m++] = idx;
  }
  return m;
}

/* build -- tree.py:190-220 (recursive median split) */
static void build_rec(build_ctx* c, int32_t* idx, int64_t m, const double* clo,
                      const double* chi, const int32_t* z, int64_t nz,
                      int64_t node, int depth) {
  int k = c->k;
  if (m == 1) {
    emit_leaf(c, node - (c->n - 1), idx[0], clo, chi, z, nz);
    return;
  }
  int d = depth % k;
  int64_t half = m / 2;
  /* np.argpartition(coords, half-1); ties broken by original index here */
  sort_arg sa = {c, d};
  qsort_r(idx, (size_t)m, sizeof(int32_t), cmp_coord_idx, &sa);
  double t = c->work[(int64_t)idx[half - 1] * k + d];
  double t_next = c->work[(int64_t)idx[half] * k + d];
  if (t == t_next && isfinite(t)) {
#ifdef _OPENMP
#pragma omp atomic
#endif
    c->ties++;
  }
  c->tests[node] = (float)t;
  double lo1[KMAX], hi1[KMAX], lo2[KMAX], hi2[KMAX];
  memcpy(lo1, clo, sizeof(double) * k);
  memcpy(hi1, chi, sizeof(double) * k);
  memcpy(lo2, clo, sizeof(double) * k);
  memcpy(hi2, chi, sizeof(double) * k);
  hi1[d] = t;
  lo2[d] = t;
  int32_t* left = idx;
  int32_t* right = idx + half;
  int64_t mr = m - half;
  /* finite members of each half, in partition order */
  int32_t* fin = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
  int64_t nfr = 0;
  for (int64_t i = 0; i < mr; ++i)
    if (c->finite[right[i]]) fin[nfr++] = right[i];
  int32_t* zc = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nz + m + 1));
  int64_t nz1 = afforded(c, z, nz, fin, nfr, lo1, hi1, zc);
  /* the left subtree permutes only its own idx range */
  int32_t* z1 = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nz1 + 1));
  memcpy(z1, zc, sizeof(int32_t) * nz1);
  /* left-half finite points must be captured before the left recursion
   * reorders the range (only the multiset matters; order is canonicalised) */
  int64_t nfl = 0;
  for (int64_t i = 0; i < half; ++i)
    if (c->finite[left[i]]) fin[nfl++] = left[i];
  int64_t nz2 = afforded(c, z, nz, fin, nfl, lo2, hi2, zc);
  free(fin);
  /* the two subtrees touch disjoint idx ranges, leaves and nodes: the top
   * levels run as parallel tasks (the result does not depend on the order) */
#ifdef _OPENMP
#pragma omp task if (depth < 12) firstprivate(left, half, z1, nz1, node, depth) \
    shared(lo1, hi1)
#endif
  {
    build_rec(c, left, half, lo1, hi1, z1, nz1, 2 * node + 1, depth + 1);
    free(z1);
  }
  build_rec(c, right, mr, lo2, hi2, zc, nz2, 2 * node + 2, depth + 1);
  free(zc);
#ifdef _OPENMP
#pragma omp taskwait
#endif
}

static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

static int64_t next_pow2(int64_t n) {
  int64_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

oracle_tree* oracle_construct(int k, int64_t n0, const float* pts, double r_min,
                              double r_max, int use_rmin_shortcut,
                              int64_t* n_ties) {
  if (n0 <= 0 || k <= 0 || k > KMAX) return NULL;
  int64_t n = next_pow2(n0);
  double* work = (double*)malloc(sizeof(double) * n * k);
  uint8_t* finite = (uint8_t*)calloc((size_t)n, 1);
  for (int64_t i = 0; i < n * k; ++i)
    work[i] = i < n0 * k ? (double)pts[i] : INFINITY;
  for (int64_t i = 0; i < n0; ++i) finite[i] = 1;
  build_ctx c;
  memset(&c, 0, sizeof(c));
  c.k = k;
  c.n = n;
  c.work = work;
  c.finite = finite;
  c.r_min_sq = r_min * r_min;
  c.r_max_sq = r_max * r_max;
  c.shortcut = use_rmin_shortcut;
  c.tests = (float*)malloc(sizeof(float) * (size_t)(n > 1 ? n - 1 : 1));
  for (int64_t i = 0; i < n - 1; ++i) c.tests[i] = INFINITY;
  c.sets = (int32_t**)calloc((size_t)n, sizeof(int32_t*));
  c.set_len = (int32_t*)calloc((size_t)n, sizeof(int32_t));
  c.leaf_lo = (double*)malloc(sizeof(double) * n * k);
  c.leaf_hi = (double*)malloc(sizeof(double) * n * k);
  double rlo[KMAX], rhi[KMAX];
  for (int d = 0; d < k; ++d) {
    rlo[d] = -INFINITY;
    rhi[d] = INFINITY;
  }
  if (n == 1) {
    emit_leaf(&c, 0, 0, rlo, rhi, NULL, 0);
  } else {
    int32_t* idx = (int32_t*)malloc(sizeof(int32_t) * n);
    for (int64_t i = 0; i < n; ++i) idx[i] = (int32_t)i;
#ifdef _OPENMP
#pragma omp parallel
#pragma omp single
#endif
    build_rec(&c, idx, n, rlo, rhi, NULL, 0, 0, 0);
    free(idx);
  }
  oracle_tree* t = (oracle_tree*)calloc(1, sizeof(oracle_tree));
  t->k = k;
  t->n = n;
  t->tests = c.tests;
  t->offsets = (int64_t*)malloc(sizeof(int64_t) * (n + 1));
  t->offsets[0] = 0;
  for (int64_t j = 0; j < n; ++j) t->offsets[j + 1] = t->offsets[j] + c.set_len[j];
  t->total = t->offsets[n];
  t->values = (float*)malloc(sizeof(float) * (size_t)(t->total * k + 1));
  t->lo = (float*)malloc(sizeof(float) * n * k);
  t->hi = (float*)malloc(sizeof(float) * n * k);
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 256)
#endif
  for (int64_t j = 0; j < n; ++j) {
    int64_t a = t->offsets[j], m = c.set_len[j];
    int32_t* set = c.sets[j];
    /* rows 1.. in ascending original index (deterministic) */
    if (m > 2) qsort(set + 1, (size_t)(m - 1), sizeof(int32_t), cmp_i32);
    for (int d = 0; d < k; ++d)
      for (int64_t i = 0; i < m; ++i)
        t->values[a * k + d * m + i] =
            set[i] < 0 ? INFINITY : (float)work[(int64_t)set[i] * k + d];
    for (int d = 0; d < k; ++d) {
      t->lo[j * k + d] = (float)c.leaf_lo[j * k + d];
      t->hi[j * k + d] = (float)c.leaf_hi[j * k + d];
    }
    free(set);
  }
  if (n_ties) *n_ties = c.ties;
  free(c.sets);
  free(c.set_len);
  free(c.leaf_lo);
  free(c.leaf_hi);
  free(work);
  free(finite);
  return t;
}

void oracle_tree_sizes(const oracle_tree* t, int64_t* n_leaves, int64_t* total) {
  *n_leaves = t->n;
  *total = t->total;
}

void oracle_tree_export(const oracle_tree* t, float* tests, float* lo, float* hi,
                        int64_t* offsets, float* values) {
  if (t->n > 1) memcpy(tests, t->tests, sizeof(float) * (t->n - 1));
  memcpy(lo, t->lo, sizeof(float) * t->n * t->k);
  memcpy(hi, t->hi, sizeof(float) * t->n * t->k);
  memcpy(offsets, t->offsets, sizeof(int64_t) * (t->n + 1));
  memcpy(values, t->values, sizeof(float) * t->total * t->k);
}

void oracle_tree_free(oracle_tree* t) {
  if (!t) return;
  free(t->tests);
  free(t->lo);
  free(t->hi);
  free(t->offsets);
  free(t->values);
  free(t);
}

/* ------------------------------------------------------------------ */
/* canonical order                                                     */
/* ------------------------------------------------------------------ */

static inline uint32_t f32_order(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

typedef struct {
  uint32_t key[KMAX];
} row_key;
static int cmp_row(const void* a, const void* b, void* arg) {
  const row_key* x = (const row_key*)a;
  const row_key* y = (const row_key*)b;
  const int k = *(const int*)arg;
  for (int d = 0; d < k; ++d) {
    if (x->key[d] < y->key[d]) return -1;
    if (x->key[d] > y->key[d]) return 1;
  }
  return 0;
}

void oracle_canonicalize(int k, int64_t n_leaves, const int64_t* offsets,
                         float* values) {
#ifdef _OPENMP
#pragma omp parallel
#endif
  {
  row_key* rows = NULL;
  int64_t cap = 0;
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 256)
#endif
  for (int64_t j = 0; j < n_leaves; ++j) {
    int64_t a = offsets[j], m = offsets[j + 1] - a;
    if (m <= 2) continue;
    if (m > cap) {
      cap = m;
      rows = (row_key*)realloc(rows, sizeof(row_key) * cap);
    }
    float* base = values + a * k;
    for (int64_t i = 1; i < m; ++i)
      for (int d = 0; d < k; ++d) rows[i - 1].key[d] = f32_order(base[d * m + i]);
    qsort_r(rows, (size_t)(m - 1), sizeof(row_key), cmp_row, &k);
    for (int64_t i = 1; i < m; ++i)
      for (int d = 0; d < k; ++d) {
        uint32_t u = rows[i - 1].key[d];
        u = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
        float f;
        memcpy(&f, &u, 4);
        base[d * m + i] = f;
      }
  }
  free(rows);
  }
}

/* ------------------------------------------------------------------ */
/* query -- tree.py:266-273, query.py:96-99, 184-219, 126-167          */
/* ------------------------------------------------------------------ */

static inline int64_t descend(int k, int64_t n, const float* tests,
                              const double* c) {
  int depth = 0;
  while (((int64_t)1 << depth) < n) ++depth;
  int64_t i = 0;
  for (int s = 0; s < depth; ++s)
    i = 2 * i + 1 + (c[s % k] > (double)tests[i] ? 1 : 0);
  return i - (n - 1);
}

void oracle_leaf_indices(int k, int64_t n_leaves, const float* tests,
                         const double* centers, int64_t n, int64_t* out) {
  for (int64_t q = 0; q < n; ++q)
    out[q] = descend(k, n_leaves, tests, centers + q * k);
}

/* AABB prefilter: query.py:202-208 (fp64 copies of the fp32 boxes) */
static inline int aabb_keep(int k, const float* lo, const float* hi,
                            const double* c, double r_sq) {
  double l[KMAX], h[KMAX];
  for (int d = 0; d < k; ++d) {
    l[d] = (double)lo[d];
    h[d] = (double)hi[d];
  }
  return dist_sq_point_box(k, c, l, h) <= r_sq;
}

/* _scan_leaf / per-group distance matrix: query.py:96-99, 214-218.
 * returns hit; *boundary |= some |d^2 - r^2| < 1e-6 */
static inline int scan_leaf(int k, const int64_t* offsets, const float* values,
                            int64_t leaf, const double* c, double r_sq,
                            int* boundary) {
  int64_t a = offsets[leaf], m = offsets[leaf + 1] - a;
  const float* base = values + a * k;
  int hit = 0;
  for (int64_t i = 0; i < m; ++i) {
    double s = 0.0;
    for (int d = 0; d < k; ++d) {
      double t = c[d] - (double)base[d * m + i];
      double sq = t * t;
      s = (d == 0) ? sq : s + sq;
    }
    if (s <= r_sq) hit = 1;
    if (boundary && fabs(s - r_sq) < 1e-6) *boundary = 1;
    if (hit && !boundary) break;
  }
  return hit;
}

void oracle_collides_many(int k, int64_t n_leaves, const float* tests,
                          const float* lo, const float* hi,
                          const int64_t* offsets, const float* values,
                          const double* centers, const double* radii, int64_t n,
                          int use_aabb_prefilter, uint8_t* out,
                          int64_t* counters, int nthreads) {
  int64_t hits = 0, bnd = 0, scanned = 0;
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 4096) \
    reduction(+ : hits, bnd, scanned)
#endif
  for (int64_t q = 0; q < n; ++q) {
    const double* c = centers + q * k;
    double r_sq = radii[q] * radii[q];
    int64_t leaf = descend(k, n_leaves, tests, c);
    int keep = 1;
    if (use_aabb_prefilter)
      keep = aabb_keep(k, lo + leaf * k, hi + leaf * k, c, r_sq);
    int hit = 0;
    if (keep) {
      int b = 0;
      hit = scan_leaf(k, offsets, values, leaf, c, r_sq, counters ? &b : NULL);
      bnd += b;
      scanned += offsets[leaf + 1] - offsets[leaf];
    }
    out[q] = (uint8_t)hit;
    hits += hit;
  }
  if (counters) {
    counters[0] = hits;
    counters[1] = bnd;
    counters[2] = scanned;
  }
}

void oracle_collides_groups(int k, int64_t n_leaves, const float* tests,
                            const float* lo, const float* hi,
                            const int64_t* offsets, const float* values,
                            const double* centers, const double* radii,
                            const uint8_t* mask, int64_t n_groups,
                            int lane_width, int use_aabb_prefilter,
                            uint8_t* out, int64_t* counters, int nthreads) {
  int64_t hits = 0, rej = 0, scanned = 0;
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 1024) \
    reduction(+ : hits, rej, scanned)
#endif
  for (int64_t g = 0; g < n_groups; ++g) {
    int any = 0;
    int64_t leaves[64];
    int active[64];
    /* lockstep phase: descent + AABB over all valid lanes (query.py:138-150) */
    for (int l = 0; l < lane_width; ++l) {
      int64_t q = g * lane_width + l;
      const double* c = centers + q * k;
      double r_sq = radii[q] * radii[q];
      leaves[l] = descend(k, n_leaves, tests, c);
      active[l] = mask ? (mask[q] != 0) : 1;
      if (active[l] && use_aabb_prefilter) {
        int keep = aabb_keep(k, lo + leaves[l] * k, hi + leaves[l] * k, c, r_sq);
        if (!keep) {
          ++rej;
          active[l] = 0;
        }
      }
    }
    /* lane loop with early exit (query.py:152-160) */
    for (int l = 0; l < lane_width && !any; ++l) {
      if (!active[l]) continue;
      int64_t q = g * lane_width + l;
      scanned += offsets[leaves[l] + 1] - offsets[leaves[l]];
      any = scan_leaf(k, offsets, values, leaves[l], centers + q * k,
                      radii[q] * radii[q], NULL);
    }
    out[g] = (uint8_t)any;
    hits += any;
  }
  if (counters) {
    counters[0] = hits;
    counters[1] = rej;
    counters[2] = scanned;
  }
}

/* brute_collides_many -- oracle.py:34-49 */
void oracle_brute_collides_many(int k, int64_t n_pts, const float* pts,
                                const double* centers, const double* radii,
                                int64_t n, uint8_t* out, int nthreads) {
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 256)
#endif
  for (int64_t q = 0; q < n; ++q) {
    const double* c = centers + q * k;
    double r_sq = radii[q] * radii[q];
    int hit = 0;
    for (int64_t i = 0; i < n_pts && !hit; ++i) {
      double s = 0.0;
      for (int d = 0; d < k; ++d) {
        double t = c[d] - (double)pts[i * k + d];
        double sq = t * t;
        s = (d == 0) ? sq : s + sq;
      }
      hit = s <= r_sq;
    }
    out[q] = (uint8_t)hit;
  }
}

/* ------------------------------------------------------------------ */
/* Morton filter -- morton.py:36-236                                   */
/* ------------------------------------------------------------------ */

static inline int axis_bits(int k) { return 63 / k < 21 ? 63 / k : 21; }

static inline uint64_t spread_bits(uint64_t v, int k, int bits) {
  uint64_t out = 0;
  for (int b = 0; b < bits; ++b) out |= ((v >> b) & 1ull) << (b * k);
  return out;
}

/* quantize + morton_keys -- morton.py:95-126 */
static void morton_keys_impl(int k, int64_t n, const float* pts,
                             const double* lo, const double* hi, const int* perm,
                             uint64_t* keys) {
  int bits = axis_bits(k);
  uint64_t amax = (1ull << bits) - 1;
  double span[KMAX];
  int degen[KMAX];
  for (int d = 0; d < k; ++d) {
    span[d] = hi[d] - lo[d];
    degen[d] = span[d] == 0.0;
    if (degen[d]) span[d] = 1.0;
  }
  for (int64_t i = 0; i < n; ++i) {
    uint64_t q[KMAX];
    for (int d = 0; d < k; ++d) {
      double frac = ((double)pts[i * k + d] - lo[d]) / span[d];
      double f = floor(frac * (double)amax);
      uint64_t v = (uint64_t)f;
      if (v > amax) v = amax;
      q[d] = degen[d] ? 0 : v;
    }
    uint64_t key = 0;
    for (int j = 0; j < k; ++j) key |= spread_bits(q[perm[j]], k, bits) << (k - 1 - j);
    keys[i] = key;
  }
}

void oracle_morton_keys(int k, int64_t n, const float* pts, const double* lo,
                        const double* hi, const int* perm, uint64_t* keys) {
  morton_keys_impl(k, n, pts, lo, hi, perm, keys);
}

typedef struct {
  uint64_t key;
  int64_t idx;
  int64_t pos;
} key_rec;

static int cmp_key_rec(const void* a, const void* b) {
  const key_rec* x = (const key_rec*)a;
  const key_rec* y = (const key_rec*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return (x->idx > y->idx) - (x->idx < y->idx);
}

static inline double dist_sq_pts(int k, const float* a, const float* b) {
  double s = 0.0;
  for (int d = 0; d < k; ++d) {
    double t = (double)a[d] - (double)b[d];
    double sq = t * t;
    s = (d == 0) ? sq : s + sq;
  }
  return s;
}

/* lexicographic next permutation (itertools.permutations order) */
static int next_perm(int* p, int k) {
  int i = k - 2;
  while (i >= 0 && p[i] > p[i + 1]) --i;
  if (i < 0) return 0;
  int j = k - 1;
  while (p[j] < p[i]) --j;
  int t = p[i];
  p[i] = p[j];
  p[j] = t;
  for (int a = i + 1, b = k - 1; a < b; ++a, --b) {
    t = p[a];
    p[a] = p[b];
    p[b] = t;
  }
  return 1;
}

int64_t oracle_filter_cloud(int k, int64_t n_in, const float* pts_in,
                            double r_filter, int has_reach, const double* base,
                            double max_reach, float* out) {
  /* reach_filter -- morton.py:173-182 */
  float* pts0 = (float*)malloc(sizeof(float) * (size_t)(n_in * k + 1));
  int64_t n0 = 0;
  double reach_sq = max_reach * max_reach;
  for (int64_t i = 0; i < n_in; ++i) {
    int keep = 1;
    if (has_reach) {
      double s = 0.0;
      for (int d = 0; d < k; ++d) {
        double t = (double)pts_in[i * k + d] - base[d];
        double sq = t * t;
        s = (d == 0) ? sq : s + sq;
      }
      keep = s <= reach_sq;
    }
    if (keep) {
      memcpy(pts0 + n0 * k, pts_in + i * k, sizeof(float) * k);
      ++n0;
    }
  }
  if (n0 == 0) {
    free(pts0);
    return 0;
  }
  int64_t m = n0;
  int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * n0);
  int64_t* anchor_of = (int64_t*)malloc(sizeof(int64_t) * n0);
  float* pts = (float*)malloc(sizeof(float) * n0 * k);
  float* tmp = (float*)malloc(sizeof(float) * n0 * k);
  int64_t* tidx = (int64_t*)malloc(sizeof(int64_t) * n0);
  uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * n0);
  key_rec* recs = (key_rec*)malloc(sizeof(key_rec) * n0);
  memcpy(pts, pts0, sizeof(float) * n0 * k);
  for (int64_t i = 0; i < n0; ++i) {
    idx[i] = i;
    anchor_of[i] = -1;
  }
  double r2 = r_filter * r_filter;
  int perm[KMAX];
  for (int d = 0; d < k; ++d) perm[d] = d;
  do {
    if (m <= 1) break;
    double lo[KMAX], hi[KMAX];
    for (int d = 0; d < k; ++d) {
      float mn = pts[d], mx = pts[d];
      for (int64_t i = 1; i < m; ++i) {
        float v = pts[i * k + d];
        if (v < mn) mn = v;
        if (v > mx) mx = v;
      }
      lo[d] = mn;
      hi[d] = mx;
    }
    morton_keys_impl(k, m, pts, lo, hi, perm, keys);
    for (int64_t i = 0; i < m; ++i) {
      recs[i].key = keys[i];
      recs[i].idx = idx[i];
      recs[i].pos = i;
    }
    qsort(recs, (size_t)m, sizeof(key_rec), cmp_key_rec); /* np.lexsort((idx, keys)) */
    for (int64_t i = 0; i < m; ++i) {
      memcpy(tmp + i * k, pts + recs[i].pos * k, sizeof(float) * k);
      tidx[i] = recs[i].idx;
    }
    /* _gap_scan -- morton.py:141-170 */
    int64_t nk = 0;
    int64_t last = 0;
    for (int64_t j = 0; j < m; ++j) {
      if (j == 0 || dist_sq_pts(k, tmp + j * k, tmp + last * k) > r2) {
        last = j;
        memcpy(pts + nk * k, tmp + j * k, sizeof(float) * k);
        idx[nk] = tidx[j];
        ++nk;
      } else {
        anchor_of[tidx[j]] = tidx[last];
      }
    }
    m = nk;
  } while (next_perm(perm, k));

  /* orphan repair -- morton.py:212-235 */
  uint8_t* surviving = (uint8_t*)calloc((size_t)n0, 1);
  for (int64_t i = 0; i < m; ++i) surviving[idx[i]] = 1;
  memcpy(out, pts, sizeof(float) * m * k);
  int64_t n_out = m;
  for (int64_t i = 0; i < n0; ++i) {
    if (surviving[i] || surviving[anchor_of[i]]) continue;
    int orphan = 1;
    for (int64_t s = 0; s < m && orphan; ++s)
      if (dist_sq_pts(k, pts0 + i * k, pts + s * k) <= r2) orphan = 0;
    if (orphan) {
      memcpy(out + n_out * k, pts0 + i * k, sizeof(float) * k);
      ++n_out;
    }
  }
  free(surviving);
  free(pts0);
  free(idx);
  free(anchor_of);
  free(pts);
  free(tmp);
  free(tidx);
  free(keys);
  free(recs);
  return n_out;
}
