/*
 * bo_core.c -- ORACLE (test infrastructure): RNG, errors, partition tree.
 *
 * RNG restates /root/reference/proj/include/bfly/core.hpp:70-141 and
 * linalg.hpp:16-25.  Tree restates tree.hpp:75-201.
 */
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "bo_internal.h"

static __thread char g_err[512];

const char* bo_last_error(void) { return g_err; }

int bo_fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

/* ---------------------------------------------------------------- RNG --- */
#define BO_GAMMA 0x9e3779b97f4a7c15ULL

/* core.hpp:70-76 */
uint64_t bo_splitmix64(uint64_t* state) {
  *state += BO_GAMMA;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* core.hpp:78-88: each word folds one splitmix step into the running hash,
 * then one final step finishes the mix. */
uint64_t bo_seed_mix(uint64_t seed, int nwords, const uint64_t* words) {
  uint64_t h = seed;
  for (int i = 0; i < nwords; ++i) {
    uint64_t s = h;
    h = bo_splitmix64(&s) ^ (words[i] + BO_GAMMA);
  }
  uint64_t s = h;
  return bo_splitmix64(&s);
}

uint64_t bo_mix1(uint64_t seed, uint64_t a) { return bo_seed_mix(seed, 1, &a); }
uint64_t bo_mix2(uint64_t seed, uint64_t a, uint64_t b) {
  uint64_t w[2] = {a, b};
  return bo_seed_mix(seed, 2, w);
}
uint64_t bo_mix3(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  uint64_t w[3] = {a, b, c};
  return bo_seed_mix(seed, 3, w);
}

/* (0,1] uniform, core.hpp:119-124 */
static inline double uniform_open0(uint64_t* st) {
  uint64_t bits = bo_splitmix64(st);
  return ((double)(bits >> 11) + 1.0) * 0x1p-53;
}

/* Box-Muller pair, core.hpp:106-118: first value uses cos, spare uses sin. */
static inline void box_muller(uint64_t* st, double* c, double* s) {
  double u1 = uniform_open0(st);
  double u2 = uniform_open0(st);
  double radius = sqrt(-2.0 * log(u1));
  double angle = 2.0 * M_PI * u2;
  *s = radius * sin(angle);
  *c = radius * cos(angle);
}

/* linalg.hpp:16-25 (column-major fill, stream seeded with seed_mix(seed,"matr")).
 * Complex entries take one full Box-Muller pair (core.hpp:133-141); the real
 * stream hands out cos then the spare sin. */
int bo_gaussian(int64_t rows, int64_t cols, uint64_t seed, int is_real, bo_cplx* out) {
  if (rows < 1 || cols < 1) return bo_fail(BO_PRECONDITION, "gaussian_matrix: dimensions must be positive");
  uint64_t st = bo_mix1(seed, 0x6d617472ULL);
  int64_t total = rows * cols;
  if (!is_real) {
    for (int64_t t = 0; t < total; ++t) {
      double c, s;
      box_muller(&st, &c, &s);
      out[t] = c + I * s;
    }
  } else {
    for (int64_t t = 0; t < total; t += 2) {
      double c, s;
      box_muller(&st, &c, &s);
      out[t] = c;
      if (t + 1 < total) out[t + 1] = s;
    }
  }
  return BO_OK;
}

/* --------------------------------------------------------------- tree --- */
int bo_depth_for(int64_t n, int64_t leaf_cap) {
  if (leaf_cap < 1) return -1;
  int levels = 0;
  while ((n >> (levels + 1)) >= leaf_cap) ++levels;
  return levels;
}

static const double* g_sort_coords;
static int g_sort_axis;

/* stable merge sort of idx[0..n) keyed by coords[idx*3 + axis] */
static void merge_sort(int64_t* a, int64_t* tmp, int64_t n) {
  if (n < 2) return;
  int64_t h = n / 2;
  merge_sort(a, tmp, h);
  merge_sort(a + h, tmp, n - h);
  int64_t i = 0, j = h, k = 0;
  while (i < h && j < n) {
    double ki = g_sort_coords[a[i] * 3 + g_sort_axis];
    double kj = g_sort_coords[a[j] * 3 + g_sort_axis];
    if (kj < ki) tmp[k++] = a[j++];
    else tmp[k++] = a[i++];
  }
  while (i < h) tmp[k++] = a[i++];
  while (j < n) tmp[k++] = a[j++];
  memcpy(a, tmp, sizeof(int64_t) * (size_t)n);
}

static bo_tree* tree_alloc(int64_t n, int levels) {
  bo_tree* t = (bo_tree*)calloc(1, sizeof(bo_tree));
  t->levels = levels;
  t->n = n;
  t->perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  t->rb = (int64_t**)calloc((size_t)levels + 1, sizeof(int64_t*));
  for (int l = 0; l <= levels; ++l) t->rb[l] = (int64_t*)malloc(sizeof(int64_t) * (((size_t)1 << l) + 1));
  return t;
}

/* tree.hpp:75-101 (+ split :178-201): longest bounding-box axis, stable sort,
 * left child gets ceil(size/2). */
bo_tree* bo_tree_build(int dim, int64_t n, const double* coords, int levels) {
  if (dim < 1 || dim > 3 || n < 1) {
    bo_fail(BO_PRECONDITION, "PointSet: dim must be 1..3 and n >= 1");
    return NULL;
  }
  for (int64_t i = 0; i < n; ++i)
    for (int a = 0; a < dim; ++a)
      if (!isfinite(coords[i * 3 + a])) {
        bo_fail(BO_PRECONDITION, "PointSet: non-finite coordinate");
        return NULL;
      }
  if (levels < 0 || levels > 62 || ((int64_t)1 << levels) > n) {
    bo_fail(BO_PRECONDITION, "PartitionTree: 2^L must not exceed the point count");
    return NULL;
  }
  bo_tree* t = tree_alloc(n, levels);
  for (int64_t i = 0; i < n; ++i) t->perm[i] = i;
  t->rb[0][0] = 0;
  t->rb[0][1] = n;
  int64_t* tmp = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  g_sort_coords = coords;
  for (int l = 0; l < levels; ++l) {
    int64_t nodes = (int64_t)1 << l;
    for (int64_t j = 0; j < nodes; ++j) {
      int64_t b = t->rb[l][j], e = t->rb[l][j + 1];
      double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
      for (int a = 0; a < dim; ++a) {
        lo[a] = INFINITY;
        hi[a] = -INFINITY;
      }
      for (int64_t i = b; i < e; ++i)
        for (int a = 0; a < dim; ++a) {
          double c = coords[t->perm[i] * 3 + a];
          if (c < lo[a]) lo[a] = c;
          if (c > hi[a]) hi[a] = c;
        }
      int axis = 0;
      for (int a = 1; a < dim; ++a)
        if (hi[a] - lo[a] > hi[axis] - lo[axis]) axis = a;
      g_sort_axis = axis;
      merge_sort(t->perm + b, tmp, e - b);
      t->rb[l + 1][2 * j] = b;
      t->rb[l + 1][2 * j + 1] = b + (e - b + 1) / 2;
    }
    t->rb[l + 1][2 * nodes] = n;
  }
  free(tmp);
  return t;
}

bo_tree* bo_tree_from_table(int64_t n, int levels, const int64_t* perm, const int64_t* rb_flat) {
  bo_tree* t = tree_alloc(n, levels);
  memcpy(t->perm, perm, sizeof(int64_t) * (size_t)n);
  int64_t off = 0;
  for (int l = 0; l <= levels; ++l) {
    int64_t cnt = ((int64_t)1 << l) + 1;
    memcpy(t->rb[l], rb_flat + off, sizeof(int64_t) * (size_t)cnt);
    off += cnt;
  }
  return t;
}

bo_tree* bo_tree_copy(const bo_tree* s) {
  bo_tree* t = tree_alloc(s->n, s->levels);
  memcpy(t->perm, s->perm, sizeof(int64_t) * (size_t)s->n);
  for (int l = 0; l <= s->levels; ++l)
    memcpy(t->rb[l], s->rb[l], sizeof(int64_t) * (((size_t)1 << l) + 1));
  return t;
}

void bo_tree_free(bo_tree* t) {
  if (!t) return;
  for (int l = 0; l <= t->levels; ++l) free(t->rb[l]);
  free(t->rb);
  free(t->perm);
  free(t);
}

void bo_tree_table(const bo_tree* t, int64_t* perm_out, int64_t* rb_out) {
  if (perm_out) memcpy(perm_out, t->perm, sizeof(int64_t) * (size_t)t->n);
  if (rb_out) {
    int64_t off = 0;
    for (int l = 0; l <= t->levels; ++l) {
      int64_t cnt = ((int64_t)1 << l) + 1;
      memcpy(rb_out + off, t->rb[l], sizeof(int64_t) * (size_t)cnt);
      off += cnt;
    }
  }
}

/* ------------------------------------------------------ point sets --- */
/* Uniform points from the splitmix stream seed_mix(seed, tag): [lo, hi). */
void bo_points_uniform(int64_t n, uint64_t seed, uint64_t tag, double lo, double hi, double* out) {
  uint64_t st = bo_mix1(seed, tag);
  for (int64_t i = 0; i < n; ++i) {
    uint64_t bits = bo_splitmix64(&st);
    double u = (double)(bits >> 11) * 0x1p-53;
    out[i * 3 + 0] = lo + (hi - lo) * u;
    out[i * 3 + 1] = 0.0;
    out[i * 3 + 2] = 0.0;
  }
}

/* side x side cell-centred grid on [0,1]^2 at height z (row-major in x). */
void bo_points_plate(int64_t side, double z, double* out) {
  double h = 1.0 / (double)side;
  for (int64_t a = 0; a < side; ++a)
    for (int64_t b = 0; b < side; ++b) {
      int64_t i = a * side + b;
      out[i * 3 + 0] = ((double)b + 0.5) * h;
      out[i * 3 + 1] = ((double)a + 0.5) * h;
      out[i * 3 + 2] = z;
    }
}

/* midpoint nodes on the upper (theta in (0,pi)) or lower (pi,2pi) unit half circle */
void bo_points_half_circle(int64_t n, int upper, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    double th = ((double)i + 0.5) * M_PI / (double)n + (upper ? 0.0 : M_PI);
    out[i * 3 + 0] = cos(th);
    out[i * 3 + 1] = sin(th);
    out[i * 3 + 2] = 0.0;
  }
}
