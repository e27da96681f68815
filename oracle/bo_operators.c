/*
 * bo_operators.c -- ORACLE (test infrastructure): black-box operators.
 *
 * BlackBoxOperator contract: /root/reference/proj/include/bfly/operators.hpp:17-66
 * (apply / apply_transpose with column counters, adjoint = conj(A^T conj(Y))).
 * DenseOperator :68-85, ButterflyOperator :105-122, synth_butterfly :124-178
 * (generalised here to leaf size b and rank r for the BASELINE config 4).
 *
 * The BASELINE operators (NUFFT, 3D plates, 2D half circles, composition) are
 * new subclasses following the kernel-evaluation pattern of operators.hpp:430-439;
 * the entry formulas are written with explicit fma() so the CUDA kernels can
 * reproduce r and the phase bit-for-bit (only sin/cos differ by ulps).
 * Entries are evaluated on the fly; all-zero input rows (structured probes,
 * reconstruct.hpp:72-85) are skipped, which changes no result.
 */
#include <math.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "bo_internal.h"

#define TWO_PI 6.283185307179586476925286766559
#define FOUR_PI 12.566370614359172953850573533118

static int g_threads = 1;
void bo_set_threads(int threads) { g_threads = threads < 1 ? 1 : threads; }
int bo_threads(void) { return g_threads; }

struct bo_op {
  int kind;
  int64_t m, n;
  int is_real;
  bo_cplx* dense;
  double* tgt;
  double* src;
  double kappa;
  bo_op* f1;
  bo_op* f2;
  bo_bf* bf;
  int64_t fwd, tr;
};

bo_op* bo_op_dense(int64_t m, int64_t n, const bo_cplx* a, int is_real) {
  bo_op* op = (bo_op*)calloc(1, sizeof(bo_op));
  op->kind = BO_OP_DENSE;
  op->m = m;
  op->n = n;
  op->is_real = is_real;
  op->dense = (bo_cplx*)malloc(sizeof(bo_cplx) * (size_t)(m * n > 0 ? m * n : 1));
  memcpy(op->dense, a, sizeof(bo_cplx) * (size_t)(m * n));
  return op;
}

bo_op* bo_op_kernel(int kind, int64_t m, int64_t n, const double* tgt, const double* src,
                    double wavenumber) {
  bo_op* op = (bo_op*)calloc(1, sizeof(bo_op));
  op->kind = kind;
  op->m = m;
  op->n = n;
  op->tgt = (double*)malloc(sizeof(double) * 3 * (size_t)m);
  op->src = (double*)malloc(sizeof(double) * 3 * (size_t)n);
  memcpy(op->tgt, tgt, sizeof(double) * 3 * (size_t)m);
  memcpy(op->src, src, sizeof(double) * 3 * (size_t)n);
  op->kappa = wavenumber;
  return op;
}

bo_op* bo_op_compose(bo_op* f2, bo_op* f1) {
  bo_op* op = (bo_op*)calloc(1, sizeof(bo_op));
  op->kind = BO_OP_COMPOSE;
  op->m = f2->m;
  op->n = f1->n;
  op->f1 = f1;
  op->f2 = f2;
  return op;
}

bo_op* bo_op_butterfly(bo_bf* bf) {
  bo_op* op = (bo_op*)calloc(1, sizeof(bo_op));
  op->kind = BO_OP_BUTTERFLY;
  op->m = bf->row_tree->n;
  op->n = bf->col_tree->n;
  op->bf = bf;
  op->is_real = bf->is_real;
  return op;
}

void bo_op_free(bo_op* op) {
  if (!op) return;
  free(op->dense);
  free(op->tgt);
  free(op->src);
  bo_op_free(op->f1);
  bo_op_free(op->f2);
  bo_bf_free(op->bf);
  free(op);
}

int64_t bo_op_rows(const bo_op* op) { return op->m; }
int64_t bo_op_cols(const bo_op* op) { return op->n; }
int bo_op_is_real(const bo_op* op) { return op->is_real; }
void bo_op_counters(const bo_op* op, int64_t* fwd, int64_t* tr) {
  *fwd = op->fwd;
  *tr = op->tr;
}
void bo_op_reset_counters(bo_op* op) { op->fwd = op->tr = 0; }

/* kernel entry K(i, j), i a target (row) index, j a source (column) index,
 * both in the operator's (tree) ordering. */
static inline bo_cplx kernel_entry(const bo_op* op, int64_t i, int64_t j) {
  const double* t = op->tgt + 3 * i;
  const double* s = op->src + 3 * j;
  if (op->kind == BO_OP_NUFFT) {
    double ph = t[0] * s[0];
    double f = ph - rint(ph);
    double ang = TWO_PI * f;
    return cos(ang) + I * sin(ang);
  }
  double dx = t[0] - s[0], dy = t[1] - s[1];
  double r;
  if (op->kind == BO_OP_PLATES) {
    double dz = t[2] - s[2];
    r = sqrt(fma(dz, dz, fma(dy, dy, dx * dx)));
    double ph = op->kappa * r;
    double sc = 1.0 / (FOUR_PI * r);
    return cos(ph) * sc + I * (sin(ph) * sc);
  }
  r = sqrt(fma(dy, dy, dx * dx));
  double ph = op->kappa * r;
  double sc = 1.0 / r;
  return cos(ph) * sc + I * (sin(ph) * sc);
}

int bo_op_entry(const bo_op* op, int64_t i, int64_t j, bo_cplx* out) {
  if (op->kind == BO_OP_DENSE) {
    *out = op->dense[i + j * op->m];
    return BO_OK;
  }
  if (op->kind == BO_OP_NUFFT || op->kind == BO_OP_PLATES || op->kind == BO_OP_CIRCLE) {
    *out = kernel_entry(op, i, j);
    return BO_OK;
  }
  return bo_fail(BO_PRECONDITION, "entry: operator has no explicit entries");
}

/* Y (nout x k) = sum over nonzero input rows: trans 0 -> K(i,j) X(j,:), trans 1 -> K(j,i) X(j,:) */
static void kernel_apply(const bo_op* op, int trans, const bo_cplx* x, int64_t k, bo_cplx* y) {
  int64_t nin = trans ? op->m : op->n, nout = trans ? op->n : op->m;
  int64_t* nz = (int64_t*)malloc(sizeof(int64_t) * (size_t)nin);
  int64_t nnz = 0;
  for (int64_t j = 0; j < nin; ++j) {
    int any = 0;
    for (int64_t c = 0; c < k && !any; ++c) any = x[j + c * nin] != 0;
    if (any) nz[nnz++] = j;
  }
  /* row-major copy of the nonzero input rows for a contiguous inner loop */
  bo_cplx* xr = (bo_cplx*)malloc(sizeof(bo_cplx) * (size_t)(nnz * k > 0 ? nnz * k : 1));
  for (int64_t t = 0; t < nnz; ++t)
    for (int64_t c = 0; c < k; ++c) xr[t * k + c] = x[nz[t] + c * nin];
#pragma omp parallel num_threads(g_threads)
  {
    bo_cplx* acc = (bo_cplx*)malloc(sizeof(bo_cplx) * (size_t)(k > 0 ? k : 1));
#pragma omp for schedule(dynamic, 16)
    for (int64_t i = 0; i < nout; ++i) {
      for (int64_t c = 0; c < k; ++c) acc[c] = 0;
      for (int64_t t = 0; t < nnz; ++t) {
        bo_cplx e = trans ? kernel_entry(op, nz[t], i) : kernel_entry(op, i, nz[t]);
        const bo_cplx* xt = xr + t * k;
        for (int64_t c = 0; c < k; ++c) acc[c] += e * xt[c];
      }
      for (int64_t c = 0; c < k; ++c) y[i + c * nout] = acc[c];
    }
    free(acc);
  }
  free(xr);
  free(nz);
}

static void do_apply(const bo_op* op, int trans, const bo_cplx* x, int64_t k, bo_cplx* y) {
  int64_t nout = trans ? op->n : op->m, nin = trans ? op->m : op->n;
  switch (op->kind) {
    case BO_OP_DENSE:
      if (!trans) {
        bo_gemm('N', op->m, k, op->n, op->dense, op->m, x, op->m == 0 ? 1 : op->n, y, op->m, 0);
      } else {
        /* plain transpose: conj(A^H conj(x)) */
        bo_cplx* xc = (bo_cplx*)malloc(sizeof(bo_cplx) * (size_t)(nin * k));
        for (int64_t i = 0; i < nin * k; ++i) xc[i] = conj(x[i]);
        bo_gemm('H', op->n, k, op->m, op->dense, op->m, xc, op->m, y, op->n, 0);
        for (int64_t i = 0; i < nout * k; ++i) y[i] = conj(y[i]);
        free(xc);
      }
      break;
    case BO_OP_NUFFT:
    case BO_OP_PLATES:
    case BO_OP_CIRCLE:
      kernel_apply(op, trans, x, k, y);
      break;
    case BO_OP_COMPOSE: {
      /* A = F2 F1 ; A^T = F1^T F2^T (two sequential black-box products) */
      const bo_op* first = trans ? op->f2 : op->f1;
      const bo_op* second = trans ? op->f1 : op->f2;
      int64_t mid = trans ? op->f2->n : op->f1->m;
      bo_cplx* tmp = (bo_cplx*)malloc(sizeof(bo_cplx) * (size_t)(mid * k));
      bo_op_apply(first, trans, x, k, tmp);
      bo_op_apply(second, trans, tmp, k, y);
      free(tmp);
      break;
    }
    case BO_OP_BUTTERFLY:
      bo_bf_apply(op->bf, trans ? 1 : 0, x, k, y);
      break;
  }
}

int bo_op_apply(const bo_op* op, int trans, const bo_cplx* x, int64_t k, bo_cplx* y) {
  bo_op* mop = (bo_op*)op; /* counters are logically mutable (operators.hpp:54-55) */
  if (trans) mop->tr += k;
  else mop->fwd += k;
  do_apply(op, trans, x, k, y);
  return BO_OK;
}

int bo_op_apply_adjoint(const bo_op* op, const bo_cplx* y, int64_t k, bo_cplx* x) {
  if (op->is_real) return bo_op_apply(op, 1, y, k, x);
  int64_t m = op->m, n = op->n;
  bo_cplx* yc = (bo_cplx*)malloc(sizeof(bo_cplx) * (size_t)(m * k > 0 ? m * k : 1));
  for (int64_t i = 0; i < m * k; ++i) yc[i] = conj(y[i]);
  bo_op_apply(op, 1, yc, k, x);
  for (int64_t i = 0; i < n * k; ++i) x[i] = conj(x[i]);
  free(yc);
  return BO_OK;
}

/* ------------------------------------------------ synthetic butterfly --- */
static void random_orthonormal(int64_t rows, int64_t cols, uint64_t seed, int is_real, bo_mat* out) {
  bo_cplx* g = (bo_cplx*)malloc(sizeof(bo_cplx) * (size_t)(rows * cols));
  bo_gaussian(rows, cols, seed, is_real, g);
  *out = bo_mat_new(rows, cols);
  bo_householder_q(rows, cols, g, out->a);
  free(g);
}

static uint64_t synth_mix(uint64_t seed, uint64_t kind, uint64_t level, uint64_t idx) {
  uint64_t w[4] = {6 /* probe_phase::synthetic */, kind, level, idx};
  return bo_seed_mix(seed, 4, w);
}

/* seeded relative Gaussian perturbation ||dX||_F = rel * ||X||_F */
static void perturb_block(bo_mat* x, uint64_t seed, uint64_t kind, uint64_t level, uint64_t idx,
                          double rel, int is_real) {
  int64_t sz = x->rows * x->cols;
  if (sz == 0 || rel == 0.0) return;
  uint64_t w[4] = {7, kind, level, idx};
  bo_cplx* e = (bo_cplx*)malloc(sizeof(bo_cplx) * (size_t)sz);
  bo_gaussian(x->rows, x->cols, bo_seed_mix(seed, 4, w), is_real, e);
  double nx = 0, ne = 0;
  for (int64_t i = 0; i < sz; ++i) {
    nx += bo_abs2(x->a[i]);
    ne += bo_abs2(e[i]);
  }
  double f = rel * sqrt(nx) / sqrt(ne);
  for (int64_t i = 0; i < sz; ++i) x->a[i] += f * e[i];
  free(e);
}

bo_bf* bo_synth_butterfly(int levels, int64_t leaf, int64_t rank, uint64_t seed, int is_real,
                          double perturb) {
  if (rank < 1 || rank > leaf) {
    bo_fail(BO_PRECONDITION, "synth_butterfly: rank must lie in [1, leaf]");
    return NULL;
  }
  if (levels < 2) {
    bo_fail(BO_PRECONDITION, "synth_butterfly: at least 2 levels required");
    return NULL;
  }
  int64_t n = ((int64_t)1 << levels) * leaf;
  bo_bf* bf = bo_bf_alloc(levels, levels / 2);
  bf->is_real = is_real;
  double* line = (double*)calloc((size_t)(3 * n), sizeof(double));
  for (int64_t i = 0; i < n; ++i) line[3 * i] = (double)i;
  bf->row_tree = bo_tree_build(1, n, line, levels);
  bf->col_tree = bo_tree_build(1, n, line, levels);
  free(line);
  int64_t nb = (int64_t)1 << levels;
  int threads = bo_threads();
#pragma omp parallel for schedule(dynamic, 8) num_threads(threads)
  for (int64_t i = 0; i < nb; ++i) {
    random_orthonormal(leaf, rank, synth_mix(seed, 1, 0, (uint64_t)i), is_real, &bf->u_leaf[i]);
    random_orthonormal(leaf, rank, synth_mix(seed, 2, 0, (uint64_t)i), is_real, &bf->v_leaf[i]);
    perturb_block(&bf->u_leaf[i], seed, 1, 0, (uint64_t)i, perturb, is_real);
    perturb_block(&bf->v_leaf[i], seed, 2, 0, (uint64_t)i, perturb, is_real);
  }
  for (int l = bf->center; l < levels; ++l) {
#pragma omp parallel for schedule(dynamic, 8) num_threads(threads)
    for (int64_t i = 0; i < nb; ++i) {
      bo_mat* b = &bf->r_blocks[l - bf->center][i];
      random_orthonormal(2 * rank, rank, synth_mix(seed, 3, (uint64_t)l, (uint64_t)i), is_real, b);
      perturb_block(b, seed, 3, (uint64_t)l, (uint64_t)i, perturb, is_real);
    }
  }
  for (int l = 1; l <= bf->center; ++l) {
#pragma omp parallel for schedule(dynamic, 8) num_threads(threads)
    for (int64_t i = 0; i < nb; ++i) {
      bo_mat* b = &bf->w_blocks[l - 1][i];
      random_orthonormal(2 * rank, rank, synth_mix(seed, 4, (uint64_t)l, (uint64_t)i), is_real, b);
      perturb_block(b, seed, 4, (uint64_t)l, (uint64_t)i, perturb, is_real);
    }
  }
#pragma omp parallel for schedule(dynamic, 8) num_threads(threads)
  for (int64_t i = 0; i < nb; ++i) {
    bf->b_blocks[i] = bo_mat_new(rank, rank);
    bo_gaussian(rank, rank, synth_mix(seed, 5, 0, (uint64_t)i), is_real, bf->b_blocks[i].a);
    perturb_block(&bf->b_blocks[i], seed, 5, 0, (uint64_t)i, perturb, is_real);
  }
  if (bo_bf_validate(bf) != BO_OK) {
    bo_bf_free(bf);
    return NULL;
  }
  return bf;
}
