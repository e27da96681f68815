/*
 * bo_butterfly.c -- ORACLE (test infrastructure): hybrid butterfly container.
 *
 * Restates /root/reference/proj/include/bfly/butterfly.hpp:
 *   layout and rank accessors :20-66, apply :71-118, apply_adjoint :122-184,
 *   apply_transpose :187-193 (block-parallel over a level with OpenMP; each
 *   output block sums its contributions in the reference's sequential order), to_dense/expand_* :199-242, validate :290-326,
 *   v/u chain coefficients :330-354;
 * and the .bfh container of serialize.hpp:103-177 (format in
 * proj/docs/formats.md:3-54).
 */
#include <math.h>
#include <string.h>

#include "bo_internal.h"

bo_bf* bo_bf_alloc(int levels, int center) {
  bo_bf* bf = (bo_bf*)calloc(1, sizeof(bo_bf));
  bf->levels = levels;
  bf->center = center;
  int64_t nb = (int64_t)1 << levels;
  bf->u_leaf = (bo_mat*)calloc((size_t)nb, sizeof(bo_mat));
  bf->v_leaf = (bo_mat*)calloc((size_t)nb, sizeof(bo_mat));
  bf->b_blocks = (bo_mat*)calloc((size_t)nb, sizeof(bo_mat));
  int nr = levels - center, nw = center;
  bf->r_blocks = (bo_mat**)calloc((size_t)(nr > 0 ? nr : 1), sizeof(bo_mat*));
  for (int i = 0; i < nr; ++i) bf->r_blocks[i] = (bo_mat*)calloc((size_t)nb, sizeof(bo_mat));
  bf->w_blocks = (bo_mat**)calloc((size_t)(nw > 0 ? nw : 1), sizeof(bo_mat*));
  for (int i = 0; i < nw; ++i) bf->w_blocks[i] = (bo_mat*)calloc((size_t)nb, sizeof(bo_mat));
  return bf;
}

void bo_bf_free(bo_bf* bf) {
  if (!bf) return;
  int64_t nb = (int64_t)1 << bf->levels;
  for (int64_t i = 0; i < nb; ++i) {
    bo_mat_free(&bf->u_leaf[i]);
    bo_mat_free(&bf->v_leaf[i]);
    bo_mat_free(&bf->b_blocks[i]);
  }
  for (int l = 0; l < bf->levels - bf->center; ++l) {
    for (int64_t i = 0; i < nb; ++i) bo_mat_free(&bf->r_blocks[l][i]);
    free(bf->r_blocks[l]);
  }
  for (int l = 0; l < bf->center; ++l) {
    for (int64_t i = 0; i < nb; ++i) bo_mat_free(&bf->w_blocks[l][i]);
    free(bf->w_blocks[l]);
  }
  free(bf->u_leaf); free(bf->v_leaf); free(bf->b_blocks); free(bf->r_blocks); free(bf->w_blocks);
  bo_tree_free(bf->row_tree);
  bo_tree_free(bf->col_tree);
  free(bf);
}

bo_mat* bo_r_block(const bo_bf* bf, int l, int64_t tau, int64_t nu) {
  return &bf->r_blocks[l - bf->center][bo_bidx(bf->levels, l, tau, nu)];
}
bo_mat* bo_w_block(const bo_bf* bf, int l, int64_t tau, int64_t nu) {
  return &bf->w_blocks[l - 1][bo_bidx(bf->levels, l, tau, nu)];
}
int64_t bo_u_rank(const bo_bf* bf, int l, int64_t tau, int64_t nu) {
  if (l == bf->levels) return bf->u_leaf[tau].cols;
  return bo_r_block(bf, l, tau, nu)->cols;
}
int64_t bo_v_rank(const bo_bf* bf, int l, int64_t tau, int64_t nu) {
  if (l == 0) return bf->v_leaf[nu].cols;
  return bo_w_block(bf, l, tau, nu)->cols;
}

static void gather_rows(const bo_tree* t, const bo_cplx* x, int64_t k, bo_cplx* out) {
  int64_t n = t->n;
  for (int64_t c = 0; c < k; ++c)
    for (int64_t i = 0; i < n; ++i) out[i + c * n] = x[t->perm[i] + c * n];
}
static void scatter_rows(const bo_tree* t, const bo_cplx* x, int64_t k, bo_cplx* out) {
  int64_t n = t->n;
  for (int64_t c = 0; c < k; ++c)
    for (int64_t i = 0; i < n; ++i) out[t->perm[i] + c * n] = x[i + c * n];
}

/* [a; b] stacked into a fresh matrix */
static bo_mat stack2(const bo_mat* a, const bo_mat* b, int64_t k) {
  bo_mat s = bo_mat_new(a->rows + b->rows, k);
  for (int64_t c = 0; c < k; ++c) {
    if (a->rows) memcpy(s.a + c * s.rows, a->a + c * a->rows, sizeof(bo_cplx) * (size_t)a->rows);
    if (b->rows) memcpy(s.a + c * s.rows + a->rows, b->a + c * b->rows, sizeof(bo_cplx) * (size_t)b->rows);
  }
  return s;
}

void bo_v_chain(const bo_bf* bf, int level, int64_t tau, int64_t nu, const bo_cplx* x, int64_t ldx,
                int64_t k, bo_mat* out) {
  if (level == 0) {
    const bo_mat* v = &bf->v_leaf[nu];
    *out = bo_mat_new(v->cols, k);
    bo_gemm('H', v->cols, k, v->rows, v->a, v->rows, x, ldx, out->a, out->rows, 0);
    return;
  }
  const bo_tree* ct = bf->col_tree;
  int cl = bf->levels - level + 1;
  int64_t top = bo_node_e(ct, cl, 2 * nu) - bo_node_b(ct, cl, 2 * nu);
  bo_mat a, b;
  bo_v_chain(bf, level - 1, tau / 2, 2 * nu, x, ldx, k, &a);
  bo_v_chain(bf, level - 1, tau / 2, 2 * nu + 1, x + top, ldx, k, &b);
  bo_mat s = stack2(&a, &b, k);
  const bo_mat* w = bo_w_block(bf, level, tau, nu);
  *out = bo_mat_new(w->cols, k);
  bo_gemm('H', w->cols, k, w->rows, w->a, w->rows, s.a, s.rows, out->a, out->rows, 0);
  bo_mat_free(&a); bo_mat_free(&b); bo_mat_free(&s);
}

void bo_u_chain(const bo_bf* bf, int level, int64_t tau, int64_t nu, const bo_cplx* x, int64_t ldx,
                int64_t k, bo_mat* out) {
  if (level == bf->levels) {
    const bo_mat* u = &bf->u_leaf[tau];
    *out = bo_mat_new(u->cols, k);
    bo_gemm('H', u->cols, k, u->rows, u->a, u->rows, x, ldx, out->a, out->rows, 0);
    return;
  }
  const bo_tree* rt = bf->row_tree;
  int64_t top = bo_node_e(rt, level + 1, 2 * tau) - bo_node_b(rt, level + 1, 2 * tau);
  bo_mat a, b;
  bo_u_chain(bf, level + 1, 2 * tau, nu / 2, x, ldx, k, &a);
  bo_u_chain(bf, level + 1, 2 * tau + 1, nu / 2, x + top, ldx, k, &b);
  bo_mat s = stack2(&a, &b, k);
  const bo_mat* r = bo_r_block(bf, level, tau, nu);
  *out = bo_mat_new(r->cols, k);
  bo_gemm('H', r->cols, k, r->rows, r->a, r->rows, s.a, s.rows, out->a, out->rows, 0);
  bo_mat_free(&a); bo_mat_free(&b); bo_mat_free(&s);
}

static void free_vec(bo_mat* v, int64_t nb) {
  for (int64_t i = 0; i < nb; ++i) bo_mat_free(&v[i]);
  free(v);
}

/* K x (butterfly.hpp:71-118) */
static void apply_n(const bo_bf* bf, const bo_cplx* x, int64_t k, bo_cplx* y) {
  int L = bf->levels, lm = bf->center;
  int64_t nb = (int64_t)1 << L, n = bf->col_tree->n, m = bf->row_tree->n;
  bo_cplx* xt = (bo_cplx*)malloc(sizeof(bo_cplx) * (size_t)(n * k));
  gather_rows(bf->col_tree, x, k, xt);
  bo_mat* coef = (bo_mat*)calloc((size_t)nb, sizeof(bo_mat));
  const int nt = bo_threads();
#pragma omp parallel for schedule(static) num_threads(nt)
  for (int64_t nu = 0; nu < nb; ++nu) {
    const bo_mat* v = &bf->v_leaf[nu];
    int64_t b = bo_node_b(bf->col_tree, L, nu);
    coef[nu] = bo_mat_new(v->cols, k);
    bo_gemm('H', v->cols, k, v->rows, v->a, v->rows, xt + b, n, coef[nu].a, coef[nu].rows, 0);
  }
  for (int l = 1; l <= lm; ++l) {
    bo_mat* next = (bo_mat*)calloc((size_t)nb, sizeof(bo_mat));
#pragma omp parallel for schedule(static) num_threads(nt)
    for (int64_t e = 0; e < nb; ++e) {
      {
        const int64_t tau = e >> (L - l), nu = e & (((int64_t)1 << (L - l)) - 1);
        bo_mat s = stack2(&coef[bo_bidx(L, l - 1, tau / 2, 2 * nu)], &coef[bo_bidx(L, l - 1, tau / 2, 2 * nu + 1)], k);
        const bo_mat* w = bo_w_block(bf, l, tau, nu);
        bo_mat* o = &next[bo_bidx(L, l, tau, nu)];
        *o = bo_mat_new(w->cols, k);
        bo_gemm('H', w->cols, k, w->rows, w->a, w->rows, s.a, s.rows, o->a, o->rows, 0);
        bo_mat_free(&s);
      }
    }
    free_vec(coef, nb);
    coef = next;
  }
  bo_mat* g = (bo_mat*)calloc((size_t)nb, sizeof(bo_mat));
#pragma omp parallel for schedule(static) num_threads(nt)
  for (int64_t i = 0; i < nb; ++i) {
    const bo_mat* b = &bf->b_blocks[i];
    g[i] = bo_mat_new(b->rows, k);
    bo_gemm('N', b->rows, k, b->cols, b->a, b->rows, coef[i].a, coef[i].rows, g[i].a, g[i].rows, 0);
  }
  free_vec(coef, nb);
  for (int l = lm; l < L; ++l) {
    bo_mat* next = (bo_mat*)calloc((size_t)nb, sizeof(bo_mat));
    int64_t wide = (int64_t)1 << (L - l - 1);
    for (int64_t tau = 0; tau < ((int64_t)1 << (l + 1)); ++tau)
      for (int64_t nu = 0; nu < wide; ++nu)
        next[bo_bidx(L, l + 1, tau, nu)] = bo_mat_new(bo_u_rank(bf, l + 1, tau, nu), k);
    /* each (tau, parent nu) pair owns its two outputs; the two children nu
     * are added in the sequential order (2 pnu, then 2 pnu + 1) */
#pragma omp parallel for schedule(static) num_threads(nt)
    for (int64_t e = 0; e < (nb >> 1); ++e) {
      const int64_t tau = e / wide, pnu = e % wide;
      for (int64_t nu = 2 * pnu; nu <= 2 * pnu + 1; ++nu) {
        const bo_mat* r = bo_r_block(bf, l, tau, nu);
        bo_mat h = bo_mat_new(r->rows, k);
        const bo_mat* gi = &g[bo_bidx(L, l, tau, nu)];
        bo_gemm('N', r->rows, k, r->cols, r->a, r->rows, gi->a, gi->rows, h.a, h.rows, 0);
        bo_mat* t0 = &next[bo_bidx(L, l + 1, 2 * tau, pnu)];
        bo_mat* t1 = &next[bo_bidx(L, l + 1, 2 * tau + 1, pnu)];
        int64_t top = t0->rows;
        for (int64_t c = 0; c < k; ++c) {
          for (int64_t i = 0; i < top; ++i) t0->a[i + c * t0->rows] += h.a[i + c * h.rows];
          for (int64_t i = 0; i < t1->rows; ++i) t1->a[i + c * t1->rows] += h.a[top + i + c * h.rows];
        }
        bo_mat_free(&h);
      }
    }
    free_vec(g, nb);
    g = next;
  }
  bo_cplx* yt = (bo_cplx*)calloc((size_t)(m * k), sizeof(bo_cplx));
#pragma omp parallel for schedule(static) num_threads(nt)
  for (int64_t tau = 0; tau < nb; ++tau) {
    const bo_mat* u = &bf->u_leaf[tau];
    int64_t b = bo_node_b(bf->row_tree, L, tau);
    bo_gemm('N', u->rows, k, u->cols, u->a, u->rows, g[tau].a, g[tau].rows, yt + b, m, 0);
  }
  free_vec(g, nb);
  scatter_rows(bf->row_tree, yt, k, y);
  free(yt);
  free(xt);
}

/* K^H y (butterfly.hpp:122-184) */
static void apply_h(const bo_bf* bf, const bo_cplx* y, int64_t k, bo_cplx* x) {
  int L = bf->levels, lm = bf->center;
  int64_t nb = (int64_t)1 << L, n = bf->col_tree->n, m = bf->row_tree->n;
  bo_cplx* yt = (bo_cplx*)malloc(sizeof(bo_cplx) * (size_t)(m * k));
  gather_rows(bf->row_tree, y, k, yt);
  bo_mat* a = (bo_mat*)calloc((size_t)nb, sizeof(bo_mat));
  const int nt = bo_threads();
#pragma omp parallel for schedule(static) num_threads(nt)
  for (int64_t tau = 0; tau < nb; ++tau) {
    const bo_mat* u = &bf->u_leaf[tau];
    int64_t b = bo_node_b(bf->row_tree, L, tau);
    a[tau] = bo_mat_new(u->cols, k);
    bo_gemm('H', u->cols, k, u->rows, u->a, u->rows, yt + b, m, a[tau].a, a[tau].rows, 0);
  }
  for (int l = L - 1; l >= lm; --l) {
    bo_mat* cur = (bo_mat*)calloc((size_t)nb, sizeof(bo_mat));
#pragma omp parallel for schedule(static) num_threads(nt)
    for (int64_t e = 0; e < nb; ++e) {
      {
        const int64_t tau = e >> (L - l), nu = e & (((int64_t)1 << (L - l)) - 1);
        int64_t pnu = nu / 2;
        bo_mat s = stack2(&a[bo_bidx(L, l + 1, 2 * tau, pnu)], &a[bo_bidx(L, l + 1, 2 * tau + 1, pnu)], k);
        const bo_mat* r = bo_r_block(bf, l, tau, nu);
        bo_mat* o = &cur[bo_bidx(L, l, tau, nu)];
        *o = bo_mat_new(r->cols, k);
        bo_gemm('H', r->cols, k, r->rows, r->a, r->rows, s.a, s.rows, o->a, o->rows, 0);
        bo_mat_free(&s);
      }
    }
    free_vec(a, nb);
    a = cur;
  }
#pragma omp parallel for schedule(static) num_threads(nt)
  for (int64_t i = 0; i < nb; ++i) {
    const bo_mat* b = &bf->b_blocks[i];
    bo_mat o = bo_mat_new(b->cols, k);
    bo_gemm('H', b->cols, k, b->rows, b->a, b->rows, a[i].a, a[i].rows, o.a, o.rows, 0);
    bo_mat_free(&a[i]);
    a[i] = o;
  }
  for (int l = lm; l >= 1; --l) {
    bo_mat* prev = (bo_mat*)calloc((size_t)nb, sizeof(bo_mat));
    for (int64_t tau = 0; tau < ((int64_t)1 << (l - 1)); ++tau)
      for (int64_t nu = 0; nu < ((int64_t)1 << (L - l + 1)); ++nu)
        prev[bo_bidx(L, l - 1, tau, nu)] = bo_mat_new(bo_v_rank(bf, l - 1, tau, nu), k);
    /* each (parent tau, nu) pair owns its two outputs; the two children tau
     * are added in the sequential order (2 ptau, then 2 ptau + 1) */
    const int64_t wide = (int64_t)1 << (L - l);
#pragma omp parallel for schedule(static) num_threads(nt)
    for (int64_t q = 0; q < (nb >> 1); ++q) {
      const int64_t ptau = q / wide, nu = q % wide;
      for (int64_t tau = 2 * ptau; tau <= 2 * ptau + 1; ++tau) {
        const bo_mat* w = bo_w_block(bf, l, tau, nu);
        const bo_mat* ai = &a[bo_bidx(L, l, tau, nu)];
        bo_mat e = bo_mat_new(w->rows, k);
        bo_gemm('N', w->rows, k, w->cols, w->a, w->rows, ai->a, ai->rows, e.a, e.rows, 0);
        bo_mat* t0 = &prev[bo_bidx(L, l - 1, ptau, 2 * nu)];
        bo_mat* t1 = &prev[bo_bidx(L, l - 1, ptau, 2 * nu + 1)];
        int64_t top = t0->rows;
        for (int64_t c = 0; c < k; ++c) {
          for (int64_t i = 0; i < top; ++i) t0->a[i + c * t0->rows] += e.a[i + c * e.rows];
          for (int64_t i = 0; i < t1->rows; ++i) t1->a[i + c * t1->rows] += e.a[top + i + c * e.rows];
        }
        bo_mat_free(&e);
      }
    }
    free_vec(a, nb);
    a = prev;
  }
  bo_cplx* xt = (bo_cplx*)calloc((size_t)(n * k), sizeof(bo_cplx));
#pragma omp parallel for schedule(static) num_threads(nt)
  for (int64_t nu = 0; nu < nb; ++nu) {
    const bo_mat* v = &bf->v_leaf[nu];
    int64_t b = bo_node_b(bf->col_tree, L, nu);
    bo_gemm('N', v->rows, k, v->cols, v->a, v->rows, a[nu].a, a[nu].rows, xt + b, n, 0);
  }
  free_vec(a, nb);
  scatter_rows(bf->col_tree, xt, k, x);
  free(xt);
  free(yt);
}

int bo_bf_apply(const bo_bf* bf, int trans, const bo_cplx* x, int64_t k, bo_cplx* y) {
  int64_t m = bf->row_tree->n, n = bf->col_tree->n;
  if (trans == 0) {
    apply_n(bf, x, k, y);
  } else if (trans == 2) {
    apply_h(bf, x, k, y);
  } else {
    bo_cplx* xc = (bo_cplx*)malloc(sizeof(bo_cplx) * (size_t)(m * k));
    for (int64_t i = 0; i < m * k; ++i) xc[i] = conj(x[i]);
    apply_h(bf, xc, k, y);
    for (int64_t i = 0; i < n * k; ++i) y[i] = conj(y[i]);
    free(xc);
  }
  return BO_OK;
}

int bo_bf_validate(const bo_bf* bf) {
  int L = bf->levels, lm = bf->center;
  int64_t nb = (int64_t)1 << L;
  if (lm < 0 || lm > L) return bo_fail(BO_DIMENSION, "HybridButterfly: center level out of range");
  for (int64_t t = 0; t < nb; ++t)
    if (bf->u_leaf[t].rows != bo_node_e(bf->row_tree, L, t) - bo_node_b(bf->row_tree, L, t))
      return bo_fail(BO_DIMENSION, "HybridButterfly: U leaf height mismatch");
  for (int64_t t = 0; t < nb; ++t)
    if (bf->v_leaf[t].rows != bo_node_e(bf->col_tree, L, t) - bo_node_b(bf->col_tree, L, t))
      return bo_fail(BO_DIMENSION, "HybridButterfly: V leaf height mismatch");
  for (int l = lm; l < L; ++l)
    for (int64_t tau = 0; tau < ((int64_t)1 << l); ++tau)
      for (int64_t nu = 0; nu < ((int64_t)1 << (L - l)); ++nu)
        if (bo_r_block(bf, l, tau, nu)->rows !=
            bo_u_rank(bf, l + 1, 2 * tau, nu / 2) + bo_u_rank(bf, l + 1, 2 * tau + 1, nu / 2))
          return bo_fail(BO_DIMENSION, "HybridButterfly: R block height mismatch");
  for (int l = 1; l <= lm; ++l)
    for (int64_t tau = 0; tau < ((int64_t)1 << l); ++tau)
      for (int64_t nu = 0; nu < ((int64_t)1 << (L - l)); ++nu)
        if (bo_w_block(bf, l, tau, nu)->rows !=
            bo_v_rank(bf, l - 1, tau / 2, 2 * nu) + bo_v_rank(bf, l - 1, tau / 2, 2 * nu + 1))
          return bo_fail(BO_DIMENSION, "HybridButterfly: W block height mismatch");
  for (int64_t tau = 0; tau < ((int64_t)1 << lm); ++tau)
    for (int64_t nu = 0; nu < ((int64_t)1 << (L - lm)); ++nu) {
      const bo_mat* b = &bf->b_blocks[bo_bidx(L, lm, tau, nu)];
      if (b->rows != bo_u_rank(bf, lm, tau, nu) || b->cols != bo_v_rank(bf, lm, tau, nu))
        return bo_fail(BO_DIMENSION, "HybridButterfly: B block shape mismatch");
    }
  return BO_OK;
}

int64_t bo_bf_nnz(const bo_bf* bf) {
  int64_t nb = (int64_t)1 << bf->levels, s = 0;
  for (int64_t i = 0; i < nb; ++i)
    s += bf->u_leaf[i].rows * bf->u_leaf[i].cols + bf->v_leaf[i].rows * bf->v_leaf[i].cols +
         bf->b_blocks[i].rows * bf->b_blocks[i].cols;
  for (int l = 0; l < bf->levels - bf->center; ++l)
    for (int64_t i = 0; i < nb; ++i) s += bf->r_blocks[l][i].rows * bf->r_blocks[l][i].cols;
  for (int l = 0; l < bf->center; ++l)
    for (int64_t i = 0; i < nb; ++i) s += bf->w_blocks[l][i].rows * bf->w_blocks[l][i].cols;
  return s;
}

int64_t bo_bf_max_rank(const bo_bf* bf) {
  int64_t nb = (int64_t)1 << bf->levels, r = 0;
#define UPD(x) if ((x) > r) r = (x)
  for (int64_t i = 0; i < nb; ++i) {
    UPD(bf->u_leaf[i].cols);
    UPD(bf->v_leaf[i].cols);
  }
  for (int l = 0; l < bf->levels - bf->center; ++l)
    for (int64_t i = 0; i < nb; ++i) UPD(bf->r_blocks[l][i].cols);
  for (int l = 0; l < bf->center; ++l)
    for (int64_t i = 0; i < nb; ++i) UPD(bf->w_blocks[l][i].cols);
#undef UPD
  return r;
}

/* u ranks for levels center..L then v ranks for levels 0..center, 2^L each */
int64_t bo_bf_rank_profile(const bo_bf* bf, int32_t* out) {
  int L = bf->levels, lm = bf->center;
  int64_t nb = (int64_t)1 << L, off = 0;
  for (int l = lm; l <= L; ++l) {
    for (int64_t tau = 0; tau < ((int64_t)1 << l); ++tau)
      for (int64_t nu = 0; nu < ((int64_t)1 << (L - l)); ++nu)
        if (out) out[off + bo_bidx(L, l, tau, nu)] = (int32_t)bo_u_rank(bf, l, tau, nu);
    off += nb;
  }
  for (int l = 0; l <= lm; ++l) {
    for (int64_t tau = 0; tau < ((int64_t)1 << l); ++tau)
      for (int64_t nu = 0; nu < ((int64_t)1 << (L - l)); ++nu)
        if (out) out[off + bo_bidx(L, l, tau, nu)] = (int32_t)bo_v_rank(bf, l, tau, nu);
    off += nb;
  }
  return off;
}

/* ----------------------------------------------------- .bfh container --- */
typedef struct {
  uint8_t* buf;
  int64_t pos;
} wr_t;
static void put(wr_t* w, const void* p, int64_t n) {
  if (w->buf) memcpy(w->buf + w->pos, p, (size_t)n);
  w->pos += n;
}
static void put_u32(wr_t* w, uint32_t v) { put(w, &v, 4); }
static void put_u64(wr_t* w, uint64_t v) { put(w, &v, 8); }
static void put_tree(wr_t* w, const bo_tree* t) {
  put_u64(w, (uint64_t)t->n);
  put_u32(w, (uint32_t)t->levels);
  for (int64_t i = 0; i < t->n; ++i) put_u64(w, (uint64_t)t->perm[i]);
  for (int l = 0; l <= t->levels; ++l)
    for (int64_t j = 0; j <= ((int64_t)1 << l); ++j) put_u64(w, (uint64_t)t->rb[l][j]);
}
static void put_block(wr_t* w, const bo_mat* m, int is_real) {
  put_u64(w, (uint64_t)m->rows);
  put_u64(w, (uint64_t)m->cols);
  int64_t sz = m->rows * m->cols;
  if (!is_real) {
    put(w, m->a, sz * 16);
  } else {
    for (int64_t i = 0; i < sz; ++i) {
      double re = creal(m->a[i]);
      put(w, &re, 8);
    }
  }
}

int64_t bo_bf_serialize(const bo_bf* bf, uint8_t* buf) {
  wr_t w = {buf, 0};
  int64_t nb = (int64_t)1 << bf->levels;
  put_u32(&w, 0x31484642u);
  put_u32(&w, 1);
  uint8_t tag = bf->is_real ? 0 : 1;
  put(&w, &tag, 1);
  put_u32(&w, (uint32_t)bf->levels);
  put_u32(&w, (uint32_t)bf->center);
  put_u64(&w, (uint64_t)bf->row_tree->n);
  put_u64(&w, (uint64_t)bf->col_tree->n);
  put_u64(&w, (uint64_t)bo_bf_nnz(bf));
  put_u64(&w, (uint64_t)bo_bf_max_rank(bf));
  put_tree(&w, bf->row_tree);
  put_tree(&w, bf->col_tree);
  for (int64_t i = 0; i < nb; ++i) put_block(&w, &bf->u_leaf[i], bf->is_real);
  for (int l = 0; l < bf->levels - bf->center; ++l)
    for (int64_t i = 0; i < nb; ++i) put_block(&w, &bf->r_blocks[l][i], bf->is_real);
  for (int64_t i = 0; i < nb; ++i) put_block(&w, &bf->b_blocks[i], bf->is_real);
  for (int l = 0; l < bf->center; ++l)
    for (int64_t i = 0; i < nb; ++i) put_block(&w, &bf->w_blocks[l][i], bf->is_real);
  for (int64_t i = 0; i < nb; ++i) put_block(&w, &bf->v_leaf[i], bf->is_real);
  return w.pos;
}

typedef struct {
  const uint8_t* buf;
  int64_t pos, n;
  int bad;
} rd_t;
static void get(rd_t* r, void* p, int64_t n) {
  if (r->bad || r->pos + n > r->n) {
    r->bad = 1;
    memset(p, 0, (size_t)n);
    return;
  }
  memcpy(p, r->buf + r->pos, (size_t)n);
  r->pos += n;
}
static uint64_t get_u64(rd_t* r) {
  uint64_t v;
  get(r, &v, 8);
  return v;
}
static uint32_t get_u32(rd_t* r) {
  uint32_t v;
  get(r, &v, 4);
  return v;
}
static bo_tree* get_tree(rd_t* r) {
  int64_t n = (int64_t)get_u64(r);
  int levels = (int)get_u32(r);
  if (r->bad || levels < 0 || levels > 40 || n < 0 || n > (int64_t)1 << 40) {
    r->bad = 1;
    return NULL;
  }
  int64_t total = 0;
  for (int l = 0; l <= levels; ++l) total += ((int64_t)1 << l) + 1;
  int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  int64_t* rb = (int64_t*)malloc(sizeof(int64_t) * (size_t)total);
  for (int64_t i = 0; i < n; ++i) perm[i] = (int64_t)get_u64(r);
  for (int64_t i = 0; i < total; ++i) rb[i] = (int64_t)get_u64(r);
  bo_tree* t = r->bad ? NULL : bo_tree_from_table(n, levels, perm, rb);
  free(perm);
  free(rb);
  return t;
}
static void get_block(rd_t* r, bo_mat* m, int is_real) {
  int64_t rows = (int64_t)get_u64(r), cols = (int64_t)get_u64(r);
  if (r->bad || rows < 0 || cols < 0 || rows * cols * (is_real ? 8 : 16) > r->n - r->pos) {
    r->bad = 1;
    *m = bo_mat_new(0, 0);
    return;
  }
  *m = bo_mat_new(rows, cols);
  if (!is_real) {
    get(r, m->a, rows * cols * 16);
  } else {
    for (int64_t i = 0; i < rows * cols; ++i) {
      double v;
      get(r, &v, 8);
      m->a[i] = v;
    }
  }
}

bo_bf* bo_bf_deserialize(const uint8_t* buf, int64_t nbytes) {
  rd_t r = {buf, 0, nbytes, 0};
  uint32_t magic = get_u32(&r);
  if (r.bad) { bo_fail(BO_FORMAT, "container truncated in section header"); return NULL; }
  if (magic != 0x31484642u) { bo_fail(BO_FORMAT, "bad container magic"); return NULL; }
  uint32_t version = get_u32(&r);
  if (!r.bad && version != 1) { bo_fail(BO_FORMAT, "unsupported container version %u", version); return NULL; }
  uint8_t tag = 0;
  get(&r, &tag, 1);
  int levels = (int)get_u32(&r), center = (int)get_u32(&r);
  get_u64(&r); get_u64(&r); get_u64(&r); get_u64(&r);
  if (r.bad || levels < 0 || levels > 30 || center < 0 || center > levels) {
    bo_fail(BO_FORMAT, "container truncated in section header");
    return NULL;
  }
  bo_bf* bf = bo_bf_alloc(levels, center);
  bf->is_real = tag == 0;
  bf->row_tree = get_tree(&r);
  bf->col_tree = get_tree(&r);
  int64_t nb = (int64_t)1 << levels;
  for (int64_t i = 0; i < nb; ++i) get_block(&r, &bf->u_leaf[i], bf->is_real);
  for (int l = 0; l < levels - center; ++l)
    for (int64_t i = 0; i < nb; ++i) get_block(&r, &bf->r_blocks[l][i], bf->is_real);
  for (int64_t i = 0; i < nb; ++i) get_block(&r, &bf->b_blocks[i], bf->is_real);
  for (int l = 0; l < center; ++l)
    for (int64_t i = 0; i < nb; ++i) get_block(&r, &bf->w_blocks[l][i], bf->is_real);
  for (int64_t i = 0; i < nb; ++i) get_block(&r, &bf->v_leaf[i], bf->is_real);
  if (r.bad || !bf->row_tree || !bf->col_tree) {
    bo_bf_free(bf);
    bo_fail(BO_FORMAT, "container truncated");
    return NULL;
  }
  if (bo_bf_validate(bf) != BO_OK) {
    bo_bf_free(bf);
    return NULL;
  }
  return bf;
}

/* dense nested bases (butterfly.hpp:218-242) */
static bo_mat expand_u(const bo_bf* bf, int level, int64_t tau, int64_t nu) {
  if (level == bf->levels) {
    const bo_mat* u = &bf->u_leaf[tau];
    bo_mat o = bo_mat_new(u->rows, u->cols);
    if (u->rows * u->cols > 0) memcpy(o.a, u->a, sizeof(bo_cplx) * (size_t)(u->rows * u->cols));
    return o;
  }
  bo_mat top = expand_u(bf, level + 1, 2 * tau, nu / 2);
  bo_mat bot = expand_u(bf, level + 1, 2 * tau + 1, nu / 2);
  const bo_mat* r = bo_r_block(bf, level, tau, nu);
  bo_mat o = bo_mat_new(top.rows + bot.rows, r->cols);
  bo_gemm('N', top.rows, r->cols, top.cols, top.a, top.rows, r->a, r->rows, o.a, o.rows, 0);
  bo_gemm('N', bot.rows, r->cols, bot.cols, bot.a, bot.rows, r->a + top.cols, r->rows, o.a + top.rows, o.rows, 0);
  bo_mat_free(&top);
  bo_mat_free(&bot);
  return o;
}
static bo_mat expand_v(const bo_bf* bf, int level, int64_t tau, int64_t nu) {
  if (level == 0) {
    const bo_mat* v = &bf->v_leaf[nu];
    bo_mat o = bo_mat_new(v->rows, v->cols);
    if (v->rows * v->cols > 0) memcpy(o.a, v->a, sizeof(bo_cplx) * (size_t)(v->rows * v->cols));
    return o;
  }
  bo_mat top = expand_v(bf, level - 1, tau / 2, 2 * nu);
  bo_mat bot = expand_v(bf, level - 1, tau / 2, 2 * nu + 1);
  const bo_mat* w = bo_w_block(bf, level, tau, nu);
  bo_mat o = bo_mat_new(top.rows + bot.rows, w->cols);
  bo_gemm('N', top.rows, w->cols, top.cols, top.a, top.rows, w->a, w->rows, o.a, o.rows, 0);
  bo_gemm('N', bot.rows, w->cols, bot.cols, bot.a, bot.rows, w->a + top.cols, w->rows, o.a + top.rows, o.rows, 0);
  bo_mat_free(&top);
  bo_mat_free(&bot);
  return o;
}

int bo_bf_to_dense(const bo_bf* bf, bo_cplx* out) {
  int L = bf->levels, lm = bf->center;
  int64_t m = bf->row_tree->n, n = bf->col_tree->n;
  bo_cplx* d = (bo_cplx*)calloc((size_t)(m * n), sizeof(bo_cplx));
  for (int64_t tau = 0; tau < ((int64_t)1 << lm); ++tau)
    for (int64_t nu = 0; nu < ((int64_t)1 << (L - lm)); ++nu) {
      bo_mat u = expand_u(bf, lm, tau, nu), v = expand_v(bf, lm, tau, nu);
      const bo_mat* b = &bf->b_blocks[bo_bidx(L, lm, tau, nu)];
      bo_mat ub = bo_mat_new(u.rows, b->cols);
      bo_gemm('N', u.rows, b->cols, u.cols, u.a, u.rows, b->a, b->rows, ub.a, ub.rows, 0);
      int64_t rb = bo_node_b(bf->row_tree, lm, tau), cb = bo_node_b(bf->col_tree, L - lm, nu);
      /* block = ub * v^H */
      for (int64_t j = 0; j < v.rows; ++j)
        for (int64_t i = 0; i < ub.rows; ++i) {
          bo_cplx s = 0;
          for (int64_t c = 0; c < ub.cols; ++c) s += ub.a[i + c * ub.rows] * conj(v.a[j + c * v.rows]);
          d[(rb + i) + (cb + j) * m] = s;
        }
      bo_mat_free(&u); bo_mat_free(&v); bo_mat_free(&ub);
    }
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i)
      out[bf->row_tree->perm[i] + bf->col_tree->perm[j] * m] = d[i + j * m];
  free(d);
  return BO_OK;
}
