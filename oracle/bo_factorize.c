/*
 * bo_factorize.c -- ORACLE (test infrastructure): Algorithm 2 driver.
 *
 * Restates /root/reference/proj/include/bfly/reconstruct.hpp:
 *   ReconstructionConfig :10-36, StructuredProbe/probe_with :41-85,
 *   PhaseStat/FactorizationLog :87-120, core_block :125-138,
 *   Factorizer :145-410 (leaf phases :352-399, W levels :193-240,
 *   R levels + core fit :245-305, run :308-317), estimate_error :423-434.
 * Per-node work inside a level runs under OpenMP (the reference's
 * parallel_for, core.hpp:145-163); every node writes a disjoint block, so
 * results do not depend on the thread count.
 */
#include <math.h>
#include <stdio.h>
#include <string.h>
#include <time.h>

#include "bo_internal.h"

#define TRUNCATION_SAFETY 0.25 /* reconstruct.hpp:342 */

void bo_cfg_default(bo_cfg* c) {
  c->tolerance = 1e-6;
  c->oversampling = 2;
  c->rank_guess = 4;
  c->levels = 4;
  c->center = -1;
  c->seed = 0;
  c->hard_cap = -1;
  c->threads = 1;
  c->literal_transpose_core = 0;
}

static int cfg_validate(const bo_cfg* c) {
  if (!(c->tolerance > 0.0 && c->tolerance < 1.0))
    return bo_fail(BO_PRECONDITION, "ReconstructionConfig: tolerance must lie in (0,1)");
  if (c->oversampling < 0) return bo_fail(BO_PRECONDITION, "ReconstructionConfig: oversampling >= 0");
  if (c->rank_guess < 1) return bo_fail(BO_PRECONDITION, "ReconstructionConfig: rank_guess >= 1");
  if (c->levels < 1) return bo_fail(BO_PRECONDITION, "ReconstructionConfig: levels >= 1");
  if (c->center > c->levels)
    return bo_fail(BO_PRECONDITION, "ReconstructionConfig: center level must not exceed levels");
  if (c->threads < 1) return bo_fail(BO_PRECONDITION, "ReconstructionConfig: threads >= 1");
  return BO_OK;
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

struct bo_factorizer {
  const bo_op* op;
  bo_cfg cfg;
  bo_bf* bf;
  bo_log log;
  int v_done, u_done, next_w, next_r, core_done;
  int64_t scalar_bytes;
};

bo_factorizer* bo_factorizer_new(const bo_op* op, const bo_tree* rt, const bo_tree* ct,
                                 const bo_cfg* cfg_in) {
  bo_cfg cfg = *cfg_in;
  if (cfg_validate(&cfg) != BO_OK) return NULL;
  if (rt->levels != cfg.levels || ct->levels != cfg.levels) {
    bo_fail(BO_PRECONDITION, "Factorizer: tree depth must equal the configured level count");
    return NULL;
  }
  if (rt->n != bo_op_rows(op) || ct->n != bo_op_cols(op)) {
    bo_fail(BO_DIMENSION, "Factorizer: tree sizes must match the operator dimensions");
    return NULL;
  }
  bo_factorizer* f = (bo_factorizer*)calloc(1, sizeof(bo_factorizer));
  f->op = op;
  f->cfg = cfg;
  int center = cfg.center < 0 ? cfg.levels / 2 : cfg.center;
  f->bf = bo_bf_alloc(cfg.levels, center);
  f->bf->row_tree = bo_tree_copy(rt);
  f->bf->col_tree = bo_tree_copy(ct);
  f->bf->is_real = bo_op_is_real(op);
  f->next_w = 1;
  f->next_r = cfg.levels - 1;
  f->scalar_bytes = f->bf->is_real ? 8 : 16;
  return f;
}

void bo_factorizer_free(bo_factorizer* f) {
  if (!f) return;
  bo_bf_free(f->bf);
  free(f);
}

static void note_probe_bytes(bo_factorizer* f, int64_t scalars) {
  uint64_t bytes = (uint64_t)scalars * (uint64_t)f->scalar_bytes;
  if (bytes > f->log.peak_probe_bytes) f->log.peak_probe_bytes = bytes;
  if (f->log.peak_concurrent_probes < 1) f->log.peak_concurrent_probes = 1;
}

/* Rank margin at the truncation cut (diagnostic, SURVEY 7 hard part 1): how
 * far the last kept and the first dropped pivot |R_kk| lie from the threshold
 * eps |R_00| (linalg.hpp:74-77), relative to it:
 *   min(|R_{k-1}| / thr - 1, 1 - |R_k| / thr);  +inf for a zero block.
 * A margin near 0 means a rank that rounding could flip. */
double bo_cut_margin(const double* rd, int64_t size, int64_t k, double eps) {
  if (k <= 0 || size <= 0 || rd[0] == 0.0) return HUGE_VAL;
  double thr = eps * rd[0], m = rd[k - 1] / thr - 1.0;
  if (k < size && 1.0 - rd[k] / thr < m) m = 1.0 - rd[k] / thr;
  return m;
}

/* truncate_basis (reconstruct.hpp:344-348): rank-0 for empty or all-zero input;
 * *margin = the block's cut margin */
static void truncate_basis(const bo_factorizer* f, int64_t rows, int64_t cols, const bo_cplx* z,
                           int64_t ldz, bo_mat* out, double* margin) {
  int64_t size = rows < cols ? rows : cols;
  *margin = HUGE_VAL;
  if (rows == 0 || cols == 0) {
    *out = bo_mat_new(rows, 0);
    return;
  }
  bo_cplx* q = (bo_cplx*)malloc(sizeof(bo_cplx) * (size_t)(rows * size));
  double* rd = (double*)malloc(sizeof(double) * (size_t)size);
  int64_t k = 0;
  const double eps = TRUNCATION_SAFETY * f->cfg.tolerance;
  rd[0] = 0.0;
  bo_cpqr_truncate(rows, cols, z, ldz, eps, q, &k, NULL, rd);
  *margin = bo_cut_margin(rd, size, k, eps);
  *out = bo_mat_new(rows, k);
  if (k) memcpy(out->a, q, sizeof(bo_cplx) * (size_t)(rows * k));
  free(q);
  free(rd);
}

static bo_phase* new_phase(bo_factorizer* f, const char* name) {
  bo_phase* p = &f->log.phases[f->log.nphases++];
  memset(p, 0, sizeof *p);
  snprintf(p->name, sizeof p->name, "%s", name);
  return p;
}

static void gather(const bo_tree* t, const bo_cplx* x, int64_t k, bo_cplx* out) {
  for (int64_t c = 0; c < k; ++c)
    for (int64_t i = 0; i < t->n; ++i) out[i + c * t->n] = x[t->perm[i] + c * t->n];
}

/* probe_with (reconstruct.hpp:72-85): pad the tree-ordered core into the
 * original ordering, one black-box product. */
static bo_cplx* probe_with(const bo_factorizer* f, const bo_tree* t, int level, int64_t node,
                           const bo_cplx* core, int64_t width, int forward) {
  int64_t b = bo_node_b(t, level, node), e = bo_node_e(t, level, node), h = t->n;
  bo_cplx* padded = (bo_cplx*)calloc((size_t)(h * width), sizeof(bo_cplx));
  for (int64_t i = b; i < e; ++i)
    for (int64_t c = 0; c < width; ++c) padded[t->perm[i] + c * h] = core[(i - b) + c * (e - b)];
  int64_t out_rows = forward ? bo_op_rows(f->op) : bo_op_cols(f->op);
  bo_cplx* y = (bo_cplx*)malloc(sizeof(bo_cplx) * (size_t)(out_rows * width));
  if (forward) bo_op_apply(f->op, 0, padded, width, y);
  else bo_op_apply_adjoint(f->op, padded, width, y);
  free(padded);
  return y;
}

/* run_leaf_phase (reconstruct.hpp:352-399) */
static void leaf_phase(bo_factorizer* f, const char* name, int row_side) {
  double t0 = now_s();
  int64_t f0, tr0;
  bo_op_counters(f->op, &f0, &tr0);
  bo_phase* st = new_phase(f, name);
  bo_bf* bf = f->bf;
  const bo_tree* slice = row_side ? bf->col_tree : bf->row_tree;
  int64_t m = bo_op_rows(f->op), n = bo_op_cols(f->op);
  int64_t height = row_side ? m : n, out_h = row_side ? n : m;
  int64_t hard_cap = f->cfg.hard_cap > 0 ? f->cfg.hard_cap : (m < n ? m : n);
  int64_t nb = (int64_t)1 << bf->levels;
  bo_mat* out = row_side ? bf->v_leaf : bf->u_leaf;
  uint64_t tag = row_side ? 1 : 2;
  int64_t r = f->cfg.rank_guess;
  for (int round = 0;; ++round) {
    int64_t width = r + f->cfg.oversampling;
    if (width > st->probe_width) st->probe_width = width;
    bo_cplx* omega = (bo_cplx*)malloc(sizeof(bo_cplx) * (size_t)(height * width));
    bo_gaussian(height, width, bo_mix2(f->cfg.seed, tag, (uint64_t)round), bf->is_real, omega);
    bo_cplx* prod = (bo_cplx*)malloc(sizeof(bo_cplx) * (size_t)(out_h * width));
    if (row_side) bo_op_apply_adjoint(f->op, omega, width, prod);
    else bo_op_apply(f->op, 0, omega, width, prod);
    note_probe_bytes(f, height * width + out_h * width);
    bo_cplx* pt = (bo_cplx*)malloc(sizeof(bo_cplx) * (size_t)(out_h * width));
    gather(slice, prod, width, pt);
    int64_t max_rank = 0;
    double mg = HUGE_VAL;
#pragma omp parallel for schedule(dynamic) num_threads(f->cfg.threads) reduction(max : max_rank) reduction(min : mg)
    for (int64_t leaf = 0; leaf < nb; ++leaf) {
      int64_t b = bo_node_b(slice, bf->levels, leaf), e = bo_node_e(slice, bf->levels, leaf);
      bo_mat_free(&out[leaf]);
      double m1;
      truncate_basis(f, e - b, width, pt + b, out_h, &out[leaf], &m1);
      if (m1 < mg) mg = m1;
      if (out[leaf].cols > max_rank) max_rank = out[leaf].cols;
    }
    free(omega);
    free(prod);
    free(pt);
    st->rounds = round;
    st->rank_margin = mg; /* the kept (last) round's blocks */
    if (r > max_rank) break;
    if (r >= hard_cap) {
      f->log.rank_capped = 1;
      break;
    }
    r = 2 * r < hard_cap ? 2 * r : hard_cap;
  }
  int64_t f1, tr1;
  bo_op_counters(f->op, &f1, &tr1);
  st->forward_columns = f1 - f0;
  st->transpose_columns = tr1 - tr0;
  st->seconds = now_s() - t0;
}

int bo_factorizer_leaf_row(bo_factorizer* f) {
  if (f->v_done) return bo_fail(BO_SEQUENCING, "Factorizer: leaf_row_bases already ran");
  leaf_phase(f, "leaf_v", 1);
  f->v_done = 1;
  return BO_OK;
}

int bo_factorizer_leaf_col(bo_factorizer* f) {
  if (!f->v_done) return bo_fail(BO_SEQUENCING, "Factorizer: leaf_row_bases must run first");
  if (f->u_done) return bo_fail(BO_SEQUENCING, "Factorizer: leaf_col_bases already ran");
  leaf_phase(f, "leaf_u", 0);
  f->u_done = 1;
  return BO_OK;
}

/* stack [top; bot] (each rows x k with their own ld) */
static bo_mat stack_mats(const bo_mat* a, const bo_mat* b, int64_t k) {
  bo_mat s = bo_mat_new(a->rows + b->rows, k);
  for (int64_t c = 0; c < k; ++c) {
    if (a->rows) memcpy(s.a + c * s.rows, a->a + c * a->rows, sizeof(bo_cplx) * (size_t)a->rows);
    if (b->rows) memcpy(s.a + c * s.rows + a->rows, b->a + c * b->rows, sizeof(bo_cplx) * (size_t)b->rows);
  }
  return s;
}

/* transfer_level_w (reconstruct.hpp:193-240) */
int bo_factorizer_transfer_w(bo_factorizer* f, int l) {
  if (!f->u_done) return bo_fail(BO_SEQUENCING, "Factorizer: leaf phases must run first");
  if (l != f->next_w) return bo_fail(BO_SEQUENCING, "Factorizer: W levels must run in order 1..l_m");
  double t0 = now_s();
  int64_t f0, tr0;
  bo_op_counters(f->op, &f0, &tr0);
  char name[32];
  snprintf(name, sizeof name, "transfer_w_%d", l);
  bo_phase* st = new_phase(f, name);
  bo_bf* bf = f->bf;
  int L = bf->levels;
  int64_t ntau = (int64_t)1 << l, nnu = (int64_t)1 << (L - l), n = bf->col_tree->n;
  double mg = HUGE_VAL;
  for (int64_t tau = 0; tau < ntau; ++tau) {
    int64_t bound = 0;
    for (int64_t nu = 0; nu < nnu; ++nu) {
      int64_t s = bo_v_rank(bf, l - 1, tau / 2, 2 * nu) + bo_v_rank(bf, l - 1, tau / 2, 2 * nu + 1);
      if (s > bound) bound = s;
    }
    if (bound == 0) {
      for (int64_t nu = 0; nu < nnu; ++nu) {
        bo_mat* w = bo_w_block(bf, l, tau, nu);
        bo_mat_free(w);
        *w = bo_mat_new(0, 0);
      }
      continue;
    }
    int64_t width = bound + f->cfg.oversampling;
    if (width > st->probe_width) st->probe_width = width;
    int64_t hb = bo_node_b(bf->row_tree, l, tau), he = bo_node_e(bf->row_tree, l, tau);
    bo_cplx* core = (bo_cplx*)malloc(sizeof(bo_cplx) * (size_t)((he - hb) * width));
    bo_gaussian(he - hb, width, bo_mix3(f->cfg.seed, 3, (uint64_t)l, (uint64_t)tau), bf->is_real, core);
    bo_cplx* x = probe_with(f, bf->row_tree, l, tau, core, width, 0);
    note_probe_bytes(f, (he - hb) * width + n * width);
    bo_cplx* xt = (bo_cplx*)malloc(sizeof(bo_cplx) * (size_t)(n * width));
    gather(bf->col_tree, x, width, xt);
#pragma omp parallel for schedule(dynamic) num_threads(f->cfg.threads) reduction(min : mg)
    for (int64_t nu = 0; nu < nnu; ++nu) {
      int cl = L - l + 1;
      int64_t b1 = bo_node_b(bf->col_tree, cl, 2 * nu), b2 = bo_node_b(bf->col_tree, cl, 2 * nu + 1);
      bo_mat top, bot;
      bo_v_chain(bf, l - 1, tau / 2, 2 * nu, xt + b1, n, width, &top);
      bo_v_chain(bf, l - 1, tau / 2, 2 * nu + 1, xt + b2, n, width, &bot);
      bo_mat z = stack_mats(&top, &bot, width);
      bo_mat* w = bo_w_block(bf, l, tau, nu);
      bo_mat_free(w);
      double m1;
      truncate_basis(f, z.rows, z.cols, z.a, z.rows, w, &m1);
      if (m1 < mg) mg = m1;
      bo_mat_free(&top); bo_mat_free(&bot); bo_mat_free(&z);
    }
    free(core);
    free(x);
    free(xt);
  }
  st->rank_margin = mg;
  int64_t f1, tr1;
  bo_op_counters(f->op, &f1, &tr1);
  st->forward_columns = f1 - f0;
  st->transpose_columns = tr1 - tr0;
  st->seconds = now_s() - t0;
  ++f->next_w;
  return BO_OK;
}

/* core_block (reconstruct.hpp:125-138) */
static int core_block(const bo_mat* z, const bo_mat* u, const bo_mat* coeff, int literal, bo_mat* out) {
  if (u->rows != z->rows) return bo_fail(BO_DIMENSION, "core_block: U height mismatch");
  if (coeff->cols != z->cols) return bo_fail(BO_DIMENSION, "core_block: probe width mismatch between sides");
  if (coeff->cols < coeff->rows)
    return bo_fail(BO_PRECONDITION,
                   "core_block: underdetermined fit; the probe needs at least as many columns as the V rank");
  int64_t w = z->cols;
  bo_mat proj = bo_mat_new(u->cols, w);
  bo_gemm('H', u->cols, w, u->rows, u->a, u->rows, z->a, z->rows, proj.a, proj.rows, 0);
  if (coeff->rows == 0) {
    *out = bo_mat_new(proj.rows, 0);
    bo_mat_free(&proj);
    return BO_OK;
  }
  *out = bo_mat_new(proj.rows, coeff->rows);
  if (literal) {
    /* projected * coeff^T (no conjugation) */
    for (int64_t j = 0; j < coeff->rows; ++j)
      for (int64_t i = 0; i < proj.rows; ++i) {
        bo_cplx s = 0;
        for (int64_t c = 0; c < w; ++c) s += proj.a[i + c * proj.rows] * coeff->a[j + c * coeff->rows];
        out->a[i + j * out->rows] = s;
      }
  } else {
    bo_cplx* pinv = (bo_cplx*)malloc(sizeof(bo_cplx) * (size_t)(w * coeff->rows));
    bo_pinv(coeff->rows, w, coeff->a, 1e-12, pinv);
    bo_gemm('N', proj.rows, coeff->rows, w, proj.a, proj.rows, pinv, w, out->a, out->rows, 0);
    free(pinv);
  }
  bo_mat_free(&proj);
  return BO_OK;
}

/* exported for tests: core_block on plain arrays; out is (u_cols x coeff_rows) */
int bo_core_block(int64_t zr, int64_t w, const bo_cplx* z, int64_t ur, int64_t uc, const bo_cplx* u, int64_t cr,
                  int64_t cc, const bo_cplx* coeff, int literal, bo_cplx* out) {
  bo_mat Z = {zr, w, (bo_cplx*)z}, U = {ur, uc, (bo_cplx*)u}, Cf = {cr, cc, (bo_cplx*)coeff}, B;
  int e = core_block(&Z, &U, &Cf, literal, &B);
  if (e != BO_OK) return e;
  if (B.rows * B.cols > 0) memcpy(out, B.a, sizeof(bo_cplx) * (size_t)(B.rows * B.cols));
  bo_mat_free(&B);
  return BO_OK;
}

/* exported for tests: probe_with (reconstruct.hpp:72-85) */
int bo_probe_with(const bo_op* op, const bo_tree* t, int level, int64_t node, const bo_cplx* core, int64_t core_rows,
                  int64_t width, int forward, bo_cplx* out) {
  if (core_rows != bo_node_e(t, level, node) - bo_node_b(t, level, node))
    return bo_fail(BO_DIMENSION, "probe_with: core height does not match the owner node");
  if (t->n != (forward ? bo_op_cols(op) : bo_op_rows(op)))
    return bo_fail(BO_DIMENSION, "probe_with: tree size does not match the operator");
  bo_factorizer tmp;
  memset(&tmp, 0, sizeof tmp);
  tmp.op = op;
  bo_cplx* y = probe_with(&tmp, t, level, node, core, width, forward);
  int64_t rows = forward ? bo_op_rows(op) : bo_op_cols(op);
  memcpy(out, y, sizeof(bo_cplx) * (size_t)(rows * width));
  free(y);
  return BO_OK;
}

/* transfer_level_r (reconstruct.hpp:245-305) */
int bo_factorizer_transfer_r(bo_factorizer* f, int l) {
  bo_bf* bf = f->bf;
  if (f->next_w <= bf->center) return bo_fail(BO_SEQUENCING, "Factorizer: W levels must finish first");
  if (l != f->next_r) return bo_fail(BO_SEQUENCING, "Factorizer: R levels must run in order L-1..l_m");
  double t0 = now_s();
  int64_t f0, tr0;
  bo_op_counters(f->op, &f0, &tr0);
  char name[32];
  snprintf(name, sizeof name, "transfer_r_%d", l);
  bo_phase* st = new_phase(f, name);
  int L = bf->levels;
  int at_center = l == bf->center;
  int64_t ntau = (int64_t)1 << l, nnu = (int64_t)1 << (L - l), m = bf->row_tree->n;
  int err = BO_OK;
  double mg = HUGE_VAL;
  for (int64_t nu = 0; nu < nnu && err == BO_OK; ++nu) {
    int64_t bound = 0;
    for (int64_t tau = 0; tau < ntau; ++tau) {
      int64_t s = bo_u_rank(bf, l + 1, 2 * tau, nu / 2) + bo_u_rank(bf, l + 1, 2 * tau + 1, nu / 2);
      if (s > bound) bound = s;
    }
    if (bound == 0) {
      for (int64_t tau = 0; tau < ntau; ++tau) {
        bo_mat* r = bo_r_block(bf, l, tau, nu);
        bo_mat_free(r);
        *r = bo_mat_new(0, 0);
        if (at_center) {
          bo_mat* b = &bf->b_blocks[bo_bidx(L, l, tau, nu)];
          bo_mat_free(b);
          *b = bo_mat_new(0, bo_v_rank(bf, bf->center, tau, nu));
        }
      }
      continue;
    }
    int64_t width = bound + f->cfg.oversampling;
    if (width > st->probe_width) st->probe_width = width;
    int cl = L - l;
    int64_t sb = bo_node_b(bf->col_tree, cl, nu), se = bo_node_e(bf->col_tree, cl, nu);
    bo_cplx* core = (bo_cplx*)malloc(sizeof(bo_cplx) * (size_t)((se - sb) * width));
    bo_gaussian(se - sb, width, bo_mix3(f->cfg.seed, 4, (uint64_t)l, (uint64_t)nu), bf->is_real, core);
    bo_cplx* y = probe_with(f, bf->col_tree, cl, nu, core, width, 1);
    note_probe_bytes(f, (se - sb) * width + m * width);
    bo_cplx* yt = (bo_cplx*)malloc(sizeof(bo_cplx) * (size_t)(m * width));
    gather(bf->row_tree, y, width, yt);
#pragma omp parallel for schedule(dynamic) num_threads(f->cfg.threads) reduction(min : mg)
    for (int64_t tau = 0; tau < ntau; ++tau) {
      int64_t b1 = bo_node_b(bf->row_tree, l + 1, 2 * tau), b2 = bo_node_b(bf->row_tree, l + 1, 2 * tau + 1);
      bo_mat top, bot;
      bo_u_chain(bf, l + 1, 2 * tau, nu / 2, yt + b1, m, width, &top);
      bo_u_chain(bf, l + 1, 2 * tau + 1, nu / 2, yt + b2, m, width, &bot);
      bo_mat z = stack_mats(&top, &bot, width);
      bo_mat r;
      double m1;
      truncate_basis(f, z.rows, z.cols, z.a, z.rows, &r, &m1);
      if (m1 < mg) mg = m1;
      if (at_center) {
        bo_mat coeff;
        bo_v_chain(bf, bf->center, tau, nu, core, se - sb, width, &coeff);
        bo_mat* b = &bf->b_blocks[bo_bidx(L, l, tau, nu)];
        bo_mat_free(b);
        int e = core_block(&z, &r, &coeff, f->cfg.literal_transpose_core, b);
        if (e != BO_OK) {
#pragma omp critical
          err = e;
        }
        bo_mat_free(&coeff);
      }
      bo_mat* rr = bo_r_block(bf, l, tau, nu);
      bo_mat_free(rr);
      *rr = r;
      bo_mat_free(&top); bo_mat_free(&bot); bo_mat_free(&z);
    }
    free(core);
    free(y);
    free(yt);
  }
  if (err != BO_OK) return err;
  st->rank_margin = mg;
  int64_t f1, tr1;
  bo_op_counters(f->op, &f1, &tr1);
  st->forward_columns = f1 - f0;
  st->transpose_columns = tr1 - tr0;
  st->seconds = now_s() - t0;
  --f->next_r;
  if (f->next_r < bf->center) f->core_done = 1;
  return BO_OK;
}

int bo_factorizer_complete(const bo_factorizer* f) { return f->core_done; }

bo_bf* bo_factorizer_take(bo_factorizer* f, bo_log* log) {
  bo_bf* bf = f->bf;
  f->bf = NULL;
  if (log) *log = f->log;
  return bf;
}

int bo_factorize(const bo_op* op, const bo_tree* rt, const bo_tree* ct, const bo_cfg* cfg,
                 bo_bf** bf_out, bo_log* log) {
  *bf_out = NULL;
  bo_factorizer* f = bo_factorizer_new(op, rt, ct, cfg);
  if (!f) return BO_PRECONDITION;
  double t0 = now_s();
  int e = bo_factorizer_leaf_row(f);
  if (e == BO_OK) e = bo_factorizer_leaf_col(f);
  for (int l = 1; e == BO_OK && l <= f->bf->center; ++l) e = bo_factorizer_transfer_w(f, l);
  for (int l = f->bf->levels - 1; e == BO_OK && l >= f->bf->center; --l) e = bo_factorizer_transfer_r(f, l);
  if (e == BO_OK) {
    f->log.total_seconds = now_s() - t0;
    e = bo_bf_validate(f->bf);
  }
  if (e == BO_OK) *bf_out = bo_factorizer_take(f, log);
  bo_factorizer_free(f);
  return e;
}

/* estimate_error (reconstruct.hpp:423-434) */
int bo_estimate_error(const bo_op* op, const bo_bf* bf, int64_t k, uint64_t seed, double* err) {
  if (k < 1) return bo_fail(BO_PRECONDITION, "estimate_error: k >= 1 required");
  int64_t m = bo_op_rows(op), n = bo_op_cols(op);
  bo_cplx* om = (bo_cplx*)malloc(sizeof(bo_cplx) * (size_t)(n * k));
  bo_gaussian(n, k, bo_mix1(seed, 5), bo_op_is_real(op), om);
  bo_cplx* ex = (bo_cplx*)malloc(sizeof(bo_cplx) * (size_t)(m * k));
  bo_cplx* ap = (bo_cplx*)malloc(sizeof(bo_cplx) * (size_t)(m * k));
  bo_op_apply(op, 0, om, k, ex);
  bo_bf_apply(bf, 0, om, k, ap);
  double num = 0, den = 0;
  for (int64_t i = 0; i < m * k; ++i) {
    den += bo_abs2(ex[i]);
    num += bo_abs2(ex[i] - ap[i]);
  }
  free(om); free(ex); free(ap);
  if (den == 0.0) return bo_fail(BO_CONDITIONING, "estimate_error: ||A Omega||_F is zero, relative error undefined");
  *err = sqrt(num) / sqrt(den);
  return BO_OK;
}
