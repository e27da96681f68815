/*
 * bfly_oracle.h -- CPU ORACLE for the butterfly construction loop.
 *
 * TEST INFRASTRUCTURE ONLY.  This is a plain-C restatement of the reference's
 * algorithm (arXiv 2002.03400, Algorithm 2, as implemented in
 * /root/reference/proj/include/bfly/{core,linalg,tree,butterfly,operators,
 * reconstruct,serialize}.hpp).  It is the checker used by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference
 * legs.  The product (paper_2002_03400_b200/) never links or calls it.
 *
 * Storage: every matrix is column-major complex double.  Real-scalar mode
 * (the reference's BlackBoxOperator<double>) is represented with zero
 * imaginary parts; the only behavioural difference is the Gaussian draw
 * (one N(0,1) per entry instead of one Box-Muller pair), because conjugation
 * and adjoints are exact no-ops on real-valued data.
 *
 * Third-party arithmetic restated here (Eigen3, unpinned, not vendored --
 * see DESIGN.md "Oracle"): ColPivHouseholderQR (+householderQ),
 * HouseholderQR, JacobiSVD-based pseudo-inverse.
 */
#ifndef BFLY_ORACLE_H
#define BFLY_ORACLE_H

#include <complex.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef double _Complex bo_cplx;

/* status codes mirror the reference's error hierarchy (core.hpp:43-60) */
enum {
  BO_OK = 0,
  BO_PRECONDITION = 1,
  BO_DIMENSION = 2,
  BO_SEQUENCING = 3,
  BO_FORMAT = 4,
  BO_CONDITIONING = 5,
};

const char* bo_last_error(void);

/* ---------------- RNG (core.hpp:70-141, linalg.hpp:16-25) ---------------- */
uint64_t bo_splitmix64(uint64_t* state);
uint64_t bo_seed_mix(uint64_t seed, int nwords, const uint64_t* words);
/* rows x cols column-major Gaussian block; is_real selects the real stream. */
int bo_gaussian(int64_t rows, int64_t cols, uint64_t seed, int is_real, bo_cplx* out);

/* ---------------- tree (tree.hpp:75-201) ---------------- */
typedef struct bo_tree {
  int levels;
  int64_t n;
  int64_t* perm;     /* tree slot -> original index */
  int64_t** rb;      /* rb[l] has 2^l + 1 entries */
} bo_tree;

/* coords: n x 3 row-major (unused axes 0).  Returns NULL on error. */
bo_tree* bo_tree_build(int dim, int64_t n, const double* coords, int levels);
bo_tree* bo_tree_from_table(int64_t n, int levels, const int64_t* perm, const int64_t* rb_flat);
bo_tree* bo_tree_copy(const bo_tree* t);
void bo_tree_free(bo_tree* t);
int bo_depth_for(int64_t n, int64_t leaf_cap);
/* flattened range table: sum_l (2^l + 1) entries */
void bo_tree_table(const bo_tree* t, int64_t* perm_out, int64_t* rb_out);

/* ---------------- dense numerics (linalg.hpp:62-139) ---------------- */
/* Truncated column-pivoted QR: keeps k leading pivots with
 * |R_kk| > eps*|R_00|.  q_out must hold rows*min(rows,cols); *k_out = k.
 * piv_out (cols) and rdiag_out (min(rows,cols)) are optional diagnostics. */
int bo_cpqr_truncate(int64_t rows, int64_t cols, const bo_cplx* z, int64_t ldz, double eps,
                     bo_cplx* q_out, int64_t* k_out, int64_t* piv_out, double* rdiag_out);
/* Moore-Penrose pseudo-inverse (rows x cols) -> (cols x rows), cutoff tol*smax */
int bo_pinv(int64_t rows, int64_t cols, const bo_cplx* m, double tol, bo_cplx* out);
/* Q factor (rows x cols) of an unpivoted Householder QR (operators.hpp:124-129) */
int bo_householder_q(int64_t rows, int64_t cols, const bo_cplx* g, bo_cplx* q_out);

/* ---------------- butterfly (butterfly.hpp:20-387) ---------------- */
typedef struct bo_mat {
  int64_t rows, cols;
  bo_cplx* a; /* column-major, ld = rows */
} bo_mat;

typedef struct bo_bf {
  int levels, center;
  bo_tree* row_tree;
  bo_tree* col_tree;
  bo_mat* u_leaf;    /* 2^L */
  bo_mat* v_leaf;    /* 2^L */
  bo_mat** r_blocks; /* [l - center][2^L], l in [center, L-1] */
  bo_mat** w_blocks; /* [l - 1][2^L], l in [1, center] */
  bo_mat* b_blocks;  /* 2^L */
  int is_real;
} bo_bf;

void bo_bf_free(bo_bf* bf);
int bo_bf_validate(const bo_bf* bf);
int64_t bo_bf_nnz(const bo_bf* bf);
int64_t bo_bf_max_rank(const bo_bf* bf);
/* trans: 0 = K x, 1 = K^T y, 2 = K^H y.  X/Y column-major original order. */
int bo_bf_apply(const bo_bf* bf, int trans, const bo_cplx* x, int64_t k, bo_cplx* y);
/* rank profile: u ranks for levels center..L, v ranks for levels 0..center,
 * each 2^L entries (layout documented in DESIGN.md). */
int64_t bo_bf_rank_profile(const bo_bf* bf, int32_t* out);
/* .bfh container bytes (serialize.hpp:103-127); returns byte count, fills buf if non-NULL */
int64_t bo_bf_serialize(const bo_bf* bf, uint8_t* buf);
bo_bf* bo_bf_deserialize(const uint8_t* buf, int64_t nbytes);
/* dense expansion (butterfly.hpp:199-216), original ordering */
int bo_bf_to_dense(const bo_bf* bf, bo_cplx* out);

/* ---------------- operators (operators.hpp:17-122 + BASELINE configs) ---------------- */
enum {
  BO_OP_DENSE = 0,
  BO_OP_NUFFT = 1,       /* config 0 */
  BO_OP_PLATES = 2,      /* config 1 */
  BO_OP_CIRCLE = 3,      /* config 2 */
  BO_OP_COMPOSE = 4,     /* config 3 */
  BO_OP_BUTTERFLY = 5,   /* config 4 / synthetic */
};

typedef struct bo_op bo_op;
bo_op* bo_op_dense(int64_t m, int64_t n, const bo_cplx* a, int is_real);
/* kernel operators: tgt/src point arrays are n x 3 row-major in TREE order */
bo_op* bo_op_kernel(int kind, int64_t m, int64_t n, const double* tgt, const double* src,
                    double wavenumber);
bo_op* bo_op_compose(bo_op* f2, bo_op* f1); /* takes ownership */
bo_op* bo_op_butterfly(bo_bf* bf);          /* takes ownership */
void bo_op_free(bo_op* op);
int64_t bo_op_rows(const bo_op* op);
int64_t bo_op_cols(const bo_op* op);
int bo_op_is_real(const bo_op* op);
/* trans 0: Y(m x k) = A X ; 1: Y(n x k) = A^T X (plain transpose); counts columns */
int bo_op_apply(const bo_op* op, int trans, const bo_cplx* x, int64_t k, bo_cplx* y);
int bo_op_apply_adjoint(const bo_op* op, const bo_cplx* y, int64_t k, bo_cplx* x);
void bo_op_counters(const bo_op* op, int64_t* fwd, int64_t* tr);
void bo_op_reset_counters(bo_op* op);
int bo_op_entry(const bo_op* op, int64_t i, int64_t j, bo_cplx* out);
void bo_set_threads(int threads);

/* point generators for the BASELINE configs (host, shared definition with
 * the product's generators) */
void bo_points_uniform(int64_t n, uint64_t seed, uint64_t tag, double lo, double hi, double* out);
void bo_points_plate(int64_t side, double z, double* out);
void bo_points_half_circle(int64_t n, int upper, double* out);

/* synthetic butterflies (operators.hpp:124-178, generalised to leaf b, rank r) */
bo_bf* bo_synth_butterfly(int levels, int64_t leaf, int64_t rank, uint64_t seed, int is_real,
                          double perturb);

/* ---------------- reconstruction (reconstruct.hpp) ---------------- */
typedef struct bo_cfg {
  double tolerance;
  int64_t oversampling;
  int64_t rank_guess;
  int levels;
  int center;
  uint64_t seed;
  int64_t hard_cap;
  int threads;
  int literal_transpose_core;
} bo_cfg;

void bo_cfg_default(bo_cfg* cfg);

/* CPQR cut margin min(|R_{k-1}|/thr - 1, 1 - |R_k|/thr), thr = eps |R_00| (+inf: zero block) */
double bo_cut_margin(const double* rdiag, int64_t size, int64_t k, double eps);

#define BO_MAX_PHASES 64
typedef struct bo_phase {
  char name[32];
  int64_t forward_columns, transpose_columns;
  double seconds;
  int rounds;
  int64_t probe_width;
  double rank_margin; /* min CPQR cut margin over the phase's blocks (bo_cut_margin) */
} bo_phase;

typedef struct bo_log {
  int nphases;
  bo_phase phases[BO_MAX_PHASES];
  uint64_t peak_probe_bytes;
  int64_t peak_concurrent_probes;
  int rank_capped;
  double total_seconds;
} bo_log;

typedef struct bo_factorizer bo_factorizer;
bo_factorizer* bo_factorizer_new(const bo_op* op, const bo_tree* rt, const bo_tree* ct,
                                 const bo_cfg* cfg);
int bo_factorizer_leaf_row(bo_factorizer* f);
int bo_factorizer_leaf_col(bo_factorizer* f);
int bo_factorizer_transfer_w(bo_factorizer* f, int l);
int bo_factorizer_transfer_r(bo_factorizer* f, int l);
int bo_factorizer_complete(const bo_factorizer* f);
/* releases the butterfly to the caller (factorizer keeps no reference) */
bo_bf* bo_factorizer_take(bo_factorizer* f, bo_log* log);
void bo_factorizer_free(bo_factorizer* f);

int bo_factorize(const bo_op* op, const bo_tree* rt, const bo_tree* ct, const bo_cfg* cfg,
                 bo_bf** bf_out, bo_log* log);
int bo_core_block(int64_t zr, int64_t w, const bo_cplx* z, int64_t ur, int64_t uc, const bo_cplx* u, int64_t cr,
                  int64_t cc, const bo_cplx* coeff, int literal, bo_cplx* out);
int bo_probe_with(const bo_op* op, const bo_tree* t, int level, int64_t node, const bo_cplx* core, int64_t core_rows,
                  int64_t width, int forward, bo_cplx* out);
int bo_estimate_error(const bo_op* op, const bo_bf* bf, int64_t k, uint64_t seed, double* err);

#ifdef __cplusplus
}
#endif
#endif
