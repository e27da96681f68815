/* bo_internal.h -- ORACLE (test infrastructure) private helpers. */
#ifndef BO_INTERNAL_H
#define BO_INTERNAL_H

#include <complex.h>
#include <stdint.h>
#include <stdlib.h>

#include "bfly_oracle.h"

int bo_fail(int code, const char* fmt, ...);
uint64_t bo_mix1(uint64_t seed, uint64_t a);
uint64_t bo_mix2(uint64_t seed, uint64_t a, uint64_t b);
uint64_t bo_mix3(uint64_t seed, uint64_t a, uint64_t b, uint64_t c);

int bo_threads(void);

static inline int64_t bo_node_b(const bo_tree* t, int l, int64_t j) { return t->rb[l][j]; }
static inline int64_t bo_node_e(const bo_tree* t, int l, int64_t j) { return t->rb[l][j + 1]; }

static inline double bo_abs2(bo_cplx z) {
  double r = creal(z), i = cimag(z);
  return r * r + i * i;
}

/* C (m x n) = op(A) * B, op in {N, H}; A is (m x k) for N, (k x m) for H.
 * ld* are leading dimensions.  beta_zero: overwrite C instead of accumulate. */
void bo_gemm(char opa, int64_t m, int64_t n, int64_t k, const bo_cplx* a, int64_t lda,
             const bo_cplx* b, int64_t ldb, bo_cplx* c, int64_t ldc, int accumulate);

bo_mat bo_mat_new(int64_t rows, int64_t cols);
void bo_mat_free(bo_mat* m);

/* butterfly block index tau * 2^(L-l) + nu (butterfly.hpp:38-43) */
static inline int64_t bo_bidx(int L, int l, int64_t tau, int64_t nu) {
  return tau * ((int64_t)1 << (L - l)) + nu;
}
int64_t bo_u_rank(const bo_bf* bf, int l, int64_t tau, int64_t nu);
int64_t bo_v_rank(const bo_bf* bf, int l, int64_t tau, int64_t nu);
bo_mat* bo_r_block(const bo_bf* bf, int l, int64_t tau, int64_t nu);
bo_mat* bo_w_block(const bo_bf* bf, int l, int64_t tau, int64_t nu);

/* chain coefficients (butterfly.hpp:330-354); x_sub is (node rows x k), ld = ldx;
 * result allocated into *out */
void bo_v_chain(const bo_bf* bf, int level, int64_t tau, int64_t nu, const bo_cplx* x, int64_t ldx,
                int64_t k, bo_mat* out);
void bo_u_chain(const bo_bf* bf, int level, int64_t tau, int64_t nu, const bo_cplx* x, int64_t ldx,
                int64_t k, bo_mat* out);

bo_bf* bo_bf_alloc(int levels, int center);

#endif
