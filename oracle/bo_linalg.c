/*
 * bo_linalg.c -- ORACLE (test infrastructure): dense numerics.
 *
 * pivoted_qr_truncate: /root/reference/proj/include/bfly/linalg.hpp:62-80, which
 * calls Eigen::ColPivHouseholderQR + householderQ().  Eigen is not vendored in
 * the reference and is absent here, so its published algorithm is restated:
 *   - pivot = first column with the largest *updated* norm;
 *   - Householder with beta = -sign(Re c0) * ||x||, tau = conj((beta - c0)/beta),
 *     essential = tail / (c0 - beta); skipped when the tail is below DBL_MIN;
 *   - LAWN-176 norm downdating, direct recomputation when the downdate ratio
 *     (times (updated/direct)^2) falls to sqrt(DBL_EPSILON) or below;
 *   - Q = H_0 ... H_{k-1} [I_k; 0] with H_j = I - conj(tau_j) v_j v_j^H.
 * pinv_solve: linalg.hpp:128-139 (JacobiSVD, thin U/V, cutoff tol*sigma_max);
 * restated as a one-sided (Hestenes) Jacobi SVD -- the pseudo-inverse is unique,
 * so any accurate SVD reproduces it.
 * random_orthonormal: operators.hpp:124-129 (HouseholderQR + householderQ).
 */
#include <float.h>
#include <math.h>
#include <string.h>

#include "bo_internal.h"

bo_mat bo_mat_new(int64_t rows, int64_t cols) {
  bo_mat m;
  m.rows = rows;
  m.cols = cols;
  m.a = (rows * cols > 0) ? (bo_cplx*)calloc((size_t)(rows * cols), sizeof(bo_cplx)) : NULL;
  return m;
}

void bo_mat_free(bo_mat* m) {
  free(m->a);
  m->a = NULL;
  m->rows = m->cols = 0;
}

void bo_gemm(char opa, int64_t m, int64_t n, int64_t k, const bo_cplx* a, int64_t lda,
             const bo_cplx* b, int64_t ldb, bo_cplx* c, int64_t ldc, int accumulate) {
  if (!accumulate)
    for (int64_t j = 0; j < n; ++j) memset(c + j * ldc, 0, sizeof(bo_cplx) * (size_t)m);
  if (m == 0 || n == 0 || k == 0) return;
  if (opa == 'N') {
    for (int64_t j = 0; j < n; ++j)
      for (int64_t l = 0; l < k; ++l) {
        bo_cplx bl = b[l + j * ldb];
        const bo_cplx* al = a + l * lda;
        bo_cplx* cj = c + j * ldc;
        for (int64_t i = 0; i < m; ++i) cj[i] += al[i] * bl;
      }
  } else {
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < m; ++i) {
        const bo_cplx* ai = a + i * lda;
        const bo_cplx* bj = b + j * ldb;
        bo_cplx s = 0;
        for (int64_t l = 0; l < k; ++l) s += conj(ai[l]) * bj[l];
        c[i + j * ldc] += s;
      }
  }
}

static double col_norm(const bo_cplx* x, int64_t n) {
  double s = 0;
  for (int64_t i = 0; i < n; ++i) s += bo_abs2(x[i]);
  return sqrt(s);
}

/* makeHouseholderInPlace on x[0..n): returns tau, writes beta; x[1..] <- essential */
static bo_cplx make_householder(bo_cplx* x, int64_t n, double* beta) {
  double tail_sq = 0;
  for (int64_t i = 1; i < n; ++i) tail_sq += bo_abs2(x[i]);
  bo_cplx c0 = x[0];
  double im = cimag(c0);
  if (tail_sq <= DBL_MIN && im * im <= DBL_MIN) {
    *beta = creal(c0);
    for (int64_t i = 1; i < n; ++i) x[i] = 0;
    return 0;
  }
  double b = sqrt(bo_abs2(c0) + tail_sq);
  if (creal(c0) >= 0) b = -b;
  bo_cplx d = c0 - b;
  for (int64_t i = 1; i < n; ++i) x[i] = x[i] / d;
  *beta = b;
  return conj((b - c0) / b);
}

/* (I - tau v v^H) applied to the (n x ncols) block at m (ld), v = (1; ess) */
static void apply_householder_left(bo_cplx* m, int64_t ld, int64_t n, int64_t ncols,
                                   const bo_cplx* ess, bo_cplx tau) {
  if (n == 1) {
    for (int64_t j = 0; j < ncols; ++j) m[j * ld] *= (1.0 - tau);
    return;
  }
  if (tau == 0) return;
  for (int64_t j = 0; j < ncols; ++j) {
    bo_cplx* col = m + j * ld;
    bo_cplx tmp = col[0];
    for (int64_t i = 1; i < n; ++i) tmp += conj(ess[i - 1]) * col[i];
    bo_cplx t = tau * tmp;
    col[0] -= t;
    for (int64_t i = 1; i < n; ++i) col[i] -= ess[i - 1] * t;
  }
}

/* Q(:, 0:k) = H_0 ... H_{k-1} [I_k; 0] from the compact factor qr (ld = rows) */
static void form_q(const bo_cplx* qr, int64_t rows, const bo_cplx* hc, int64_t k, bo_cplx* q) {
  memset(q, 0, sizeof(bo_cplx) * (size_t)(rows * k));
  for (int64_t i = 0; i < k; ++i) q[i + i * rows] = 1.0;
  for (int64_t j = k - 1; j >= 0; --j)
    apply_householder_left(q + j + j * rows, rows, rows - j, k - j, qr + j + 1 + j * rows, conj(hc[j]));
}

int bo_cpqr_truncate(int64_t rows, int64_t cols, const bo_cplx* z, int64_t ldz, double eps,
                     bo_cplx* q_out, int64_t* k_out, int64_t* piv_out, double* rdiag_out) {
  if (rows == 0 || cols == 0) return bo_fail(BO_PRECONDITION, "pivoted_qr_truncate: empty input");
  int64_t size = rows < cols ? rows : cols;
  bo_cplx* qr = (bo_cplx*)malloc(sizeof(bo_cplx) * (size_t)(rows * cols));
  for (int64_t j = 0; j < cols; ++j) memcpy(qr + j * rows, z + j * ldz, sizeof(bo_cplx) * (size_t)rows);
  double total = 0;
  for (int64_t j = 0; j < cols; ++j) {
    double nj = col_norm(qr + j * rows, rows);
    total += nj * nj;
  }
  if (total == 0.0) {
    *k_out = 0;
    free(qr);
    return BO_OK;
  }
  double* nu = (double*)malloc(sizeof(double) * (size_t)cols);
  double* nd = (double*)malloc(sizeof(double) * (size_t)cols);
  int64_t* piv = (int64_t*)malloc(sizeof(int64_t) * (size_t)cols);
  bo_cplx* hc = (bo_cplx*)malloc(sizeof(bo_cplx) * (size_t)size);
  double* rd = (double*)malloc(sizeof(double) * (size_t)size);
  for (int64_t j = 0; j < cols; ++j) {
    nu[j] = nd[j] = col_norm(qr + j * rows, rows);
    piv[j] = j;
  }
  const double downdate_thresh = sqrt(DBL_EPSILON);
  for (int64_t k = 0; k < size; ++k) {
    int64_t big = k;
    for (int64_t j = k + 1; j < cols; ++j)
      if (nu[j] > nu[big]) big = j;
    if (big != k) {
      for (int64_t i = 0; i < rows; ++i) {
        bo_cplx t = qr[i + k * rows];
        qr[i + k * rows] = qr[i + big * rows];
        qr[i + big * rows] = t;
      }
      double t = nu[k]; nu[k] = nu[big]; nu[big] = t;
      t = nd[k]; nd[k] = nd[big]; nd[big] = t;
      int64_t p = piv[k]; piv[k] = piv[big]; piv[big] = p;
    }
    double beta;
    hc[k] = make_householder(qr + k + k * rows, rows - k, &beta);
    qr[k + k * rows] = beta;
    rd[k] = fabs(beta);
    apply_householder_left(qr + k + (k + 1) * rows, rows, rows - k, cols - k - 1, qr + k + 1 + k * rows, hc[k]);
    for (int64_t j = k + 1; j < cols; ++j) {
      if (nu[j] != 0.0) {
        double temp = cabs(qr[k + j * rows]) / nu[j];
        temp = (1.0 + temp) * (1.0 - temp);
        if (temp < 0) temp = 0;
        double ratio = nu[j] / nd[j];
        double temp2 = temp * ratio * ratio;
        if (temp2 <= downdate_thresh) {
          nd[j] = col_norm(qr + k + 1 + j * rows, rows - k - 1);
          nu[j] = nd[j];
        } else {
          nu[j] *= sqrt(temp);
        }
      }
    }
  }
  double head = rd[0];
  int64_t k = 0;
  while (k < size && rd[k] > eps * head) ++k;
  if (k > 0 && q_out) form_q(qr, rows, hc, k, q_out);
  *k_out = k;
  if (piv_out) memcpy(piv_out, piv, sizeof(int64_t) * (size_t)cols);
  if (rdiag_out) memcpy(rdiag_out, rd, sizeof(double) * (size_t)size);
  free(qr); free(nu); free(nd); free(piv); free(hc); free(rd);
  return BO_OK;
}

/* unpivoted Householder QR, Q(:,0:cols) (operators.hpp:124-129) */
int bo_householder_q(int64_t rows, int64_t cols, const bo_cplx* g, bo_cplx* q_out) {
  if (cols > rows) return bo_fail(BO_PRECONDITION, "householder_q: cols > rows");
  bo_cplx* qr = (bo_cplx*)malloc(sizeof(bo_cplx) * (size_t)(rows * cols));
  memcpy(qr, g, sizeof(bo_cplx) * (size_t)(rows * cols));
  bo_cplx* hc = (bo_cplx*)malloc(sizeof(bo_cplx) * (size_t)cols);
  for (int64_t k = 0; k < cols; ++k) {
    double beta;
    hc[k] = make_householder(qr + k + k * rows, rows - k, &beta);
    qr[k + k * rows] = beta;
    apply_householder_left(qr + k + (k + 1) * rows, rows, rows - k, cols - k - 1, qr + k + 1 + k * rows, hc[k]);
  }
  form_q(qr, rows, hc, cols, q_out);
  free(qr);
  free(hc);
  return BO_OK;
}

/* One-sided Jacobi SVD of a tall p x q matrix a (p >= q), in place:
 * on exit a = U * diag(s) (columns), v = V (q x q); A = U S V^H. */
static void jacobi_svd(bo_cplx* a, int64_t p, int64_t q, bo_cplx* v, double* s) {
  memset(v, 0, sizeof(bo_cplx) * (size_t)(q * q));
  for (int64_t i = 0; i < q; ++i) v[i + i * q] = 1.0;
  for (int sweep = 0; sweep < 80; ++sweep) {
    int rotated = 0;
    for (int64_t i = 0; i < q - 1; ++i)
      for (int64_t j = i + 1; j < q; ++j) {
        bo_cplx* ai = a + i * p;
        bo_cplx* aj = a + j * p;
        double alpha = 0, beta = 0;
        bo_cplx gamma = 0;
        for (int64_t r = 0; r < p; ++r) {
          alpha += bo_abs2(ai[r]);
          beta += bo_abs2(aj[r]);
          gamma += conj(ai[r]) * aj[r];
        }
        double g = cabs(gamma);
        if (g == 0.0 || g <= 1e-15 * sqrt(alpha * beta)) continue;
        rotated = 1;
        bo_cplx ph = gamma / g; /* e^{i phi} */
        double zeta = (beta - alpha) / (2.0 * g);
        double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        double c = 1.0 / sqrt(1.0 + t * t);
        double sn = c * t;
        /* [a_i, a_j] <- [a_i, a_j] [[c, s], [-s conj(ph), c conj(ph)]] */
        bo_cplx cph = conj(ph);
        for (int64_t r = 0; r < p; ++r) {
          bo_cplx x = ai[r], y = aj[r] * cph;
          ai[r] = c * x - sn * y;
          aj[r] = sn * x + c * y;
        }
        bo_cplx* vi = v + i * q;
        bo_cplx* vj = v + j * q;
        for (int64_t r = 0; r < q; ++r) {
          bo_cplx x = vi[r], y = vj[r] * cph;
          vi[r] = c * x - sn * y;
          vj[r] = sn * x + c * y;
        }
      }
    if (!rotated) break;
  }
  for (int64_t i = 0; i < q; ++i) s[i] = col_norm(a + i * p, p);
}

int bo_pinv(int64_t rows, int64_t cols, const bo_cplx* m, double tol, bo_cplx* out) {
  if (rows == 0 || cols == 0) return bo_fail(BO_PRECONDITION, "pinv_solve: empty input");
  int wide = rows <= cols;
  int64_t p = wide ? cols : rows, q = wide ? rows : cols;
  bo_cplx* a = (bo_cplx*)malloc(sizeof(bo_cplx) * (size_t)(p * q));
  /* tall matrix A = M^H (wide) or M (tall) */
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < cols; ++j) {
      if (wide) a[j + i * p] = conj(m[i + j * rows]);
      else a[i + j * p] = m[i + j * rows];
    }
  bo_cplx* v = (bo_cplx*)malloc(sizeof(bo_cplx) * (size_t)(q * q));
  double* s = (double*)malloc(sizeof(double) * (size_t)q);
  jacobi_svd(a, p, q, v, s);
  double smax = 0;
  for (int64_t i = 0; i < q; ++i)
    if (s[i] > smax) smax = s[i];
  double cutoff = tol * smax;
  /* a columns hold U*S; scale column i by 1/s_i^2 (to get U/s) when kept, else drop */
  for (int64_t i = 0; i < q; ++i) {
    double f = (s[i] > cutoff && s[i] > 0) ? 1.0 / (s[i] * s[i]) : 0.0;
    for (int64_t r = 0; r < p; ++r) a[r + i * p] *= f;
  }
  /* out is cols x rows.
   * wide:  M = V S U^H  => pinv = U S^+ V^H  = (a) (p x q) * V^H (q x q)  -> p=cols, q=rows
   * tall:  M = U S V^H  => pinv = V S^+ U^H  = V (q x q) * (a)^H (q x p) -> q=cols, p=rows */
  memset(out, 0, sizeof(bo_cplx) * (size_t)(rows * cols));
  if (wide) {
    for (int64_t c = 0; c < rows; ++c)
      for (int64_t i = 0; i < q; ++i) {
        bo_cplx f = conj(v[c + i * q]);
        if (f == 0) continue;
        for (int64_t r = 0; r < p; ++r) out[r + c * cols] += a[r + i * p] * f;
      }
  } else {
    for (int64_t c = 0; c < rows; ++c)
      for (int64_t i = 0; i < q; ++i) {
        bo_cplx f = conj(a[c + i * p]);
        if (f == 0) continue;
        for (int64_t r = 0; r < q; ++r) out[r + c * cols] += v[r + i * q] * f;
      }
  }
  free(a); free(v); free(s);
  return BO_OK;
}
