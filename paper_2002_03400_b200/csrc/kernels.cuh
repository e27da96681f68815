// kernels.cuh -- launchers of the sm_100a kernels.
#pragma once

#include <cstdint>

#include "common.cuh"
#include "context.h"

namespace bfly {

enum Op { OP_N = 0, OP_T = 1, OP_H = 2 };

// ------------------------------------------------------------ K1: RNG
// One seeded Gaussian block (gaussian_matrix, linalg.hpp:16-25) per entry.
struct GaussEnt {
  int64_t dst;    // element offset into the output base
  int64_t ld;
  int64_t rows, cols;
  uint64_t s0;    // seed_mix(seed, "matr")
};
template <typename R>
void launch_gauss(Ctx* c, cx<R>* base, const GaussEnt* ents_dev, int nent, int64_t max_elems, bool is_real);

// --------------------------------------------------- K2: kernel matvec
enum KernelKind { KK_NUFFT = 1, KK_PLATES = 2, KK_CIRCLE = 3 };
// Y[:, col0:col0+ncols] (all output points) = sum over the segment's input
// rows of op(K) * X_seg.  X_seg row t corresponds to input point row0 + t.
struct MatvecSeg {
  int64_t row0, rows;   // input point range
  int64_t x_off;        // element offset of X_seg(0,0) in the X base
  int64_t ldx;
  int64_t col0;         // first output column in Y
  int32_t ncols;
  int32_t pad_;
};
struct Points {
  const double* x;
  const double* y;
  const double* z;
};
template <typename R>
void launch_kernel_matvec(Ctx* c, int kind, int mode, Points out_pts, Points in_pts, double kappa, int64_t m_out,
                          const cx<R>* X, cx<R>* Y, int64_t ldy, const MatvecSeg* segs_host, int nseg);
// complex128 contraction on tcgen05 int8 (exact integer-slice scheme,
// k_matvec_oz.cu); returns false if an entry fell outside the representable
// range (the caller then recomputes on the FP64 DMMA path).  BFLY_MATVEC=fp64
// selects the FP64 path.
bool matvec_oz_enabled();
// widest probe block one kernel-evaluation pass covers (40 on CTA pairs, else 32)
int kernel_matvec_pass_cols();
bool launch_kernel_matvec_oz(Ctx* c, int kind, int mode, Points out_pts, Points in_pts, double kappa, int64_t m_out,
                             const double2* X, double2* Y, int64_t ldy, const MatvecSeg* segs_host, int nseg);

// ------------------------------------------ K3/K4: batched block GEMM
// C_e (M x ncols_e) (+)= sum_{s<S} op(A + a_s) (M x K) * (B + b_s) (K x ncols_e)
// Per-entry mrows/krows (<= M/K) bound the rows of C written and of B read
// (ragged leaves); ncols_all > 0 overrides every entry's ncols.
struct GemmEnt {
  int64_t a0, a1, b0, b1, c;
  int32_t ncols, mrows, krows, pad_;
};
// L2 prefetch of the NEXT chain stage's factor level: entry e of this launch
// prefetches [base + e*stride, +len) bytes (stage kernel only)
struct L2Prefetch {
  const void* base = nullptr;
  int64_t stride = 0, len = 0;
};
template <typename R>
void launch_bgemm(Ctx* c, int op, int M, int K, int S, const cx<R>* A, int64_t lda, const cx<R>* B, int64_t ldb,
                  cx<R>* C, int64_t ldc, const GemmEnt* ents_dev, int nent, int max_ncols, bool accumulate,
                  int ncols_all = 0, bool pdl = false, L2Prefetch pf = L2Prefetch());
// pdl: programmatic dependent launch for chains whose A operand is NOT written
// by the preceding kernel (butterfly apply stages): A is staged before the
// dependency wait, overlapping the previous stage's tail.

// ------------------------------------------ K5: batched truncated CPQR
// Compact input rows: [0, r1) from src, [r1, r1+r2) from src + src_gap.
// Output Q (r1+r2 x k) written padded-stacked into a ld_dst x cap block:
// rows [0,r1) -> [0,r1), rows [r1, r1+r2) -> [dst_gap, dst_gap+r2).
struct QrEnt {
  int64_t src, dst;
  int32_t r1, r2;
  int32_t src_gap, dst_gap;
  int32_t cols;
  int32_t rank_slot;
};
template <typename R>
void launch_cpqr(Ctx* c, const cx<R>* src, int64_t ld_src, cx<R>* dst, int64_t ld_dst, int cap, const QrEnt* ents_dev,
                 int nent, int max_rows, int max_cols, int32_t* ranks, double eps, double* margins = nullptr);

// ------------------------------------------ K6: batched core fit
// B = (Q^H z) * pinv(coeff) (core_block, reconstruct.hpp:125-138)
struct CoreEnt {
  int64_t q, z, coeff, b;  // element offsets
  int32_t r1, r2;          // compact rows of z / Q
  int32_t q_gap, z_gap;    // second-child row offsets in Q / z storage
  int32_t ku, kv;          // ranks
  int32_t w;               // probe width
  int32_t pad_;
};
// saturated centre blocks (kv >= 64): B = P G^-1 by Newton-Schulz on batched
// DMMA GEMMs (k_corefit.cu); returns the blocks fitted, the rest (not
// converged: ill-conditioned coefficients) in `fallback` for launch_core_fit
template <typename R>
int64_t core_fit_big(Ctx* c, const cx<R>* Q, int64_t ldq, const cx<R>* Z, int64_t ldz, const cx<R>* Cf, int64_t ldc,
                     cx<R>* B, int64_t ldb, int bcap, const std::vector<CoreEnt>& ents,
                     std::vector<CoreEnt>& fallback);
template <typename R>
void launch_core_fit(Ctx* c, const cx<R>* Q, int64_t ldq, const cx<R>* Z, int64_t ldz, const cx<R>* Cf, int64_t ldc,
                     cx<R>* B, int64_t ldb, int bcap, const CoreEnt* ents_dev, int nent, int max_ku, int max_kv,
                     int max_w, bool literal, int32_t* err_flag);

// ------------------------------------------------------------ utilities
template <typename R>
void launch_conj(Ctx* c, cx<R>* p, int64_t rows, int64_t cols, int64_t ld);
// dst[i] = src[idx[i]] (gather) or dst[idx[i]] = src[i] (scatter), rows x cols
template <typename R>
void launch_permute_rows(Ctx* c, cx<R>* dst, int64_t ldd, const cx<R>* src, int64_t lds, int64_t rows, int64_t cols,
                         const int64_t* idx, bool scatter);
template <typename R>
void launch_copy2d(Ctx* c, cx<R>* dst, int64_t ldd, const cx<R>* src, int64_t lds, int64_t rows, int64_t cols);
// out[0] += ||a - b||_F^2, out[1] += ||a||_F^2 (double accumulators)
template <typename R>
void launch_diff_norms(Ctx* c, const cx<R>* a, const cx<R>* b, int64_t n, double* out);
// dst block idx_dst[i] <- src block idx_src[i] (blocks of `stride` elements);
// null index arrays mean the identity
template <typename R>
void launch_copy_blocks(Ctx* c, cx<R>* dst, const int64_t* idx_dst, const cx<R>* src, const int64_t* idx_src,
                        int64_t nblocks, int64_t stride);
// int32 gather / scatter: dst[idx_dst[t] or t] = src[idx_src[t] or t], t < n
void launch_copy_idx_i32(Ctx* c, int32_t* dst, const int64_t* idx_dst, const int32_t* src, const int64_t* idx_src,
                         int64_t n);
// real-valued copy-converters between precisions
void launch_d2f(Ctx* c, const double2* src, float2* dst, int64_t n);
void launch_f2d(Ctx* c, const float2* src, double2* dst, int64_t n);

}  // namespace bfly
