// operators.h -- device black-box operators (BlackBoxOperator,
// reference operators.hpp:17-66).
//
// The factorizer hands an operator a batch of structured probes: probe s has
// nonzero input rows [row0, row0+rows) (operator index space) whose values
// live at X + x_off (ld ldx), and owns output columns [col0, col0+ncols) of Y.
// Built-in kinds exploit the zero rows (the reference pads and multiplies
// the zeros, reconstruct.hpp:72-85); generic kinds see the padded probe.
#pragma once

#include <memory>
#include <vector>

#include "butterfly.h"
#include "context.h"
#include "kernels.cuh"

#include "../../include/bfly_b200.h"

namespace bfly {

// A transfer level never uses a product y = op(A) X itself, only its
// coefficients in the NEW factorization's nested basis one level above the
// probes: B_new(level)^H y, which the reference obtains by projecting y on
// the leaf bases and running the partial V / U chain (butterfly.hpp:330-354).
// A kind that knows y in a nested basis of its own can answer directly: the
// butterfly black box stops its apply at `level` and multiplies
// G = B_new(level)^H B_in(level) (one P x P block per butterfly block), so
// its remaining stages, the n x w product and the caller's whole chain
// disappear.  The coefficients go to the chain buffer C of that level (slot
// = column node for OP_H products / row node for OP_N, P_new(level) rows per
// slot, ld ldc, same columns as Y); done reports it, and Y is then not written.
template <typename R>
struct BasisProj {
  const DevButterfly<R>* nbf = nullptr;  // the factorization in progress
  uint64_t gen = 0;                      // changes with every factorization (cached G levels)
  int level = 0;                         // V side 0..lm-1 (OP_H products), U side lm+1..L (OP_N)
  cx<R>* C = nullptr;
  int64_t ldc = 0;
  bool done = false;
};

template <typename R>
struct DevOp {
  int kind = 0;
  int64_t m = 0, n = 0;
  bool is_real = false;
  Ctx* ctx = nullptr;
  int64_t fwd = 0, tr = 0;  // column counters (operators.hpp:41-47)
  double flops = 0, evals = 0;  // algorithmic work of every product so far

  virtual ~DevOp() = default;
  // true when do_apply computes only the requested output rows (work and
  // counted flops proportional to them)
  virtual bool restricts_rows() const { return false; }
  // whether the last apply_segs produced only the requested rows (a kind may
  // restrict some products only: the butterfly black box's structured path)
  bool last_restricted = false;
  int64_t in_dim(int mode) const { return mode == OP_N ? n : m; }
  int64_t out_dim(int mode) const { return mode == OP_N ? m : n; }

  // Y(:, seg cols) = op(A) X_seg for every segment; mode N, T or H (the
  // adjoint, derived exactly as apply_adjoint in the reference).
  // [o0, o1) restricts the output rows that must be produced (the rank's
  // leaves in a sharded leaf phase); kinds that cannot restrict compute all.
  // count_cols >= 0 overrides the columns added to the counters
  BasisProj<R>* cur_lp = nullptr;  // the running apply_segs' projection request
  // whether this kind would answer the request (the caller then does not
  // allocate the product; a group that still comes back unanswered is
  // multiplied again the plain way)
  virtual bool can_project(int mode, const BasisProj<R>& lp) { return false; }
  void apply_segs(int mode, const cx<R>* X, const std::vector<MatvecSeg>& segs, cx<R>* Y, int64_t ldy,
                  int64_t o0 = 0, int64_t o1 = -1, int64_t count_cols = -1, BasisProj<R>* lp = nullptr) {
    int64_t cols = 0;
    for (const auto& s : segs) cols += s.ncols;
    if (count_cols >= 0) cols = count_cols;
    if (mode == OP_N) fwd += cols;
    else tr += cols;
    if (o1 < 0) o1 = out_dim(mode);
    last_restricted = restricts_rows();
    cur_lp = lp;
    do_apply(mode, X, segs, Y, ldy, o0, o1);
    cur_lp = nullptr;
  }
  void apply_dense(int mode, const cx<R>* X, int64_t ldx, cx<R>* Y, int64_t ldy, int64_t k) {
    MatvecSeg s{0, in_dim(mode), 0, ldx, 0, (int32_t)k, 0};
    apply_segs(mode, X, {s}, Y, ldy);
  }

 protected:
  virtual void do_apply(int mode, const cx<R>* X, const std::vector<MatvecSeg>& segs, cx<R>* Y, int64_t ldy,
                        int64_t o0, int64_t o1) = 0;
  // materialise the padded probes (zeros outside the segment rows) as one
  // in_dim x w buffer whose column t lines up with column c0 + t of Y
  // (c0 / w: the column span of the segments)
  DBuf<cx<R>> pad_probes(int mode, const cx<R>* X, const std::vector<MatvecSeg>& segs, int64_t& c0, int64_t& w);
};

// segments grouped into runs that tile a column range without gaps
std::vector<std::vector<MatvecSeg>> column_runs(std::vector<MatvecSeg> segs);

template <typename R>
std::unique_ptr<DevOp<R>> make_kernel_op(Ctx* c, int kind, int64_t m, int64_t n, const double* tgt, const double* src,
                                         double kappa);
template <typename R>
std::unique_ptr<DevOp<R>> make_dense_op(Ctx* c, int64_t m, int64_t n, const std::vector<cx<R>>& a, bool is_real);
template <typename R>
std::unique_ptr<DevOp<R>> make_compose_op(Ctx* c, std::unique_ptr<DevOp<R>> f2, std::unique_ptr<DevOp<R>> f1);
template <typename R>
std::unique_ptr<DevOp<R>> make_butterfly_op(Ctx* c, std::unique_ptr<DevButterfly<R>> bf);
template <typename R>
std::unique_ptr<DevOp<R>> make_callback_op(Ctx* c, int64_t m, int64_t n, bool is_real, bfly_apply_fn fn, void* user);
template <typename R>
std::unique_ptr<DevOp<R>> make_callback_range_op(Ctx* c, int64_t m, int64_t n, bool is_real, bfly_apply_range_fn fn,
                                                 void* user);
template <typename R>
DevButterfly<R>* butterfly_of(DevOp<R>* op);

}  // namespace bfly
