// butterfly.h -- hybrid butterfly on the device (level-major padded layout)
// and its host (reference-layout) twin.
//
// Reference container: HybridButterfly (butterfly.hpp:20-66): per level 2^L
// blocks, flat index tau*2^(L-l)+nu; u_leaf, r_blocks[l-lm], b_blocks,
// w_blocks[l-1], v_leaf.  On the device every level is ONE buffer of 2^L
// equally-strided blocks (ld x cap, column major, zero padded):
//   * leaves: ld = max leaf size, rows beyond the leaf are zero;
//   * R/W transfer blocks are stored "padded-stacked": the first child's rows
//     at [0, r1), the second child's at [gap, gap + r2) with gap = P(child
//     level), so a stacked pair of child coefficient vectors is simply two
//     adjacent P-row slots of a level-major coefficient buffer;
//   * columns beyond the block's rank are zero; P = max rank of the level.
// Zero padding contributes exact zeros to every product, so all blocks of a
// level run as one uniform batched GEMM.
#pragma once

#include <complex>
#include <memory>
#include <vector>

#include "context.h"
#include "kernels.cuh"
#include "tree.h"

namespace bfly {

inline int64_t bidx(int L, int l, int64_t tau, int64_t nu) { return tau * (int64_t(1) << (L - l)) + nu; }

// --------------------------------------------------------- host layout
struct HostBlock {
  int64_t rows = 0, cols = 0;
  std::vector<std::complex<double>> a;  // column major
};

struct HostButterfly {
  int L = 0, lm = 0;
  bool is_real = false;
  Tree rt, ct;
  std::vector<HostBlock> u, v, b;
  std::vector<std::vector<HostBlock>> r, w;  // r[l-lm], w[l-1]

  int64_t u_rank(int l, int64_t tau, int64_t nu) const {
    return l == L ? u[tau].cols : r[l - lm][bidx(L, l, tau, nu)].cols;
  }
  int64_t v_rank(int l, int64_t tau, int64_t nu) const {
    return l == 0 ? v[nu].cols : w[l - 1][bidx(L, l, tau, nu)].cols;
  }
  void validate() const;  // butterfly.hpp:290-326
  int64_t nnz() const;
  int64_t max_rank() const;
  std::vector<uint8_t> serialize(int scalar_tag) const;  // serialize.hpp:103-127
  static HostButterfly deserialize(const uint8_t* buf, int64_t n);
};

// -------------------------------------------------------- device layout
template <typename R>
struct Level {
  DBuf<cx<R>> data;
  int64_t ld = 0, cap = 0;  // padded rows / column capacity per block
  int P = 0;                // max rank of the level (columns used by products)
  int gap = 0;              // second-child row offset (transfer blocks)
  std::vector<int32_t> ranks, rows;  // per block (host)
  DBuf<int32_t> dranks;

  int64_t stride() const { return ld * cap; }
  cx<R>* block(int64_t i) const { return data.p + i * stride(); }
  // cap_blocks >= nb reserves room for an in-place all-gather whose per-rank
  // chunks overhang the last block
  void alloc(Ctx* c, int64_t nb, int64_t ld_, int64_t cap_, int64_t cap_blocks = 0) {
    ld = std::max<int64_t>(ld_, 1);
    cap = std::max<int64_t>(cap_, 1);
    const int64_t nblk = std::max(nb, cap_blocks);
    data.reset(c, (size_t)(nblk * ld * cap));
    ranks.assign(nb, 0);
    rows.assign(nb, 0);
    dranks.reset(c, nblk);
  }
  void finish_ranks(Ctx* c);  // download ranks, set P
};

template <typename R>
struct DevButterfly {
  Ctx* ctx = nullptr;
  int L = 0, lm = 0;
  bool is_real = false;
  Tree rt, ct;
  Level<R> uleaf, vleaf, b;
  std::vector<Level<R>> r, w;  // r[l-lm] (l in [lm, L-1]), w[l-1] (l in [1, lm])
  DBuf<int64_t> rperm, cperm;  // device permutations (non-identity trees)
  bool leaves_uniform_r = true, leaves_uniform_c = true;

  int64_t m() const { return rt.n; }
  int64_t n() const { return ct.n; }
  int64_t nb() const { return int64_t(1) << L; }
  int PU(int l) const { return l == L ? uleaf.P : r[l - lm].P; }
  int PV(int l) const { return l == 0 ? vleaf.P : w[l - 1].P; }
  int u_rank(int l, int64_t tau, int64_t nu) const {
    return l == L ? uleaf.ranks[tau] : r[l - lm].ranks[bidx(L, l, tau, nu)];
  }
  int v_rank(int l, int64_t tau, int64_t nu) const {
    return l == 0 ? vleaf.ranks[nu] : w[l - 1].ranks[bidx(L, l, tau, nu)];
  }
  const Level<R>& ulevel(int l) const { return l == L ? uleaf : r[l - lm]; }
  const Level<R>& vlevel(int l) const { return l == 0 ? vleaf : w[l - 1]; }

  void setup_trees(Ctx* c, const Tree& row, const Tree& col, int levels, int center);
  // K x / K^T y / K^H y ; device buffers, original ordering
  void apply(int trans, const cx<R>* x, int64_t ldx, cx<R>* y, int64_t ldy, int64_t k);
  // Structured probes (the recompression black box, config 4).  Probe j is
  // nonzero only on node `node` of level `plevel` of the input-side tree
  // (row tree for OP_H, column tree for OP_N); its compact values (node rows
  // x ncols, leading dimension ldx) sit at X + x_off and it owns output
  // columns [col0, col0 + ncols) of y.  The reference pads every probe to
  // full height and multiplies the zeros (reconstruct.hpp:72-85,
  // ButterflyOperator operators.hpp:106-122); here a block is multiplied only
  // for the columns of the probes whose support reaches it, so the stages
  // before the supports merge cost one apply for the whole batch.  Column
  // arithmetic is unchanged: results equal the padded apply's.  segs sorted
  // by node with contiguous columns; returns false (nothing launched) when
  // the batch does not fit the scheme (non-identity trees, OP_T, gaps).
  struct ProbeSeg {
    int64_t node, x_off, col0;
    int32_t ncols;
  };
  // [o0, o1) (output tree order; o1 < 0: all) are the output rows that must be
  // produced: blocks whose output-side node holds none of them are skipped
  // too (a probe split across ranks needs only its partner nodes' rows).
  // G / glevel / proj_c / proj_ldc (optional): instead of y, write the
  // product's coefficients in ANOTHER butterfly's nested basis of level
  // glevel on the output side (V side for OP_H, U side for OP_N).  With
  // G(tau,nu) = B_other(glevel,tau,nu)^H B_this(glevel,tau,nu) (P_other x P_this
  // per block; G.ranks = the other's ranks, G.rows = this one's) the chain
  // stops at level glevel -- the stages between it and the leaves, the
  // leaf stage and the caller's whole projection chain back up disappear --
  // and block (tau,nu) writes G c into slot nu (OP_H) / tau (OP_N) of proj_c
  // (P_other rows per slot, ld proj_ldc, same columns as y).  The caller
  // guarantees both butterflies share trees and centre level.
  bool apply_structured(int trans, int plevel, const std::vector<ProbeSeg>& segs, const cx<R>* X, int64_t ldx,
                        cx<R>* y, int64_t ldy, int64_t o0, int64_t o1, double* flops_done,
                        const Level<R>* G = nullptr, int glevel = 0, cx<R>* proj_c = nullptr, int64_t proj_ldc = 0);
  int64_t nnz() const;
  int64_t max_rank() const;
  double apply_flops(int64_t k) const;   // 8 * nnz * k (complex)
  double apply_bytes(int64_t k) const;   // nnz*s + (m+n)*k*s

  HostButterfly to_host() const;
  // .bfh bytes straight from the padded device levels (one pinned staging
  // copy per level); returns the size, writes only when out != nullptr.
  int64_t serialize(int scalar_tag, uint8_t* out) const;
  static std::unique_ptr<DevButterfly> from_host(Ctx* c, const HostButterfly& h);

 private:
  // One stage of the apply chain: C_e = sum_s op(A_s) B_s over its entries.
  struct StageDesc {
    int op = 0, M = 0, K = 0, S = 1;
    const cx<R>* A = nullptr;
    int64_t lda = 0;
    int64_t ld_out = 0;  // ld of its coefficient output (NB * M); 0 for the last stage
    std::vector<GemmEnt> h;
    DBuf<GemmEnt> d;
    L2Prefetch pf;  // its factor level, prefetched into L2 by the kernel before it
    // block whose owner runs entry e in a process layout (layout.h):
    // side (0 V, 1 U), level, and per entry (tau, nu)
    int own_side = 0, own_level = 0;
    std::vector<int64_t> own_tau, own_nu;
  };
  struct Plan {
    std::vector<StageDesc> st;
  };
  Plan plan_n_, plan_h_;
  bool have_n_ = false, have_h_ = false;
  void build_plan_n();
  void build_plan_h();
  void upload_plan(Plan& plan);
  void run_plan(Plan& plan, const cx<R>* x, int64_t ldx, cx<R>* y, int64_t ldy, int64_t k, cx<R>* buf0,
                cx<R>* buf1);
  // per (trans, layout, p): every stage's entries split by owner, and the
  // block transfers feeding each stage (producer != consumer owner)
  struct DistXfer {
    int src = 0, dst = 0;
    std::vector<int64_t> offs;  // producer output row offsets (M rows each)
    DBuf<int64_t> d_offs;
  };
  struct DistPlan {
    int trans = 0, kind = 0, p = 1;
    std::vector<std::vector<std::vector<GemmEnt>>> h;  // [stage][rank]
    std::vector<std::vector<DBuf<GemmEnt>>> d;         // [stage][rank]
    std::vector<std::vector<DistXfer>> xfers;          // [stage]
    double report[6] = {0, 0, 0, 0, 0, 0};
  };
  std::vector<std::unique_ptr<DistPlan>> dist_plans_;
  DistPlan& dist_plan(int trans, int kind, int p);

 public:
  // Distributed apply over a process layout (dist.cu; reference
  // inc/layout.hpp:139-261): p = ctx world size (one process per GPU, NCCL
  // point-to-point exchanges), or p virtual processes run in turn on this GPU
  // when the context has no communicator.  trans: OP_N or OP_H; x is the full
  // input on every process, y the full output.  report[6]: exchange volume,
  // exchange messages, all-to-all volume, all-to-all messages (reference
  // counting, scalars per column and process), then the measured scalars
  // per column received by the busiest process and by all processes.
  void apply_layout(int trans, int kind, int p, const cx<R>* x, int64_t ldx, cx<R>* y, int64_t ldy, int64_t k,
                    double* report);

 private:
  // buf0/buf1: level coefficient buffers (NB*maxP*k each); null -> allocate
  void apply_n(const cx<R>* xt, int64_t ldx, cx<R>* yt, int64_t ldy, int64_t k, cx<R>* buf0 = nullptr,
               cx<R>* buf1 = nullptr);
  void apply_h(const cx<R>* yt, int64_t ldy, cx<R>* xt, int64_t ldx, int64_t k, cx<R>* buf0 = nullptr,
               cx<R>* buf1 = nullptr);
  int max_p() const;
  // CUDA graphs of repeated device-resident applies (same buffers, same k):
  // the ~2L+2 dependent stage launches replay as one graph launch.
  struct GraphEntry {
    int trans;
    const void* x;
    void* y;
    int64_t ldx, ldy, k;
    int uses = 0;
    int64_t kernels = 0;
    cudaGraphExec_t exec = nullptr;
    DBuf<cx<R>> b0, b1;
  };
  std::vector<std::unique_ptr<GraphEntry>> graphs_;
  bool apply_graph(int trans, const cx<R>* x, int64_t ldx, cx<R>* y, int64_t ldy, int64_t k);

 public:
  ~DevButterfly();
};

// Builds a HostButterfly from a seeded generator (synth_butterfly,
// operators.hpp:131-178, generalised to leaf b / rank r) + perturbation.
HostButterfly synth_host(int levels, int64_t leaf, int64_t rank, uint64_t seed, bool is_real, double perturb);
// host Gaussian block (same stream as the device K1 kernel)
void host_gaussian(int64_t rows, int64_t cols, uint64_t seed, bool is_real, std::complex<double>* out);

}  // namespace bfly
