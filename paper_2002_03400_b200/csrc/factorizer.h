// factorizer.h -- Algorithm 2 driver on the GPU (reference Factorizer,
// reconstruct.hpp:145-410): same phase order, seeds, probe widths,
// truncation and stop rule; every level runs as a handful of batched launches.
//
// Multi-GPU: every level's units (leaves, W probes tau, R probes nu) are split
// into contiguous per-rank chunks.  Leaf and W blocks of a chunk are
// contiguous in the tau-major level layout and are all-gathered in place;
// R/B blocks of a nu chunk are strided and go through pack -> all-gather ->
// unpack.  With virtual_ranks > 1 one process executes every rank's chunk
// through the same pack/unpack path (single-GPU test of the sharding).
#pragma once

#include <chrono>
#include <memory>
#include <string>
#include <vector>

#include "../../include/bfly_b200.h"
#include "butterfly.h"
#include "shard.h"
#include "operators.h"

namespace bfly {

// per-(phase, rank) device milliseconds of the last virtual-rank factorization
// run with BFLY_VRANK_TIMING=1 (row-major, world entries per phase)
std::vector<double>& vrank_table();

template <typename R>
class Factorizer {
 public:
  Factorizer(Ctx* c, DevOp<R>* op, const Tree& rt, const Tree& ct, const bfly_recon_cfg& cfg);
  void leaf_row_bases();
  void leaf_col_bases();
  void transfer_level_w(int l);
  void transfer_level_r(int l);
  bool complete() const { return core_done_; }
  void run();
  std::unique_ptr<DevButterfly<R>> take(bfly_log* log);
  const bfly_log& log() const { return log_; }

 private:
  using V = cx<R>;
  using clock = std::chrono::steady_clock;
  Ctx* c_;
  DevOp<R>* op_;
  bfly_recon_cfg cfg_;
  std::unique_ptr<DevButterfly<R>> bf_;
  bfly_log log_{};
  bool v_done_ = false, u_done_ = false, core_done_ = false;
  int next_w_ = 1, next_r_ = 0;
  double flops_ = 0;  // chain + QR + core-fit work (black box counted by the operator)
  // CPQR cut margin of every block of the current phase (bfly_phase::rank_margin)
  DBuf<double> margin_;
  double* margins_reset();
  // memory guard: probes per launch that fit next to the level (0: no limit)
  int64_t guard_batch_ = 0;
  void memory_guard(const std::string& what, double level_bytes, double per_probe_bytes, int64_t nprobes);
  // sharding
  int world_ = 1, rank_ = 0;
  bool virtual_ = false;

  // per-(phase, virtual rank) device time of each rank's share
  // (BFLY_VRANK_TIMING=1 with virtual ranks; diagnostics for a scaling
  // projection, see vrank_table())
  bool vr_timing_ = false;
  uint64_t gen_ = 0;  // distinct per Factorizer (operators cache per-factorization state by it)
  struct VrTimer {
    Factorizer* f;
    int rank;
    cudaEvent_t a = nullptr, b = nullptr;
    VrTimer(Factorizer* f_, int r);
    ~VrTimer();
  };
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> vr_events_;
  std::vector<int> vr_rank_;
  void vr_flush(int phase);  // accumulate the phase's rank timings into the table

  std::vector<int> my_ranks() const;
  static std::pair<int64_t, int64_t> chunk(int64_t n, int world, int r);
  bfly_phase& new_phase(const std::string& name);
  void end_phase(bfly_phase& st, clock::time_point t0, int64_t f0, int64_t tr0);
  void note_probe_bytes(double scalars, int64_t probes);
  void run_leaf_phase(const char* name, bool row_side);
  // orange[p]: output rows probe p needs ([o0, o1) in tree order of the
  // output side); counted[p]: its columns go into the operator counters (a
  // probe split across ranks is counted by the rank holding its first piece)
  void probe_products(int mode, const Tree& probe_tree, int level, const std::vector<int64_t>& nodes,
                      const std::vector<int>& widths, const std::vector<int64_t>& col0, const std::vector<int64_t>& goff,
                      const V* G, int64_t wtot, DBuf<V>& Y, const std::vector<std::pair<int64_t, int64_t>>& orange,
                      const std::vector<char>& counted, BasisProj<R>* lp = nullptr, std::vector<char>* fused = nullptr);
  // W level: probe pieces (tau, partner nodes nu in [p0, p1)) of one rank
  void w_probes(int l, const std::vector<int>& width, const std::vector<ProbePiece>& pieces, int maxw);
  // R level: probe pieces (nu, partner nodes tau in [p0, p1)) of one rank
  void r_probes(int l, const std::vector<int>& width, const std::vector<ProbePiece>& pieces, int maxw,
                int32_t* err_flag);
  // in-place all-gather of `per_rank` consecutive blocks per rank (+ ranks)
  void gather_inplace(Level<R>& lv, int64_t per_rank);
  // pack/all-gather/unpack of block index lists (one list per rank)
  void gather_packed(std::vector<Level<R>*> lvs, const std::vector<std::vector<int64_t>>& owned);
  double qr_flops(double a, double w, double k) const;
};

}  // namespace bfly
